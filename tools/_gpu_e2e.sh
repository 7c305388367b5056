# e2e (host-buffer C-ABI step) across pipeline shapes + raw PCIe copy rates
python - > gpurun_out/pcie.log 2>&1 <<'PY'
import torch, time
n = 52 * 1024 * 1024 // 4
d = torch.empty(n, device="cuda"); h = torch.empty(n, pin_memory=True)
for name, f in [("d2h", lambda: h.copy_(d, non_blocking=True)), ("h2d", lambda: d.copy_(h, non_blocking=True))]:
    for _ in range(3): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): f()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 20
    print(name, f"{n * 4 / dt / 1e9:.1f} GB/s")
PY
for cs in "4 2" "1 1" "2 2" "4 4" "8 2" "8 4" "8 8" "16 4" "16 8" "32 8"; do
  set -- $cs
  MSK_HOST_CHUNKS=$1 MSK_HOST_STREAMS=$2 timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$1_$2.log 2>&1
  echo "$1 $2 $(tail -1 gpurun_out/e2e_$1_$2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"], d["value"])')"
done
cat gpurun_out/pcie.log
