# GPU tests + c4 rollout bench with/without the on-device discriminator training step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
for dt in "" fp32 bf16; do
  timeout 600 python bench.py --config c4 --rollout --steps 48 --warmup 9 --no-cpu-baseline --no-e2e ${dt:+--disc-train $dt} > gpurun_out/c4_dt_${dt:-none}.log 2>&1; echo c4 $dt rc=$?
done
for f in gpurun_out/c4_dt_*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phases_ms_per_step'])"; done
tail -3 gpurun_out/pytest_gpu.log
