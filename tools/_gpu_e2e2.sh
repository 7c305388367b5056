for E in 1024 1536 2048 3072 4096; do
  timeout 300 python bench.py --steps 100 --warmup 3 --envs $E --no-cpu-baseline --no-e2e > gpurun_out/envs_$E.log 2>&1
  echo "E=$E $(tail -1 gpurun_out/envs_$E.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["step_kernel_ms"])')"
done
for cs in "2 1" "3 1" "3 3" "4 4" "2 2"; do
  set -- $cs
  MSK_HOST_CHUNKS=$1 MSK_HOST_STREAMS=$2 timeout 300 python bench.py --steps 60 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$1_$2.log 2>&1
  echo "$1 $2 $(tail -1 gpurun_out/e2e_$1_$2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"], d["value"])')"
done
