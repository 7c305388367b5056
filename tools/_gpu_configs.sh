# GPU tests + bench lines for every BASELINE config (c2 default, c3-c5 rollout-shaped)
mkdir -p gpurun_out
# (tests skipped in this script variant)
for c in ${CFGS:-c2 c3 c4 c5}; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], d.get('disc_kernel'), d['clocks'], d['gpu_launches'])" 2>&1 | tail -1
done
