# Bench lines for every BASELINE config (c2 default, c3-c5 rollout-shaped) and the on-device loop variants
mkdir -p gpurun_out
for c in ${CFGS:-c3 c4 c5}; do
  timeout 900 python bench.py --config $c --steps 200 --warmup 9 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], d.get('disc_kernel'), d['clocks'], d['gpu_launches'])" 2>&1 | tail -1
done
timeout 900 python bench.py --config c2 --policy-width 1024 --rollout --steps 96 --warmup 9 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2_policy.log 2>&1; echo "c2 policy rc=$?"
timeout 900 python bench.py --config c4 --policy-width 1024 --rollout --disc-train fp32 --steps 48 --warmup 9 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_full.log 2>&1; echo "c4 full loop rc=$?"
for f in gpurun_out/bench_c2_policy.log gpurun_out/bench_c4_full.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phases_ms_per_step'])"; done
