for c in ${CFGS:-c3 c4}; do
  timeout 900 python bench.py --config $c --steps 64 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.log 2>&1; echo "$c rc=$?"
  tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phases_ms_per_step'])" 2>&1 | tail -1
done
