timeout 600 python -m pytest tests/test_policy.py -q --timeout 500 > gpurun_out/pytest_policy.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/pytest_policy.log
timeout 600 python tools/policy_check.py 1024 4096 > gpurun_out/policy.log 2>&1; cat gpurun_out/policy.log
for cw in "c2 1024" "c2 256" "c4 1024"; do set -- $cw
  timeout 900 python bench.py --config $1 --policy-width $2 --steps 60 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_pol_$1_$2.log 2>&1; echo "$1 W=$2 rc=$?"
  tail -1 gpurun_out/bench_pol_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phases_ms_per_step'])" 2>&1 | tail -1
done
