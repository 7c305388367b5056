# A/B every variants/*.so (bench, no cpu/e2e legs), phase timers for lib_timers, then GPU tests on the in-tree lib.
set -x
mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log gpurun_out/phases.log
for rep in 1 2; do
for v in variants/*.so; do
  [ "$(basename $v)" = lib_timers.so ] && continue
  MSK_B200_LIB=$PWD/$v timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab_$(basename $v .so)_$rep.log 2>&1; echo $v rc=$?
done
done
[ -f variants/lib_timers.so ] && MSK_B200_LIB=$PWD/variants/lib_timers.so timeout 300 python tools/phase_timers.py wb700_fixed 4096 >> gpurun_out/phases.log 2>&1
[ -n "$AB_TESTS" ] && { timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log; }
for f in gpurun_out/ab_*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d.get('clocks'))"; done
cat gpurun_out/phases.log
