mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x --timeout 600 > gpurun_out/ab4_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ab4_tests.log
for r in 1 2 3; do for v in base simple; do
  MSK_B200_LIB=$PWD/variants/$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/ab_$v_$r.log 2>&1
  tail -1 gpurun_out/ab_$v_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['roofline']['step_kernel_ms']))"
done; done
