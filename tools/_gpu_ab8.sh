mkdir -p gpurun_out
MSK_B200_LIB=$PWD/variants/dofsort.so timeout 900 python -m pytest tests/test_gpu.py -q -x --timeout 600 > gpurun_out/ab8_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/ab8_tests.log
for r in 1 2 3; do for v in base dofsort; do
  MSK_B200_LIB=$PWD/variants/$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['roofline']['step_kernel_ms']))"
done; done
for v in base dofsort; do MSK_B200_LIB=$PWD/variants/$v.so timeout 300 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 60 > gpurun_out/ab4_$v.log 2>&1; tail -1 gpurun_out/ab4_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $v: %.4g M'%(d['value']/1e6))"; done
