# A/B of variants/*.so vs the in-tree library on c2 and c4 (2 reps), then the GPU tests on variants/$AB_TEST_LIB.
mkdir -p gpurun_out; rm -f gpurun_out/ab12_*.log
for rep in 1 2; do
  for v in cur ${AB_VARIANTS}; do
    if [ $v = cur ]; then L=; else L=MSK_B200_LIB=$PWD/variants/$v.so; fi
    env $L timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab12_${v}_c2_$rep.log 2>&1
    env $L timeout 300 python bench.py --config c4 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab12_${v}_c4_$rep.log 2>&1
  done
done
for f in gpurun_out/ab12_*.log; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['roofline']['step_kernel_ms'],4))" 2>/dev/null); done
if [ -n "$AB_TEST_LIB" ]; then
  MSK_B200_LIB=$PWD/variants/$AB_TEST_LIB.so timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
fi
