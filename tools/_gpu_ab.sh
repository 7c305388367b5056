set -x
for v in variants/*.so; do
  MSK_B200_LIB=$PWD/$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_$(basename $v .so).log 2>&1; echo $v rc=$?
done
timeout 600 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
for f in gpurun_out/ab_*.log; do echo $f; tail -1 $f | cut -c1-120; done
tail -3 gpurun_out/pytest_gpu.log
