set -x
rm -f gpurun_out/phases.log
MSK_B200_LIB=$PWD/variants/lib_timers.so timeout 300 python tools/phase_timers.py wb700_fixed 4096 >> gpurun_out/phases.log 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 400 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
cat gpurun_out/phases.log; tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/bench.log | cut -c1-200
