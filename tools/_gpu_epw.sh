rm -f gpurun_out/phases.log
for v in variants/*.so; do
  echo "== $v" >> gpurun_out/phases.log
  MSK_B200_LIB=$PWD/$v timeout 300 python tools/phase_timers.py wb700_fixed 4096 >> gpurun_out/phases.log 2>&1
done
MSK_B200_LIB=$PWD/variants/lib_kform.so timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_k.log 2>&1; echo pytest rc=$?
cat gpurun_out/phases.log; tail -3 gpurun_out/pytest_k.log
