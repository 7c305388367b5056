for v in variants/*.so; do
  echo "== $v" >> gpurun_out/phases.log
  MSK_B200_LIB=$PWD/$v timeout 300 python tools/phase_timers.py wb700_fixed 4096 >> gpurun_out/phases.log 2>&1
done
cat gpurun_out/phases.log
