# ncu --set full of the step kernel (c2 headline workload) + the launch list of the same command.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -f -o gpurun_out/prof_step_r2 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
timeout 300 $CMD > gpurun_out/plain_prof2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
tail -2 gpurun_out/ncu_full.log
