# ncu --set full (source view) of the c2 step kernel only.
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain_prof.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -f -o gpurun_out/prof_step3 $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_full.log
