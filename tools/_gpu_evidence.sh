# Full round evidence: tests (+parity margins), default bench, reference arm, configs c3-c5,
# phase timers, ncu launch list, ncu --set full of the step kernel and of the discriminator kernel.
set -x
mkdir -p gpurun_out
MSK_PARITY_REPORT=gpurun_out/parity_report.json timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --steps 160 --warmup 8 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c rc=$?; done
[ -f variants/lib_timers.so ] && MSK_B200_LIB=$PWD/variants/lib_timers.so timeout 300 python tools/phase_timers.py wb700_fixed 4096 > gpurun_out/phases.log 2>&1
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -f -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
CMD4="python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $CMD4 > gpurun_out/plain4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:disc_reward -s 3 -c 1 -f -o gpurun_out/prof_disc $CMD4 > gpurun_out/ncu_disc.log 2>&1; echo ncu3 rc=$?
tail -2 gpurun_out/pytest_gpu.log
