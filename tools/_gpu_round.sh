# Round evidence: GPU tests (+parity report), headline bench, reference arm (c2, c4), smoke,
# configs c2g/c3/c4/c5 + on-device loops, D-training timing, policy, ncu launch list + step-kernel capture.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
# the step-kernel capture first: bench.py's roofline.issue reads profiles/step_kernel_traffic.json
timeout 300 $CMD > gpurun_out/plain2.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 3 -c 1 -f -o gpurun_out/prof_step $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
python tools/ncu_summary.py gpurun_out/prof_step.ncu-rep gpurun_out/prof_summary > gpurun_out/ncu_summary.log 2>&1
python tools/ncu_source_breakdown.py gpurun_out/prof_step.ncu-rep > gpurun_out/step_kernel_source_breakdown.txt 2>&1
MSK_PARITY_REPORT=gpurun_out/parity_report.json timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$?
timeout 600 python bench.py --impl reference --config c4 --steps 3 --warmup 3 > gpurun_out/bench_ref_c4.log 2>&1; echo ref4 rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
CFGS="c2g c3 c4 c5" bash tools/_gpu_configs.sh > gpurun_out/configs.log 2>&1; echo configs rc=$?
timeout 900 python bench.py --config c4 --rollout --disc-train fp32 --steps 48 --warmup 9 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_dt.log 2>&1; echo c4dt rc=$?
for m in 0 1; do timeout 120 python tools/disc_train_bench.py 131072 $m 20 > gpurun_out/dt_bench$m.log 2>&1; done
timeout 120 python tools/policy_check.py 1024 4096 > gpurun_out/policy_check.log 2>&1
timeout 120 python tools/gemm_bench.py 4096 1024 > gpurun_out/gemm_bench.log 2>&1
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 120 python tools/disc_train_bench.py 131072 0 3 > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dt_launches.csv python tools/disc_train_bench.py 131072 0 1 > gpurun_out/dt_ncu.log 2>&1; echo ncu3 rc=$?
tail -2 gpurun_out/pytest_gpu.log; tail -5 gpurun_out/smoke.log; cat gpurun_out/configs.log; tail -1 gpurun_out/dt_bench0.log; tail -1 gpurun_out/dt_bench1.log; tail -2 gpurun_out/policy_check.log
