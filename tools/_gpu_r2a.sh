# GPU tests + D-training timing/launch list + c4 loop with on-device D training
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
for m in 0 1; do timeout 120 python tools/disc_train_bench.py 131072 $m 20 > gpurun_out/dt_bench$m.log 2>&1; echo bench$m rc=$?; tail -1 gpurun_out/dt_bench$m.log; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dt_launches.csv python tools/disc_train_bench.py 131072 0 1 > gpurun_out/dt_ncu.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/dt_launches.csv --skip 66 2>&1 | tail -24
timeout 900 python bench.py --config c4 --rollout --disc-train fp32 --steps 48 --warmup 9 --no-cpu-baseline --no-e2e > gpurun_out/c4_dt.log 2>&1; echo c4dt rc=$?; tail -1 gpurun_out/c4_dt.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['phases_ms_per_step'])"
