# Discriminator training (own tcgen05 GEMMs): per-block gradient check, tests, c4-batch timing, launch list.
mkdir -p gpurun_out
timeout 120 python tools/disc_train_check.py 0 > gpurun_out/dt_check0.log 2>&1; echo check0 rc=$?; cat gpurun_out/dt_check0.log | tail -8
timeout 300 python -m pytest tests/test_disc_train.py -q --timeout 120 > gpurun_out/dt_tests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/dt_tests.log
for m in 0 1; do timeout 120 python tools/disc_train_bench.py 131072 $m 20 > gpurun_out/dt_bench$m.log 2>&1; echo bench$m rc=$?; tail -1 gpurun_out/dt_bench$m.log; done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dt_launches.csv python tools/disc_train_bench.py 131072 0 1 > gpurun_out/dt_ncu.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/dt_launches.csv --skip 90 2>&1 | tail -32
