mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_disc_train.py -q --timeout 120 > gpurun_out/dt_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/dt_tests.log
for m in 0 1; do timeout 120 python tools/disc_train_bench.py 131072 $m 20 2>&1 | tail -1; done
timeout 120 python tools/disc_train_bench.py 131072 0 3 > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dt_launches.csv python tools/disc_train_bench.py 131072 0 1 > gpurun_out/dt_ncu.log 2>&1; echo ncu rc=$?
n=$(python tools/launch_table.py gpurun_out/dt_launches.csv | grep -c " us "); python tools/launch_table.py gpurun_out/dt_launches.csv --skip $((n-23)) | grep -E "pack_input|reduce|total"
