mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_disc_train.py -q --timeout 120 > gpurun_out/dt_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/dt_tests.log
timeout 120 python tools/disc_train_check.py 0 2>&1 | tail -4
for m in 0 1; do timeout 120 python tools/disc_train_bench.py 131072 $m 20 2>&1 | tail -1; done
