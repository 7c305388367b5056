# GPU tests (all failures listed) + parity report + smoke + parity diag + default bench line.
bash tools/_gpu_tests.sh
python tools/parity_diag.py wb700_fixed 3 > gpurun_out/pdiag.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | cut -c1-400
