# Quick check: GPU tests (+parity margins) and the default bench line.
mkdir -p gpurun_out
MSK_PARITY_REPORT=gpurun_out/parity_report.json timeout 900 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log | cut -c1-600
