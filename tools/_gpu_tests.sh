# GPU tests without -x (every failure listed) + the parity report + smoke.
mkdir -p gpurun_out
MSK_PARITY_REPORT=gpurun_out/parity_report.json timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -30
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -4 gpurun_out/smoke.log
