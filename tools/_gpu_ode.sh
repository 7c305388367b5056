mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_policy.py -q --timeout 120 -x > gpurun_out/ode_tests.log 2>&1; echo tests rc=$?; tail -5 gpurun_out/ode_tests.log
for i in 1 2; do timeout 120 python tools/policy_check.py 1024 4096 2>&1 | tail -2; MSK_POLICY_LAYERS=1 timeout 120 python tools/policy_check.py 1024 4096 2>&1 | tail -2 | head -1; done
timeout 120 python tools/policy_check.py 1024 16384 2>&1 | tail -2
