export MSK_GEMM_2CTA=1
timeout 300 python -m pytest tests/test_policy.py -q --timeout 250 > gpurun_out/pytest_policy2.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pytest_policy2.log
timeout 300 python tools/policy_check.py 1024 4096; echo rc=$?
unset MSK_GEMM_2CTA
timeout 300 python tools/policy_check.py 1024 4096
