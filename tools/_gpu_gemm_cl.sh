timeout 600 python -m pytest tests/test_policy.py -q --timeout 500 > gpurun_out/pytest_policy.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/pytest_policy.log
MSK_GEMM_CLUSTER=1 timeout 600 python -m pytest tests/test_policy.py -q --timeout 500 > gpurun_out/pytest_policy1.log 2>&1; echo tests-cl1 rc=$?
for c in 1 2 4; do echo "cluster=$c"; MSK_GEMM_CLUSTER=$c timeout 600 python tools/policy_check.py 1024 4096; done
