for v in e8 e16; do echo "== $v"; MSK_B200_LIB=$PWD/variants/$v.so timeout 120 python tools/gemm_bench.py 4096 1024 2>&1 | head -4; MSK_B200_LIB=$PWD/variants/$v.so timeout 120 python tools/policy_check.py 1024 4096 2>&1 | tail -2 | head -1; done
MSK_B200_LIB=$PWD/variants/e16.so timeout 300 python -m pytest tests/test_policy.py -q -x --timeout 200 2>&1 | tail -1
