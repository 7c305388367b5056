mkdir -p gpurun_out
for v in g128s3 g128s4; do MSK_B200_LIB=$PWD/variants/$v.so timeout 600 python -m pytest tests/test_policy.py -q --timeout 300 2>&1 | tail -1; done
for r in 1 2; do for v in g256 g128s3 g128s4; do
  echo -n "$v round $r: "; MSK_B200_LIB=$PWD/variants/$v.so timeout 120 python tools/policy_check.py 1024 4096 2>&1 | tail -2 | head -1
done; done
for v in g256 g128s3; do echo -n "$v 16384: "; MSK_B200_LIB=$PWD/variants/$v.so timeout 120 python tools/policy_check.py 1024 16384 2>&1 | tail -2 | head -1; done
