# Parity report of an A/B library variant: MSK_B200_LIB=variants/$1.so
mkdir -p gpurun_out
MSK_B200_LIB=$PWD/variants/$1.so MSK_PARITY_REPORT=gpurun_out/parity_$1.json timeout 900 python -m pytest tests/test_gpu.py -q -k "single_step or full_size or general or contact" > gpurun_out/pytest_$1.log 2>&1; echo rc=$?
grep -E "^E  .*ratio|passed|failed" gpurun_out/pytest_$1.log | head -20
