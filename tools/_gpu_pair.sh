bash tools/_gpu_ab.sh > gpurun_out/ab_summary.txt 2>&1
MSK_B200_LIB=$PWD/variants/lib_pair.so timeout 600 python -m pytest tests/test_gpu.py -q -x --timeout 500 > gpurun_out/pytest_pair.log 2>&1; echo pair-tests rc=$?; tail -3 gpurun_out/pytest_pair.log
grep -v "^+" gpurun_out/ab_summary.txt | grep -v rc=
