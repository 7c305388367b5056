mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 205 -c 1 -f -o gpurun_out/prof_gemm python tools/policy_check.py 1024 4096 > gpurun_out/ncu_gemm.log 2>&1; echo rc=$?
ncu -i gpurun_out/prof_gemm.ncu-rep --page details --csv > gpurun_out/gemm_details.csv 2>/dev/null; echo det rc=$?
