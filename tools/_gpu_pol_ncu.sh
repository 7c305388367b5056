CMD="python tools/policy_check.py 1024 4096"
timeout 600 $CMD > gpurun_out/pol_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pol_launches.csv -c 120 $CMD > gpurun_out/pol_ncu.log 2>&1; echo ncu rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 10 -c 1 -f -o gpurun_out/prof_gemm $CMD > gpurun_out/pol_ncu2.log 2>&1; echo ncu2 rc=$?
# discriminator training step (c4 batch, TF32): one --set full capture of its heaviest own kernel
CMD2="python tools/disc_train_bench.py 131072 1 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rev_elem_kernel -s 2 -c 1 -f -o gpurun_out/prof_dt $CMD2 > gpurun_out/dt_ncu.log 2>&1; echo ncu3 rc=$?
