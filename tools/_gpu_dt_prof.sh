# Launch list of one discriminator training step on the c4 batch (own tcgen05 GEMMs).
mkdir -p gpurun_out
timeout 120 python tools/disc_train_bench.py 131072 0 3 > gpurun_out/dt_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/dt_launches.csv python tools/disc_train_bench.py 131072 0 1 > gpurun_out/dt_ncu.log 2>&1; echo ncu rc=$?
python tools/launch_table.py gpurun_out/dt_launches.csv 2>&1 | tail -42
