# A/B: variants/base.so (HEAD) vs the in-tree library on c2 and c4, then the GPU tests.
mkdir -p gpurun_out; rm -f gpurun_out/ab10_*.log
for rep in 1 2; do
  for v in base tree; do
    for cfg in c2 c4; do
      if [ $v = base ]; then L=MSK_B200_LIB=$PWD/variants/base.so; else L=; fi
      env $L timeout 300 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ab10_${v}_${cfg}_$rep.log 2>&1; echo $v $cfg rc=$?
    done
  done
done
for f in gpurun_out/ab10_*.log; do echo $f $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,3), round(d['roofline']['step_kernel_ms'],4))" 2>/dev/null); done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
