mkdir -p gpurun_out
for r in 1 2 3; do for v in a bc; do
  MSK_B200_LIB=$PWD/variants/$v.so timeout 300 python bench.py --config c2g --no-cpu-baseline --no-e2e --steps 200 > gpurun_out/ab_$v_$r.log 2>&1
  tail -1 gpurun_out/ab_$v_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['phases_ms_per_step']['step']))"
done; done
