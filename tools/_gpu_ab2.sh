# A/B of library variants on one box: bench.py (device value + step kernel ms), alternating, 3 rounds.
mkdir -p gpurun_out
for r in 1 2 3; do for v in "$@"; do
  MSK_B200_LIB=$PWD/variants/$v.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/ab_$v_$r.log 2>&1
  python -c "import json,sys;d=json.loads(open('gpurun_out/ab_$v_$r.log').read().strip().splitlines()[-1]);print('$v round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['roofline']['step_kernel_ms']))"
done; done
