# A/B: base (NE=1), rolled children loop (NE=1), NE=2 at 144 registers
mkdir -p gpurun_out
for r in 1 2; do
for spec in "base 1" "rolled 1" "ne144 2"; do set -- $spec
  MSK_NE=$2 MSK_B200_LIB=$PWD/variants/$1.so timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/ab_$1_$r.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ab_$1_$r.log').read().strip().splitlines()[-1]);print('$1 NE=$2 round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['roofline']['step_kernel_ms']))"
done; done
