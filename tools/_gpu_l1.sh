mkdir -p gpurun_out
for r in 1 2; do
for spec in "w28 4144" "w24 3552" "w20 2960"; do set -- $spec
  MSK_B200_LIB=$PWD/variants/$1.so timeout 300 python bench.py --envs $2 --no-cpu-baseline --no-e2e --steps 200 > gpurun_out/l1_$1.log 2>&1
  tail -1 gpurun_out/l1_$1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 envs $2 round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['phases_ms_per_step']['step']))"
done; done
