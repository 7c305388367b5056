# Env-vectorised step kernel: parity subset and bench for MSK_NE = 2, 4, 1
mkdir -p gpurun_out
for ne in 2 4; do
  MSK_NE=$ne timeout 900 python -m pytest tests/test_gpu.py -q -x --timeout 600 > gpurun_out/ne${ne}_tests.log 2>&1; echo ne$ne tests rc=$?; tail -3 gpurun_out/ne${ne}_tests.log
done
for r in 1 2; do for ne in 1 2 4; do
  MSK_NE=$ne timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/ne${ne}_bench$r.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/ne${ne}_bench$r.log').read().strip().splitlines()[-1]);print('NE=$ne round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['roofline']['step_kernel_ms']))"
done; done
