mkdir -p gpurun_out
for q in 4 2; do
  MSK_TREEQ=$q timeout 900 python -m pytest tests/test_gpu.py -q -x --timeout 600 > gpurun_out/tq${q}_tests.log 2>&1; echo tq$q tests rc=$?; tail -2 gpurun_out/tq${q}_tests.log
done
for r in 1 2; do for q in 1 2 4; do
  MSK_TREEQ=$q timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 300 > gpurun_out/tq${q}_b$r.log 2>&1
  tail -1 gpurun_out/tq${q}_b$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TREEQ=$q round $r: %.4g M  step %.4f ms'%(d['value']/1e6,d['roofline']['step_kernel_ms']))"
done; done
for q in 1 4; do MSK_TREEQ=$q timeout 600 python bench.py --config c4 --no-cpu-baseline --no-e2e --steps 100 > gpurun_out/tq${q}_c4.log 2>&1; tail -1 gpurun_out/tq${q}_c4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 TREEQ=$q: %.4g M  step %.4f ms'%(d['value']/1e6,d['phases_ms_per_step']['step']))"; done
