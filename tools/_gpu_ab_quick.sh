# Fast iteration: a parity subset + the default bench line (device value only).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "single_step or substep or general or contact" > gpurun_out/pytest_q.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_q.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_q$i.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/bench_q$i.log').read().strip().splitlines()[-1]);print('value %.4g M  step_kernel_ms %.4f'%(d['value']/1e6,d['roofline']['step_kernel_ms']))"; done
