mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py -q -x --timeout 600 > gpurun_out/gen_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gen_tests.log
timeout 600 python -m pytest tests/test_dist.py tests/test_capi.py -q -m gpu --timeout 300 > gpurun_out/gen_tests2.log 2>&1; echo tests2 rc=$?; tail -2 gpurun_out/gen_tests2.log
for c in c2g c2; do timeout 600 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo $c rc=$?; tail -1 gpurun_out/bench_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d['e2e']['value'])"; done
