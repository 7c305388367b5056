mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -q -k "disc or reward" --timeout 300 > gpurun_out/disc_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/disc_tests.log
timeout 300 python -m pytest tests/test_disc_train.py -q -k publish --timeout 300 2>&1 | tail -1
timeout 600 python bench.py --config c4 --steps 60 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/c4d.log 2>&1; tail -1 gpurun_out/c4d.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['disc_kernel']['ms'], d['disc_kernel']['frac'])"
