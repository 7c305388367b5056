for c in c2 c3 c4 c5; do timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/e2e5_$c.log 2>&1
echo "$c $(tail -1 gpurun_out/e2e5_$c.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"])' 2>&1 | tail -1)"; done
