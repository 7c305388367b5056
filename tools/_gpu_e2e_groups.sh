for c in c4 c5; do for g in 2 4; do
timeout 900 python bench.py --config $c --steps 100 --warmup 9 --no-cpu-baseline --e2e-groups $g 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $g, d['value'], d['e2e']['value'])"
done; done
