# e2e (host-buffer C-ABI loop) vs the number of env groups
for c in ${CFGS:-c2}; do for g in ${NGROUPS:-2 4 8}; do
timeout 900 python bench.py --config $c --steps 100 --warmup 9 --no-cpu-baseline --e2e-groups $g 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', $g, d['value'], d['e2e']['value'])"
done; done
