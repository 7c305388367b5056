for c in c2 c4; do for g in 1 2 4; do
  timeout 600 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --e2e-groups $g > gpurun_out/e2e_${c}_$g.log 2>&1
  echo "$c groups=$g $(tail -1 gpurun_out/e2e_${c}_$g.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"], d["value"])' 2>&1 | tail -1)"
done; done
