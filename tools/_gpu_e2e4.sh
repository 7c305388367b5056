for gc in "4 1" "6 1" "8 1" "4 2" "16 1"; do set -- $gc
  MSK_HOST_CHUNKS=$2 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-groups $1 > gpurun_out/e2e4_$1_$2.log 2>&1
  echo "groups=$1 chunks=$2 $(tail -1 gpurun_out/e2e4_$1_$2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["e2e"]["value"])' 2>&1 | tail -1)"
done
