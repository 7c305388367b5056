# A/B of policy-GEMM variants: policy_check at 4096 / 16384 envs and the c4 full loop.
mkdir -p gpurun_out
for v in cur ${AB_VARIANTS}; do
  if [ $v = cur ]; then L=; else L=MSK_B200_LIB=$PWD/variants/$v.so; fi
  for E in 4096 16384; do env $L timeout 300 python tools/policy_check.py 1024 $E 2>&1 | grep "ms per sample" | sed "s/^/$v /"; done
  env $L timeout 600 python bench.py --config c4 --policy-width 1024 --rollout --disc-train fp32 --steps 24 --warmup 9 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v c4_full', d['value'], d['phases_ms_per_step']['actions'])"
done
