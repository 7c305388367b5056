mkdir -p gpurun_out
timeout 300 python tools/policy_check.py 1024 4096 > gpurun_out/pol1.log 2>&1; tail -2 gpurun_out/pol1.log
MSK_GEMM_2CTA=1 timeout 300 python tools/policy_check.py 1024 4096 > gpurun_out/pol2.log 2>&1; tail -2 gpurun_out/pol2.log
M=gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__cycles_active.avg
for v in 1 2; do
  E=""; [ $v = 2 ] && E="MSK_GEMM_2CTA=1"
  env $E timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 200 -c 12 --csv python tools/policy_check.py 1024 4096 > gpurun_out/pol_ncu$v.csv 2>/dev/null; echo v$v rc=$?
done
python - <<'PY'
import csv
for v in (1,2):
    rows=list(csv.reader(open(f'gpurun_out/pol_ncu{v}.csv')))
    h=next(i for i,r in enumerate(rows) if 'Metric Name' in r); hdr=rows[h]
    mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ki=hdr.index('Kernel Name'); ii=hdr.index('ID')
    from collections import OrderedDict
    L=OrderedDict()
    for r in rows[h+1:]:
        if len(r)>vi: L.setdefault(r[ii],{'k':r[ki][:40]})[r[mi]]=r[vi]
    print('variant',v)
    for d in L.values(): print('  ', d['k'], {k[:28]:v for k,v in d.items() if k!='k'})
PY
