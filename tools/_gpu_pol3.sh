mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_policy.py -q --timeout 300 > gpurun_out/pol_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pol_tests.log
for i in 1 2; do timeout 120 python tools/policy_check.py 1024 4096 2>&1 | tail -2; MSK_GEMM_1CTA=1 timeout 120 python tools/policy_check.py 1024 4096 2>&1 | tail -2; done
timeout 300 python tools/policy_check.py 1024 16384 2>&1 | tail -2
M=gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 300 ncu --metrics $M --clock-control none -k regex:gemm -s 200 -c 6 --csv python tools/policy_check.py 1024 4096 > gpurun_out/pol_ncu4.csv 2>/dev/null
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/pol_ncu4.csv')))
h=next(i for i,r in enumerate(rows) if 'Metric Name' in r); hdr=rows[h]
mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ki=hdr.index('Kernel Name'); ii=hdr.index('ID')
from collections import OrderedDict
L=OrderedDict()
for r in rows[h+1:]:
    if len(r)>vi: L.setdefault(r[ii],{'k':r[ki][:40]})[r[mi]]=r[vi]
for d in L.values(): print('  ', d['k'], {k[:28]:v for k,v in d.items() if k!='k'})
PY
