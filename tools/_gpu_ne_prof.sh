mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_long_scoreboard,smsp__average_warp_latency_issue_stalled_short_scoreboard,smsp__average_warp_latency_issue_stalled_wait,smsp__average_warp_latency_issue_stalled_math_pipe_throttle,smsp__average_warp_latency_issue_stalled_mio_throttle,smsp__average_warp_latency_issue_stalled_lg_throttle,smsp__average_warp_latency_issue_stalled_not_selected,smsp__average_warp_latency_issue_stalled_barrier,smsp__average_warp_latency_issue_stalled_membar,smsp__average_warp_latency_issue_stalled_branch_resolving,smsp__average_warp_latency_issue_stalled_dispatch_stall,smsp__average_warp_latency_issue_stalled_no_instruction,smsp__average_warp_latency_issue_stalled_selected,smsp__thread_inst_executed_per_inst_executed.ratio,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_global_ld.sum
for ne in 1 2; do
  MSK_NE=$ne timeout 600 ncu --metrics $M --clock-control none -k regex:step -s 3 -c 1 --csv $CMD > gpurun_out/ne${ne}_ncu.csv 2> gpurun_out/ne${ne}_ncu.err; echo ne$ne rc=$?
done
python - <<'PY'
import csv
for ne in (1,2):
    rows=list(csv.reader(open(f'gpurun_out/ne{ne}_ncu.csv')))
    h=next(i for i,r in enumerate(rows) if 'Metric Name' in r); hdr=rows[h]
    mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ki=hdr.index('Kernel Name')
    print('NE',ne, rows[h+1][ki][:50])
    for r in rows[h+1:]:
        if len(r)>vi: print(f"   {r[mi][:75]:75s} {r[vi]}")
PY
