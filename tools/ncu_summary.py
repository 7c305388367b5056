#!/usr/bin/env python3
"""Summarise an ncu --set full capture of the step kernel into profiles/.

  python tools/ncu_summary.py gpurun_out/prof_step.ncu-rep profiles/r01
writes <out>/step_kernel_ncu_details.csv (details page) and refreshes
profiles/step_kernel_traffic.json (per-launch DRAM bytes read by bench.py)."""
import csv
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(rep, out_dir):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {k: [v, u] for k, u, v in zip(hdr, units, vals) if k in KEYS}
    name = vals[hdr.index("Kernel Name")]

    def nbytes(k):
        v, u = m[k]
        return float(v.replace(",", "")) * SCALE.get(u, 1)

    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    out = {"kernel": name, "source": os.path.basename(rep), "bytes_per_launch": rd + wr, "dram_read_bytes": rd,
           "dram_write_bytes": wr, "metrics": m}
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(root, "profiles", "step_kernel_traffic.json"), "w") as f:
        json.dump(out, f, indent=1)
    os.makedirs(out_dir, exist_ok=True)
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    with open(os.path.join(out_dir, "step_kernel_ncu_details.csv"), "w") as f:
        f.write(det)
    for k in KEYS:
        if k in m:
            print(f"{k:60s} {m[k][0]:>16s} {m[k][1]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
