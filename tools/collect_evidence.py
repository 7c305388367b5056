#!/usr/bin/env python3
"""Copy a tools/_gpu_round.sh run (gpurun_out/) into profiles/<round>/ and
refresh profiles/step_kernel_traffic.json (python tools/collect_evidence.py r02)."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINES = {"bench.log": "bench_line.json", "bench_ref.log": "bench_ref_line.json",
         "bench_ref_c4.log": "bench_ref_c4_line.json", "bench_c2g.log": "bench_c2g_line.json",
         "bench_c3.log": "bench_c3_line.json", "bench_c4.log": "bench_c4_line.json", "bench_c5.log": "bench_c5_line.json",
         "bench_c2_policy.log": "bench_c2_policy_line.json", "bench_c4_full.log": "bench_c4_full_line.json",
         "bench_c4_dt.log": "bench_c4_dt_line.json", "dt_bench0.log": "disc_train_fp32_line.json",
         "dt_bench1.log": "disc_train_bf16_line.json"}
COPIES = {"parity_report.json": "parity_report.json", "smoke.log": "smoke.log", "launches.csv": "launches_bench.csv",
          "dt_launches.csv": "disc_train_launches.csv", "policy_check.log": "policy_check.txt",
          "gemm_bench.log": "gemm_bench.txt"}


def main(rnd):
    g, p = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", rnd)
    os.makedirs(p, exist_ok=True)
    for a, b in LINES.items():
        line = open(os.path.join(g, a)).read().strip().splitlines()[-1]
        with open(os.path.join(p, b), "w") as f:
            f.write(json.dumps(json.loads(line), indent=1) + "\n")
    for a, b in COPIES.items():
        shutil.copy(os.path.join(g, a), os.path.join(p, b))
    with open(os.path.join(p, "disc_train_launch_table.txt"), "w") as f:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_table.py"),
                        os.path.join(p, "disc_train_launches.csv")], stdout=f, check=True)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"),
                    os.path.join(g, "prof_step.ncu-rep"), p], stdout=subprocess.DEVNULL, check=True)
    print("evidence copied to", p)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
