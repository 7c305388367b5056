#!/usr/bin/env python3
"""Per-source-line view of an ncu report: stall samples, instructions, L1 shared
wavefronts and global tag requests (ncu -i REP --page source --csv --print-source cuda,sass)."""
import csv
import subprocess
import sys


def main(rep, top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    col = {}
    for i, n in enumerate(hdr):
        col.setdefault(n, i)
    want = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared",
            "L1 Wavefronts Shared Ideal", "L1 Tag Requests Global", "L2 Theoretical Sectors Global"]
    lines = []
    for r in rows:
        if not r or not r[0].isdigit() or len(r) < len(hdr):
            continue
        vals = []
        for w in want:
            try:
                vals.append(float(r[col[w]] or 0))
            except ValueError:
                vals.append(0.0)
        lines.append((int(r[0]), r[1].strip()[:70], vals))
    tot = [sum(l[2][i] for l in lines) for i in range(len(want))]
    print("totals:", {w: f"{t:.3g}" for w, t in zip(want, tot)})
    print(f"{'line':>5} {'samp%':>6} {'inst%':>6} {'shWF%':>6} {'shIdeal':>8} {'gTag%':>6}  source")
    for ln, src, v in sorted(lines, key=lambda l: -l[2][0])[:top]:
        print(f"{ln:5d} {100 * v[0] / tot[0]:6.2f} {100 * v[1] / tot[1]:6.2f} {100 * v[2] / max(tot[2], 1):6.2f} "
              f"{v[3] / max(v[2], 1):8.2f} {100 * v[4] / max(tot[4], 1):6.2f}  {src}")
    print("\n-- top shared-wavefront lines --")
    for ln, src, v in sorted(lines, key=lambda l: -l[2][2])[:20]:
        print(f"{ln:5d} {100 * v[0] / tot[0]:6.2f} {100 * v[1] / tot[1]:6.2f} {100 * v[2] / max(tot[2], 1):6.2f} "
              f"{v[3] / max(v[2], 1):8.2f} {100 * v[4] / max(tot[4], 1):6.2f}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
