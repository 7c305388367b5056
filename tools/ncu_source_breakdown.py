#!/usr/bin/env python3
"""Per-function instruction / stall attribution of the step kernel from an ncu
--set full --import-source capture: joins ncu's SASS source page with the
library's own line table (nvdisasm -g) and sums per inlined device function.

  python tools/ncu_source_breakdown.py gpurun_out/prof_step.ncu-rep [kernel-mangled-name] > out.txt
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2603_29332_b200", "libmsk_b200.so")
SRC = os.path.join(ROOT, "paper_2603_29332_b200", "csrc", "kernels.cu")
DEFAULT = "_ZN8msk_b20011step_kernelILi28ELi1ELi3ELi1ELi3EEEvNS_8DevModelENS_8DevStateEiiPKfPfS5_S5_PhS5_S5_i"


def sass_lines(func):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "kernels.sm_100a.cubin", LIB], cwd=d, check=True,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, "kernels.sm_100a.cubin")], capture_output=True,
                             text=True, check=True).stdout
    out, line, on = [], None, False
    for s in txt.splitlines():
        if s.startswith(func + ":"):
            on = True
            continue
        if on and s.startswith(".text.") and not s.startswith(".text." + func):
            break
        if not on:
            continue
        m = re.search(r"line (\d+)", s)
        if m and "//##" in s:
            line = int(m.group(1))
            continue
        if re.match(r"\s*/\*[0-9a-f]+\*/\s+", s):
            out.append(line)
    return out


def main(rep, func=DEFAULT):
    page = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(page)))
    hdr, data = rows[1], rows[2:]
    lines = sass_lines(func)
    if len(lines) != len(data):
        sys.exit(f"SASS of the library ({len(lines)}) does not match the capture ({len(data)}): rebuild or recapture")
    i_e, i_s = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    src = open(SRC).read().split("\n")
    fns = [(i + 1, m.group(1)) for i, l in enumerate(src)
           for m in [re.match(r"^(?:__device__|__global__).*?\b(\w+)\(", l)] if m]

    def owner(ln):
        name = "?"
        for a, n in fns:
            if ln and a <= ln:
                name = n
        return name

    agg = collections.defaultdict(lambda: [0, 0])
    for ln, r in zip(lines, data):
        a = agg[owner(ln)]
        a[0] += int(r[i_e])
        a[1] += int(r[i_s])
    tot_i, tot_s = sum(v[0] for v in agg.values()), sum(v[1] for v in agg.values())
    print(f"{os.path.basename(rep)}: {tot_i} warp-instructions, {tot_s} stall samples")
    print(f"{'function (inlined)':26s} {'inst %':>7s} {'stall %':>8s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0]):
        if v[0] / tot_i < 0.003:
            continue
        print(f"{k:26s} {100 * v[0] / tot_i:7.1f} {100 * v[1] / tot_s:8.1f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
