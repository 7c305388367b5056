#!/usr/bin/env python3
"""Per-kernel table of an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes]).

  python tools/launch_table.py launches.csv [--skip N]   (skip the first N launches)"""
import csv
import sys
from collections import OrderedDict


def main(path, skip=0):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, ii, mi, vi = hdr.index("Kernel Name"), hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
    launches = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    items = list(launches.values())[skip:]
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in items)
    for d in items:
        t = d.get("gpu__time_duration.sum", 0)
        rb, wb = d.get("dram__bytes_read.sum", 0), d.get("dram__bytes_write.sum", 0)
        print(f"{t / 1e3:9.1f} us {100 * t / max(tot, 1):5.1f}%  dram r {rb / 1e6:8.1f} MB w {wb / 1e6:8.1f} MB "
              f"{(rb + wb) / max(t, 1):7.0f} GB/s  {d['name'][:90]}")
    print(f"total {tot / 1e3:.1f} us over {len(items)} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[2] == "--skip" else 0)
