#!/usr/bin/env python3
"""Aggregate an ncu source page (--print-source=cuda,sass CSV) by source line and by kernel region."""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    cur, agg, src = None, {}, {}
    for r in rows:
        if len(r) < 8:
            continue
        if r[0] != "":
            try:
                cur = int(r[0])
                src[cur] = r[1]
            except ValueError:
                pass
            continue
        try:
            s, ie = float(r[4] or 0), float(r[7] or 0)
        except ValueError:
            continue
        a = agg.setdefault(cur, [0.0, 0.0])
        a[0] += s
        a[1] += ie
    return agg, src


if __name__ == "__main__":
    agg, src = load(sys.argv[1])
    units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    S = sum(v[0] for v in agg.values())
    I = sum(v[1] for v in agg.values())
    print(f"stall samples {S:.0f}, instructions {I:.0f} ({I / units:.0f} per unit)")
    key = 1 if "--inst" in sys.argv else 0
    for ln, (s, ie) in sorted(agg.items(), key=lambda x: -x[1][key])[:40]:
        print(f"{s / S * 100:5.1f}% stall  {ie / I * 100:5.1f}% inst  L{ln}: {src.get(ln, '').strip()[:100]}")
