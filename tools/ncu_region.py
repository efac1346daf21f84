"""Stall-reason breakdown of an ncu source page over SASS index ranges.
usage: python tools/ncu_region.py source.csv a:b [c:d ...]   (indices as printed by ncu_phases)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
iW = h.index("Warp Stall Sampling (All Samples)")
iE = h.index("Instructions Executed")
tot = sum(float(r[iW] or 0) for r in data) or 1
for rg in sys.argv[2:]:
    a, b = map(int, rg.split(":"))
    seg = data[a:b + 1]
    s = {h[c][6:]: sum(float(r[c] or 0) for r in seg) for c in cols}
    n = sum(s.values()) or 1
    inst = sum(float(r[iE] or 0) for r in seg)
    print(f"[{a}:{b}] {100 * sum(float(r[iW] or 0) for r in seg) / tot:.1f}% of samples, inst {inst:.3e}: "
          + ", ".join(f"{k} {100 * v / n:.0f}%" for k, v in sorted(s.items(), key=lambda t: -t[1])[:7]))
