"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.
usage: python tools/launch_summary.py raw.csv "<command description>" > summary.csv"""
import csv
import io
import sys
from collections import OrderedDict

raw = open(sys.argv[1]).read().splitlines()
rows = list(csv.reader(io.StringIO("\n".join(l for l in raw if not l.startswith("==")))))
h = rows[0]
iK, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = OrderedDict()
for r in rows[1:]:
    name = r[iK].split("(")[0].replace("void ", "").strip()
    name = name.split("<")[0] if name.startswith("at::") else name
    v = float(r[iV].replace(",", ""))
    ms = v / 1e6 if r[iU] == "ns" else (v / 1e3 if r[iU] in ("us", "usecond") else v)
    n, t = agg.get(name, (0, 0.0))
    agg[name] = (n + 1, t + ms)
eng = {k: v for k, v in agg.items() if not k.startswith("at::")}
tot = sum(t for _, t in eng.values())
n_eng = sum(n for n, _ in eng.values())
print(f"# ncu launch list of `{sys.argv[2]}`, metric gpu__time_duration.sum, --clock-control none")
print("# ncu serializes launches and runs them cold-cache: compare SHARES, not absolute times.")
print("# at::* kernels are torch fills (the L2 flush between timed steps), not part of the engine.")
print(f"# engine launches: {n_eng}; engine kernel time {tot:.3f} ms")
print("kernel,launches,total_ms,ms_per_launch,share_of_engine")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    share = t / tot if k in eng and tot else 0.0
    print(f"{k},{n},{t:.4f},{t / n:.4f},{share:.3f}")
