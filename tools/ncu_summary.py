"""Text summary of one kernel of an ncu --set full report (key metrics, stall mix, hot SASS
regions): python tools/ncu_summary.py report.ncu-rep kernel_regex "title" > summary.txt"""
import csv
import io
import re
import subprocess
import sys

rep, kre, title = sys.argv[1], sys.argv[2], sys.argv[3]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size"]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, units = raw[0], raw[1]
row = next(r for r in raw[2:] if re.search(kre, r[h.index("Kernel Name")]))
print(f"# {title}")
print(f"# kernel: {row[h.index('Kernel Name')][:100]}")
for k in KEYS:
    if k in h:
        print(f"{k:<80} {row[h.index(k)]} {units[h.index(k)]}")
st = {}
for i, name in enumerate(h):
    m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", name)
    if m and not name.endswith("_not_issued"):
        try:
            st[m.group(1)] = float(row[i] or 0)
        except ValueError:
            pass
tot = sum(st.values()) or 1.0
print("stalls: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in
                             sorted(st.items(), key=lambda kv: -kv[1])[:8]))
# hot SASS regions (100-instruction windows with >= 3% of the samples)
src = ncu("--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kre}")
lines = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(lines) if r and r[0] == "Address")
hs = lines[hi]
end = next((i for i in range(hi + 1, len(lines)) if lines[i] and lines[i][0] == "Kernel Name"),
           len(lines))
data = lines[hi + 1:end]
iS, iW, iE = hs.index("Source"), hs.index("Warp Stall Sampling (All Samples)"), \
    hs.index("Instructions Executed")
wt = sum(float(r[iW] or 0) for r in data) or 1.0
for a in range(0, len(data), 100):
    seg = data[a:a + 100]
    w = sum(float(r[iW] or 0) for r in seg)
    if w / wt < 0.03:
        continue
    ops = {}
    for r in seg:
        t = r[iS].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
        ops[op] = ops.get(op, 0.0) + float(r[iW] or 0)
    top = " ".join(f"{k}:{100 * v / wt:.1f}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    inst = sum(float(r[iE] or 0) for r in seg)
    print(f"[{a:5d}-{a + len(seg) - 1:5d}] samples {100 * w / wt:5.1f}%  inst {inst:.3e}  {top}")
