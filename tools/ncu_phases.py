"""Summarise an ncu report of k_couple: SOL numbers, stall reasons, and SASS samples per
barrier-delimited phase. Usage: python tools/ncu_phases.py report.ncu-rep [kernel-name regex]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = ["--kernel-name", "regex:" + sys.argv[2]] if len(sys.argv) > 2 else []


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *kfilter, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, vals = raw[0], raw[2]
d = dict(zip(hdr, vals))
for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__warps_active.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "launch__registers_per_thread", "launch__block_size"]:
    if k in d:
        print(f"{k:80s} {d[k]}")
items = []
for k in hdr:
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
        try:
            items.append((float(d[k]), k))
        except ValueError:
            pass
tot = sum(v for v, _ in items) or 1
print("stalls:", ", ".join(f"{k.split('stalled_')[1]} {100*v/tot:.1f}%" for v, k in sorted(items, reverse=True)[:8]))
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = rows[1]
data = [r for r in rows[2:] if r != h and len(r) == len(h)]
iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[iW] or 0) for r in data) or 1
acc = ex = 0.0
start = 0
for i, r in enumerate(data):
    acc += float(r[iW] or 0)
    ex += float(r[iE] or 0)
    if "BAR.SYNC" in r[iS] or i == len(data) - 1:
        ops = {}
        for q in data[start:i + 1]:
            tok = q[iS].split()
            if not tok:
                continue
            op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
            op = op.split(".")[0]
            ops[op] = ops.get(op, 0) + float(q[iW] or 0)
        top = sorted(ops.items(), key=lambda t: -t[1])[:6]
        print(f"[{start:4d}-{i:4d}] samples {100*acc/tot:5.1f}%  inst {ex:.3e}  "
              + " ".join(f"{k}:{100*v/tot:.1f}" for k, v in top))
        acc = ex = 0.0
        start = i + 1
