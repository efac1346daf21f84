"""profiles/traffic_config<k>.json from the raw ncu CSV of tools/refresh_profiles_r02.sh (DRAM
bytes and duration of every coupling launch of one step, summed per kernel):
python tools/traffic_json.py raw.csv config > profiles/traffic_config<k>.json"""
import csv
import io
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from paper_1207_5558_b200 import configs as C  # noqa: E402

raw = open(sys.argv[1]).read().splitlines()
cfg_i = int(sys.argv[2])
rows = list(csv.reader(io.StringIO("\n".join(l for l in raw if not l.startswith("==")))))
h = rows[0]
iK, iM, iV, iU, iI = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
agg = {}
for r in rows[1:]:
    name = r[iK].split("<")[0].split("(")[0].replace("void ", "").strip().split("::")[-1]
    v = float(r[iV].replace(",", ""))
    unit = r[iU]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
             "ms": 1.0, "msecond": 1.0}.get(unit, 1)
    d = agg.setdefault(name, {"ids": set(), "dram_bytes_read": 0.0, "dram_bytes_write": 0.0, "ncu_ms_per_step": 0.0})
    d["ids"].add(r[iI])
    if r[iM] == "dram__bytes_read.sum":
        d["dram_bytes_read"] += v * scale
    elif r[iM] == "dram__bytes_write.sum":
        d["dram_bytes_write"] += v * scale
    elif r[iM] == "gpu__time_duration.sum":
        d["ncu_ms_per_step"] += v * scale
cfg = C.CONFIGS[cfg_i] if hasattr(C, "CONFIGS") else C.make_inputs(cfg_i)[2]
out = {"config": cfg_i,
       "source": ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                  "--clock-control none over every launch of one forward_device step with the bench's "
                  "plan (tools/one_step.py; tools/refresh_profiles_r02.sh; tools/traffic_json.py); "
                  "per-launch values summed over the step's chunks"),
       "algorithmic_bytes_per_step": int(cfg.samples() * 16)}
for name, d in agg.items():
    out[name] = {"launches_per_step": len(d["ids"]), "dram_bytes_read": d["dram_bytes_read"],
                 "dram_bytes_write": d["dram_bytes_write"],
                 "dram_bytes_per_step": d["dram_bytes_read"] + d["dram_bytes_write"],
                 "ncu_ms_per_step": d["ncu_ms_per_step"]}
print(json.dumps(out, indent=1))
