"""Host-sink throughput of the drop-in's product (bench.py's host_sink leg) for a thread sweep:
python tools/host_sink_time.py config [threads ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import bench  # noqa: E402
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

cfg_i = int(sys.argv[1])
f, h, cfg = C.make_inputs(cfg_i)
for t in sys.argv[2:] or ["0"]:
    if int(t):
        os.environ["SLSHT_CUDA_HOST_THREADS"] = t
    else:
        os.environ.pop("SLSHT_CUDA_HOST_THREADS", None)
    r = bench.host_sink_sample(S, C, cfg, f, h, 0)
    print(json.dumps({"config": cfg_i, "threads": r["host_copy_threads"], "gb_per_s": round(r["gb_per_s"], 2),
                      "samples_per_s": r["value"], "components": r["components"]}), flush=True)
