"""Time one BASELINE config on cuda:0: step ms (events), stage split, digest check vs default.

usage: python tools/stage_times.py [config] [reps]
Env knobs of the engine (SLSHT_CUDA_LINES, SLSHT_CUDA_NO_WS, ...) select the coupling kernel;
the digests are compared against a second plan built with those knobs removed.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
f, h, cfg = C.make_inputs(cfg_i)
dev = torch.device("cuda:0")
fd = torch.from_numpy(np.ascontiguousarray(f).view(np.float64)).to(dev)
hd = torch.from_numpy(np.ascontiguousarray(h).view(np.float64)).to(dev)


def run(env_on):
    saved = {k: os.environ.pop(k) for k in list(os.environ) if k.startswith("SLSHT_CUDA_")
             and not env_on}
    try:
        with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, materialize=False) as p:
            dig = torch.zeros((S.coeff_count(cfg.L_g), 8), dtype=torch.float64, device=dev)
            st = torch.cuda.ExternalStream(p.stream_handle) if hasattr(p, "stream_handle") else None
            for _ in range(2):
                p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                                 digests_ptr=dig.data_ptr(), digests_on_device=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(reps):
                e0.record()
                p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                                 digests_ptr=dig.data_ptr(), digests_on_device=True)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            p.set_profiling(True)
            p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                             digests_ptr=dig.data_ptr(), digests_on_device=True)
            stages = p.stage_times()
            p.set_profiling(False)
            return float(np.median(ts)), stages, dig.cpu().numpy()
    finally:
        os.environ.update(saved)


ms, stages, d1 = run(True)
print(f"config {cfg_i}: step {ms:.3f} ms  stages {['%.3f' % x for x in stages]}  "
      f"samples/s {cfg.samples(cfg.L_g) / ms * 1e3:.4g}")
if any(k.startswith("SLSHT_CUDA_") for k in os.environ):
    ms0, stages0, d0 = run(False)
    scale = np.abs(d0).max(axis=0)
    rel = np.abs(d1 - d0).max(axis=0) / np.where(scale > 0, scale, 1)
    print(f"default: step {ms0:.3f} ms stages {['%.3f' % x for x in stages0]}")
    print("digest field max rel diff vs default:", ["%.2e" % x for x in rel])
