"""Run `reps` forward calls of one BASELINE config on cuda:0 (for ncu / compute-sanitizer)."""
import argparse
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--lmax", type=int, default=-1)
ap.add_argument("--ring-mb", type=int, default=2048)
a = ap.parse_args()
f, h, cfg = C.make_inputs(a.config)
lmax = cfg.L_g if a.lmax < 0 else a.lmax
mat = cfg.samples(lmax) * 16 < 40e9
with S.Plan(cfg.L_f, cfg.L_h, lmax=lmax, real_mode=cfg.real_mode, materialize=mat,
            ring_bytes=a.ring_mb << 20) as plan:
    for _ in range(a.reps):
        d = plan.forward_digests(f, h)
    print("ok", cfg.index, lmax, plan.computed_count, plan.emitted_count, np.nansum(d[:, 0]))
