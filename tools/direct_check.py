"""Cross-engine check at a BASELINE config: the device direct engine (forward_direct) at `ncells`
seeded cells against full volumes of the fast engine for a few components.
usage: python tools/direct_check.py config ncells"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

cfg_i, ncells = int(sys.argv[1]), int(sys.argv[2])
f, h, cfg = C.make_inputs(cfg_i)
rng = np.random.default_rng(cfg_i)
cells = np.sort(rng.choice(cfg.volume, min(ncells, cfg.volume), replace=False)).astype(np.int64)
L_g = cfg.L_g
lm = [(0, 0), (L_g // 3, L_g // 5), (L_g // 2, -(L_g // 2)), (L_g, L_g), (L_g, -L_g), (L_g - 1, 0)]
fs, hs = S.SphCoeffs(cfg.L_f, f), S.SphCoeffs(cfg.L_h, h)
S.forward_direct(S.SphCoeffs(2, f[:9]), S.SphCoeffs(1, h[:4]))  # CUDA/cuBLAS start-up
t = time.perf_counter()
direct = S.forward_direct(fs, hs, cells=cells)
dt = time.perf_counter() - t
with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, ring_bytes=4 << 30) as p:
    _, vols = p.forward_capture(f, h, lm)
scale = max(np.abs(vols[k]).max() for k in lm)
err = max(np.max(np.abs(direct[S.coeff_index(l, m)] - vols[(l, m)].reshape(-1)[cells])) for (l, m) in lm)
print(f"config {cfg_i}: direct engine, {len(cells)} cells x {direct.shape[0]} components in {dt:.2f} s "
      f"(sphere band {L_g}); max |direct - fast| / max |g| over {len(lm)} components = {err / scale:.2e}")
