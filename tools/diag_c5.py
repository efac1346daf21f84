"""Diagnostics of the config-5 live-volume parity: the worst components (vs the reference's
component chain) and their modulated SHT (GPU vs reference). python tools/diag_c5.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle  # noqa: E402
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from test_gpu import live_sample  # noqa: E402

R = oracle.Reference()
f, h, cfg = C.make_inputs(5)
lm = live_sample(cfg, 200, 105)
with S.Plan(cfg.L_f, cfg.L_h, ring_bytes=4 << 30) as plan:
    _, vols = plan.forward_capture(f, h, lm)
exp = R.components_mt(f, cfg.L_f, h, cfg.L_h, lm)
gmax = float(np.max(np.abs(exp)))
rows = []
for i, k in enumerate(lm):
    d = float(np.max(np.abs(vols[k] - exp[i])))
    rows.append((d / gmax, float(np.max(np.abs(exp[i]))) / gmax, k))
rows.sort(reverse=True)
for r in rows[:10]:
    print("abs err / gmax %.2e  |g|/gmax %.2e  (l, m) %s" % r)
worst = [r[2] for r in rows[:4]]
mg = S.modulated_sht(S.SphCoeffs(cfg.L_f, f), worst, cfg.L_h)
for i, (l, m) in enumerate(worst):
    mr = R.modulated_sht(f, cfg.L_f, l, m, cfg.L_h)
    print((l, m), "mod: |mod| %.3e, max diff %.3e" % (np.max(np.abs(mr)), np.max(np.abs(mg[i] - mr))))
np.savez("gpurun_out/diag_c5.npz", worst=np.array(worst), mod_gpu=mg,
         mod_ref=np.stack([R.modulated_sht(f, cfg.L_f, l, m, cfg.L_h) for l, m in worst]))
