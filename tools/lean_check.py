"""k_qfft_lean (SLSHT_CUDA_QFFT_LEAN=<CTAs per SM>) against k_qfft over a degree range: time per
call and the largest digest difference.  python tools/lean_check.py config l0 l1 [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

cfg_i, l0, l1 = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
f, h, cfg = C.make_inputs(cfg_i)
dev = torch.device("cuda:0")
fd = torch.from_numpy(np.ascontiguousarray(f).view(np.float64)).to(dev)
hd = torch.from_numpy(np.ascontiguousarray(h).view(np.float64)).to(dev)
ring = int(os.environ.get("RING_MB", "16384")) << 20


def run():
    dig = torch.zeros((S.coeff_count(cfg.L_g), 8), dtype=torch.float64, device=dev)
    with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, l_begin=l0, l_end=l1,
                materialize=False, ring_bytes=ring) as p:
        best = 1e30
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                             digests_ptr=dig.data_ptr(), digests_on_device=True)
            torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best, p.computed_count, dig.cpu().numpy()


os.environ["SLSHT_CUDA_QFFT_LEAN"] = "0"
ms0, comps, d0 = run()
print(f"config {cfg_i} l in [{l0},{l1}): {comps} comps; k_qfft {ms0:.3f} ms", flush=True)
r0, r1 = l0 * l0, l1 * l1
for mb in os.environ.get("LEAN", "4,6,8").split(","):
    os.environ["SLSHT_CUDA_QFFT_LEAN"] = mb
    ms, _, d1 = run()
    a, b = d0[r0:r1], d1[r0:r1]
    rel = float(np.max(np.abs(a - b) / np.maximum(np.max(np.abs(a), axis=0, keepdims=True), 1e-300)))
    print(f"  k_qfft_lean at {mb} CTAs per SM: {ms:.3f} ms ({ms / ms0:.3f}x), max column-relative "
          f"digest difference {rel:.2e}", flush=True)
