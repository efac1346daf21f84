"""Device time of one whole forward_device call over a degree range (no per-stage events, so the
overlapped two-pass schedule runs as in bench.py): python tools/range_time.py config l0 l1 [reps]
Env: RING_MB (default 16384); the digests of the first call are compared with those of a plan
built with SLSHT_CUDA_TP_OVERLAP=0 when CHECK=1."""
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
        p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                         digests_ptr=dig.data_ptr(), digests_on_device=True)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                             digests_ptr=dig.data_ptr(), digests_on_device=True)
            torch.cuda.synchronize()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best, p.emitted_count * p.volume_elems, p.computed_count, dig.cpu().numpy()


ms, samples, comps, d1 = run()
print(f"config {cfg_i} l in [{l0},{l1}): {comps} comps, {ms:.3f} ms, {samples / ms * 1e3:.4g} samples/s"
      f" (env: {' '.join(k + '=' + v for k, v in os.environ.items() if k.startswith('SLSHT_CUDA'))})")
if os.environ.get("CHECK") == "1":
    os.environ["SLSHT_CUDA_TP_OVERLAP"] = "0"
    _, _, _, d2 = run()
    r0, r1 = l0 * l0, l1 * l1
    print("digests bitwise equal to the serial schedule:", np.array_equal(d1[r0:r1], d2[r0:r1]))
