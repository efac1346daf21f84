"""k_tpipe (SLSHT_CUDA_TP_PIPE=1) against the two-pass kernels over a degree range: time per
call and bitwise equality of the digests.  python tools/pipe_check.py config l0 l1 [reps]
Env: RING_MB (default 16384); SHAPES="ct,nqg,nslot,fb,lag;..." pipe shapes to try (0 = default)."""
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
KEYS = ["SLSHT_CUDA_TP_CT", "SLSHT_CUDA_TP_NQG", "SLSHT_CUDA_TP_NSLOT", "SLSHT_CUDA_TP_FB", "SLSHT_CUDA_TP_LAG"]


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
        return best, p.computed_count, dig.cpu().numpy()


os.environ["SLSHT_CUDA_TP_PIPE"] = "0"
ms0, comps, d0 = run()
print(f"config {cfg_i} l in [{l0},{l1}): {comps} comps; two-pass {ms0:.3f} ms", flush=True)
r0, r1 = l0 * l0, l1 * l1
os.environ["SLSHT_CUDA_TP_PIPE"] = "1"
for shape in os.environ.get("SHAPES", "0,0,0,0,0").split(";"):
    vals = [int(x) for x in shape.split(",")]
    for k, v in zip(KEYS, vals):
        if v:
            os.environ[k] = str(v)
        else:
            os.environ.pop(k, None)
    ms, _, d1 = run()
    print(f"  pipe ct,nqg,nslot,fb,lag={shape}: {ms:.3f} ms ({ms / ms0:.3f}x), digests bitwise equal: "
          f"{np.array_equal(d0[r0:r1], d1[r0:r1])}", flush=True)
