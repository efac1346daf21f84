"""Stage split of one degree range of a config on cuda:0 (a bounded sample of the big configs).
usage: python tools/shard_stage.py config l0 l1 [reps]"""
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
dig = torch.zeros((S.coeff_count(cfg.L_g), 8), dtype=torch.float64, device=dev)
with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, l_begin=l0, l_end=l1,
            materialize=False, ring_bytes=int(os.environ.get("RING_MB", "16384")) << 20) as p:
    p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                     digests_ptr=dig.data_ptr(), digests_on_device=True)
    p.set_profiling(True)
    best = None
    for _ in range(reps):
        p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                         digests_ptr=dig.data_ptr(), digests_on_device=True)
        st = p.stage_times()
        best = st if best is None or sum(st) < sum(best) else best
    samples = p.emitted_count * p.volume_elems
    print(f"config {cfg_i} l in [{l0},{l1}): {p.computed_count} comps, stages "
          f"{['%.3f' % x for x in best]} ms, {samples / sum(best) * 1e3:.4g} samples/s")
