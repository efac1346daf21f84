"""Single-GPU proxy of the N-GPU strong-scaling step: time every degree shard of an N-way split
on cuda:0 (ranks share nothing during compute) and report max over shards.

usage: python tools/shard_time.py [config] [reps]
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
dig = torch.zeros((S.coeff_count(cfg.L_g), 8), dtype=torch.float64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
base = None
for world in (1, 2, 4, 8):
    worst = 0.0
    for r in range(world):
        l0, l1 = C.shard_degrees(cfg, world, r)
        mat = cfg.samples() * 16 / world < 40e9
        with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, l_begin=l0, l_end=l1,
                    materialize=mat, ring_bytes=16384 << 20) as p:
            for _ in range(2):
                p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                                 digests_ptr=dig.data_ptr(), digests_on_device=True)
            ts = []
            for _ in range(reps):
                flush.fill_(1)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                                 digests_ptr=dig.data_ptr(), digests_on_device=True)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            p.set_profiling(True)
            p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                             digests_ptr=dig.data_ptr(), digests_on_device=True)
            st = p.stage_times()
            p.set_profiling(False)
            if float(np.median(ts)) > worst:
                worst, wst, wr = float(np.median(ts)), st, (l0, l1, p.computed_count)
            
    base = base or worst
    print(f"config {cfg_i} N={world}: max shard step {worst:.3f} ms, "
          f"strong-scaling efficiency {base / (world * worst):.3f}; worst shard {wr} stages "
          f"{['%.3f' % x for x in wst]}")
