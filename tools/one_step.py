"""One forward_device step of a BASELINE config with bench.py's plan (24 GiB ring, inputs in
HBM), for ncu: python tools/one_step.py [config] [repeats]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

cfg_i = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
f, h, cfg = C.make_inputs(cfg_i)
dev = torch.device("cuda:0")
fd = torch.from_numpy(np.ascontiguousarray(f).view(np.float64)).to(dev)
hd = torch.from_numpy(np.ascontiguousarray(h).view(np.float64)).to(dev)
dig = torch.zeros((S.coeff_count(cfg.L_g), S.DIGEST_WIDTH), dtype=torch.float64, device=dev)
materialize = cfg.samples() * 16 < 40e9
with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, emit_negative_m=True,
            materialize=materialize, ring_bytes=24576 << 20) as p:
    for _ in range(reps):
        p.forward_device(fd.data_ptr(), hd.data_ptr(), inputs_on_device=True,
                         digests_ptr=dig.data_ptr(), digests_on_device=True)
    torch.cuda.synchronize()
    print("ok", cfg_i, p.computed_count, "launches per step", p.launch_count)
