"""One forward of a degree range of a config on cuda:0 (for ncu): python tools/profile_shard.py config l0 l1"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1207_5558_b200 as S  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

cfg_i, l0, l1 = (int(x) for x in sys.argv[1:4])
f, h, cfg = C.make_inputs(cfg_i)
with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, l_begin=l0, l_end=l1,
            materialize=False, ring_bytes=16384 << 20) as p:
    d = p.forward_digests(f, h)
    print("ok", cfg_i, l0, l1, p.computed_count)
