import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1207_5558_b200._lib as L
from pathlib import Path
import os; L.LIB_PATH = Path(os.environ.get('TRACE_LIB', '/root/repo/tools/libslsht_cuda_trace.so'))
import paper_1207_5558_b200 as S
from paper_1207_5558_b200 import configs as C
f, h, cfg = C.make_inputs(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, materialize=cfg.samples() * 16 < 40e9, ring_bytes=16384 << 20) as p:
    p.forward_digests(f, h)
