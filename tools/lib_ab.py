"""A/B of two builds of the library over a degree range (best of reps, whole forward_device
call): python tools/lib_ab.py config l0 l1 libA.so libB.so [reps]"""
import os
import subprocess
import sys

if len(sys.argv) > 6 and sys.argv[6] == "--child":
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
    from pathlib import Path

    import paper_1207_5558_b200._lib as L

    L.LIB_PATH = Path(sys.argv[4]).resolve()
    import numpy as np
    import torch

    import paper_1207_5558_b200 as S
    from paper_1207_5558_b200 import configs as C

    cfg_i, l0, l1 = (int(x) for x in sys.argv[1:4])
    reps = int(sys.argv[5])
    f, h, cfg = C.make_inputs(cfg_i)
    dev = torch.device("cuda:0")
    fd = torch.from_numpy(np.ascontiguousarray(f).view(np.float64)).to(dev)
    hd = torch.from_numpy(np.ascontiguousarray(h).view(np.float64)).to(dev)
    dig = torch.zeros((S.coeff_count(cfg.L_g), 8), dtype=torch.float64, device=dev)
    with S.Plan(cfg.L_f, cfg.L_h, real_mode=cfg.real_mode, l_begin=l0, l_end=l1, materialize=False,
                ring_bytes=16 << 30) as p:
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
    print(f"{sys.argv[4]}: {best:.3f} ms")
else:
    cfg_i, l0, l1, a, b = sys.argv[1:6]
    reps = sys.argv[6] if len(sys.argv) > 6 else "3"
    for lib in (a, b, a, b):
        subprocess.run([sys.executable, __file__, cfg_i, l0, l1, lib, reps, "--child"], check=True)
