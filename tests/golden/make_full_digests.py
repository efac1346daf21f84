#!/usr/bin/env python3
"""Reference digests of EVERY emitted component of configs 3 and 4, and of the l <= 24 sample of
config 5, from the UNMODIFIED reference forward_fast (oracle/_ref, proj/src/transform.cpp:244-295)
with a digest sink ("Configs 3-4: digests of all components"; config 5: "digests
from the sampled CPU run").

Run where /root/reference exists (`make -C oracle ref` first):
    python tests/golden/make_full_digests.py [3] [4] [5]
Writes tests/golden/config{3,4,5}_digests.npz: digests[coeff_index(l, m)] (8 doubles, the
SLSHT_DIGEST definition of include/slsht_cuda.h), the f/h checksums of the regenerated inputs
and the reference's wall time. About 9 / 16 / 3 min on 8 cores.
"""
from __future__ import annotations

import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

OUT = Path(__file__).resolve().parent
LMAX = {3: -1, 4: -1, 5: 24}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    R = oracle.Reference()
    which = [int(x) for x in sys.argv[1:]] or [3, 4, 5]
    for index in which:
        t = time.time()
        f, h, cfg = C.make_inputs(index)
        dig, secs = R.forward_fast_digest(f, cfg.L_f, cfg.f_real, h, cfg.L_h, cfg.h_real,
                                          lmax=LMAX[index], threads=8)
        assert not np.isnan(dig).any()
        np.savez_compressed(OUT / f"config{index}_digests.npz", digests=dig,
                            lmax=np.array(LMAX[index]), f_sha256=np.array(sha(f)),
                            h_sha256=np.array(sha(h)), ref_seconds_8threads=np.array(secs))
        print(f"config{index}_digests.npz rows={dig.shape[0]} ref {secs:.1f}s "
              f"(total {time.time() - t:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
