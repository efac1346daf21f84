#!/usr/bin/env python3
"""Solve the Slepian windows of BASELINE configs 2, 3 and 5 with the reference's own
eigenfunction_window (proj/src/window.cpp:126-198, via oracle/_ref) and store them in
paper_1207_5558_b200/data/. Run once in a container where /root/reference exists.

Regions: an ellipse with semi-major a and semi-minor b about the north pole
has its foci at theta_c = arccos(cos a / cos b) (spherical Pythagoras), window.hpp:8-17.
"""
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = ROOT / "paper_1207_5558_b200" / "data"


def focal(a_deg: float, b_deg: float) -> float:
    return math.acos(math.cos(math.radians(a_deg)) / math.cos(math.radians(b_deg)))


def main() -> None:
    R = oracle.Reference()
    OUT.mkdir(parents=True, exist_ok=True)
    jobs = [
        ("window_cfg2", math.radians(20.0), math.radians(30.0), 16),
        ("window_cfg3", focal(15.0, 5.0), math.radians(15.0), 32),
        ("window_cfg5", focal(10.0, 3.0), math.radians(10.0), 64),
    ]
    for name, tc, a, L in jobs:
        t = time.time()
        h, lam = R.eigenfunction_window(tc, a, L, 4)
        np.save(OUT / f"{name}.npy", h)
        print(f"{name}: L={L} theta_c={tc:.6f} a={a:.6f} lambda={lam:.6f} "
              f"h00={h[0]:.6f} ({time.time() - t:.1f}s)")


if __name__ == "__main__":
    main()
