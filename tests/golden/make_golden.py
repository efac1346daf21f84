#!/usr/bin/env python3
"""Generate the committed golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in a container where /root/reference exists (`make -C oracle ref` first):
    python tests/golden/make_golden.py
Every array here comes from the reference's own code path (forward_fast, the component-level
ModulatedSht / build_c_tensor / So3Evaluator chain of proj/src/cli.cpp:94-143, DeltaTables,
theta_weights, legendre_rows, InverseAccumulator, forward_direct); inputs are either stored or regenerated
deterministically by paper_1207_5558_b200.configs (their checksums are stored).
"""
from __future__ import annotations

import hashlib
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402
from paper_1207_5558_b200 import configs as C  # noqa: E402

OUT = Path(__file__).resolve().parent
R = oracle.Reference()
O = oracle.Oracle()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_complex(L: int, seed: int) -> np.ndarray:
    # the reference tests' random_complex_coeffs (test_transform.cpp:19-26) uses mt19937_64;
    # we only need seeded inputs, so numpy PCG64 uniform [-0.5, 0.5) is used instead
    rng = np.random.default_rng(seed)
    n = C.coeff_count(L)
    return (rng.random(n) - 0.5) + 1j * (rng.random(n) - 0.5)


def synthetic_window(L: int, seed: int) -> np.ndarray:
    # test_transform.cpp:28-36: random window with h00 += 1, unit energy
    h = random_complex(L, seed)
    h[0] += 1.0
    return h / np.linalg.norm(h)


def digest_many(L_h: int, vols: dict) -> tuple[np.ndarray, np.ndarray]:
    keys = sorted(vols)
    dig = np.array([O.digest(L_h, vols[k]) for k in keys])
    return np.array(keys, dtype=np.int64), dig


def strided(vol: np.ndarray, count: int = 2048) -> tuple[np.ndarray, np.ndarray]:
    flat = vol.reshape(-1)
    stride = max(1, flat.size // count)
    idx = np.arange(0, flat.size, stride, dtype=np.int64)
    return idx, flat[idx]


def make_tables() -> None:
    d16 = R.delta_tables(16)
    d64 = R.delta_tables(64)
    thetas81 = math.pi * (2 * np.arange(81) + 1) / 161.0
    leg = {m: R.legendre_rows(m, 40, thetas81) for m in (0, 3, -5, 40)}
    np.savez_compressed(
        OUT / "tables.npz",
        delta16=d16, delta64_sha256=np.array(sha(d64)), delta64_sample=d64[::97].copy(),
        theta_weights_4=R.theta_weights(4), theta_weights_80=R.theta_weights(80),
        theta_weights_288=R.theta_weights(288),
        beta_weights_2=R.beta_weights(2), beta_weights_8=R.beta_weights(8),
        beta_weights_16=R.beta_weights(16), beta_weights_64=R.beta_weights(64),
        thetas81=thetas81, leg_m0=leg[0], leg_m3=leg[3], leg_mneg5=leg[-5], leg_m40=leg[40])
    print("tables.npz")


SMALL = [
    # name, L_f, L_h, kind, lmax, use_real_symmetry, emit_negative_m
    ("c32", 3, 2, "complex", -1, True, True),
    ("r43", 4, 3, "real", -1, True, True),
    ("c63", 6, 3, "complex", -1, True, True),
    ("r53_noneg", 5, 3, "real", 5, True, False),
    ("r43_full", 4, 3, "real", -1, False, True),
    ("trivial", 0, 0, "one", -1, True, True),
    ("c24", 2, 4, "complex", -1, True, True),
    ("c30", 3, 0, "complex", -1, True, True),
]


def small_inputs(name, L_f, L_h, kind):
    if kind == "complex":
        seed = sum(map(ord, name))
        return random_complex(L_f, seed), synthetic_window(L_h, seed + 1), False, False
    if kind == "real":
        f = R.random_coeffs(L_f, 43, True)
        h, _ = R.eigenfunction_window(0.3, 0.7, L_h, 4)
        return f, h, True, True
    f = np.ones(1, np.complex128)
    return f, np.ones(1, np.complex128), False, False


def make_small() -> None:
    arrays = {}
    for name, L_f, L_h, kind, lmax, urs, emit in SMALL:
        f, h, fr, hr = small_inputs(name, L_f, L_h, kind)
        vols = R.forward_fast(f, L_f, fr, h, L_h, hr, lmax=lmax, threads=2,
                              use_real_symmetry=urs, emit_negative_m=emit)
        keys = sorted(vols)
        arrays[f"{name}__f"] = f
        arrays[f"{name}__h"] = h
        arrays[f"{name}__meta"] = np.array([L_f, L_h, int(fr), int(hr), lmax, int(urs), int(emit)])
        arrays[f"{name}__lm"] = np.array(keys, dtype=np.int64)
        arrays[f"{name}__vol"] = np.stack([vols[k] for k in keys])
        # modulated SHT of two components through the reference's free function
        ls = [(0, 0), (min(L_f + L_h, 3), min(L_f + L_h, 3) - 1)] if L_f + L_h > 0 else [(0, 0)]
        arrays[f"{name}__mod_lm"] = np.array(ls, dtype=np.int64)
        arrays[f"{name}__mod"] = np.stack([R.modulated_sht(f, L_f, l, m, L_h) for l, m in ls])
    np.savez_compressed(OUT / "small.npz", **arrays)
    print("small.npz", len(SMALL), "cases")


def make_config(index: int, full_digests: bool, sample_lm, n_full: int = 0) -> None:
    t = time.time()
    f, h, cfg = C.make_inputs(index)
    arrays = {"f_sha256": np.array(sha(f)), "h": h, "meta": np.array(
        [cfg.L_f, cfg.L_h, int(cfg.f_real), int(cfg.h_real)])}
    if index <= 2:
        arrays["f"] = f
    if full_digests:
        dig, secs = R.forward_fast_digest(f, cfg.L_f, cfg.f_real, h, cfg.L_h, cfg.h_real,
                                          threads=8)
        arrays["digests"] = dig
        arrays["ref_seconds_8threads"] = np.array(secs)
    vols = R.components(f, cfg.L_f, h, cfg.L_h, sample_lm)
    keys = sorted(vols)
    arrays["sample_lm"] = np.array(keys, dtype=np.int64)
    arrays["sample_digest"] = np.array([O.digest(cfg.L_h, vols[k]) for k in keys])
    idx, vals = zip(*(strided(vols[k]) for k in keys))
    arrays["sample_idx"] = np.stack(idx)
    arrays["sample_vals"] = np.stack(vals)
    if n_full:
        arrays["full_lm"] = np.array(keys[:n_full], dtype=np.int64)
        arrays["full_vol"] = np.stack([vols[k] for k in keys[:n_full]])
    np.savez_compressed(OUT / f"config{index}.npz", **arrays)
    print(f"config{index}.npz ({time.time() - t:.1f}s)")


def make_roundtrip() -> None:
    # acceptance criterion 1 shape (acceptance_main.cpp:87-107): L_h = 18 eigenfunction window
    # on R(pi/6, pi/6 + pi/240), random real f
    h, lam = R.eigenfunction_window(math.pi / 6.0, math.pi / 6.0 + math.pi / 240.0, 18, 4)
    arrays = {"h": h, "lambda": np.array(lam)}
    for L_f in (18, 32, 48, 64):  # acceptance_main.cpp:87-107
        f = R.random_coeffs(L_f, 100 + L_f, True)
        arrays[f"f{L_f}"] = f
        arrays[f"frec{L_f}"] = R.roundtrip(f, L_f, True, h, 18, True)
    np.savez_compressed(OUT / "roundtrip.npz", **arrays)
    print("roundtrip.npz")


def make_direct() -> None:
    # the reference's independent direct engine forward_direct (transform.cpp:313-388): full
    # distributions of small cases (lmax = L_g, lmax < L_g, lmax > L_g: sphere band lmax)
    arrays = {}
    for name, L_f, L_h, lmax, seed in (("a", 6, 3, -1, 61), ("b", 9, 4, 5, 62), ("c", 3, 2, 7, 63)):
        f = random_complex(L_f, seed)
        h = synthetic_window(L_h, seed + 100)
        arrays[f"{name}_f"] = f
        arrays[f"{name}_h"] = h
        arrays[f"{name}_meta"] = np.array([L_f, L_h, lmax])
        arrays[f"{name}_g"] = R.forward_direct(f, L_f, h, L_h, lmax)
    np.savez_compressed(OUT / "direct.npz", **arrays)
    print("direct.npz")


def main() -> None:
    which = set(sys.argv[1:]) or {"tables", "small", "1", "2", "3", "4", "5", "rt", "direct"}
    if "direct" in which:
        make_direct()
    if "tables" in which:
        make_tables()
    if "small" in which:
        make_small()
    if "1" in which:
        make_config(1, True, [(0, 0), (1, -1), (8, 3), (17, -9), (25, 25), (40, 0), (40, -40),
                              (33, 12)], n_full=8)
    if "2" in which:
        make_config(2, True, [(0, 0), (5, 2), (16, -7), (77, 31), (144, 144), (144, 0),
                              (120, -61), (3, -3)], n_full=4)
    if "3" in which:
        make_config(3, False, [(0, 0), (31, 4), (200, 100), (288, 288), (288, 0), (150, -75)])
    if "4" in which:
        make_config(4, False, [(0, 0), (24, -20), (300, 150), (536, 536), (536, -536), (411, 0)])
    if "5" in which:
        make_config(5, False, [(0, 0), (64, 10), (700, -350), (1088, 1088), (1088, -1)])
    if "rt" in which:
        make_roundtrip()


if __name__ == "__main__":
    main()
