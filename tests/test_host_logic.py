"""Host-side logic that needs no GPU: the BASELINE workloads, degree sharding, the alpha-axis
FFT plan (digit-reversed DIF, as built in slsht_cuda.cu) and the stored Slepian windows."""
from __future__ import annotations

import math

import numpy as np
import pytest

from paper_1207_5558_b200 import configs as C


@pytest.mark.parametrize("index,samples,fps", [(1, 4.372e6, 132.9), (2, 3.892e8, 96.9),
                                               (3, 1.164e10, 138.4), (4, 1.731e10, 264.0),
                                               (5, 1.283e12, 439.9)])
def test_workload_sizes_match_survey(index, samples, fps):
    cfg = C.CONFIGS[index]
    assert abs(cfg.samples() / samples - 1) < 1e-3
    assert abs(cfg.flops_per_sample() / fps - 1) < 2e-3


@pytest.mark.parametrize("index", [1, 2, 3, 5])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_degree_shards_cover_and_balance(index, world):
    cfg = C.CONFIGS[index]
    bounds = [C.shard_degrees(cfg, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == cfg.L_g + 1
    for (a0, a1), (b0, b1) in zip(bounds, bounds[1:]):
        assert a1 == b0
    w = lambda l: (l + 1) if cfg.real_mode else (2 * l + 1)
    loads = [sum(w(l) for l in range(a, b)) for a, b in bounds]
    assert max(loads) - min(loads) <= 2 * w(cfg.L_g)


@pytest.mark.parametrize("index", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_engine_shard_rule_equals_host_rule(index, world):
    """slsht_cuda_shard_bounds (the multi-GPU plan's split, C ABI, host only) is the same rule as
    configs.shard_degrees, which bench.py's ranks use."""
    import paper_1207_5558_b200 as S

    cfg = C.CONFIGS[index]
    eng = S.shard_bounds(0, cfg.L_g + 1, cfg.real_mode, world)
    host = [C.shard_degrees(cfg, world, r)[0] for r in range(world)] + [cfg.L_g + 1]
    assert eng == host


def test_config5_shards_match_survey_boundaries():
    cfg = C.CONFIGS[5]
    got = [C.shard_degrees(cfg, 8, r)[0] for r in range(8)] + [cfg.L_g + 1]
    survey = [0, 384, 543, 666, 769, 860, 942, 1018, 1089]
    assert max(abs(a - b) for a, b in zip(got, survey)) <= 2


def fft_plan(n):
    fac, x, p = [], n, 3
    while x > 1:
        while x % p == 0:
            fac.append(p)
            x //= p
        p += 2
    perm = np.zeros(n, int)
    for pos in range(n):
        rem, freq, mult, mm = pos, 0, 1, n
        for r in fac:
            mp = mm // r
            k = rem // mp
            rem %= mp
            freq += k * mult
            mult *= r
            mm = mp
        perm[freq] = pos
    return fac, perm


def dif(x, n):
    fac, perm = fft_plan(n)
    x = x.astype(complex).copy()
    w = np.exp(-2j * np.pi * np.arange(n) / n)
    span = n
    for r in fac:
        mp = span // r
        F = np.exp(-2j * np.pi * np.outer(np.arange(r), np.arange(r)) / r)
        for blk in range(n // span):
            for t in range(mp):
                idx = blk * span + t + mp * np.arange(r)
                y = F @ x[idx]
                x[idx] = y * w[(t * np.arange(r) * (n // span)) % n]
        span = mp
    return x[perm]


@pytest.mark.parametrize("n", [1, 3, 5, 9, 15, 17, 25, 27, 33, 45, 49, 63, 65, 75, 81, 99, 105, 129])
def test_alpha_fft_plan_is_a_dft(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    assert np.max(np.abs(dif(x, n) - np.fft.fft(x))) < 1e-12 * n


def test_q_mod_n_rows_give_the_reference_alpha_sum():
    # g[a] = sum_q e^{-i q alpha_a} T_q (transform.cpp:81-85,111-122) == DFT of rows q mod n
    L = 7
    n = 2 * L + 1
    rng = np.random.default_rng(1)
    T = rng.standard_normal(n) + 1j * rng.standard_normal(n)  # index q + L
    q = np.arange(-L, L + 1)
    a = np.arange(n)
    ref = np.exp(-2j * np.pi * np.outer(a, q) / n) @ T
    rows = np.zeros(n, complex)
    rows[q % n] = T
    assert np.max(np.abs(np.fft.fft(rows) - ref)) < 1e-12


@pytest.mark.parametrize("name,L,lam", [("window_cfg2", 16, 0.999933), ("window_cfg3", 32, 0.966555),
                                        ("window_cfg5", 64, 0.982500)])
def test_stored_windows(name, L, lam):
    h = C.load_window(name)
    assert h.size == (L + 1) ** 2
    assert abs(np.linalg.norm(h) - 1.0) < 1e-10  # unit energy (window.cpp:176-189)
    assert abs(h[0].imag) < 1e-15 and h[0].real > 0
    for l in range(L + 1):  # conjugate-symmetric (real-valued window)
        for m in range(1, l + 1):
            assert abs(h[l * l + l - m] - (-1) ** m * np.conj(h[l * l + l + m])) < 1e-12


def test_real_inputs_are_conjugate_symmetric():
    for index in (2, 3):
        f, h, cfg = C.make_inputs(index)
        L = cfg.L_f
        l = np.repeat(np.arange(L + 1), np.arange(L + 1))
        m = np.concatenate([np.arange(1, k + 1) for k in range(L + 1)])
        assert np.max(np.abs(f[l * l + l - m] - (-1.0) ** m * np.conj(f[l * l + l + m]))) == 0.0
