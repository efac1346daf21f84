"""The CPU oracle (oracle/slsht_oracle.c) pinned against the reference: the committed golden
fixtures (generated from the unmodified reference by tests/golden/make_golden.py) and, where
oracle/_ref is built, the live reference library. Mirrors the reference's own pins in
proj/tests/test_transform.cpp, test_wigner.cpp, test_harmonics.cpp and test_grids.cpp."""
from __future__ import annotations

import hashlib
import math

import numpy as np
import pytest

from conftest import rel_err


def coeff_count(L):
    return (L + 1) ** 2


def coeff_index(l, m):
    return l * l + l + m


# --------------------------------------------------------------------------- Delta tables
def test_delta_tables_match_reference_bitwise(oracle_lib, gold):
    t = gold("tables")
    assert np.array_equal(oracle_lib.delta_tables(16), t["delta16"])
    d64 = oracle_lib.delta_tables(64)
    assert hashlib.sha256(d64.tobytes()).hexdigest() == str(t["delta64_sha256"])


def test_delta_seeds(oracle_lib):
    # test_wigner.cpp:44-55
    d1 = oracle_lib.delta_tables(1)
    at = lambda q, qp: d1[1 + (q + 1) * 3 + (qp + 1)]
    assert d1[0] == 1.0
    assert abs(at(0, 0)) < 1e-15
    assert abs(at(1, 1) - 0.5) < 1e-15
    assert abs(at(1, 0) + 1 / math.sqrt(2)) < 1e-15
    assert abs(at(0, 1) - 1 / math.sqrt(2)) < 1e-15
    assert abs(at(-1, 0) - 1 / math.sqrt(2)) < 1e-15
    assert abs(at(1, -1) - 0.5) < 1e-15


def _levels(d, L):
    off = 0
    for p in range(L + 1):
        w = 2 * p + 1
        yield p, d[off:off + w * w].reshape(w, w)
        off += w * w


def test_delta_symmetries_and_unit_rows(oracle_lib):
    # test_wigner.cpp:57-83
    for p, lev in _levels(oracle_lib.delta_tables(64), 64):
        q = np.arange(-p, p + 1)
        sign = np.where((q[:, None] - q[None, :]) % 2 == 0, 1.0, -1.0)
        if p <= 32:
            assert np.max(np.abs(lev - sign * lev.T)) < 1e-12
            assert np.max(np.abs(lev - lev[::-1, ::-1].T)) < 1e-12
        assert np.max(np.abs((lev ** 2).sum(1) - 1.0)) < 1e-12


# --------------------------------------------------------------------------- grids, Legendre
def test_theta_and_beta_weights_match_reference(oracle_lib, gold):
    t = gold("tables")
    for N in (4, 80, 288):
        assert np.max(np.abs(oracle_lib.theta_weights(N) - t[f"theta_weights_{N}"])) < 1e-15
    for L in (2, 8, 16, 64):
        assert np.max(np.abs(oracle_lib.beta_weights(L) - t[f"beta_weights_{L}"])) < 1e-12


def test_theta_weights_integrate_sin(oracle_lib):
    # test_grids.cpp:115-129 analogue: sum_t v_t u(theta_t) = int_0^pi u sin for even trig u
    N = 40
    w = oracle_lib.theta_weights(N)
    th = math.pi * (2 * np.arange(N + 1) + 1) / (2 * N + 1)
    assert abs(w.sum() - 2.0) < 1e-13
    assert abs((w * np.cos(2 * th)).sum() - (-2.0 / 3.0)) < 1e-13


def test_legendre_rows_match_reference(oracle_lib, gold):
    t = gold("tables")
    th = t["thetas81"]
    for m, key in ((0, "leg_m0"), (3, "leg_m3"), (-5, "leg_mneg5"), (40, "leg_m40")):
        assert rel_err(oracle_lib.legendre_rows(m, 40, th), t[key])[0] < 1e-14


def test_eval_ylm_pinned_value(oracle_lib):
    # test_harmonics.cpp:92-93: Y_1^1(pi/2, 0) = -sqrt(3/(8 pi))
    rows = oracle_lib.legendre_rows(1, 1, np.array([math.pi / 2]))
    assert abs(rows[0, 0] + math.sqrt(3 / (8 * math.pi))) < 1e-15


# --------------------------------------------------------------------------- transform path
SMALL = ["c32", "r43", "c63", "r53_noneg", "r43_full", "trivial", "c24", "c30"]


@pytest.mark.parametrize("name", SMALL)
def test_forward_small_cases_match_reference(oracle_lib, gold, name):
    g = gold("small")
    L_f, L_h, fr, hr, lmax, urs, emit = (int(x) for x in g[f"{name}__meta"])
    vols = oracle_lib.forward_fast(g[f"{name}__f"], L_f, fr, g[f"{name}__h"], L_h, hr, lmax=lmax,
                                   use_real_symmetry=urs, emit_negative_m=emit)
    keys = [tuple(k) for k in g[f"{name}__lm"]]
    assert sorted(vols) == keys  # every component exactly once (test_transform.cpp:331-348)
    got = np.stack([vols[k] for k in keys])
    assert rel_err(got, g[f"{name}__vol"])[0] < 1e-13


@pytest.mark.parametrize("name", SMALL)
def test_modulated_sht_matches_reference(oracle_lib, gold, name):
    g = gold("small")
    L_f, L_h = int(g[f"{name}__meta"][0]), int(g[f"{name}__meta"][1])
    for (l, m), ref in zip(g[f"{name}__mod_lm"], g[f"{name}__mod"]):
        got = oracle_lib.modulated_sht(g[f"{name}__f"], L_f, int(l), int(m), L_h)
        assert np.max(np.abs(got - ref)) < 1e-14


def test_trivial_distribution_is_one_over_sqrt_4pi(oracle_lib):
    # test_transform.cpp:178-194
    vols = oracle_lib.forward_fast(np.ones(1), 0, False, np.ones(1), 0, False)
    assert abs(vols[(0, 0)].ravel()[0] - 1 / math.sqrt(4 * math.pi)) < 1e-12


def test_modulated_constant_signal_is_shifted_delta(oracle_lib):
    # test_transform.cpp:70-92
    f = np.zeros(1, np.complex128)
    f[0] = 1.0
    for l in (0, 2, 4):
        for m in range(-l, l + 1):
            mod = oracle_lib.modulated_sht(f, 0, l, m, 4)
            exp = np.zeros(coeff_count(4))
            exp[coeff_index(l, m)] = 1 / math.sqrt(4 * math.pi)
            assert np.max(np.abs(mod - exp)) < 1e-13


def test_config1_digests_match_reference(oracle_lib, gold):
    g = gold("config1")
    L_f, L_h, fr, hr = (int(x) for x in g["meta"])
    dig = np.full((coeff_count(L_f + L_h), 8), np.nan)

    def sink(l, m, v):
        dig[coeff_index(l, m)] = oracle_lib.digest(L_h, v)

    oracle_lib.forward_fast(g["f"], L_f, fr, g["h"], L_h, hr, on_component=sink)
    ref = g["digests"]
    assert np.max(np.abs(dig[:, 0] - ref[:, 0]) / ref[:, 0]) < 1e-12
    assert rel_err(dig[:, 2:8], ref[:, 2:8])[0] < 1e-12
    for (l, m), vol in zip(g["full_lm"], g["full_vol"]):
        pass  # full volumes are compared through the components below
    vols = oracle_lib.components(g["f"], L_f, g["h"], L_h, [tuple(map(int, k)) for k in g["full_lm"]])
    got = np.stack([vols[tuple(map(int, k))] for k in g["full_lm"]])
    assert rel_err(got, g["full_vol"])[0] < 1e-13


@pytest.mark.parametrize("index", [2, 3])
def test_sampled_components_match_reference(oracle_lib, gold, index):
    from paper_1207_5558_b200 import configs as C

    g = gold(f"config{index}")
    f, h, cfg = C.make_inputs(index)
    assert hashlib.sha256(f.tobytes()).hexdigest() == str(g["f_sha256"])
    keys = [tuple(map(int, k)) for k in g["sample_lm"]]
    vols = oracle_lib.components(f, cfg.L_f, h, cfg.L_h, keys)
    for i, k in enumerate(keys):
        got = vols[k].reshape(-1)[g["sample_idx"][i]]
        assert rel_err(got, g["sample_vals"][i])[0] < 1e-11, k


def test_roundtrip_reference_and_oracle(oracle_lib, gold):
    # acceptance_main.cpp:87-107: inverse(forward_fast(f)) == f  (< 1e-9; we pin 1e-10)
    g = gold("roundtrip")
    h = g["h"]
    h00 = h[0]
    scale = math.sqrt(16 * math.pi ** 3)
    for L_f in (18, 32):
        f = g[f"f{L_f}"]
        assert np.max(np.abs(g[f"frec{L_f}"] - f)) < 1e-10
        if L_f != 18:
            continue
        rec = np.zeros_like(f)

        def sink(l, m, v):
            d = oracle_lib.digest(18, v)
            rec[coeff_index(l, m)] = complex(d[6], d[7]) / (scale * h00)
            if m > 0:  # InverseAccumulator::finish fills m < 0 by symmetry (transform.cpp:530-533)
                rec[coeff_index(l, -m)] = (-1) ** m * np.conj(rec[coeff_index(l, m)])

        oracle_lib.forward_fast(f, L_f, True, h, 18, True, lmax=L_f, emit_negative_m=False,
                                on_component=sink)
        assert np.max(np.abs(rec - f)) < 1e-10


def test_oracle_validation_errors(oracle_lib):
    with pytest.raises(ValueError):
        oracle_lib.forward_fast(np.ones(4), 1, False, np.ones(1), 0, False, lmax=5)
    with pytest.raises(ValueError):
        oracle_lib.modulated_sht(np.ones(4), 1, 1, 2, 1)


def test_oracle_matches_live_reference(oracle_lib, reference_lib):
    rng = np.random.default_rng(5)
    for L_f, L_h, real in ((5, 2, False), (7, 4, True), (9, 1, False)):
        if real:
            f = reference_lib.random_coeffs(L_f, 9, True)
            h, _ = reference_lib.eigenfunction_window(0.2, 0.5, L_h, 4)
        else:
            f = rng.standard_normal(coeff_count(L_f)) + 1j * rng.standard_normal(coeff_count(L_f))
            h = rng.standard_normal(coeff_count(L_h)) + 1j * rng.standard_normal(coeff_count(L_h))
        a = oracle_lib.forward_fast(f, L_f, real, h, L_h, real)
        b = reference_lib.forward_fast(f, L_f, real, h, L_h, real, threads=3)
        assert sorted(a) == sorted(b)
        assert max(np.max(np.abs(a[k] - b[k])) for k in b) == 0.0  # bit-identical restatement


def test_gauss_legendre_half_rule_equals_reference_quadrature(oracle_lib):
    """The engine integrates the modulated SHT over theta with the x >= 0 half of the
    (L_g + 1)-point Gauss-Legendre rule instead of the reference's S_{2L_g}
    rule (transform.cpp:151-156, 206-219): both are exact for the integrand, so in long double
    they agree to roundoff, and in double the engine's rule is at least as accurate
    (tools/quadrature_check.py, CPU)."""
    import sys
    from pathlib import Path

    import numpy as np

    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
    import quadrature_check as Q

    LD = np.longdouble
    rng = np.random.default_rng(5)
    L_f, L_h = 40, 6
    L_g = L_f + L_h
    f = np.concatenate([(rng.standard_normal(2 * p + 1) + 1j * rng.standard_normal(2 * p + 1))
                        / (p + 1) for p in range(L_f + 1)])
    cL, sL, wL = Q.gl_full(L_g + 1, LD)
    keep = cL > 1e-12
    if (L_g + 1) % 2:
        keep[int(np.argmin(np.abs(cL)))] = True
    cD, sD, wD = (a[keep].astype(np.float64) for a in (cL, sL, wL))
    if (L_g + 1) % 2:
        j = int(np.argmin(np.abs(cD)))
        cD[j], sD[j], wD[j] = 0.0, 1.0, wD[j] * 0.5
    for l, m in [(L_g, -1), (L_g - 2, 7), (10, 3), (0, 0)]:
        truth = Q.modulated(f, L_f, L_h, l, m, cL, sL, wL, LD, False)
        truth_mw = Q.modulated(f, L_f, L_h, l, m, *Q.mw(2 * L_g, LD), LD, False)
        eng = Q.modulated(f, L_f, L_h, l, m, cD, sD, wD, np.float64, True)
        ref = oracle_lib.modulated_sht(f, L_f, l, m, L_h)
        sc = float(np.max(np.abs(truth)))
        assert float(np.max(np.abs(truth - truth_mw))) / sc < 1e-15  # both rules exact
        e_eng = float(np.max(np.abs(eng - truth))) / sc
        e_ref = float(np.max(np.abs(ref - truth))) / sc
        assert e_eng < 1e-13 and e_eng <= max(2 * e_ref, 1e-15), (l, m, e_eng, e_ref)
