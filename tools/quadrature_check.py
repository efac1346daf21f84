"""The θ-quadrature evidence of DESIGN.md §2 (CPU only, ~20 s): the modulated SHT of a few
components (L_f = 100, L_h = 8) by
  * the reference (oracle/_ref modulated_sht: the S_{2L_g} rule, transform.cpp:189-220),
  * the engine's rule (x >= 0 half of the (L_g+1)-point Gauss-Legendre rule, I_0 / I_1 fold),
    emulated in double,
  * both rules in long double (the "truth"),
and the errors relative to max |mod|. python tools/quadrature_check.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle  # noqa: E402  (test infrastructure: this is a checker, not the product)

LD = np.longdouble
PI = LD("3.14159265358979323846264338327950288")


def lam_rows(m, lmax, c, s, T):
    am = abs(m)
    sect = np.ones_like(c) / np.sqrt(4 * (PI if T is LD else np.pi))
    for k in range(1, am + 1):
        sect = sect * (-s * np.sqrt(T(2 * k + 1) / T(2 * k)))
    if m < 0 and am & 1:
        sect = -sect
    rows = [sect]
    if lmax > am:
        rows.append(c * np.sqrt(T(2 * am + 3)) * sect)
    for l in range(am + 2, lmax + 1):
        a = np.sqrt(T(4 * l * l - 1) / T(l * l - am * am))
        b = np.sqrt(T((l - 1) ** 2 - am * am) / T(4 * (l - 1) ** 2 - 1))
        rows.append(a * (c * rows[-1] - b * rows[-2]))
    return rows


def gl_full(NG, T):
    x0, _ = np.polynomial.legendre.leggauss(NG)
    th = np.arccos(x0).astype(T)
    for _ in range(5):
        c, s = np.cos(th), np.sin(th)
        p0, p1 = np.ones_like(c), c.copy()
        for k in range(2, NG + 1):
            p0, p1 = p1, ((2 * k - 1) * c * p1 - (k - 1) * p0) / T(k)
        th = th - p1 * s / (NG * (c * p1 - p0))
    c, s = np.cos(th), np.sin(th)
    p0, p1 = np.ones_like(c), c.copy()
    for k in range(2, NG + 1):
        p0, p1 = p1, ((2 * k - 1) * c * p1 - (k - 1) * p0) / T(k)
    return c, s, 2 * s * s / (NG * (c * p1 - p0)) ** 2


def mw(N, T):
    t = np.arange(N + 1)
    th = (PI if T is LD else np.pi) * (2 * t.astype(T) + 1) / (2 * N + 1)
    w = np.zeros(N + 1, dtype=T)
    for k in range(-N, N + 1):
        if k % 2 == 0:
            w += (T(2) if k == 0 else T(2) / (1 - T(k) * k)) * np.cos(k * th)
    w = 2 * w / (2 * N + 1)
    w[N] *= 0.5
    return np.cos(th), np.sin(th), w


def modulated(f, L_f, L_h, l, m, c, s, w, T, half):
    ff = f.astype(np.clongdouble if T is LD else np.complex128)
    lm = lam_rows(m, l, c, s, T)[l - abs(m)]
    out = np.zeros((L_h + 1) ** 2, dtype=ff.dtype)
    for q in range(-L_h, L_h + 1):
        mu = m - q
        if abs(mu) > L_f:
            continue
        rows = lam_rows(mu, L_f, c, s, T)
        acc = [np.zeros_like(c, dtype=ff.dtype), np.zeros_like(c, dtype=ff.dtype)]
        for lp in range(abs(mu), L_f + 1):
            acc[(lp + mu) & 1] = acc[(lp + mu) & 1] + ff[lp * lp + lp + mu] * rows[lp - abs(mu)]
        hr = lam_rows(q, L_h, c, s, T)
        for p in range(abs(q), L_h + 1):
            I = 4 * np.pi * np.conj(acc[(l + m + p + q) & 1]) if half else \
                2 * np.pi * np.conj(acc[0] + acc[1])
            out[p * p + p + q] = np.sum(w * lm * hr[p - abs(q)] * I)
    return out


def main():
    rng = np.random.default_rng(3)
    L_f, L_h = 100, 8
    L_g = L_f + L_h
    f = np.concatenate([(rng.standard_normal(2 * p + 1) + 1j * rng.standard_normal(2 * p + 1))
                        / (p + 1) for p in range(L_f + 1)])
    R = oracle.Reference() if oracle.reference_available() else oracle.Oracle()
    cL, sL, wL = gl_full(L_g + 1, LD)
    keep = cL > 1e-12
    if (L_g + 1) % 2:  # the x = 0 node of an odd rule: half weight, exact zero
        keep[int(np.argmin(np.abs(cL)))] = True
    cD, sD, wD = (a[keep].astype(np.float64) for a in (cL, sL, wL))
    if (L_g + 1) % 2:
        j = int(np.argmin(np.abs(cD)))
        cD[j], sD[j], wD[j] = 0.0, 1.0, wD[j] * 0.5
    for l, m in [(L_g, -1), (L_g, 5), (L_g - 3, 40), (0, 0)]:
        truth = modulated(f, L_f, L_h, l, m, cL, sL, wL, LD, False)
        truth_mw = modulated(f, L_f, L_h, l, m, *mw(2 * L_g, LD), LD, False)
        eng = modulated(f, L_f, L_h, l, m, cD, sD, wD, np.float64, True)
        ref = R.modulated_sht(f, L_f, l, m, L_h)
        sc = float(np.max(np.abs(truth)))
        print(f"(l, m) = ({l:3d}, {m:3d})  |mod| {sc:.3e}   GL vs S_2Lg rule in long double "
              f"{float(np.max(np.abs(truth - truth_mw))) / sc:.1e}   engine rule (double) "
              f"{float(np.max(np.abs(eng - truth))) / sc:.1e}   reference (double) "
              f"{float(np.max(np.abs(ref - truth))) / sc:.1e}")


if __name__ == "__main__":
    main()
