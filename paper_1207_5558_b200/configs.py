"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: the paper's planetary topographies are replaced by synthetic
fields of the stated spectra. All generators are deterministic (numpy PCG64 with fixed
seeds). The Slepian windows (configs 2, 3, 5) were solved once with the reference's own
eigenfunction_window (proj/src/window.cpp:126-198) by tools/make_windows.py and are stored in
data/ (the L_h = 64 solve takes ~47 s on a CPU core).

This module is input preparation for tests and bench.py, not part of the timed hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from pathlib import Path

import numpy as np

DATA = Path(__file__).resolve().parent / "data"


def coeff_count(L: int) -> int:
    return (L + 1) * (L + 1)


def coeff_index(l: int, m: int) -> int:
    return l * l + l + m


@dataclass(frozen=True)
class Config:
    index: int
    L_f: int
    L_h: int
    f_real: bool
    h_real: bool
    description: str

    @property
    def L_g(self) -> int:
        return self.L_f + self.L_h

    @property
    def real_mode(self) -> bool:
        return self.f_real and self.h_real

    @property
    def n(self) -> int:
        return 2 * self.L_h + 1

    @property
    def volume(self) -> int:
        return self.n * self.n * (self.L_h + 1)

    def computed(self, lmax: int | None = None) -> int:
        lm = self.L_g if lmax is None else lmax
        return (lm + 1) * (lm + 2) // 2 if self.real_mode else (lm + 1) ** 2

    def emitted(self, lmax: int | None = None) -> int:
        lm = self.L_g if lmax is None else lmax
        return (lm + 1) ** 2

    def samples(self, lmax: int | None = None) -> int:
        return self.emitted(lmax) * self.volume

    def flops_per_component(self) -> float:
        """Canonical FP64 work per computed component."""
        Lh, n, nb = self.L_h, self.n, self.L_h + 1
        n_theta = 2 * self.L_g + 1
        f_mod = n_theta * (4 * nb * nb + 3 * n) + 5 * n_theta
        f_c = sum(8 * (2 * p + 1) ** 3 + 4 * (2 * p + 1) ** 2 for p in range(Lh + 1))
        f_fft = 5 * n * math.log2(n) * (n * n + 2 * nb * n) if n > 1 else 0.0
        return float(f_mod + f_c + f_fft)

    def flops_per_sample(self) -> float:
        return self.flops_per_component() * self.computed() / self.samples()


CONFIGS = {
    1: Config(1, 32, 8, False, False, "complex CN(0,1) f and h"),
    2: Config(2, 128, 16, True, True,
              "real f, C_p=(p+1)^-2; Slepian window, ellipse theta_c=20deg a=30deg"),
    3: Config(3, 256, 32, True, True,
              "real f, C_p=(p+1)^-2.5 + 1% white floor; Slepian window a=15deg b=5deg rotated 30deg"),
    4: Config(4, 512, 24, True, False,
              "real field of 50 elongated Gaussian blobs; complex window |h_st| ~ exp(-s^2/128)"),
    5: Config(5, 1024, 64, False, True,
              "complex f, C_p=(p+1)^-2; Slepian window a=10deg b=3deg"),
}


def _cn(rng: np.random.Generator, size, var) -> np.ndarray:
    """Complex normal with E|z|^2 = var."""
    s = np.sqrt(np.asarray(var, dtype=np.float64) / 2.0)
    return s * (rng.standard_normal(size) + 1j * rng.standard_normal(size))


def complex_gaussian(L: int, seed: int, power=None) -> np.ndarray:
    """f_l^m ~ CN(0, C_l) for all |m| <= l <= L (C_l = 1 without a power law)."""
    rng = np.random.default_rng(seed)
    ls = np.repeat(np.arange(L + 1), 2 * np.arange(L + 1) + 1)
    var = np.ones(ls.size) if power is None else power(ls)
    return _cn(rng, ls.size, var)


def real_gaussian(L: int, seed: int, power) -> np.ndarray:
    """Real-signal coefficients: f_l^0 ~ N(0, C_l), f_l^m ~ CN(0, C_l) for m > 0,
    f_l^{-m} = (-1)^m conj(f_l^m) (harmonics.hpp:18-20)."""
    rng = np.random.default_rng(seed)
    out = np.zeros(coeff_count(L), np.complex128)
    for l in range(L + 1):
        c = power(l)
        out[coeff_index(l, 0)] = math.sqrt(c) * rng.standard_normal()
        if l:
            v = _cn(rng, l, c)
            m = np.arange(1, l + 1)
            out[l * l + l + m] = v
            out[l * l + l - m] = np.where(m % 2 == 1, -1.0, 1.0) * np.conj(v)
    return out


def load_window(name: str) -> np.ndarray:
    return np.load(DATA / f"{name}.npy")


def rotate_azimuth(h: np.ndarray, L: int, alpha: float) -> np.ndarray:
    """h_l^m <- e^{-i m alpha} h_l^m: rotate_coeffs with rho = (alpha, 0, 0)
    (harmonics.cpp:207-231; D^l_{mm'}(alpha,0,0) = e^{-i m alpha} delta_{mm'})."""
    out = h.copy()
    for l in range(L + 1):
        m = np.arange(-l, l + 1)
        out[l * l + l + m] *= np.exp(-1j * m * alpha)
    return out


def blob_field(L: int, seed: int, n_blobs: int = 50) -> np.ndarray:
    """Config 4 signal: 50 seeded elongated Gaussian blobs on the sphere (uniform centres,
    uniform orientations, major width U[4,8] deg, minor width U[2, major/2] deg, N(0,1)
    amplitudes), analysed by Gauss-Legendre quadrature in theta and an FFT in phi, truncated
    at degree L and made exactly conjugate-symmetric (a real field)."""
    rng = np.random.default_rng(seed)
    cen = rng.standard_normal((n_blobs, 3))
    cen /= np.linalg.norm(cen, axis=1, keepdims=True)
    tmp = rng.standard_normal((n_blobs, 3))
    e1 = tmp - (tmp * cen).sum(1, keepdims=True) * cen
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    e2 = np.cross(cen, e1)
    s1 = np.radians(rng.uniform(4.0, 8.0, n_blobs))
    s2 = np.radians(2.0) + rng.uniform(0.0, 1.0, n_blobs) * (s1 / 2.0 - np.radians(2.0))
    amp = rng.standard_normal(n_blobs)
    n_theta, n_phi = L + 64, 2 * L + 128
    x, w = np.polynomial.legendre.leggauss(n_theta)
    theta = np.arccos(x)
    phi = 2.0 * np.pi * np.arange(n_phi) / n_phi
    st = np.sin(theta)[:, None]
    pts = np.stack([st * np.cos(phi)[None, :], st * np.sin(phi)[None, :],
                    np.repeat(x[:, None], n_phi, axis=1)], axis=-1)
    field = np.zeros((n_theta, n_phi))
    for i in range(n_blobs):
        dot = pts @ cen[i]
        u1 = pts @ e1[i]
        u2 = pts @ e2[i]
        g = amp[i] * np.exp(-0.5 * ((u1 / s1[i]) ** 2 + (u2 / s2[i]) ** 2))
        field += np.where(dot > 0.0, g, 0.0)
    # F_m(theta) = int f e^{-i m phi} dphi
    Fm = np.fft.fft(field, axis=1) * (2.0 * np.pi / n_phi)
    out = np.zeros(coeff_count(L), np.complex128)
    sq = np.sqrt(np.maximum(0.0, 1.0 - x * x))
    sect = np.full(x.size, 1.0 / math.sqrt(4.0 * math.pi))
    for m in range(L + 1):
        # lambda_l^m on the Gauss nodes by the recursion of harmonics.cpp:60-89
        if m:
            sect = sect * (-sq * math.sqrt((2.0 * m + 1.0) / (2.0 * m)))
        rows = np.zeros((L + 1 - m, x.size))
        rows[0] = sect
        if m < L:
            rows[1] = x * math.sqrt(2.0 * m + 3.0) * sect
        for l in range(m + 2, L + 1):
            a = math.sqrt((4.0 * l * l - 1.0) / (l * l - m * m))
            b = math.sqrt(((l - 1) ** 2 - m * m) / (4.0 * (l - 1) ** 2 - 1.0))
            rows[l - m] = a * (x * rows[l - m - 1] - b * rows[l - m - 2])
        vals = rows @ (w * Fm[:, m])  # sum_k w_k lambda_l^m(theta_k) F_m(theta_k)
        ls = np.arange(m, L + 1)
        out[ls * ls + ls + m] = vals
        if m:
            out[ls * ls + ls - m] = (-1.0) ** m * np.conj(vals)
        else:
            out[ls * ls + ls] = vals.real
    return out


def make_inputs(index: int) -> tuple[np.ndarray, np.ndarray, Config]:
    """(f, h, config) for BASELINE configuration `index` (1-based)."""
    cfg = CONFIGS[index]
    if index == 1:
        f = complex_gaussian(cfg.L_f, 1)
        h = complex_gaussian(cfg.L_h, 2)
    elif index == 2:
        f = real_gaussian(cfg.L_f, 1, lambda p: (p + 1.0) ** -2)
        h = load_window("window_cfg2")
    elif index == 3:
        total = sum((2 * p + 1) * (p + 1.0) ** -2.5 for p in range(cfg.L_f + 1))
        floor = 0.01 * total / coeff_count(cfg.L_f)
        f = real_gaussian(cfg.L_f, 1, lambda p: (p + 1.0) ** -2.5 + floor)
        h = rotate_azimuth(load_window("window_cfg3"), cfg.L_h, math.pi / 6.0)
    elif index == 4:
        f = blob_field(cfg.L_f, 1)
        s = np.repeat(np.arange(cfg.L_h + 1), 2 * np.arange(cfg.L_h + 1) + 1)
        h = complex_gaussian(cfg.L_h, 2) * np.exp(-(s ** 2) / 128.0)
    elif index == 5:
        f = complex_gaussian(cfg.L_f, 1, lambda ls: (ls + 1.0) ** -2)
        h = load_window("window_cfg5")
    else:
        raise KeyError(index)
    return f, h, cfg


def shard_degrees(cfg: Config, world: int, rank: int, lmax: int | None = None) -> tuple[int, int]:
    """Contiguous degree range [l0, l1) of `rank`, balanced by computed components
    (c(l) = 2l+1 in full-m mode, l+1 in real mode)."""
    lm = cfg.L_g if lmax is None else lmax
    w = np.array([(l + 1) if cfg.real_mode else (2 * l + 1) for l in range(lm + 1)], float)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    bounds = [0]
    for k in range(1, world):
        bounds.append(int(np.searchsorted(cum, total * k / world)))
    bounds.append(lm + 1)
    bounds = [min(max(b, 0), lm + 1) for b in bounds]
    for k in range(1, len(bounds)):
        bounds[k] = max(bounds[k], bounds[k - 1])
    return bounds[rank], bounds[rank + 1]
