"""CPU oracle bindings — TEST INFRASTRUCTURE ONLY.

Python (ctypes + numpy) access to
  * ``liboracle_slsht.so`` — our plain-C restatement of the reference's forward_fast
    path (``oracle/slsht_oracle.c``), and
  * ``_ref/libslsht_ref.so`` — the unmodified reference sources compiled by
    ``oracle/Makefile`` (only present where /root/reference was available at build time;
    the built file travels with the repo snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg import
this module, and only as the checker / baseline. The product path
(``paper_1207_5558_b200``) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle_slsht.so"
REF_SO = HERE / "_ref" / "libslsht_ref.so"
REF_SRC = Path("/root/reference/proj")

SINK = C.CFUNCTYPE(None, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_void_p)
_dp = C.POINTER(C.c_double)


def coeff_index(l: int, m: int) -> int:
    return l * l + l + m


def coeff_count(L: int) -> int:
    return (L + 1) * (L + 1)


def volume_shape(L_h: int) -> tuple[int, int, int]:
    n = 2 * L_h + 1
    return (n, L_h + 1, n)


def _ptr(a: np.ndarray):
    assert a.dtype in (np.float64, np.complex128) and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def build(reference: bool | None = None) -> None:
    """Build the oracle (always) and the reference library (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if reference is None:
        reference = REF_SRC.is_dir()
    if reference:
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


class _Lib:
    def __init__(self, path: Path, prefix: str):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run oracle.build())")
        self.lib = C.CDLL(str(path))
        self.prefix = prefix
        getattr(self.lib, f"{prefix}last_error").restype = C.c_char_p

    def err(self) -> str:
        return getattr(self.lib, f"{self.prefix}last_error")().decode()

    def check(self, rc: int) -> None:
        if rc == 2:
            raise ValueError(self.err())
        if rc == 3:
            raise ArithmeticError(self.err())
        if rc != 0:
            raise RuntimeError(self.err())


class Oracle(_Lib):
    """Our C restatement of the reference (the parity checker)."""

    def __init__(self, path: Path = ORACLE_SO):
        super().__init__(path, "oracle_")
        L = self.lib
        L.oracle_ctx_create.restype = C.c_void_p
        L.oracle_ctx_create.argtypes = [C.c_int, _dp, C.c_int]
        L.oracle_ctx_destroy.argtypes = [C.c_void_p]
        L.oracle_modulated_sht.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp]
        L.oracle_component.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.c_int, _dp]
        L.oracle_delta_size.restype = C.c_size_t
        L.oracle_forward_fast.argtypes = [C.c_int, _dp, C.c_int, C.c_int, _dp, C.c_int,
                                          C.c_int, C.c_int, C.c_int, SINK, C.c_void_p]

    def theta_weights(self, N: int) -> np.ndarray:
        out = np.zeros(N + 1)
        self.check(self.lib.oracle_theta_weights(N, _ptr(out)))
        return out

    def beta_weights(self, L: int) -> np.ndarray:
        out = np.zeros(L + 1)
        self.check(self.lib.oracle_beta_weights(L, _ptr(out)))
        return out

    def legendre_rows(self, m: int, lmax: int, thetas: np.ndarray) -> np.ndarray:
        thetas = np.ascontiguousarray(thetas, dtype=np.float64)
        out = np.zeros((lmax - abs(m) + 1, thetas.size))
        self.check(self.lib.oracle_legendre_rows(m, lmax, _ptr(thetas), thetas.size, _ptr(out)))
        return out

    def delta_tables(self, L: int) -> np.ndarray:
        out = np.zeros(int(self.lib.oracle_delta_size(L)))
        self.check(self.lib.oracle_delta_tables(L, _ptr(out)))
        return out

    def modulated_sht(self, f: np.ndarray, L_f: int, l: int, m: int, L_h: int) -> np.ndarray:
        f = np.ascontiguousarray(f, dtype=np.complex128)
        ctx = self.lib.oracle_ctx_create(L_f, _ptr(f), L_h)
        try:
            out = np.zeros(coeff_count(L_h), dtype=np.complex128)
            self.check(self.lib.oracle_modulated_sht(ctx, l, m, _ptr(out)))
            return out
        finally:
            self.lib.oracle_ctx_destroy(ctx)

    def c_tensor(self, L_h: int, mod: np.ndarray, h: np.ndarray) -> np.ndarray:
        n = 2 * L_h + 1
        delta = self.delta_tables(L_h)
        out = np.zeros((n, n, n), dtype=np.complex128)
        self.check(self.lib.oracle_c_tensor(L_h, _ptr(np.ascontiguousarray(mod)),
                                            _ptr(np.ascontiguousarray(h)), _ptr(delta), _ptr(out)))
        return out

    def evaluate(self, L_h: int, ct: np.ndarray) -> np.ndarray:
        out = np.zeros(volume_shape(L_h), dtype=np.complex128)
        self.check(self.lib.oracle_evaluate(L_h, _ptr(np.ascontiguousarray(ct)), _ptr(out)))
        return out

    def digest(self, L_h: int, vol: np.ndarray) -> np.ndarray:
        out = np.zeros(8)
        self.lib.oracle_digest(L_h, _ptr(np.ascontiguousarray(vol, dtype=np.complex128)), _ptr(out))
        return out

    def components(self, f: np.ndarray, L_f: int, h: np.ndarray, L_h: int, lm) -> dict:
        """Volumes for selected (l, m) (lazy I-table: cheap at large L_f)."""
        f = np.ascontiguousarray(f, dtype=np.complex128)
        h = np.ascontiguousarray(h, dtype=np.complex128)
        delta = self.delta_tables(L_h)
        ctx = self.lib.oracle_ctx_create(L_f, _ptr(f), L_h)
        out = {}
        try:
            for l, m in sorted(lm, key=lambda t: (t[1], t[0])):
                vol = np.zeros(volume_shape(L_h), dtype=np.complex128)
                self.check(self.lib.oracle_component(ctx, _ptr(h), _ptr(delta), l, m, _ptr(vol)))
                out[(l, m)] = vol
        finally:
            self.lib.oracle_ctx_destroy(ctx)
        return out

    def forward_fast(self, f, L_f, f_real, h, L_h, h_real, lmax=-1, use_real_symmetry=True,
                     emit_negative_m=True, on_component=None) -> dict:
        """Full forward_fast; returns {(l, m): volume} unless on_component is given."""
        f = np.ascontiguousarray(f, dtype=np.complex128)
        h = np.ascontiguousarray(h, dtype=np.complex128)
        shape = volume_shape(L_h)
        count = int(np.prod(shape))
        out = {}

        def cb(l, m, ptr, _user):
            vol = np.ctypeslib.as_array(ptr, shape=(count * 2,)).view(np.complex128).reshape(shape)
            if on_component is None:
                out[(l, m)] = vol.copy()
            else:
                on_component(l, m, vol)

        self.check(self.lib.oracle_forward_fast(L_f, _ptr(f), int(f_real), L_h, _ptr(h),
                                                int(h_real), lmax, int(use_real_symmetry),
                                                int(emit_negative_m), SINK(cb), None))
        return out


class Reference(_Lib):
    """The unmodified reference library (oracle/_ref), reached through ref_capi.cpp."""

    def __init__(self, path: Path = REF_SO):
        super().__init__(path, "ref_")
        L = self.lib
        L.ref_forward_fast.argtypes = [C.c_int, _dp, C.c_int, C.c_int, _dp, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, SINK, C.c_void_p]
        L.ref_forward_fast_digest.argtypes = [C.c_int, _dp, C.c_int, C.c_int, _dp, C.c_int,
                                              C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp]
        L.ref_eigenfunction_window.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int, _dp, _dp]
        L.ref_random_coeffs.argtypes = [C.c_int, C.c_uint64, C.c_int, _dp]
        L.ref_components.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_int, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), _dp]
        L.ref_components_mt.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_int, C.POINTER(C.c_int),
                                        C.POINTER(C.c_int), C.c_int, _dp]
        L.ref_setup_seconds.argtypes = [C.c_int, _dp, C.c_int, C.c_int, _dp, C.c_int, _dp]
        L.ref_rotate_coeffs.argtypes = [C.c_int, _dp, C.c_double, C.c_double, C.c_double, _dp]
        L.ref_forward_direct.argtypes = [C.c_int, _dp, C.c_int, _dp, C.c_int, C.c_int, _dp]

    def delta_tables(self, L: int) -> np.ndarray:
        size = sum((2 * p + 1) ** 2 for p in range(L + 1))
        out = np.zeros(size)
        self.check(self.lib.ref_delta_tables(L, _ptr(out)))
        return out

    def theta_weights(self, N: int) -> np.ndarray:
        out = np.zeros(N + 1)
        self.check(self.lib.ref_theta_weights(N, _ptr(out)))
        return out

    def beta_weights(self, L: int) -> np.ndarray:
        out = np.zeros(L + 1)
        self.check(self.lib.ref_beta_weights(L, _ptr(out)))
        return out

    def legendre_rows(self, m: int, lmax: int, thetas: np.ndarray) -> np.ndarray:
        thetas = np.ascontiguousarray(thetas, dtype=np.float64)
        out = np.zeros((lmax - abs(m) + 1, thetas.size))
        self.check(self.lib.ref_legendre_rows(m, lmax, _ptr(thetas), thetas.size, _ptr(out)))
        return out

    def modulated_sht(self, f, L_f, l, m, L_h) -> np.ndarray:
        out = np.zeros(coeff_count(L_h), dtype=np.complex128)
        self.check(self.lib.ref_modulated_sht(L_f, _ptr(np.ascontiguousarray(f, dtype=np.complex128)),
                                              l, m, L_h, _ptr(out)))
        return out

    def c_tensor(self, L_h, mod, h) -> np.ndarray:
        n = 2 * L_h + 1
        out = np.zeros((n, n, n), dtype=np.complex128)
        self.check(self.lib.ref_build_c_tensor(L_h, _ptr(np.ascontiguousarray(mod)),
                                               _ptr(np.ascontiguousarray(h)), _ptr(out)))
        return out

    def evaluate(self, L_h, ct) -> np.ndarray:
        out = np.zeros(volume_shape(L_h), dtype=np.complex128)
        self.check(self.lib.ref_evaluate(L_h, _ptr(np.ascontiguousarray(ct)), _ptr(out)))
        return out

    def integrate_volume(self, L_h, vol) -> complex:
        out = np.zeros(2)
        self.check(self.lib.ref_integrate_volume(L_h, _ptr(np.ascontiguousarray(vol)), _ptr(out)))
        return complex(out[0], out[1])

    def forward_fast(self, f, L_f, f_real, h, L_h, h_real, lmax=-1, threads=0,
                     use_real_symmetry=True, emit_negative_m=True) -> dict:
        f = np.ascontiguousarray(f, dtype=np.complex128)
        h = np.ascontiguousarray(h, dtype=np.complex128)
        shape = volume_shape(L_h)
        count = int(np.prod(shape))
        out = {}

        def cb(l, m, ptr, _user):
            out[(l, m)] = np.ctypeslib.as_array(ptr, shape=(count * 2,)).view(
                np.complex128).reshape(shape).copy()

        self.check(self.lib.ref_forward_fast(L_f, _ptr(f), int(f_real), L_h, _ptr(h), int(h_real),
                                             lmax, threads, int(use_real_symmetry),
                                             int(emit_negative_m), SINK(cb), None))
        return out

    def forward_fast_digest(self, f, L_f, f_real, h, L_h, h_real, lmax=-1, threads=0,
                            use_real_symmetry=True, emit_negative_m=True):
        """(digests[coeff_count(lmax), 8], seconds) — the CPU-baseline measurement."""
        f = np.ascontiguousarray(f, dtype=np.complex128)
        h = np.ascontiguousarray(h, dtype=np.complex128)
        lm = (L_f + L_h) if lmax < 0 else lmax
        dig = np.full((coeff_count(lm), 8), np.nan)
        secs = np.zeros(1)
        self.check(self.lib.ref_forward_fast_digest(L_f, _ptr(f), int(f_real), L_h, _ptr(h),
                                                    int(h_real), lmax, threads,
                                                    int(use_real_symmetry), int(emit_negative_m),
                                                    _ptr(dig), _ptr(secs)))
        return dig, float(secs[0])

    def roundtrip(self, f, L_f, f_real, h, L_h, h_real) -> np.ndarray:
        out = np.zeros(coeff_count(L_f), dtype=np.complex128)
        self.check(self.lib.ref_roundtrip(L_f, _ptr(np.ascontiguousarray(f, dtype=np.complex128)),
                                          int(f_real), L_h,
                                          _ptr(np.ascontiguousarray(h, dtype=np.complex128)),
                                          int(h_real), _ptr(out)))
        return out

    def components(self, f, L_f, h, L_h, lm) -> dict:
        """Volumes of the listed (l, m) through ModulatedSht/build_c_tensor/So3Evaluator."""
        lm = list(lm)
        ls = (C.c_int * len(lm))(*[l for l, _ in lm])
        ms = (C.c_int * len(lm))(*[m for _, m in lm])
        out = np.zeros((len(lm),) + volume_shape(L_h), dtype=np.complex128)
        self.check(self.lib.ref_components(L_f, _ptr(np.ascontiguousarray(f, dtype=np.complex128)), L_h,
                                           _ptr(np.ascontiguousarray(h, dtype=np.complex128)),
                                           len(lm), ls, ms, _ptr(out)))
        return {k: out[i] for i, k in enumerate(lm)}

    def components_mt(self, f, L_f, h, L_h, lm, threads: int = 0) -> np.ndarray:
        """Volumes [len(lm), n, L_h+1, n] of the listed (l, m) through the component chain on
        `threads` host threads (0: all cores)."""
        lm = list(lm)
        ls = (C.c_int * len(lm))(*[l for l, _ in lm])
        ms = (C.c_int * len(lm))(*[m for _, m in lm])
        out = np.zeros((len(lm),) + volume_shape(L_h), dtype=np.complex128)
        nt = threads or os.cpu_count() or 1
        self.check(self.lib.ref_components_mt(
            L_f, _ptr(np.ascontiguousarray(f, dtype=np.complex128)), L_h,
            _ptr(np.ascontiguousarray(h, dtype=np.complex128)), len(lm), ls, ms, nt, _ptr(out)))
        return out

    def setup_seconds(self, f, L_f, f_real, h, L_h, h_real) -> float:
        """Wall time of forward_fast's per-call setup (ModulatedSht + DeltaTables +
        So3Evaluator, transform.cpp:256-258)."""
        secs = np.zeros(1)
        self.check(self.lib.ref_setup_seconds(
            L_f, _ptr(np.ascontiguousarray(f, dtype=np.complex128)), int(f_real), L_h,
            _ptr(np.ascontiguousarray(h, dtype=np.complex128)), int(h_real), _ptr(secs)))
        return float(secs[0])

    def forward_direct(self, f, L_f, h, L_h, lmax=-1, threads=0) -> np.ndarray:
        """forward_direct (transform.cpp:313-388): [coeff_count(lmax), V] complex."""
        lm = L_f + L_h if lmax < 0 else lmax
        V = int(np.prod(volume_shape(L_h)))
        out = np.zeros((coeff_count(lm), V), np.complex128)
        f = np.ascontiguousarray(f, np.complex128)
        h = np.ascontiguousarray(h, np.complex128)
        self.check(self.lib.ref_forward_direct(L_f, _ptr(f), L_h, _ptr(h), lm, threads, _ptr(out)))
        return out

    def eigenfunction_window(self, theta_c: float, a: float, L: int, oversample: int = 4):
        out = np.zeros(coeff_count(L), dtype=np.complex128)
        lam = np.zeros(1)
        self.check(self.lib.ref_eigenfunction_window(theta_c, a, L, oversample, _ptr(out), _ptr(lam)))
        return out, float(lam[0])

    def random_coeffs(self, L: int, seed: int, real_signal: bool = True) -> np.ndarray:
        out = np.zeros(coeff_count(L), dtype=np.complex128)
        self.check(self.lib.ref_random_coeffs(L, seed, int(real_signal), _ptr(out)))
        return out

    def rotate_coeffs(self, c, L, alpha, beta, gamma) -> np.ndarray:
        out = np.zeros(coeff_count(L), dtype=np.complex128)
        self.check(self.lib.ref_rotate_coeffs(L, _ptr(np.ascontiguousarray(c, dtype=np.complex128)),
                                              alpha, beta, gamma, _ptr(out)))
        return out


def reference_available() -> bool:
    return REF_SO.exists()
