"""Host-side mirror of the reference's forward_fast interface over the C ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/slsht:
  * SphCoeffs            harmonics.hpp:18-33   (coeff_index(l, m) = l*l + l + m)
  * So3Volume layout     transform.hpp:13-29   ((a*(L_h+1)+b)*n + c, n = 2 L_h + 1)
  * ForwardOptions       transform.hpp:145-157
  * forward_fast (x2)    transform.hpp:159-165, transform.cpp:244-311
  * ValidationError / NumericError  errors.hpp:7-16
Every call runs the sm_100a kernels of libslsht_cuda.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class ValidationError(ValueError):
    """slsht::ValidationError (std::invalid_argument); CLI exit code 2."""


class NumericError(ArithmeticError):
    """slsht::NumericError (std::runtime_error); CLI exit code 3."""


class DeviceError(RuntimeError):
    """CUDA runtime failure or no sm_100a device (status 4)."""


def coeff_index(l: int, m: int) -> int:
    return l * l + l + m


def coeff_count(band_limit: int) -> int:
    return (band_limit + 1) * (band_limit + 1)


def volume_shape(L_h: int) -> tuple[int, int, int]:
    n = 2 * L_h + 1
    return (n, L_h + 1, n)


@dataclass
class SphCoeffs:
    band_limit: int
    data: np.ndarray
    real_signal: bool = False

    @staticmethod
    def zeros(band_limit: int, real_signal: bool = False) -> "SphCoeffs":
        return SphCoeffs(band_limit, np.zeros(coeff_count(band_limit), np.complex128), real_signal)

    def at(self, l: int, m: int) -> complex:
        return complex(self.data[coeff_index(l, m)])

    def __post_init__(self):
        self.data = np.ascontiguousarray(self.data, dtype=np.complex128)
        if self.data.size != coeff_count(self.band_limit):
            raise ValidationError("coefficient array size does not match the band limit")


@dataclass
class ForwardOptions:
    lmax: int = -1
    threads: int = 0
    use_real_symmetry: bool = True
    emit_negative_m: bool = True


@dataclass
class SlshtDistribution:
    L_f: int
    L_h: int
    L_g: int
    lmax: int
    components: np.ndarray = field(repr=False)  # [coeff_count(lmax), n, L_h+1, n]

    def component(self, l: int, m: int) -> np.ndarray:
        return self.components[coeff_index(l, m)]


def _raise(code: int, plan) -> None:
    if code == L.SLSHT_OK:
        return
    lib = L.load()
    msg = lib.slsht_cuda_last_error(plan).decode(errors="replace")
    if code == L.SLSHT_ERR_VALIDATION:
        raise ValidationError(msg)
    if code == L.SLSHT_ERR_NUMERIC:
        raise NumericError(msg)
    raise DeviceError(msg)


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class Plan:
    """Owns one slsht_cuda_plan (device tables, chunk schedule, output ring or buffer)."""

    def __init__(self, L_f: int, L_h: int, *, lmax: int = -1, real_mode: bool = False,
                 emit_negative_m: bool = True, device: int = 0, l_begin: int = 0,
                 l_end: int = -1, materialize: bool = False, ring_bytes: int = 0,
                 stream: int | None = None, devices: list[int] | None = None):
        """devices: a multi-GPU plan, one balanced degree shard per entry (an ordinal may
        repeat); the shards' digests are gathered into the caller's table."""
        self.lib = L.load()
        d = L.slsht_cuda_desc()
        d.L_f, d.L_h, d.lmax = L_f, L_h, lmax
        d.real_mode, d.emit_negative_m = int(real_mode), int(emit_negative_m)
        d.device, d.l_begin, d.l_end = device, l_begin, l_end
        d.materialize, d.ring_bytes = int(materialize), int(ring_bytes)
        d.stream = stream
        if devices is not None and len(devices) > 1:
            self._devices = (C.c_int * len(devices))(*devices)
            d.n_devices = len(devices)
            d.devices = self._devices
        handle = C.c_void_p()
        rc = self.lib.slsht_cuda_plan_create(C.byref(d), C.byref(handle))
        _raise(rc, None)
        self.handle = handle
        self.L_f, self.L_h = L_f, L_h
        self.lmax = (L_f + L_h) if lmax < 0 else lmax
        self.real_mode = real_mode
        self.materialize = materialize

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.slsht_cuda_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- queries
    @property
    def volume_elems(self) -> int:
        return int(self.lib.slsht_cuda_volume_elems(self.handle))

    @property
    def computed_count(self) -> int:
        return int(self.lib.slsht_cuda_computed_count(self.handle))

    @property
    def emitted_count(self) -> int:
        return int(self.lib.slsht_cuda_emitted_count(self.handle))

    @property
    def stream(self) -> int:
        return int(self.lib.slsht_cuda_stream(self.handle) or 0)

    @property
    def device_output(self) -> int:
        return int(self.lib.slsht_cuda_device_output(self.handle) or 0)

    @property
    def launch_count(self) -> int:
        return int(self.lib.slsht_cuda_launch_count(self.handle))

    def set_profiling(self, enable: bool) -> None:
        self.lib.slsht_cuda_set_profiling(self.handle, int(enable))

    def kernel_time(self) -> float | None:
        """Coupling-kernel device time (ms) of the last forward_device (single-chunk plans)."""
        out = C.c_double(0.0)
        rc = self.lib.slsht_cuda_kernel_time(self.handle, C.byref(out))
        return float(out.value) if rc == 0 else None

    def stage_times(self) -> list[float]:
        out = (C.c_double * 8)()
        k = self.lib.slsht_cuda_stage_times(self.handle, out, 8)
        return list(out[:k])

    # ---- compute
    def forward_device(self, f_ptr: int, h_ptr: int, *, inputs_on_device: bool,
                       digests_ptr: int | None, digests_on_device: bool,
                       synchronize: bool = True) -> None:
        rc = self.lib.slsht_cuda_forward_device(self.handle, C.c_void_p(f_ptr), C.c_void_p(h_ptr),
                                                int(inputs_on_device),
                                                C.c_void_p(digests_ptr or 0),
                                                int(digests_on_device), int(synchronize))
        _raise(rc, self.handle)

    def forward_digests(self, f: np.ndarray, h: np.ndarray) -> np.ndarray:
        """Host f, h -> host digests [coeff_count(lmax), 8] (NaN rows not in this plan)."""
        f = np.ascontiguousarray(f, np.complex128)
        h = np.ascontiguousarray(h, np.complex128)
        dig = np.full((coeff_count(self.lmax), L.DIGEST_WIDTH), np.nan)
        self.forward_device(f.ctypes.data, h.ctypes.data, inputs_on_device=False,
                            digests_ptr=dig.ctypes.data, digests_on_device=False)
        return dig

    def forward_capture(self, f: np.ndarray, h: np.ndarray, lm) -> tuple[np.ndarray, dict]:
        """Device-mode forward returning (digests, {(l, m): volume}) for the listed components."""
        f = np.ascontiguousarray(f, np.complex128)
        h = np.ascontiguousarray(h, np.complex128)
        lm = list(lm)
        dig = np.full((coeff_count(self.lmax), L.DIGEST_WIDTH), np.nan)
        vols = np.zeros((max(1, len(lm)),) + volume_shape(self.L_h), np.complex128)
        ls = (C.c_int * max(1, len(lm)))(*[l for l, _ in lm])
        ms = (C.c_int * max(1, len(lm)))(*[m for _, m in lm])
        rc = self.lib.slsht_cuda_forward_capture(self.handle, _dptr(f), _dptr(h), _dptr(dig),
                                                 len(lm), ls, ms, _dptr(vols))
        _raise(rc, self.handle)
        return dig, {k: vols[i] for i, k in enumerate(lm)}

    def inverse(self, f: np.ndarray, h: np.ndarray, h00: complex,
                signal_band_limit: int) -> np.ndarray:
        """inverse_slsht(forward_fast(f, h), h00, L) (transform.cpp:469-544) on the device: the
        forward's digest epilogue already holds every integrate_volume; returns f_rec."""
        f = np.ascontiguousarray(f, np.complex128)
        h = np.ascontiguousarray(h, np.complex128)
        out = np.zeros(coeff_count(signal_band_limit), np.complex128)
        rc = self.lib.slsht_cuda_inverse(self.handle, _dptr(f), _dptr(h), float(np.real(h00)),
                                         float(np.imag(h00)), int(signal_band_limit),
                                         _dptr(out))
        _raise(rc, self.handle)
        return out

    def forward_sink(self, f: np.ndarray, h: np.ndarray, sink) -> None:
        """Stream every emitted component to sink(l, m, volume) (volume valid during the call)."""
        f = np.ascontiguousarray(f, np.complex128)
        h = np.ascontiguousarray(h, np.complex128)
        shape = volume_shape(self.L_h)
        count = int(np.prod(shape))
        err: list[BaseException] = []

        def cb(l, m, ptr, _user):
            if err:
                return
            try:
                vol = np.ctypeslib.as_array(ptr, shape=(2 * count,)).view(np.complex128)
                sink(l, m, vol.reshape(shape))
            except BaseException as e:  # re-raised after the C call returns
                err.append(e)

        cfn = L.SINK(cb)
        rc = self.lib.slsht_cuda_forward(self.handle, _dptr(f), _dptr(h),
                                         C.cast(cfn, C.c_void_p), None)
        if err:
            raise err[0]
        _raise(rc, self.handle)

    def forward_copy(self, f: np.ndarray, h: np.ndarray, out: np.ndarray,
                     first_index: int = 0) -> tuple[int, int]:
        """Host-sink forward with the library's native copy sink (slsht_cuda_copy_sink): the
        volume of (l, m) lands in out[coeff_index(l, m) - first_index] (out: [rows, n, L_h+1, n]
        complex, C-contiguous). Returns (delivered, dropped)."""
        f = np.ascontiguousarray(f, np.complex128)
        h = np.ascontiguousarray(h, np.complex128)
        if out.dtype != np.complex128 or not out.flags.c_contiguous:
            raise ValidationError("out must be a C-contiguous complex128 array")
        tgt = L.slsht_copy_target(out.ctypes.data, int(first_index), int(out.shape[0]),
                                  int(self.volume_elems), 0, 0)
        sink = C.cast(self.lib.slsht_cuda_copy_sink, C.c_void_p)
        rc = self.lib.slsht_cuda_forward(self.handle, _dptr(f), _dptr(h), sink, C.byref(tgt))
        _raise(rc, self.handle)
        return int(tgt.delivered), int(tgt.dropped)

    def forward_scatter(self, f: np.ndarray, h: np.ndarray, targets: dict, lmax: int,
                        threads: int = 0) -> int:
        """The materializing forward (slsht_cuda_forward_scatter): the volume of every emitted
        (l, m) in `targets` ({(l, m): C-contiguous complex128 array of volume_elems}) is copied
        into its array by several host threads. Returns the number of volumes copied."""
        f = np.ascontiguousarray(f, np.complex128)
        h = np.ascontiguousarray(h, np.complex128)
        n = coeff_count(lmax)
        table = (C.c_void_p * n)()
        for (l, m), a in targets.items():
            if a.dtype != np.complex128 or not a.flags.c_contiguous or a.size != self.volume_elems:
                raise ValidationError("targets must be C-contiguous complex128 volumes")
            table[coeff_index(l, m)] = a.ctypes.data
        got = C.c_longlong(0)
        rc = self.lib.slsht_cuda_forward_scatter(self.handle, _dptr(f), _dptr(h), table, n,
                                                 int(threads), C.byref(got))
        _raise(rc, self.handle)
        return int(got.value)


def _real_mode(f: SphCoeffs, h: SphCoeffs, opts: ForwardOptions) -> bool:
    # transform.cpp:253-254
    return bool(opts.use_real_symmetry and f.real_signal and h.real_signal)


def forward_fast(f: SphCoeffs, h: SphCoeffs, sink=None, opts: ForwardOptions | None = None,
                 *, device: int = 0, ring_bytes: int = 1 << 28):
    """slsht::forward_fast on the B200.

    With a sink: every component (l, m) is delivered once as sink(l, m, volume[n, L_h+1, n]);
    calls are serialized; in real mode (l, -m) follows (l, m) (transform.cpp:280-284).
    Without a sink: returns the materialized SlshtDistribution (transform.cpp:297-311).
    """
    opts = opts or ForwardOptions()
    L_f, L_h = f.band_limit, h.band_limit
    L_g = L_f + L_h
    lmax = L_g if opts.lmax < 0 else opts.lmax
    if lmax > L_g:  # transform.cpp:250-252
        raise ValidationError("fast engine computes components up to L_f + L_h only")
    with Plan(L_f, L_h, lmax=lmax, real_mode=_real_mode(f, h, opts),
              emit_negative_m=opts.emit_negative_m, device=device, materialize=False,
              ring_bytes=ring_bytes) as plan:
        if sink is not None:
            plan.forward_sink(f.data, h.data, sink)
            return None
        comps = np.zeros((coeff_count(lmax),) + volume_shape(L_h), np.complex128)

        def store(l, m, vol):
            comps[coeff_index(l, m)] = vol

        plan.forward_sink(f.data, h.data, store)
        return SlshtDistribution(L_f, L_h, L_g, lmax, comps)


def shard_bounds(l_begin: int, l_end: int, real_mode: bool, parts: int) -> list[int]:
    """The degree shards of a multi-GPU plan (slsht_cuda_shard_bounds; host only)."""
    lib = L.load()
    out = (C.c_int * (parts + 1))()
    rc = lib.slsht_cuda_shard_bounds(int(l_begin), int(l_end), int(real_mode), int(parts), out)
    _raise(rc, None)
    return list(out)


def theta_weights(N: int, device: int = 0) -> np.ndarray:
    """theta_weights(N) (grids.cpp:76-92) on the device: the N+1 weights of S_N."""
    lib = L.load()
    out = np.zeros(max(N + 1, 0))
    _raise(lib.slsht_cuda_theta_weights(device, N, out.ctypes.data_as(L._dp)), None)
    return out


def beta_weights(band_limit: int, device: int = 0) -> np.ndarray:
    """beta_weights(L) (grids.cpp:54-74) on the device: q(beta_b), b <= L."""
    lib = L.load()
    out = np.zeros(max(band_limit + 1, 0))
    _raise(lib.slsht_cuda_beta_weights(device, band_limit, out.ctypes.data_as(L._dp)), None)
    return out


def legendre_rows(m: int, lmax: int, thetas, device: int = 0) -> np.ndarray:
    """legendre_rows (harmonics.cpp:60-89) on the device: [lmax-|m|+1, len(thetas)]."""
    lib = L.load()
    th = np.ascontiguousarray(thetas, np.float64)
    out = np.zeros((max(lmax - abs(m) + 1, 0), th.size))
    _raise(lib.slsht_cuda_legendre_rows(device, m, lmax, th.ctypes.data_as(L._dp), th.size,
                                        out.ctypes.data_as(L._dp)), None)
    return out


def gauss_legendre_half(points: int, device: int = 0):
    """The x >= 0 half of the points-point Gauss-Legendre rule of the modulated SHT
    (DESIGN.md §2): (cos, sin, weights), (points+1)//2 nodes, decreasing x."""
    lib = L.load()
    K = (points + 1) // 2
    c, s, w = np.zeros(K), np.zeros(K), np.zeros(K)
    _raise(lib.slsht_cuda_gauss_legendre_half(device, points, c.ctypes.data_as(L._dp),
                                              s.ctypes.data_as(L._dp), w.ctypes.data_as(L._dp)),
           None)
    return c, s, w


def delta_tables(band_limit: int, device: int = 0) -> np.ndarray:
    """Delta^p = d^p(pi/2), p <= band_limit, flat in the reference's layout (wigner.hpp:20-30)."""
    lib = L.load()
    size = sum((2 * p + 1) ** 2 for p in range(band_limit + 1))
    out = np.zeros(size)
    rc = lib.slsht_cuda_delta_tables(device, band_limit, out.ctypes.data_as(L._dp))
    _raise(rc, None)
    return out


def eigenfunction_window(theta_c: float, a: float, band_limit: int, oversample: int = 4,
                         device: int = 0) -> tuple[np.ndarray, float]:
    """eigenfunction_window(EllipticalRegion{theta_c, a}, L, oversample) (window.cpp:126-198) on
    the device: (unit-norm coefficients, concentration ratio lambda)."""
    lib = L.load()
    out = np.zeros(coeff_count(band_limit), np.complex128)
    lam = C.c_double(0.0)
    rc = lib.slsht_cuda_eigenfunction_window(device, float(theta_c), float(a), int(band_limit),
                                             int(oversample), out.ctypes.data, C.byref(lam))
    _raise(rc, None)
    return out, float(lam.value)


def forward_direct(f: SphCoeffs, h: SphCoeffs, lmax: int = -1, cells=None,
                   device: int = 0) -> np.ndarray:
    """forward_direct (transform.cpp:313-388), the reference's independent direct engine, on the
    device: g(l, m; rho) = sh_analysis(sh_synthesis(f) sh_synthesis(R_rho h)) on the sphere grid
    of band max(lmax, L_g). Returns [coeff_count(lmax), cells] complex; `cells` are flat
    So3Volume indices (a (L_h+1) + b)(2 L_h+1) + c (default: every cell, in volume order, so
    row coeff_index(l, m) reshaped to volume_shape(L_h) is the component's So3Volume)."""
    lib = L.load()
    lm = f.band_limit + h.band_limit if lmax < 0 else int(lmax)
    fa = np.ascontiguousarray(f.data, np.complex128)
    ha = np.ascontiguousarray(h.data, np.complex128)
    if cells is None:
        ncell = int(np.prod(volume_shape(h.band_limit)))
        cptr = None
    else:
        cells = np.ascontiguousarray(cells, np.int64)
        ncell = int(cells.size)
        cptr = cells.ctypes.data
    out = np.zeros((coeff_count(lm), ncell), np.complex128)
    rc = lib.slsht_cuda_forward_direct(device, f.band_limit, fa.ctypes.data, h.band_limit,
                                       ha.ctypes.data, lm, cptr, ncell, out.ctypes.data)
    _raise(rc, None)
    return out


def modulated_sht(f: SphCoeffs, lm: list[tuple[int, int]], window_band_limit: int,
                  device: int = 0) -> np.ndarray:
    """ModulatedSht::compute for several (l, m): [len(lm), coeff_count(L_h)] complex."""
    with Plan(f.band_limit, window_band_limit, device=device, lmax=0, ring_bytes=1 << 24) as plan:
        ls = (C.c_int * len(lm))(*[l for l, _ in lm])
        ms = (C.c_int * len(lm))(*[m for _, m in lm])
        out = np.zeros((len(lm), coeff_count(window_band_limit)), np.complex128)
        rc = plan.lib.slsht_cuda_modulated(plan.handle, _dptr(f.data), len(lm), ls, ms,
                                           out.ctypes.data_as(L._dp))
        _raise(rc, plan.handle)
        return out
