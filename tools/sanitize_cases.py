"""Small forwards that launch every kernel of the engine, for bounds checking:
    SLSHT_CUDA_GUARD=1 python tools/sanitize_cases.py
With SLSHT_CUDA_GUARD=1 every plan-owned device buffer gets 64-KB guard bands (pattern 0xA5)
on both sides, verified after every call (a DeviceError names the buffer and the byte); the
GPU test tests/test_gpu.py::test_guard_bands_every_kernel runs these cases that way and checks
the results bitwise against unguarded plans. (compute-sanitizer is closed on this GPU pool.)
Cases: n = 17 (k_couple_reg; k_couple_ws with SLSHT_CUDA_REG=0), 33 (k_couple_lines), 49 (k_tgemm + k_qfft<49>; k_fused with
SLSHT_CUDA_FUSED=1; k_tpipe and k_qfft_lean with their knobs), 65 (k_qfft<65>), 129 (k_qfft<129>, DMMA radix-43), 225 (k_qfft_rt),
21 (runtime-plan k_couple<0>), and with them the setup kernels (k_glnodes, k_setup_main,
k_delta, k_dtab, k_wtab), k_agen, k_modgemm, k_digest, k_inverse."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1207_5558_b200 as S  # noqa: E402

CASES = [  # (L_f, L_h, real_mode, lmax, engine knobs)
    (6, 8, False, 8, {}),     # n = 17 (k_couple_reg)
    (6, 8, True, 8, {"SLSHT_CUDA_REG": "0"}),   # n = 17 on k_couple_ws
    (4, 16, True, 10, {}),    # n = 33, real mode (mirrors)
    (3, 24, False, 6, {}),    # n = 49 two-pass
    (3, 24, False, 6, {"SLSHT_CUDA_FUSED": "1"}),     # n = 49 fused
    (2, 32, True, 5, {}),     # n = 65, real mode
    (1, 64, False, 3, {}),    # n = 129
    (1, 112, False, 2, {}),   # n = 225, runtime alpha pass
    (3, 10, False, 6, {}),    # n = 21, runtime-plan single-pass kernel
    (3, 24, False, 9, {"SLSHT_CUDA_TP_PIPE": "1", "SLSHT_CUDA_TP_CT": "5"}),   # k_tpipe<49, 0>
    (2, 32, True, 9, {"SLSHT_CUDA_TP_PIPE": "1", "SLSHT_CUDA_TP_FV": "1"}),    # k_tpipe<65, 1>
    (3, 24, True, 6, {"SLSHT_CUDA_QFFT_LEAN": "6"}),                           # k_qfft_lean<49>
    (2, 32, False, 5, {"SLSHT_CUDA_QFFT_LEAN": "4"}),                          # k_qfft_lean<65>
    (3, 24, True, 6, {"SLSHT_CUDA_QFFT_HALF": "6"}),                           # k_qfft_half<49>
    (2, 32, False, 5, {"SLSHT_CUDA_QFFT_HALF": "5"}),                          # k_qfft_half<65>
]


def coeffs(rng, L, real):
    c = rng.standard_normal((L + 1) ** 2) + 1j * rng.standard_normal((L + 1) ** 2)
    if real:  # f_{l,-m} = (-1)^m conj(f_{l,m})
        for l in range(L + 1):
            c[l * l + l] = c[l * l + l].real
            for m in range(1, l + 1):
                c[l * l + l - m] = (-1) ** m * np.conj(c[l * l + l + m])
    return c


def run_cases(indices=None):
    """{case: (digests, captured volumes, inverse)} for the selected cases."""
    rng = np.random.default_rng(7)
    out = {}
    for i, (L_f, L_h, real, lmax, knobs) in enumerate(CASES):
        f, h = coeffs(rng, L_f, real), coeffs(rng, L_h, real)
        if indices is not None and i not in indices:
            continue
        os.environ["SLSHT_CUDA_FUSED"] = "0"
        os.environ.update(knobs)
        try:
            with S.Plan(L_f, L_h, real_mode=real, lmax=lmax, ring_bytes=64 << 20) as p:
                d = p.forward_digests(f, h)
                d2, v = p.forward_capture(f, h, [(0, 0), (lmax, lmax)])
                inv = p.inverse(f, h, h[0], L_f)
                seen = []
                p.forward_sink(f, h, lambda l, m, vol: seen.append((l, m)))
        finally:
            for k in ["SLSHT_CUDA_FUSED", *knobs]:
                os.environ.pop(k, None)
        assert np.array_equal(d, d2) and len(seen) == len(set(seen))
        out[i] = (d, v, inv)
    return out


if __name__ == "__main__":
    res = run_cases()
    for i, (d, _, _) in res.items():
        print(f"case {i} {CASES[i]}: digests finite {bool(np.isfinite(d).all())}")
    S.delta_tables(16)
    S.delta_tables(180)  # global-memory workspace
    print("done (guard bands intact)" if os.environ.get("SLSHT_CUDA_GUARD") == "1" else "done")
