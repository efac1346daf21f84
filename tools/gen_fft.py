#!/usr/bin/env python3
"""Generate paper_1207_5558_b200/csrc/fft_radix.cuh: straight-line prime-radix DFT
butterflies for the in-shared-memory odd-length FFT of the alpha axis.

Each butterfly is the symmetric form of a prime-length DFT
    y_k = x_0 + sum_{j=1}^{H} [ (x_j + x_{R-j}) cos(2 pi jk/R) - i (x_j - x_{R-j}) sin(2 pi jk/R) ]
with H = (R-1)/2, which needs (R-1)^2 real FMAs instead of 4 R^2. The cosines/sines are
emitted as literals (17 significant digits) so nvcc places them in the constant bank.

For R >= 11 a second form, dft_sink, streams each output to a callback as soon as it is
formed and splits every sum over two FMA chains: the last (twiddle-free) DIF stage stores
straight to shared memory without keeping all R outputs in registers.

Usage: python tools/gen_fft.py  (rewrites the header in place).
"""
from __future__ import annotations

import math
from pathlib import Path

PRIMES = [3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43]
SINK_MIN = 11  # radices that also get the streaming-output dft_sink
OUT = Path(__file__).resolve().parents[1] / "paper_1207_5558_b200" / "csrc" / "fft_radix.cuh"


def lit(v: float) -> str:
    if abs(v) < 1e-300:
        return "0.0"
    return repr(float(v))


def gen(R: int) -> str:
    H = (R - 1) // 2
    L = []
    L.append(f"template <> struct Radix<{R}> {{")
    L.append("  static constexpr bool kSupported = true;")
    L.append("  __device__ __forceinline__ static void dft(double* xr, double* xi) {")
    for j in range(1, H + 1):
        L.append(f"    const double sr{j} = xr[{j}] + xr[{R - j}], si{j} = xi[{j}] + xi[{R - j}];")
        L.append(f"    const double dr{j} = xr[{j}] - xr[{R - j}], di{j} = xi[{j}] - xi[{R - j}];")
    L.append("    const double x0r = xr[0], x0i = xi[0];")
    sum_r = " + ".join(f"sr{j}" for j in range(1, H + 1))
    sum_i = " + ".join(f"si{j}" for j in range(1, H + 1))
    L.append(f"    xr[0] = x0r + ({sum_r});")
    L.append(f"    xi[0] = x0i + ({sum_i});")
    for k in range(1, H + 1):
        ar = "x0r"
        ai = "x0i"
        br = None
        bi = None
        for j in range(1, H + 1):
            c = math.cos(2.0 * math.pi * j * k / R)
            s = math.sin(2.0 * math.pi * j * k / R)
            ar = f"fma(sr{j}, {lit(c)}, {ar})"
            ai = f"fma(si{j}, {lit(c)}, {ai})"
            br = f"di{j} * {lit(s)}" if br is None else f"fma(di{j}, {lit(s)}, {br})"
            bi = f"dr{j} * {lit(s)}" if bi is None else f"fma(dr{j}, {lit(s)}, {bi})"
        L.append("    {")
        L.append(f"      const double ar = {ar};")
        L.append(f"      const double ai = {ai};")
        L.append(f"      const double br = {br};")
        L.append(f"      const double bi = {bi};")
        L.append(f"      xr[{k}] = ar + br; xi[{k}] = ai - bi;")
        L.append(f"      xr[{R - k}] = ar - br; xi[{R - k}] = ai + bi;")
        L.append("    }")
    L.append("  }")
    if R >= SINK_MIN:
        L.extend(gen_sink(R))
    L.append("};")
    return "\n".join(L)


def gen_sink(R: int) -> list[str]:
    """dft_sink: the same DFT, each output pair handed to out(k, re, im) as soon as it is
    formed (outputs never all live at once), every sum split over two FMA chains (even and odd
    j) for instruction-level parallelism."""
    H = (R - 1) // 2
    L = ["  template <class F>",
         "  __device__ __forceinline__ static void dft_sink(const double* xr, const double* xi, F&& out) {"]
    for j in range(1, H + 1):
        L.append(f"    const double sr{j} = xr[{j}] + xr[{R - j}], si{j} = xi[{j}] + xi[{R - j}];")
        L.append(f"    const double dr{j} = xr[{j}] - xr[{R - j}], di{j} = xi[{j}] - xi[{R - j}];")
    L.append("    const double x0r = xr[0], x0i = xi[0];")
    ev = [j for j in range(1, H + 1) if j % 2 == 0]
    od = [j for j in range(1, H + 1) if j % 2 == 1]
    L.append(f"    out(0, (x0r + ({' + '.join(f'sr{j}' for j in od)})) + ({' + '.join(f'sr{j}' for j in ev)}),"
             f" (x0i + ({' + '.join(f'si{j}' for j in od)})) + ({' + '.join(f'si{j}' for j in ev)}));")

    def chain(js, v, k, trig, init):
        e = init
        for j in js:
            t = trig(2.0 * math.pi * j * k / R)
            e = f"{v}{j} * {lit(t)}" if e is None else f"fma({v}{j}, {lit(t)}, {e})"
        return e

    for k in range(1, H + 1):
        L.append("    {")
        L.append(f"      const double ar = {chain(od, 'sr', k, math.cos, 'x0r')} + {chain(ev, 'sr', k, math.cos, None)};")
        L.append(f"      const double ai = {chain(od, 'si', k, math.cos, 'x0i')} + {chain(ev, 'si', k, math.cos, None)};")
        L.append(f"      const double br = {chain(od, 'di', k, math.sin, None)} + {chain(ev, 'di', k, math.sin, None)};")
        L.append(f"      const double bi = {chain(od, 'dr', k, math.sin, None)} + {chain(ev, 'dr', k, math.sin, None)};")
        L.append(f"      out({k}, ar + br, ai - bi);")
        L.append(f"      out({R - k}, ar - br, ai + bi);")
        L.append("    }")
    L.append("  }")
    return L


def main() -> None:
    parts = [
        "// GENERATED by tools/gen_fft.py — do not edit by hand.",
        "// Prime-radix DFT butterflies y_k = sum_j x_j exp(-2 pi i jk/R), in place, natural order.",
        "#pragma once",
        "",
        "namespace slsht_cuda {",
        "",
        "template <int R> struct Radix { static constexpr bool kSupported = false; };",
        "",
    ]
    for R in PRIMES:
        parts.append(gen(R))
        parts.append("")
    parts.append(f"constexpr int kMaxGeneratedRadix = {max(PRIMES)};")
    parts.append(f"constexpr int kSinkMinRadix = {SINK_MIN};")
    parts.append("")
    parts.append("}  // namespace slsht_cuda")
    OUT.write_text("\n".join(parts) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
