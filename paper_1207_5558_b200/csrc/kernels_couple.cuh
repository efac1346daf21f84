// The coupling stage: one CTA owns 8*MG components x 8*NG grid columns
// (b, c) of the SO(3) volume and ALL q, and produces the final samples:
//
//   phase 1  T[comp][q][col] = sum_{p>=|q|} U[comp][(p,q)] W[(p,q)][col]
//            on the FP64 tensor cores (DMMA 8x8x4; complex product as 4 real MMAs), operands
//            streamed from L2 through a per-warp register ring of D k-steps;
//   phase 2  in-place mixed-radix DIF FFT over q in shared memory (alpha axis), prime
//            butterflies from fft_radix.cuh, compile-time plan for the BASELINE lengths;
//   phase 3  g[a][col] = e^{2 pi i L a/n} T[perm(a)] streamed to the output slot (and the
//            conjugate mirror (l, -m) in real mode) with st.global.cs, while the digest
//            partials (sum |g|^2, max |g|^2, sum w g, g000, sum q(beta) g) are accumulated.
//
// U = conj(mod) comes from k_modgemm; W is the window table of k_wtab, so the beta and gamma
// sums of the reference's 3-D evaluation (transform.cpp:88-135) were already applied once per
// run and only the alpha axis is transformed per component.
#pragma once

#include "common.cuh"
#include "fft_radix.cuh"

namespace slsht_cuda {

struct CoupleParams {
  const double2* U;
  const double2* W;
  double2* out;
  double* partials;  // [comp][col tile][8]
  const CompRec* comps;
  int count;
  int L, n, nb, ncol, NPQ, n_col_tiles;
  long long vol;
  int mirror;  // real mode && emit_negative_m
  const int* qoff;
  const double2* rou;
  const int* perm;
  const double2* phase;
  const double* betaw;
  FftPlan fft;
  int generic_dft;  // runtime path: n has a prime factor above kMaxGeneratedRadix
};

constexpr int smallest_prime_factor(int n) {
  for (int p = 3; p * p <= n; p += 2)
    if (n % p == 0) return p;
  return n;
}

// One DIF stage of radix R on sub-transforms of span S (compile-time N), executed by the
// NTHR threads numbered tid = 0..NTHR-1. SINK: the twiddle-free last stage of a radix with a
// streaming butterfly (Radix<R>::dft_sink) stores each output as soon as it is formed.
template <int N, int R, int S, int NT, int PAIRS, int NTHR, bool SINK = false, int TS = NT>
__device__ __forceinline__ void fft_stage_ct(double2* T, const double2* rou_s, int tid) {
  // TS: row stride of the tile in shared memory (NT unless padded against bank conflicts)
  constexpr int MP = S / R;
  constexpr int TOTAL = PAIRS * (N / R);
  double xr[R], xi[R];
  for (int item = tid; item < TOTAL; item += NTHR) {
    const int pair = item % PAIRS;
    const int bfl = item / PAIRS;
    const int blk = bfl / MP, t = bfl % MP;
    const int comp = pair / NT, col = pair % NT;
    double2* base = T + (size_t)(comp * N + blk * S + t) * TS + col;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double2 v = base[k * MP * TS];
      xr[k] = v.x;
      xi[k] = v.y;
    }
    if constexpr (SINK && MP == 1 && R >= kSinkMinRadix) {
      Radix<R>::dft_sink(xr, xi, [&](int k, double yr, double yi) {
        base[k * TS] = make_double2(yr, yi);
      });
      continue;
    }
    Radix<R>::dft(xr, xi);
    base[0] = make_double2(xr[0], xi[0]);
    if (MP == 1 || t == 0) {
#pragma unroll
      for (int k = 1; k < R; ++k) base[k * MP * TS] = make_double2(xr[k], xi[k]);
    } else {
#pragma unroll
      for (int k = 1; k < R; ++k) {
        const double2 w = rou_s[t * k * (N / S)];
        base[k * MP * TS] = make_double2(xr[k] * w.x - xi[k] * w.y, xr[k] * w.y + xi[k] * w.x);
      }
    }
  }
}

__device__ __forceinline__ void stage_sync(int bar, int count) {
  if (bar == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "r"(count) : "memory");
}

// Full DIF plan: radices = prime factors of N in ascending order (the host's perm matches).
// bar 0 synchronizes the whole CTA, bar > 0 only the NTHR participating threads.
template <int N, int S, int NT, int PAIRS, int NTHR, bool SINK = false>
struct FftDif {
  __device__ __forceinline__ static void run(double2* T, const double2* rou_s, int tid, int bar) {
    constexpr int R = smallest_prime_factor(S);
    static_assert(Radix<R>::kSupported, "no generated butterfly for this radix");
    fft_stage_ct<N, R, S, NT, PAIRS, NTHR, SINK>(T, rou_s, tid);
    stage_sync(bar, NTHR);
    FftDif<N, S / R, NT, PAIRS, NTHR, SINK>::run(T, rou_s, tid, bar);
  }
};
template <int N, int NT, int PAIRS, int NTHR, bool SINK>
struct FftDif<N, 1, NT, PAIRS, NTHR, SINK> {
  __device__ __forceinline__ static void run(double2*, const double2*, int, int) {}
};

// Runtime-length stage (any odd n whose prime factors have generated butterflies).
template <int R>
__device__ __forceinline__ void fft_stage_rt(double2* T, int NT, int n, int P, int span,
                                             const double2* rou_s, int nthr) {
  const int mp = span / R;
  const int total = P * (n / R);
  double xr[R], xi[R];
  for (int item = threadIdx.x; item < total; item += nthr) {
    const int pair = item % P;
    const int bfl = item / P;
    const int blk = bfl / mp, t = bfl % mp;
    const int comp = pair / NT, col = pair % NT;
    double2* base = T + (size_t)(comp * n + blk * span + t) * NT + col;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const double2 v = base[(size_t)k * mp * NT];
      xr[k] = v.x;
      xi[k] = v.y;
    }
    Radix<R>::dft(xr, xi);
    const int step = t * (n / span);
    base[0] = make_double2(xr[0], xi[0]);
#pragma unroll
    for (int k = 1; k < R; ++k) {
      double yr = xr[k], yi = xi[k];
      if (t != 0) {
        const double2 w = rou_s[step * k];
        const double tr = yr * w.x - yi * w.y;
        yi = yr * w.y + yi * w.x;
        yr = tr;
      }
      base[(size_t)k * mp * NT] = make_double2(yr, yi);
    }
  }
}

__device__ __forceinline__ void fft_runtime(double2* T, int NT, int n, int P, const FftPlan& fp,
                                            const double2* rou_s, int nthr) {
  for (int s = 0; s < fp.nstages; ++s) {
    const int R = fp.radix[s], span = fp.span[s];
    switch (R) {
      case 3: fft_stage_rt<3>(T, NT, n, P, span, rou_s, nthr); break;
      case 5: fft_stage_rt<5>(T, NT, n, P, span, rou_s, nthr); break;
      case 7: fft_stage_rt<7>(T, NT, n, P, span, rou_s, nthr); break;
      case 11: fft_stage_rt<11>(T, NT, n, P, span, rou_s, nthr); break;
      case 13: fft_stage_rt<13>(T, NT, n, P, span, rou_s, nthr); break;
      case 17: fft_stage_rt<17>(T, NT, n, P, span, rou_s, nthr); break;
      case 19: fft_stage_rt<19>(T, NT, n, P, span, rou_s, nthr); break;
      case 23: fft_stage_rt<23>(T, NT, n, P, span, rou_s, nthr); break;
      case 29: fft_stage_rt<29>(T, NT, n, P, span, rou_s, nthr); break;
      case 31: fft_stage_rt<31>(T, NT, n, P, span, rou_s, nthr); break;
      case 37: fft_stage_rt<37>(T, NT, n, P, span, rou_s, nthr); break;
      case 41: fft_stage_rt<41>(T, NT, n, P, span, rou_s, nthr); break;
      case 43: fft_stage_rt<43>(T, NT, n, P, span, rou_s, nthr); break;
      default: break;
    }
    __syncthreads();
  }
}

// Shared-memory footprint of k_couple (host and device agree on this layout).
__host__ __device__ constexpr size_t couple_t_bytes(int n, int MG, int NG) {
  // T tile, reused afterwards as the digest-reduction scratch (<= 512 threads x 8 doubles)
  return ((size_t)64 * MG * NG * n * 16 > 512 * 8 * 8) ? (size_t)64 * MG * NG * n * 16
                                                        : (size_t)512 * 8 * 8;
}

// Exact w = x 2^-24 - 0.5 for an integer 0 <= x < 2^24 without an I2F: the double with the
// bit pattern 0x43300000:x is 2^52 + x, and the FMA below is exact.
__device__ __forceinline__ double digest_weight(uint32_t hsh) {
  const double d = __hiloint2double(0x43300000, (int)(hsh >> 8));
  return fma(d, 1.0 / 16777216.0, -(268435456.0 + 0.5));
}

template <int N_CT, int MG, int NG, int NTHR, int MINB>
__global__ void __launch_bounds__(NTHR, MINB) k_couple(const CoupleParams P) {
  constexpr int NT = 8 * NG;        // grid columns per CTA
  constexpr int MT = 8 * MG;        // components per CTA
  constexpr int WT = MG * NG;       // 8x8 warp tiles
  constexpr int QS = (NTHR / 32) / WT;  // q split across warps
  constexpr int PAIRS = MT * NT;    // (comp, col) transforms per CTA
  constexpr int D = 65536 / (NTHR * MINB) < 100 ? 4 : (65536 / (NTHR * MINB) >= 200 ? 24 : 12);  // register prefetch depth (k-steps)
  static_assert((NTHR / 32) % WT == 0, "warp tiles must divide the warps");
  static_assert(NTHR % PAIRS == 0, "pairs must divide the block");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = N_CT > 0 ? N_CT : P.n;
  const int L = (n - 1) / 2;
  double2* T = reinterpret_cast<double2*>(smem_raw);
  double2* rou_s = reinterpret_cast<double2*>(smem_raw + couple_t_bytes(n, MG, NG));
  double2* phase_s = rou_s + n;
  double* betaw_s = reinterpret_cast<double*>(phase_s + n);
  int* perm_s = reinterpret_cast<int*>(betaw_s + (L + 1));
  int* qoff_s = perm_s + n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ct = blockIdx.x;
  const int comp0 = blockIdx.y * MT;
  const int col0 = ct * NT;
  for (int i = tid; i < n; i += NTHR) {
    rou_s[i] = P.rou[i];
    phase_s[i] = P.phase[i];
    perm_s[i] = P.perm[i];
  }
  for (int i = tid; i <= n; i += NTHR) qoff_s[i] = P.qoff[i];
  for (int i = tid; i <= L; i += NTHR) betaw_s[i] = P.betaw[i];
  __syncthreads();

  // ---------------- phase 1: coupling over p on the tensor cores
  {
    const int wt = warp % WT, qs = warp / WT;
    const int mg = wt / NG, ng = wt % NG;
    const int a_comp = comp0 + mg * 8 + (lane >> 2);
    const bool a_ok = a_comp < P.count;
    const int b_col = col0 + ng * 8 + (lane >> 2);
    const bool b_ok = b_col < P.ncol;
    const double2* __restrict__ Ub = P.U + (size_t)(a_ok ? a_comp : 0) * P.NPQ;
    const double2* __restrict__ Wb = P.W + (b_ok ? b_col : 0);
    const size_t ncol = (size_t)P.ncol;
    const int kl = lane & 3;
    const int crow = mg * 8 + (lane >> 2);
    const int ccol = ng * 8 + 2 * kl;
    // Complex product with three real MMAs (Gauss): K1 += (ar+ai) br, K2 += ar (bi-br),
    // K3 += ai (br+bi); re = K1 - K3, im = K1 + K2. The two extra adds per operand run on the
    // FP64 ALU while the tensor pipe does 3 instead of 4 DMMAs. Three independent chains.
    double c1[2], c2[2], c3[2];
    auto reset = [&]() { c1[0] = c1[1] = c2[0] = c2[1] = c3[0] = c3[1] = 0.0; };
    auto mma4 = [&](const double2& a, const double2& b) {
      dmma(c1[0], c1[1], a.x + a.y, b.x);
      dmma(c2[0], c2[1], a.x, b.y - b.x);
      dmma(c3[0], c3[1], a.y, b.x + b.y);
    };
    // T row = q mod n (q = jq - L): the alpha sum sum_q e^{-i q alpha_a} T_q is then a plain
    // length-n DFT of the rows, so no output phase shift is needed (transform.cpp:81-85).
    auto store = [&](int jq) {
      const int row = jq >= L ? jq - L : jq + L + 1;
      double2* dst = T + (size_t)(crow * n + row) * NT + ccol;
      dst[0] = make_double2(c1[0] - c3[0], c1[0] + c2[0]);
      dst[1] = make_double2(c1[1] - c3[1], c1[1] + c2[1]);
    };
    constexpr int KMAX = N_CT > 0 ? ((N_CT - 1) / 2 + 1 + 3) / 4 : 0;
    if constexpr (N_CT > 0 && KMAX <= 5) {
      // per-q fully unrolled k-steps, operands of the next q prefetched into a second buffer
      double2 A0[KMAX], B0[KMAX], A1[KMAX], B1[KMAX];
      auto load_q = [&](int jq, double2* A, double2* B) {
        const int np = L + 1 - abs(jq - L);
        const int cb = qoff_s[jq];
#pragma unroll
        for (int ks = 0; ks < KMAX; ++ks) {
          const int k = 4 * ks + kl;
          A[ks] = make_double2(0.0, 0.0);
          B[ks] = make_double2(0.0, 0.0);
          if (k < np) {
            if (a_ok) A[ks] = __ldg(Ub + cb + k);
            if (b_ok) B[ks] = __ldg(Wb + (size_t)(cb + k) * ncol);
          }
        }
      };
      auto run_q = [&](int jq, const double2* A, const double2* B) {
        const int np = L + 1 - abs(jq - L);
        reset();
#pragma unroll
        for (int ks = 0; ks < KMAX; ++ks)
          if (4 * ks < np) mma4(A[ks], B[ks]);
        store(jq);
      };
      if (qs < n) load_q(qs, A0, B0);
      for (int jq = qs; jq < n; jq += 2 * QS) {
        if (jq + QS < n) load_q(jq + QS, A1, B1);
        run_q(jq, A0, B0);
        if (jq + QS >= n) break;
        if (jq + 2 * QS < n) load_q(jq + 2 * QS, A0, B0);
        run_q(jq + QS, A1, B1);
      }
    } else {
      // generic lengths: flattened (q, k-step) stream with a register ring of D k-steps
      int ljq = qs, lks = 0;
      int lnp = (qs < n) ? L + 1 - abs(qs - L) : 0;
      int lcb = (qs < n) ? qoff_s[qs] : 0;
      auto issue = [&](double2& a, double2& b) {
        a = make_double2(0.0, 0.0);
        b = make_double2(0.0, 0.0);
        if (ljq < n) {
          const int k = 4 * lks + kl;
          if (k < lnp) {
            if (a_ok) a = __ldg(Ub + lcb + k);
            if (b_ok) b = __ldg(Wb + (size_t)(lcb + k) * ncol);
          }
          if (4 * (++lks) >= lnp) {
            ljq += QS;
            lks = 0;
            if (ljq < n) {
              lnp = L + 1 - abs(ljq - L);
              lcb = qoff_s[ljq];
            }
          }
        }
      };
      double2 ra[D], rb[D];
#pragma unroll
      for (int i = 0; i < D; ++i) issue(ra[i], rb[i]);
      int ujq = qs, uks = 0;
      int unp = (qs < n) ? L + 1 - abs(qs - L) : 0;
      reset();
      while (ujq < n) {
#pragma unroll
        for (int i = 0; i < D; ++i) {
          if (ujq < n) {
            mma4(ra[i], rb[i]);
            issue(ra[i], rb[i]);
            if (4 * (++uks) >= unp) {
              store(ujq);
              reset();
              ujq += QS;
              uks = 0;
              unp = L + 1 - abs(ujq - L);
            }
          }
        }
      }
    }
  }
  __syncthreads();

  // ---------------- phase 2: alpha FFT over q, in place
  if constexpr (N_CT > 0) {
    FftDif<N_CT, N_CT, NT, PAIRS, NTHR>::run(T, rou_s, threadIdx.x, 0);
  } else {
    if (!P.generic_dft) fft_runtime(T, NT, n, PAIRS, P.fft, rou_s, NTHR);
  }

  // ---------------- phase 3: epilogue (phase shift, stores, mirror, digest partials)
  const int pair = tid % PAIRS;
  const int cl = pair / NT, cc = pair % NT;
  const int comp = comp0 + cl, col = col0 + cc;
  const bool ok = comp < P.count && col < P.ncol;
  double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
  long long mx2 = 0;
  if (ok) {
    const CompRec rec = P.comps[comp];
    double2* o = P.out + rec.slot * P.vol + col;
    double2* om = (P.mirror && rec.m > 0) ? P.out + rec.mslot * P.vol + col : nullptr;
    const long long sbit = (long long)0x8000000000000000ULL;
    const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
    const double qb = betaw_s[col / n];
    const double2* Tp = T + (size_t)cl * n * NT + cc;
    const bool generic = (N_CT == 0) && P.generic_dft;
    const int a_first = tid / PAIRS;
    constexpr int A_STEP = NTHR / PAIRS;
    uint32_t hsh = (uint32_t)((size_t)a_first * P.ncol + col) * 0x9E3779B1u;
    const uint32_t hstep = (uint32_t)((size_t)A_STEP * P.ncol) * 0x9E3779B1u;
    if (a_first == 0 && col == 0) {
      if (!generic) {
        const double2 t = Tp[(size_t)perm_s[0] * NT];
        g0r = t.x;
        g0i = t.y;
      }
    }
    for (int a = a_first; a < n; a += A_STEP, hsh += hstep) {
      double vr, vi;
      if (!generic) {
        const double2 t = Tp[(size_t)perm_s[a] * NT];
        vr = t.x;
        vi = t.y;
      } else {
        // dense DFT for lengths with a prime factor above the generated radices
        double sr = 0.0, si = 0.0;
        int e = 0;
        for (int j = 0; j < n; ++j) {
          const double2 t = Tp[(size_t)j * NT];
          const double2 w = rou_s[e];
          sr += t.x * w.x - t.y * w.y;
          si += t.x * w.y + t.y * w.x;
          e += a;
          if (e >= n) e -= n;
        }
        vr = sr;
        vi = si;
      }
      const size_t idx = (size_t)a * P.ncol;
      __stcs(o + idx, make_double2(vr, vi));
      if (om) {
        // (-1)^m conj(g) by sign-bit flips (transform.cpp:60-66), off the FP64 pipe
        const long long br = __double_as_longlong(vr) ^ mflip_r;
        const long long bi = __double_as_longlong(vi) ^ mflip_i;
        __stcs(om + idx, make_double2(__longlong_as_double(br), __longlong_as_double(bi)));
      }
      const double a2 = fma(vr, vr, vi * vi);
      s2 += a2;
      mx2 = max(mx2, __double_as_longlong(a2));  // a2 >= 0: integer order == double order
      const double wgt = digest_weight(hsh);
      pr = fma(wgt, vr, pr);
      pi = fma(wgt, vi, pi);
      ir += vr;
      ii += vi;
      if (generic && a == 0 && col == 0) {
        g0r = vr;
        g0i = vi;
      }
    }
    ir *= qb;
    ii *= qb;
  }
  __syncthreads();  // T is reused as the reduction scratch
  double* red = reinterpret_cast<double*>(smem_raw);
  red[tid * 8 + 0] = s2;
  red[tid * 8 + 1] = __longlong_as_double(mx2);
  red[tid * 8 + 2] = pr;
  red[tid * 8 + 3] = pi;
  red[tid * 8 + 4] = g0r;
  red[tid * 8 + 5] = g0i;
  red[tid * 8 + 6] = ir;
  red[tid * 8 + 7] = ii;
  __syncthreads();
  if (tid < MT * 8) {
    // thread (component c = tid/8, field k = tid%8) sums the threads of component c in order
    const int c = tid >> 3, k = tid & 7;
    if (comp0 + c < P.count) {
      double acc = 0.0;
      for (int t = c * NT; t < NTHR; t += PAIRS)
        for (int u = 0; u < NT; ++u) {
          const double v = red[(t + u) * 8 + k];
          acc = (k == 1) ? fmax(acc, v) : acc + v;
        }
      P.partials[((size_t)(comp0 + c) * P.n_col_tiles + ct) * 8 + k] = acc;
    }
  }
}

}  // namespace slsht_cuda
