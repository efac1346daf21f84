// Two-pass coupling for the long transforms (n = 49, 65, 129):
//
//   k_tgemm  T[comp][q mod n][col] = sum_{p>=|q|} U[comp][(p,q)] W[(p,q)][col]
//            one batched complex GEMM per q on the FP64 tensor cores (DMMA 8x8x4, Gauss
//            3-product), 64 components x 32 columns per CTA (three CTAs per SM), every q of the
//            tile in one pass over the q-major (p, q) rows (each q padded to whole k-steps of
//            4), operands staged in shared memory by a cp.async ring. T goes to an HBM buffer.
//   k_qfft   reads T[comp][*][32 columns], runs the length-n alpha DIF FFT in shared memory
//            (fft_radix.cuh butterflies; for n = 129 the radix-43 stage on the tensor cores)
//            and writes the So3Volume rows (and the real-mode mirror) with the digest partials.
//
// Why two passes: the single-pass k_couple must keep all n rows of its T tile on chip, which
// caps its tile at 8 components x 8 columns for n = 129 (132 KB); each operand byte then
// feeds only 8 MACs, and the DMMA loop runs L2-bound at ~16% of the tensor pipe
// (profiles/r01_ncu_couple_c5_singlepass.txt). The T round trip costs 32 B of extra HBM
// traffic per sample, but frees the GEMM tile (8x the operand reuse).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "kernels_chunk.cuh"
#include "kernels_couple.cuh"

namespace slsht_cuda {

constexpr int TG_BM = 64;      // components per CTA
constexpr int TG_KS = 16;      // (p, q) rows per pipeline stage (4 k-steps)
constexpr int TG_ASTR = 20;    // A row stride (complex): == 4 mod 8, conflict-free fragments
// B row stride (complex) BN + 2 == 2 mod 8: conflict-free fragments

struct TgParams {
  const double2* U;      // [comp][KP]: q-major padded (p, q) rows, zero padding; KP % TG_KS == 0
  const double2* W;      // [KP][ncolp]
  double2* T;            // [comp][n][ncolp]
  const short* qend;     // per k-step: T row (q mod n) completed by it, or -1
  int count, KP, ncolp, n;
  int ustride;           // row stride of U (complex); KP may cover a sub-range of the rows
  int col_fast;          // 1: blockIdx.x = column tile (W L2-resident, U block read once)
  int t_stream;          // 1: T stored with the evict-first (.cs) hint; 2 (builds with -DSLSHT_TG_NOSTORE): no T stores
};

__host__ __device__ constexpr int tgemm_threads(int BN, int WNF, int BM = TG_BM) {
  return 32 * (BM / 32) * (BN / (8 * WNF));
}
__host__ __device__ constexpr size_t tgemm_smem_bytes(int KP, int BN, int NST, int BM = TG_BM) {
  return (size_t)NST * (BM * TG_ASTR + TG_KS * (BN + 2)) * 16 + (size_t)(KP / 4) * 2 + 16;
}

// 256-bit global store (sm_100): two consecutive complex values
__device__ __forceinline__ void st_global_v4(double2* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}
// the same with the streaming (evict-first) hint
__device__ __forceinline__ void st_global_cs_v4(double2* p, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c),
               "d"(d)
               : "memory");
}

// Warp tile 32 components x 8 WNF columns; BN columns per CTA, TG_NST pipeline stages.
// <32, 2, 2, 3> (default): 4 warps, two stages, three independent CTAs per SM (156 registers).
// <64, 2, 4, 1>: 8 warps, one CTA per SM. <32, 2, 3, 2>: 4 warps, two CTAs per SM.
// <32, 2, 4, 1>: 4 warps (117 KB), which leaves room on the SM for one k_qfft CTA of the
// previous chunk (the overlapped schedule).
template <int BN, int WNF, int TG_NST, int MINB, int BM = TG_BM>
__global__ void __launch_bounds__(tgemm_threads(BN, WNF, BM), MINB) k_tgemm(const TgParams P) {
  constexpr int TG_THREADS = tgemm_threads(BN, WNF, BM), TG_BSTR = BN + 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + TG_NST * BM * TG_ASTR;
  short* qend_s = reinterpret_cast<short*>(Bs + TG_NST * TG_KS * TG_BSTR);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // raster (host-chosen, TgParams::col_fast): with a large W (config 5: 0.6 GB) grid x is the
  // component block, so the CTAs in flight share a few W column tiles; with an L2-resident W
  // (configs 3-4: <= 40 MB) grid x is the column tile, so the CTAs in flight share one U block
  // and every U byte is read from HBM once per chunk
  const int bx = P.col_fast ? blockIdx.y : blockIdx.x, by = P.col_fast ? blockIdx.x : blockIdx.y;
  const int comp0 = bx * BM, col0 = by * BN;
  const int nks = P.KP / 4, nst = (P.KP + TG_KS - 1) / TG_KS;
  for (int i = tid; i < nks; i += TG_THREADS) qend_s[i] = P.qend[i];

  auto load_stage = [&](int st) {
    if (st < nst) {
      const int kb = st * TG_KS;
      double2* Ad = As + (st % TG_NST) * BM * TG_ASTR;
      double2* Bd = Bs + (st % TG_NST) * TG_KS * TG_BSTR;
#pragma unroll
      for (int j = 0; j < BM * TG_KS / TG_THREADS; ++j) {
        const int e = tid + j * TG_THREADS;
        const int c = e / TG_KS, k = e % TG_KS;
        const bool ok = comp0 + c < P.count && kb + k < P.KP;
        cp_async16(Ad + c * TG_ASTR + k, P.U + (ok ? (size_t)(comp0 + c) * P.ustride + kb + k : 0), ok);
      }
#pragma unroll
      for (int j = 0; j < TG_KS * BN / TG_THREADS; ++j) {
        const int e = tid + j * TG_THREADS;
        const int k = e / BN, c = e % BN;
        const bool ok = kb + k < P.KP;
        cp_async16(Bd + k * TG_BSTR + c, P.W + (ok ? (size_t)(kb + k) * P.ncolp + col0 + c : 0), ok);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < TG_NST - 1; ++s) load_stage(s);

  // warp tile: 32 components (4 MMA rows) x 16 columns (2 MMA columns)
  constexpr int WN = BN / (8 * WNF);
  const int wm = warp / WN, wn = warp % WN;
  const int arow = wm * 32 + (lane >> 2), acol = lane & 3;
  const int brow = lane & 3, bcol = wn * 8 * WNF + (lane >> 2);
  double c1[4][WNF][2], c2[4][WNF][2], c3[4][WNF][2];
  auto reset = [&]() {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < WNF; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) c1[mi][ni][e] = c2[mi][ni][e] = c3[mi][ni][e] = 0.0;
  };
  reset();
  const int scomp = comp0 + wm * 32 + (lane >> 2);
  const int scol = col0 + wn * 8 * WNF + 2 * (lane & 3);
  // T address of the thread's first component row; rows mi 8 further are tstep elements on
  double2* const tbase = P.T + (size_t)scomp * P.n * P.ncolp + scol;
  const size_t tstep = (size_t)8 * P.n * P.ncolp;

  for (int st = 0; st < nst; ++st) {
    cp_async_wait<TG_NST - 2>();
    __syncthreads();
    load_stage(st + TG_NST - 1);  // refills the buffer consumed at st - 1 (all warps passed it)
    const double2* Ab = As + (st % TG_NST) * BM * TG_ASTR;
    const double2* Bb = Bs + (st % TG_NST) * TG_KS * TG_BSTR;
#pragma unroll
    for (int kk = 0; kk < TG_KS / 4; ++kk) {
      const int ks = st * (TG_KS / 4) + kk;  // KP is a multiple of TG_KS: no partial stage
      double2 a[4], b[WNF];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = Ab[(arow + mi * 8) * TG_ASTR + kk * 4 + acol];
#pragma unroll
      for (int ni = 0; ni < WNF; ++ni) b[ni] = Bb[(kk * 4 + brow) * TG_BSTR + bcol + ni * 8];
      // Gauss: K1 += (ar+ai) br, K2 += ar (bi-br), K3 += ai (br+bi); re = K1-K3, im = K1+K2
      double as[4], bd[WNF], bs[WNF];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) as[mi] = a[mi].x + a[mi].y;
#pragma unroll
      for (int ni = 0; ni < WNF; ++ni) {
        bd[ni] = b[ni].y - b[ni].x;
        bs[ni] = b[ni].x + b[ni].y;
      }
#pragma unroll
      for (int ni = 0; ni < WNF; ++ni)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) dmma(c1[mi][ni][0], c1[mi][ni][1], as[mi], b[ni].x);
#pragma unroll
      for (int ni = 0; ni < WNF; ++ni)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) dmma(c2[mi][ni][0], c2[mi][ni][1], a[mi].x, bd[ni]);
#pragma unroll
      for (int ni = 0; ni < WNF; ++ni)
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) dmma(c3[mi][ni][0], c3[mi][ni][1], a[mi].y, bs[ni]);
      const int row = qend_s[ks];
      if (row >= 0) {
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          const int comp = scomp + mi * 8;
#ifdef SLSHT_TG_NOSTORE  // timing builds only: the sweep without the q-end sums, addresses and stores
          if (comp < P.count && P.t_stream != 2) {
#else
          if (comp < P.count) {
#endif
            double2* dst = tbase + (size_t)mi * tstep + row * P.ncolp;
#pragma unroll
            for (int ni = 0; ni < WNF; ++ni) {  // 32 B per lane: 4 lanes write one whole 128-B line
              if (P.t_stream == 1)
                st_global_cs_v4(dst + ni * 8, c1[mi][ni][0] - c3[mi][ni][0],
                                c1[mi][ni][0] + c2[mi][ni][0], c1[mi][ni][1] - c3[mi][ni][1],
                                c1[mi][ni][1] + c2[mi][ni][1]);
              else
                st_global_v4(dst + ni * 8, c1[mi][ni][0] - c3[mi][ni][0],
                             c1[mi][ni][0] + c2[mi][ni][0], c1[mi][ni][1] - c3[mi][ni][1],
                             c1[mi][ni][1] + c2[mi][ni][1]);
            }
          }
        }
      }
      // branch-free reset (a conditional reset inside the branch makes the compiler route
      // every MMA result through register copies)
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < WNF; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            c1[mi][ni][e] = row >= 0 ? 0.0 : c1[mi][ni][e];
            c2[mi][ni][e] = row >= 0 ? 0.0 : c2[mi][ni][e];
            c3[mi][ni][e] = row >= 0 ? 0.0 : c3[mi][ni][e];
          }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------------------------
// Last DIF stage of N = 3 x 43 (k_qfft<129>) on the FP64 tensor cores. For each of the 3 NT
// length-43 sub-transforms (GEMM column n = blk NT + c), X_k = sum_j x_j w^{jk} in the
// symmetric form
//   X_k = (x0r + P1 + P3, x0i + P2 - P4),  X_{43-k} = (x0r + P1 - P3, x0i + P2 + P4),
//   P1 = C SR, P2 = C SI, P3 = S DI, P4 = S DR,  C_kj = cos(2 pi jk / 43), S_kj = sin(...),
// with s_j = x_j + x_{43-j}, d_j = x_j - x_{43-j} (j = 1..21) formed in place first. The four
// (k = 0..23) x (j = 1..24, zero-padded) by (j) x (8 columns) products of an 8-column tile are
// DMMA 8x8x4 chains; a warp owns its tiles' columns, so it writes the outputs in place. Same
// FP64 work as the scalar butterflies, but ~140 registers instead of 255 and every warp busy.
// A fragments of the cos / sin matrices, [cos|sin][mt < 3][ks < 6][lane]: row k = mt 8 + lane/4,
// column j = ks 4 + lane%4 + 1 (zero for j > 21 or k > 21). Filled once per plan.
__global__ void k_r43_table(double* __restrict__ tab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * 6 * 32) return;
  const int lane = i % 32, ks = (i / 32) % 6, mt = i / 192;
  const int k = mt * 8 + (lane >> 2), j = ks * 4 + (lane & 3) + 1;
  double sn = 0.0, cs = 0.0;
  if (j <= 21 && k <= 21) sincospi(2.0 * (double)((j * k) % 43) / 43.0, &sn, &cs);
  tab[i] = cs;
  tab[576 + i] = sn;
}

// First DIF stage of N = 129 (radix 3 with twiddles, as fft_stage_ct) fused with the sums and
// differences of the radix-43 stage: a thread takes the stage-1 items t and 43 - t of a column
// together, so every sub-transform's s_j, d_j land in place without another pass.
template <int NT, int TS, int NTHR>
__device__ __forceinline__ void radix3_with_sums(double2* T, const double2* rou_s, int tid) {
  constexpr int R = 43, H = 21;
  for (int e = tid; e < NT * (H + 1); e += NTHR) {
    const int c = e % NT, t = e / NT;  // t = 0: the x_0 rows; t = 1..21: the pairs (t, 43 - t)
    double yr[2][3], yi[2][3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = h ? R - t : t;
      if (h && t == 0) break;
      double2* base = T + (size_t)u * TS + c;
      double xr[3], xi[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double2 v = base[k * R * TS];
        xr[k] = v.x;
        xi[k] = v.y;
      }
      Radix<3>::dft(xr, xi);
      yr[h][0] = xr[0];
      yi[h][0] = xi[0];
#pragma unroll
      for (int k = 1; k < 3; ++k) {
        if (u == 0) {
          yr[h][k] = xr[k];
          yi[h][k] = xi[k];
        } else {
          const double2 w = rou_s[u * k];
          yr[h][k] = xr[k] * w.x - xi[k] * w.y;
          yi[h][k] = xr[k] * w.y + xi[k] * w.x;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // sub-transform k: rows k 43 + j
      double2* col = T + (size_t)(k * R) * TS + c;
      if (t == 0) {
        col[0] = make_double2(yr[0][k], yi[0][k]);
      } else {
        col[t * TS] = make_double2(yr[0][k] + yr[1][k], yi[0][k] + yi[1][k]);
        col[(R - t) * TS] = make_double2(yr[0][k] - yr[1][k], yi[0][k] - yi[1][k]);
      }
    }
  }
}

template <int NT, int TS, int NTHR>
__device__ __forceinline__ void radix43_dmma(double2* T, int tid, const double* __restrict__ tab) {
  // TS: tile row stride; TS == 2 (mod 8) keeps the 4 rows of a B fragment in distinct banks.
  // Expects rows j / 43 - j of every sub-transform to hold s_j / d_j (radix3_with_sums).
  constexpr int R = 43, H = 21, NTILE = 3 * NT / 8, NW = NTHR / 32;
  static_assert(NT % 8 == 0, "a column tile must stay inside one sub-transform");
  const int lane = tid & 31, warp = tid >> 5;
  double ca[3][6], sa[3][6];  // A fragments (k_r43_table)
#pragma unroll
  for (int mt = 0; mt < 3; ++mt)
#pragma unroll
    for (int ks = 0; ks < 6; ++ks) {
      ca[mt][ks] = __ldg(tab + (mt * 6 + ks) * 32 + lane);
      sa[mt][ks] = __ldg(tab + 576 + (mt * 6 + ks) * 32 + lane);
    }
  for (int nt = warp; nt < NTILE; nt += NW) {
    double pp[4][3][2];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int mt = 0; mt < 3; ++mt) pp[q][mt][0] = pp[q][mt][1] = 0.0;
    const int nb = nt * 8 + (lane >> 2);  // B fragment column
    const double2* colb = T + (size_t)((nb / NT) * R) * TS + nb % NT;
#pragma unroll
    for (int ks = 0; ks < 6; ++ks) {
      const int j = ks * 4 + (lane & 3) + 1;
      double2 sv = make_double2(0.0, 0.0), dv = make_double2(0.0, 0.0);
      if (j <= H) {
        sv = colb[j * TS];
        dv = colb[(R - j) * TS];
      }
#pragma unroll
      for (int mt = 0; mt < 3; ++mt) {
        dmma(pp[0][mt][0], pp[0][mt][1], ca[mt][ks], sv.x);
        dmma(pp[1][mt][0], pp[1][mt][1], ca[mt][ks], sv.y);
        dmma(pp[2][mt][0], pp[2][mt][1], sa[mt][ks], dv.y);
        dmma(pp[3][mt][0], pp[3][mt][1], sa[mt][ks], dv.x);
      }
    }
    // outputs: lane holds k = mt 8 + lane/4 of columns n = nt 8 + 2 (lane%4) + e
    double2 x0[2];
    double2* colo[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int n = nt * 8 + 2 * (lane & 3) + e;
      colo[e] = T + (size_t)((n / NT) * R) * TS + n % NT;
      x0[e] = colo[e][0];
    }
    __syncwarp();  // every lane read its x_0 (and its B fragments) before any write
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int mt = 0; mt < 3; ++mt) {
        const int k = mt * 8 + (lane >> 2);
        if (k > H) continue;
        const double p1 = pp[0][mt][e], p2 = pp[1][mt][e], p3 = pp[2][mt][e], p4 = pp[3][mt][e];
        if (k == 0) {
          colo[e][0] = make_double2(x0[e].x + p1, x0[e].y + p2);
        } else {
          colo[e][k * TS] = make_double2(x0[e].x + p1 + p3, x0[e].y + p2 - p4);
          colo[e][(R - k) * TS] = make_double2(x0[e].x + p1 - p3, x0[e].y + p2 + p4);
        }
      }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------------
// k_qfft: one component x NT grid columns per CTA.

struct QfParams {
  const double2* T;      // [comp][n][ncolp]
  double2* out;
  double* partials;      // [comp][tile][8]
  const CompRec* comps;
  int count, n, ncol, ncolp, n_tiles;
  long long vol;  // slot stride of out (complex elements)
  int rpitch;     // row stride of out: ncol rounded up to whole 128-B lines in the ring
  int mirror;
  const double2* rou;
  const int* perm;
  const double* betaw;
  const double* r43;  // k_r43_table (n = 129)
  FftPlan fft;        // k_qfft_rt: the runtime DIF plan (radices of n)
  int generic_dft;    // k_qfft_rt: n has a prime factor without a generated butterfly
  // T rows [rc_lo, rc_hi) (the q of at most KC coupling terms, |q| > L - KC) are not stored by
  // k_tgemm: k_qfft recomputes them from U and W (rc_k[r] terms from U row rc_urow[r])
  const double2* U;
  const double2* W;
  int ustride, rc_lo, rc_hi;
  short rc_urow[16];
  signed char rc_k[16];
};

// row stride of the k_qfft tile: padded to == 2 (mod 8) for the DMMA radix-43 stage (n = 129)
__host__ __device__ constexpr int qfft_row_stride(int n, int NT) { return n == 129 ? NT + 2 : NT; }
__host__ __device__ constexpr size_t qfft_smem_bytes(int n, int NT) {
  return (size_t)n * qfft_row_stride(n, NT) * 16 + (size_t)n * 16 + (size_t)((n + 1) / 2) * 8 +
         (size_t)n * 4 + 64;
}

// The tile load of the alpha pass, shared by k_qfft and k_qfft_half: asynchronous copies of the
// stored T rows of (comp, 32 columns) into Ts, and the rows k_tgemm left out recomputed from U, W.
template <int N, int NT, int NTHR, int TS>
__device__ __forceinline__ void qfft_load_tile(const QfParams& P, double2* Ts, int comp, int col0, int tid) {
    // The rows k_tgemm left out (at most KC terms each, summed in increasing p). With KC = 2 or 4
    // every thread owns KC / 2 (row, column) items (rows g and g + 4 of a thread group g pair a
    // long row with a short one): their operands are requested right after the tile's copies,
    // all at once, and used when they arrive; the general loop serves the other KC.
    const double2* Uc = P.U + (size_t)comp * P.ustride;
    const double2* src = P.T + (size_t)comp * N * P.ncolp + col0;
    // rows [0, rc_lo) and [rc_hi, N): two plain loops (rc_lo = rc_hi = 0 when every row is stored)
    const int e_lo = N == 129 ? 0 : P.rc_lo * NT, e_hi = N == 129 ? 0 : P.rc_hi * NT;
    for (int e = tid; e < e_lo; e += NTHR) {
      const int row = e / NT, c = e % NT;
      cp_async16(Ts + row * TS + c, src + (size_t)row * P.ncolp + c, true);
    }
    for (int e = e_hi + tid; e < N * NT; e += NTHR) {
      const int row = e / NT, c = e % NT;
      cp_async16(Ts + row * TS + c, src + (size_t)row * P.ncolp + c, true);
    }
    cp_async_commit();
    if constexpr (N != 129) {
      constexpr int GR = NTHR / NT;  // rows per item round
      const int nrc = P.rc_hi - P.rc_lo;
      auto owned = [&](auto it_tag) {
        constexpr int IT = decltype(it_tag)::value, MAXK = 2 * IT;
        double2 fu[IT][MAXK], fw[IT][MAXK];
        const int c = tid % NT;
#pragma unroll
        for (int i = 0; i < IT; ++i) {
          const int r = tid / NT + i * GR;
          const int urow = P.rc_urow[r], K = P.rc_k[r];
          const double2* wp = P.W + (size_t)urow * P.ncolp + col0 + c;
#pragma unroll
          for (int k = 0; k < MAXK; ++k) {
            fu[i][k] = fw[i][k] = make_double2(0.0, 0.0);
            if (k < K) {
              fu[i][k] = __ldg(Uc + urow + k);
              fw[i][k] = __ldg(wp + (size_t)k * P.ncolp);
            }
          }
        }
#pragma unroll
        for (int i = 0; i < IT; ++i) {  // (absent terms are zeros: exact)
          double ar = 0.0, ai = 0.0;
#pragma unroll
          for (int k = 0; k < MAXK; ++k) {
            ar = fma(fu[i][k].x, fw[i][k].x, ar);
            ar = fma(-fu[i][k].y, fw[i][k].y, ar);
            ai = fma(fu[i][k].x, fw[i][k].y, ai);
            ai = fma(fu[i][k].y, fw[i][k].x, ai);
          }
          Ts[(P.rc_lo + tid / NT + i * GR) * TS + c] = make_double2(ar, ai);
        }
      };
      if (nrc == GR) {
        owned(std::integral_constant<int, 1>{});
      } else if (nrc == 2 * GR) {
        owned(std::integral_constant<int, 2>{});
      } else {
        for (int e = tid; e < nrc * NT; e += NTHR) {
          const int r = e / NT, c = e % NT;
          const int urow = P.rc_urow[r], K = P.rc_k[r];
          const double2* wp = P.W + (size_t)urow * P.ncolp + col0 + c;
          double ar = 0.0, ai = 0.0;
          for (int k = 0; k < K; ++k) {
            const double2 u = __ldg(Uc + urow + k);
            const double2 w = __ldg(wp + (size_t)k * P.ncolp);
            ar = fma(u.x, w.x, ar);
            ar = fma(-u.y, w.y, ar);
            ai = fma(u.x, w.y, ai);
            ai = fma(u.y, w.x, ai);
          }
          Ts[(P.rc_lo + r) * TS + c] = make_double2(ar, ai);
        }
      }
    }
}

template <int N, int NT, int NTHR, int MINB>
__global__ void __launch_bounds__(NTHR, MINB) k_qfft(const QfParams P) {
  constexpr int L = (N - 1) / 2;
  // epilogue: (NTHR / NT) * NT threads own (column, row-set) pairs; the rest only reduce
  static_assert(NTHR >= NT, "threads must cover the columns");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ts = reinterpret_cast<double2*>(smem_raw);
  constexpr int TS = qfft_row_stride(N, NT);  // tile row stride
  double2* rou_s = Ts + N * TS;
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  int* perm_s = reinterpret_cast<int*>(betaw_s + (L + 1));
  const int tid = threadIdx.x;
  for (int i = tid; i < N; i += NTHR) {
    rou_s[i] = P.rou[i];
    perm_s[i] = P.perm[i];
  }
  for (int i = tid; i <= L; i += NTHR) betaw_s[i] = P.betaw[i];
  const int ct = blockIdx.x, comp = blockIdx.y;
  const int col0 = ct * NT;
  qfft_load_tile<N, NT, NTHR, TS>(P, Ts, comp, col0, tid);
  cp_async_wait<0>();
  __syncthreads();

  if constexpr (N == 129) {
    radix3_with_sums<NT, TS, NTHR>(Ts, rou_s, tid);
    __syncthreads();
    radix43_dmma<NT, TS, NTHR>(Ts, tid, P.r43);
    __syncthreads();
  } else {
    static_assert(TS == NT, "the generic DIF plan assumes an unpadded tile");
    FftDif<N, N, NT, NT, NTHR, true>::run(Ts, rou_s, tid, 0);
  }

  // epilogue: thread = (column cc, first row a_first); stores row by row (a warp writes 32
  // consecutive samples of one row), the mirror volume with sign flips, digest partials
  const int cc = tid % NT, col = col0 + cc;
  const bool ok = tid < (NTHR / NT) * NT && col < P.ncol;
  double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
  long long mx2 = 0;
  if (ok) {
    const CompRec rec = P.comps[comp];
    double2* o = P.out + rec.slot * P.vol + col;
    double2* om = (P.mirror && rec.m > 0) ? P.out + rec.mslot * P.vol + col : nullptr;
    const long long sbit = (long long)0x8000000000000000ULL;
    const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
    const double qb = betaw_s[col / N];
    const double2* Tp = Ts + cc;
    const int a_first = tid / NT;
    constexpr int A_STEP = NTHR / NT;
    uint32_t hsh = (uint32_t)((size_t)a_first * P.ncol + col) * 0x9E3779B1u;
    const uint32_t hstep = (uint32_t)((size_t)A_STEP * P.ncol) * 0x9E3779B1u;
    if (a_first == 0 && col == 0) {
      const double2 t = Tp[(size_t)perm_s[0] * TS];
      g0r = t.x;
      g0i = t.y;
    }
    auto rows = [&](auto mirror_tag) {
      constexpr bool MIR = decltype(mirror_tag)::value;
#pragma unroll 4
      for (int a = a_first; a < N; a += A_STEP, hsh += hstep) {
        const double2 t = Tp[(size_t)perm_s[a] * TS];
        const double vr = t.x, vi = t.y;
        const size_t idx = (size_t)a * P.rpitch;
        __stcs(o + idx, make_double2(vr, vi));
        if constexpr (MIR) {
          const long long br = __double_as_longlong(vr) ^ mflip_r;
          const long long bi = __double_as_longlong(vi) ^ mflip_i;
          __stcs(om + idx, make_double2(__longlong_as_double(br), __longlong_as_double(bi)));
        }
        const double a2 = fma(vr, vr, vi * vi);
        s2 += a2;
        mx2 = max(mx2, __double_as_longlong(a2));
        const double wgt = digest_weight(hsh);
        pr = fma(wgt, vr, pr);
        pi = fma(wgt, vi, pi);
        ir += vr;
        ii += vi;
      }
    };
    if (om) rows(std::true_type{});
    else rows(std::false_type{});
    ir *= qb;
    ii *= qb;
  }
  // fixed-order reduction: a shuffle tree per warp, then the warps in order. g000 is held by
  // thread 0 of the first column tile alone (a = 0, column 0), so it is written, not reduced.
  // digest fields reduced: 0..3 (s2, max, pr, pi) and 6, 7 (ir, ii)
  double v[6] = {s2, __longlong_as_double(mx2), pr, pi, ir, ii};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double o = __shfl_down_sync(0xffffffffu, v[k], off);
      v[k] = (k == 1) ? fmax(v[k], o) : v[k] + o;
    }
  __syncthreads();  // T is reused as the reduction scratch
  double* red = reinterpret_cast<double*>(smem_raw);
  if ((tid & 31) == 0)
#pragma unroll
    for (int k = 0; k < 6; ++k) red[(tid >> 5) * 6 + k] = v[k];
  __syncthreads();
  double* part = P.partials + ((size_t)comp * P.n_tiles + ct) * 8;
  if (tid < 6) {
    double acc = 0.0;
    for (int w = 0; w < NTHR / 32; ++w) {
      const double x = red[w * 6 + tid];
      acc = (tid == 1) ? fmax(acc, x) : acc + x;
    }
    part[tid < 4 ? tid : tid + 2] = acc;
  }
  if (tid == 0) {
    part[4] = g0r;
    part[5] = g0i;
  }
}

// ---------------------------------------------------------------------------------------------
// k_qfft_lean: the alpha pass of N = R1 R2 (49 = 7 x 7, 65 = 5 x 13) with two shared-memory
// passes instead of six. The first DIF stage (radix R1, twiddles) reads its R1 rows of T
// straight from global memory into registers and writes the tile once; after one barrier the
// last stage (radix R2) reads its rows and its outputs go from registers to the volume rows
// (and the mirror), with the digest accumulated on the way; one digest partial per warp
// (4 per tile, reduced by k_digest in a fixed order). Same butterflies and twiddles as k_qfft:
// the volumes are bitwise equal, the digest sums are associated differently. Less on-chip
// traffic per sample, so less power under the HBM-bound T read.
template <int N, int NT, int NTHR, int MINB>
__global__ void __launch_bounds__(NTHR, MINB) k_qfft_lean(const QfParams P) {
  constexpr int L = (N - 1) / 2;
  constexpr int R1 = smallest_prime_factor(N), R2 = N / R1;
  static_assert(R1 * R2 == N && smallest_prime_factor(R2) == R2, "N must be a product of two primes");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ts = reinterpret_cast<double2*>(smem_raw);
  double2* rou_s = Ts + N * NT;
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += NTHR) rou_s[i] = P.rou[i];
  for (int i = tid; i <= L; i += NTHR) betaw_s[i] = P.betaw[i];
  const int ct = blockIdx.x, comp = blockIdx.y;
  const int col0 = ct * NT;
  const double2* src = P.T + (size_t)comp * N * P.ncolp + col0;
  // every thread's first-stage loads are issued before the table barrier
  constexpr int ITEMS_A = (NT * R2 + NTHR - 1) / NTHR;
  double xa[ITEMS_A][R1][2];
#pragma unroll
  for (int u = 0; u < ITEMS_A; ++u) {
    const int item = tid + u * NTHR;
    if (item < NT * R2) {
      const int c = item % NT, t = item / NT;
#pragma unroll
      for (int jj = 0; jj < R1; ++jj) {
        const double2 v = __ldcs(src + (size_t)(t + jj * R2) * P.ncolp + c);
        xa[u][jj][0] = v.x;
        xa[u][jj][1] = v.y;
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < ITEMS_A; ++u) {
    const int item = tid + u * NTHR;
    if (item < NT * R2) {
      const int c = item % NT, t = item / NT;
      double xr[R1], xi[R1];
#pragma unroll
      for (int jj = 0; jj < R1; ++jj) {
        xr[jj] = xa[u][jj][0];
        xi[jj] = xa[u][jj][1];
      }
      Radix<R1>::dft(xr, xi);
      double2* base = Ts + t * NT + c;
      base[0] = make_double2(xr[0], xi[0]);
      if (t == 0) {
#pragma unroll
        for (int jj = 1; jj < R1; ++jj) base[jj * R2 * NT] = make_double2(xr[jj], xi[jj]);
      } else {
#pragma unroll
        for (int jj = 1; jj < R1; ++jj) {
          const double2 w = rou_s[t * jj];
          base[jj * R2 * NT] = make_double2(xr[jj] * w.x - xi[jj] * w.y, xr[jj] * w.y + xi[jj] * w.x);
        }
      }
    }
  }
  __syncthreads();
  const CompRec rec = P.comps[comp];
  const bool mir = P.mirror && rec.m > 0;
  const long long sbit = (long long)0x8000000000000000ULL;
  const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
  double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
  long long mx2 = 0;
  for (int item = tid; item < NT * R1; item += NTHR) {
    const int c = item % NT, bl = item / NT;
    const int col = col0 + c;
    if (col >= P.ncol) continue;
    double xr[R2], xi[R2];
    const double2* base = Ts + (size_t)(bl * R2) * NT + c;
#pragma unroll
    for (int jj = 0; jj < R2; ++jj) {
      const double2 v = base[jj * NT];
      xr[jj] = v.x;
      xi[jj] = v.y;
    }
    double2* o = P.out + rec.slot * P.vol + col;
    double2* om = mir ? P.out + rec.mslot * P.vol + col : nullptr;
    const double qb = betaw_s[col / N];
    double sr = 0.0, si = 0.0;
    auto emit = [&](int jj, double vr, double vi) {
      const int a = bl + R1 * jj;  // output frequency of position bl R2 + jj
      const size_t idx = (size_t)a * P.rpitch;
      __stcs(o + idx, make_double2(vr, vi));
      if (om) {
        const long long br = __double_as_longlong(vr) ^ mflip_r;
        const long long bi = __double_as_longlong(vi) ^ mflip_i;
        __stcs(om + idx, make_double2(__longlong_as_double(br), __longlong_as_double(bi)));
      }
      const double a2 = fma(vr, vr, vi * vi);
      s2 += a2;
      mx2 = max(mx2, __double_as_longlong(a2));
      const double wgt = digest_weight((uint32_t)((size_t)a * P.ncol + col) * 0x9E3779B1u);
      pr = fma(wgt, vr, pr);
      pi = fma(wgt, vi, pi);
      sr += vr;
      si += vi;
      if (a == 0 && col == 0) {
        g0r = vr;
        g0i = vi;
      }
    };
    if constexpr (R2 >= kSinkMinRadix) {
      Radix<R2>::dft_sink(xr, xi, emit);
    } else {
      Radix<R2>::dft(xr, xi);
#pragma unroll
      for (int jj = 0; jj < R2; ++jj) emit(jj, xr[jj], xi[jj]);
    }
    ir = fma(qb, sr, ir);
    ii = fma(qb, si, ii);
  }
  double v[8] = {s2, __longlong_as_double(mx2), pr, pi, g0r, g0i, ir, ii};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double x = __shfl_down_sync(0xffffffffu, v[q], off);
      v[q] = (q == 1) ? fmax(v[q], x) : v[q] + x;
    }
  if (lane == 0) {
    double* part = P.partials + (((size_t)comp * P.n_tiles + ct) * (NTHR / 32) + warp) * 8;
#pragma unroll
    for (int q = 0; q < 8; ++q) part[q] = v[q];
  }
}

// ---------------------------------------------------------------------------------------------
// k_qfft_half: k_qfft with its last DIF stage fused into the epilogue (N = R1 R2: 49, 65). The
// tile load (cp.async, recomputed rows) and the first stage (radix R1, in shared memory) are
// k_qfft's; the last stage reads its R2 rows into registers and its outputs go straight to the
// volume rows, the mirror and the digest (as in k_qfft_lean): four shared-memory passes per
// sample instead of six, no permutation lookups, two barriers fewer; one digest partial per
// warp. Volumes bitwise equal to k_qfft's, digests associated differently.
template <int N, int NT, int NTHR, int MINB>
__global__ void __launch_bounds__(NTHR, MINB) k_qfft_half(const QfParams P) {
  constexpr int L = (N - 1) / 2;
  constexpr int R1 = smallest_prime_factor(N), R2 = N / R1;
  static_assert(R1 * R2 == N && smallest_prime_factor(R2) == R2, "N must be a product of two primes");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ts = reinterpret_cast<double2*>(smem_raw);
  constexpr int TS = NT;
  double2* rou_s = Ts + N * TS;
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += NTHR) rou_s[i] = P.rou[i];
  for (int i = tid; i <= L; i += NTHR) betaw_s[i] = P.betaw[i];
  const int ct = blockIdx.x, comp = blockIdx.y;
  const int col0 = ct * NT;
  qfft_load_tile<N, NT, NTHR, TS>(P, Ts, comp, col0, tid);
  cp_async_wait<0>();
  __syncthreads();
  fft_stage_ct<N, R1, N, NT, NT, NTHR, false>(Ts, rou_s, tid);
  __syncthreads();

  const CompRec rec = P.comps[comp];
  const bool mir = P.mirror && rec.m > 0;
  const long long sbit = (long long)0x8000000000000000ULL;
  const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
  double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
  long long mx2 = 0;
  for (int item = tid; item < NT * R1; item += NTHR) {
    const int c = item % NT, bl = item / NT;
    const int col = col0 + c;
    if (col >= P.ncol) continue;
    double xr[R2], xi[R2];
    const double2* base = Ts + (size_t)(bl * R2) * NT + c;
#pragma unroll
    for (int jj = 0; jj < R2; ++jj) {
      const double2 v = base[jj * NT];
      xr[jj] = v.x;
      xi[jj] = v.y;
    }
    double2* o = P.out + rec.slot * P.vol + col;
    double2* om = mir ? P.out + rec.mslot * P.vol + col : nullptr;
    const double qb = betaw_s[col / N];
    double sr = 0.0, si = 0.0;
    auto emit = [&](int jj, double vr, double vi) {
      const int a = bl + R1 * jj;  // output frequency of position bl R2 + jj
      const size_t idx = (size_t)a * P.rpitch;
      __stcs(o + idx, make_double2(vr, vi));
      if (om) {
        const long long br = __double_as_longlong(vr) ^ mflip_r;
        const long long bi = __double_as_longlong(vi) ^ mflip_i;
        __stcs(om + idx, make_double2(__longlong_as_double(br), __longlong_as_double(bi)));
      }
      const double a2 = fma(vr, vr, vi * vi);
      s2 += a2;
      mx2 = max(mx2, __double_as_longlong(a2));
      const double wgt = digest_weight((uint32_t)((size_t)a * P.ncol + col) * 0x9E3779B1u);
      pr = fma(wgt, vr, pr);
      pi = fma(wgt, vi, pi);
      sr += vr;
      si += vi;
      if (a == 0 && col == 0) {
        g0r = vr;
        g0i = vi;
      }
    };
    if constexpr (R2 >= kSinkMinRadix) {
      Radix<R2>::dft_sink(xr, xi, emit);
    } else {
      Radix<R2>::dft(xr, xi);
#pragma unroll
      for (int jj = 0; jj < R2; ++jj) emit(jj, xr[jj], xi[jj]);
    }
    ir = fma(qb, sr, ir);
    ii = fma(qb, si, ii);
  }
  double v[8] = {s2, __longlong_as_double(mx2), pr, pi, g0r, g0i, ir, ii};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double x = __shfl_down_sync(0xffffffffu, v[q], off);
      v[q] = (q == 1) ? fmax(v[q], x) : v[q] + x;
    }
  if (lane == 0) {
    double* part = P.partials + (((size_t)comp * P.n_tiles + ct) * (NTHR / 32) + warp) * 8;
#pragma unroll
    for (int q = 0; q < 8; ++q) part[q] = v[q];
  }
}

// ---------------------------------------------------------------------------------------------
// k_qfft_rt: the alpha pass for window band limits without a compile-time kernel and too
// large for the single-pass runtime kernel's on-chip tile (n > 129, i.e. L_h >= 65 off the
// BASELINE lengths): one component x NT columns per CTA, the n x NT tile of T in shared
// memory, the runtime mixed-radix DIF plan of k_couple (fft_runtime), or a dense DFT in the
// epilogue when n has a prime factor above the generated radices; then the same epilogue
// (stores, mirror, digest partials per (component, column tile)) as k_couple.
template <int NT, int NTHR>
__global__ void __launch_bounds__(NTHR) k_qfft_rt(const QfParams P) {
  static_assert(NTHR % NT == 0, "threads must cover the columns");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n = P.n, L = (n - 1) / 2;
  double2* Ts = reinterpret_cast<double2*>(smem_raw);
  double2* rou_s = Ts + (size_t)n * NT;
  double* betaw_s = reinterpret_cast<double*>(rou_s + n);
  int* perm_s = reinterpret_cast<int*>(betaw_s + (L + 1));
  const int tid = threadIdx.x;
  for (int i = tid; i < n; i += NTHR) {
    rou_s[i] = P.rou[i];
    perm_s[i] = P.perm[i];
  }
  for (int i = tid; i <= L; i += NTHR) betaw_s[i] = P.betaw[i];
  const int ct = blockIdx.x, comp = blockIdx.y;
  const int col0 = ct * NT;
  {
    const double2* src = P.T + (size_t)comp * n * P.ncolp + col0;
    for (int e = tid; e < n * NT; e += NTHR) {
      const int row = e / NT, c = e % NT;
      cp_async16(Ts + (size_t)row * NT + c, src + (size_t)row * P.ncolp + c, true);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
  __syncthreads();
  if (!P.generic_dft) fft_runtime(Ts, NT, n, NT, P.fft, rou_s, NTHR);

  const int cc = tid % NT, col = col0 + cc;
  const bool ok = col < P.ncol;
  double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
  long long mx2 = 0;
  if (ok) {
    const CompRec rec = P.comps[comp];
    double2* o = P.out + rec.slot * P.vol + col;
    double2* om = (P.mirror && rec.m > 0) ? P.out + rec.mslot * P.vol + col : nullptr;
    const long long sbit = (long long)0x8000000000000000ULL;
    const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
    const double qb = betaw_s[col / n];
    const double2* Tp = Ts + cc;
    const int a_first = tid / NT;
    constexpr int A_STEP = NTHR / NT;
    uint32_t hsh = (uint32_t)((size_t)a_first * P.ncol + col) * 0x9E3779B1u;
    const uint32_t hstep = (uint32_t)((size_t)A_STEP * P.ncol) * 0x9E3779B1u;
    for (int a = a_first; a < n; a += A_STEP, hsh += hstep) {
      double vr, vi;
      if (!P.generic_dft) {
        const double2 t = Tp[(size_t)perm_s[a] * NT];
        vr = t.x;
        vi = t.y;
      } else {  // dense DFT: g_a = sum_j w^(j a) T_j
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
      const size_t idx = (size_t)a * P.rpitch;
      __stcs(o + idx, make_double2(vr, vi));
      if (om) {
        const long long br = __double_as_longlong(vr) ^ mflip_r;
        const long long bi = __double_as_longlong(vi) ^ mflip_i;
        __stcs(om + idx, make_double2(__longlong_as_double(br), __longlong_as_double(bi)));
      }
      const double a2 = fma(vr, vr, vi * vi);
      s2 += a2;
      mx2 = max(mx2, __double_as_longlong(a2));
      const double wgt = digest_weight(hsh);
      pr = fma(wgt, vr, pr);
      pi = fma(wgt, vi, pi);
      ir += vr;
      ii += vi;
      if (a == 0 && col == 0) {
        g0r = vr;
        g0i = vi;
      }
    }
    ir *= qb;
    ii *= qb;
  }
  // fixed-order reduction: a shuffle tree per warp, then the warps in order
  double v[8] = {s2, __longlong_as_double(mx2), pr, pi, g0r, g0i, ir, ii};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double x = __shfl_down_sync(0xffffffffu, v[k], off);
      v[k] = (k == 1) ? fmax(v[k], x) : v[k] + x;
    }
  __syncthreads();  // T is reused as the reduction scratch
  double* red = reinterpret_cast<double*>(smem_raw);
  if ((tid & 31) == 0)
#pragma unroll
    for (int k = 0; k < 8; ++k) red[(tid >> 5) * 8 + k] = v[k];
  __syncthreads();
  if (tid < 8) {
    double acc = 0.0;
    for (int w = 0; w < NTHR / 32; ++w) {
      const double x = red[w * 8 + tid];
      acc = (tid == 1) ? fmax(acc, x) : acc + x;
    }
    P.partials[((size_t)comp * P.n_tiles + ct) * 8 + tid] = acc;
  }
}

}  // namespace slsht_cuda
