// Two-pass coupling for the long transforms (n = 49, 65, 129):
//
//   k_tgemm  T[comp][q mod n][col] = sum_{p>=|q|} U[comp][(p,q)] W[(p,q)][col]
//            one batched complex GEMM per q on the FP64 tensor cores (DMMA 8x8x4, Gauss
//            3-product), 64 components x 64 columns per CTA, every q of the tile in one pass
//            over the q-major (p, q) rows (each q padded to whole k-steps of 4), operands
//            staged in shared memory by a 4-deep cp.async ring. T goes to an HBM buffer.
//   k_qfft   reads T[comp][*][32 columns], runs the length-n alpha DIF FFT in shared memory
//            (fft_radix.cuh butterflies, the plan of k_couple) and writes the So3Volume rows
//            (and the real-mode mirror) with the digest partials.
//
// Why two passes: the single-pass k_couple must keep all n rows of its T tile on chip, which
// caps its tile at 8 components x 8 columns for n = 129 (132 KB); each operand byte then
// feeds only 8 MACs, and the DMMA loop runs L2-bound at ~16% of the tensor pipe
// (profiles/r01_ncu_couple_c5_*.txt). The T round trip costs 32 B of extra HBM traffic per
// sample, but lets the GEMM run on 64x64 tiles (8x the operand reuse).
#pragma once

#include <type_traits>

#include "common.cuh"
#include "kernels_chunk.cuh"
#include "kernels_couple.cuh"

namespace slsht_cuda {

constexpr int TG_BM = 64;      // components per CTA
constexpr int TG_BN = 64;      // column padding unit of W and T (the widest CTA tile)
constexpr int TG_KS = 16;      // (p, q) rows per pipeline stage (4 k-steps)
constexpr int TG_ASTR = 20;    // A row stride (complex): == 4 mod 8, conflict-free fragments
// B row stride (complex) BN + 2 == 2 mod 8: conflict-free fragments

struct TgParams {
  const double2* U;      // [comp][KP]: q-major padded (p, q) rows, zero padding; KP % TG_KS == 0
  const double2* W;      // [KP][ncolp]
  double2* T;            // [comp][n][ncolp]
  const short* qend;     // per k-step: T row (q mod n) completed by it, or -1
  int count, KP, ncolp, n;
};

__host__ __device__ constexpr int tgemm_threads(int BN, int WNF) { return 64 * (BN / (8 * WNF)); }
__host__ __device__ constexpr size_t tgemm_smem_bytes(int KP, int BN, int NST) {
  return (size_t)NST * (TG_BM * TG_ASTR + TG_KS * (BN + 2)) * 16 + (size_t)(KP / 4) * 2 + 16;
}

// 256-bit global store (sm_100): two consecutive complex values
__device__ __forceinline__ void st_global_v4(double2* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d)
               : "memory");
}

// Warp tile 32 components x 8 WNF columns; BN columns per CTA, TG_NST pipeline stages.
// <32, 2, 2, 3> (default): 4 warps, two stages, three independent CTAs per SM (156 registers).
// <64, 2, 4, 1>: 8 warps, one CTA per SM. <32, 2, 3, 2>: 4 warps, two CTAs per SM.
// <32, 2, 4, 1>: 4 warps (117 KB), which leaves room on the SM for one k_qfft CTA of the
// previous chunk (the overlapped schedule).
template <int BN, int WNF, int TG_NST, int MINB>
__global__ void __launch_bounds__(tgemm_threads(BN, WNF), MINB) k_tgemm(const TgParams P) {
  constexpr int TG_THREADS = tgemm_threads(BN, WNF), TG_BSTR = BN + 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + TG_NST * TG_BM * TG_ASTR;
  short* qend_s = reinterpret_cast<short*>(Bs + TG_NST * TG_KS * TG_BSTR);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // grid x = component block: the CTAs in flight share a few W column tiles (read from HBM
  // once per chunk) while the chunk's U stays L2-resident
  const int comp0 = blockIdx.x * TG_BM, col0 = blockIdx.y * BN;
  const int nks = P.KP / 4, nst = (P.KP + TG_KS - 1) / TG_KS;
  for (int i = tid; i < nks; i += TG_THREADS) qend_s[i] = P.qend[i];

  auto load_stage = [&](int st) {
    if (st < nst) {
      const int kb = st * TG_KS;
      double2* Ad = As + (st % TG_NST) * TG_BM * TG_ASTR;
      double2* Bd = Bs + (st % TG_NST) * TG_KS * TG_BSTR;
#pragma unroll
      for (int j = 0; j < TG_BM * TG_KS / TG_THREADS; ++j) {
        const int e = tid + j * TG_THREADS;
        const int c = e / TG_KS, k = e % TG_KS;
        const bool ok = comp0 + c < P.count && kb + k < P.KP;
        cp_async16(Ad + c * TG_ASTR + k, P.U + (ok ? (size_t)(comp0 + c) * P.KP + kb + k : 0), ok);
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

  for (int st = 0; st < nst; ++st) {
    cp_async_wait<TG_NST - 2>();
    __syncthreads();
    load_stage(st + TG_NST - 1);  // refills the buffer consumed at st - 1 (all warps passed it)
    const double2* Ab = As + (st % TG_NST) * TG_BM * TG_ASTR;
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
          if (comp < P.count) {
            double2* dst = P.T + ((size_t)comp * P.n + row) * P.ncolp + scol;
#pragma unroll
            for (int ni = 0; ni < WNF; ++ni)  // 32 B per lane: 4 lanes write one whole 128-B line
              st_global_v4(dst + ni * 8, c1[mi][ni][0] - c3[mi][ni][0], c1[mi][ni][0] + c2[mi][ni][0],
                           c1[mi][ni][1] - c3[mi][ni][1], c1[mi][ni][1] + c2[mi][ni][1]);
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
// k_qfft: one component x NT grid columns per CTA.

struct QfParams {
  const double2* T;      // [comp][n][ncolp]
  double2* out;
  double* partials;      // [comp][tile][8]
  const CompRec* comps;
  int count, n, ncol, ncolp, n_tiles;
  long long vol;
  int mirror;
  const double2* rou;
  const int* perm;
  const double* betaw;
};

__host__ __device__ constexpr size_t qfft_smem_bytes(int n, int NT) {
  return (size_t)n * NT * 16 + (size_t)n * 16 + (size_t)((n + 1) / 2) * 8 + (size_t)n * 4 + 64;
}

template <int N, int NT, int NTHR, int MINB>
__global__ void __launch_bounds__(NTHR, MINB) k_qfft(const QfParams P) {
  constexpr int L = (N - 1) / 2;
  // epilogue: (NTHR / NT) * NT threads own (column, row-set) pairs; the rest only reduce
  static_assert(NTHR >= NT, "threads must cover the columns");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ts = reinterpret_cast<double2*>(smem_raw);
  double2* rou_s = Ts + N * NT;
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
  {
    const double2* src = P.T + (size_t)comp * N * P.ncolp + col0;
    for (int e = tid; e < N * NT; e += NTHR) {
      const int row = e / NT, c = e % NT;
      cp_async16(Ts + e, src + (size_t)row * P.ncolp + c, true);
    }
    cp_async_commit();
  }
  cp_async_wait<0>();
  __syncthreads();

  FftDif<N, N, NT, NT, NTHR, true>::run(Ts, rou_s, tid, 0);

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
      const double2 t = Tp[(size_t)perm_s[0] * NT];
      g0r = t.x;
      g0i = t.y;
    }
    auto rows = [&](auto mirror_tag) {
      constexpr bool MIR = decltype(mirror_tag)::value;
#pragma unroll 4
      for (int a = a_first; a < N; a += A_STEP, hsh += hstep) {
        const double2 t = Tp[(size_t)perm_s[a] * NT];
        const double vr = t.x, vi = t.y;
        const size_t idx = (size_t)a * P.ncol;
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
  // fixed-order reduction: a shuffle tree per warp, then the warps in order
  double v[8] = {s2, __longlong_as_double(mx2), pr, pi, g0r, g0i, ir, ii};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double o = __shfl_down_sync(0xffffffffu, v[k], off);
      v[k] = (k == 1) ? fmax(v[k], o) : v[k] + o;
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
