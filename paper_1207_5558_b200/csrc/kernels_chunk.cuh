// Per-chunk kernels around the coupling stage: Legendre rows, the modulated-SHT GEMM on the
// FP64 tensor cores, and the deterministic digest reduction.
#pragma once

#include "common.cuh"

namespace slsht_cuda {

// ---------------------------------------------------------------------------------------------
// A[row][j] = w_j lambda_l^m(x_j) for the rows l0..l1 of one order-m segment, on the x >= 0
// Gauss-Legendre nodes (kernels_setup.cuh). The segment's rows are stored parity-sorted: first
// the degrees with l + m even, then the odd ones (each in increasing l), so every GEMM tile has
// one parity class and selects I_0 or I_1 per column (k_modgemm).
// grid (segments, node blocks of 128); dynamic smem 3 (L_g+1) doubles of recursion coefficients.
struct Seg {
  int m, l0, l1, row0;
};

__host__ __device__ __forceinline__ int seg_even_first(int m, int l0) {
  return ((l0 + m) & 1) ? l0 + 1 : l0;
}
// A row (within the segment) of degree l
__host__ __device__ __forceinline__ int seg_arow(int m, int l0, int l1, int l) {
  const int e0 = seg_even_first(m, l0);
  const int ne = e0 <= l1 ? (l1 - e0) / 2 + 1 : 0;
  return ((l + m) & 1) ? ne + (l - (e0 == l0 ? l0 + 1 : l0)) / 2 : (l - e0) / 2;
}

__global__ void __launch_bounds__(128) k_agen(const Seg* __restrict__ segs, int L_g, int n_nodes,
                                              int ldA, const double* __restrict__ ncos,
                                              const double* __restrict__ nsin,
                                              const double* __restrict__ weights,
                                              double* __restrict__ A) {
  extern __shared__ double coef[];
  double *sf = coef, *ca = coef + (L_g + 1), *cb = coef + 2 * (L_g + 1);
  const Seg s = segs[blockIdx.x];
  const int am = s.m < 0 ? -s.m : s.m;
  legendre_coeffs(am, s.l1, sf, ca, cb);
  __syncthreads();
  const int j = blockIdx.y * blockDim.x + threadIdx.x;
  if (j >= ldA) return;
  if (j >= n_nodes) {
    for (int l = s.l0; l <= s.l1; ++l) A[(size_t)(s.row0 + l - s.l0) * ldA + j] = 0.0;
    return;
  }
  const double wj = weights[j];
  LegendreIt r;
  r.seed(s.m, ncos[j], nsin[j], sf);
  while (r.l < s.l0) r.next(ca, cb);
  for (int l = s.l0; l <= s.l1; ++l) {
    if (l > s.l0) r.next(ca, cb);
    A[(size_t)(s.row0 + seg_arow(s.m, s.l0, s.l1, l)) * ldA + j] = wj * r.cur;
  }
}

// ---------------------------------------------------------------------------------------------
// The modulated SHT (transform.cpp:189-220) of every row of one order m as a GEMM on the FP64
// tensor cores, over the x >= 0 Gauss-Legendre nodes (kernels_setup.cuh):
//   mod[row][c] = sum_j A[row][j] * B_m[j][c],  B_m[j][c] = I_s(x_j, m - q_c) lambda_c(x_j),
//   s = parity of the tile's rows (l + m) xor parity of p_c + q_c
// (zero where |m - q_c| > L_f), c in q-major (p, q) order. U = conj(mod) is stored at the
// tile's natural rows nat0 + 2 r (the A rows are parity-sorted, k_agen).
// CTA tile 32 rows x 64 complex columns, K chunks of 32 nodes, 8 warps = 2 row groups x 4
// column groups, each warp 16 rows x 16 complex columns = 8 DMMA per k-step of 4.
// Operands stream through a two-stage cp.async pipeline: the A rows, the raw lambda_c rows
// and the I values of the few distinct q of the column tile (B_m = I * lambda is formed at the
// MMA, two multiplies per fragment). A, lambda and I rows have the padded node stride ldA
// (zeros past n_nodes), so every copy is a whole 16-B chunk.
struct MTile {
  int m, row0, rows;  // order, first A row, rows (one parity class)
  int nat0, par;      // natural (chunk) row of tile row 0 (stride 2), parity of l + m
};

constexpr int MG_ROWS = 32;  // rows per CTA tile
constexpr int MG_COLS = 64;  // complex columns per CTA tile
constexpr int MG_K = 32;     // nodes per K chunk
constexpr int MG_NQ = 16;    // distinct q per column tile (host-checked)
constexpr int MG_KS = MG_K + 4;  // padded row stride of the A and lambda stages (doubles)
constexpr size_t MG_STAGE = (size_t)MG_ROWS * MG_KS * 8 + (size_t)MG_COLS * MG_KS * 8 +
                            (size_t)MG_K * MG_NQ * 2 * 16;
constexpr size_t MG_SMEM = 2 * MG_STAGE;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(pred ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory");
}

template <int RG>
__device__ __forceinline__ void modgemm_tile(const MTile t, int n_nodes, int ldA, int L_f,
                                             int NPQ, const int* colq, const int* colpar,
                                             const double* __restrict__ A,
                                             const double2* __restrict__ itab,
                                             const double* __restrict__ lamh, int u_group,
                                             long long u_gs, const int* __restrict__ u_base,
                                             const int* __restrict__ u_str,
                                             double2* __restrict__ U) {
  // RG row groups of 16 rows; the 8 warps split as RG x (8 / RG), each warp 16 rows x
  // 8 RG complex columns (CF = RG column fragments)
  constexpr int CF = RG, WPR = 8 / RG;
  extern __shared__ __align__(16) unsigned char mg_smem[];
  const int cbase = blockIdx.y * MG_COLS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rg = warp / WPR, cgp = warp % WPR;
  // a warp whose columns all lie past NPQ (last column tile) has no MMA work
  const bool warp_cols = cbase + cgp * 8 * CF < NPQ;
  const int q_lo = colq[0];
  const int nq = colq[min(MG_COLS, NPQ - cbase) - 1] - q_lo + 1;
  auto stage_a = [&](int b) { return reinterpret_cast<double*>(mg_smem + b * MG_STAGE); };
  auto stage_l = [&](int b) { return stage_a(b) + MG_ROWS * MG_KS; };
  auto stage_i = [&](int b) {
    return reinterpret_cast<double2*>(stage_l(b) + MG_COLS * MG_KS);
  };
  auto issue = [&](int k0, int b) {
    double* As = stage_a(b);
    double* Ls = stage_l(b);
    double2* Is = stage_i(b);
#pragma unroll
    for (int i = 0; i < 16 * RG * MG_K / 2 / 256; ++i) {
      const int e = tid + 256 * i, r = e / (MG_K / 2), u = e % (MG_K / 2);
      const bool ok = r < t.rows;
      cp_async16(As + r * MG_KS + 2 * u, A + (size_t)(t.row0 + (ok ? r : 0)) * ldA + k0 + 2 * u, ok);
    }
#pragma unroll
    for (int i = 0; i < MG_COLS * MG_K / 2 / 256; ++i) {
      const int e = tid + 256 * i, cc = e / (MG_K / 2), u = e % (MG_K / 2);
      const bool ok = cbase + cc < NPQ;
      cp_async16(Ls + cc * MG_KS + 2 * u, lamh + (size_t)(ok ? cbase + cc : 0) * ldA + k0 + 2 * u, ok);
    }
#pragma unroll
    for (int i = 0; i < MG_K * MG_NQ * 2 / 256; ++i) {  // Is[k][sq][s] = I_s(x_k, m - q)
      const int e = tid + 256 * i, k = e % MG_K, sqs = e / MG_K, sq = sqs >> 1;
      const int mu = t.m - (q_lo + sq);
      const bool ok = sq < nq && mu >= -L_f && mu <= L_f;
      cp_async16(Is + k * MG_NQ * 2 + sqs,
                 itab + (size_t)(ok ? 2 * (mu + L_f) + (sqs & 1) : 0) * ldA + k0 + k, ok);
    }
    cp_async_commit();
  };
  double acc[2][CF][2][2];  // [row frag][col frag][re/im][e]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < CF; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;
  int qi[CF];  // the column's I entry in a stage: 2 (q - q_lo) + s
#pragma unroll
  for (int cf = 0; cf < CF; ++cf) {
    const int col = cgp * 8 * CF + cf * 8 + (lane >> 2);
    qi[cf] = 2 * (colq[col] - q_lo) + (colpar[col] ^ t.par);
  }
  const int nchunks = ldA / MG_K;
  issue(0, 0);
  for (int ch = 0; ch < nchunks; ++ch) {
    const int k0 = ch * MG_K;
    if (ch + 1 < nchunks) {
      issue(k0 + MG_K, (ch + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* As = stage_a(ch & 1);
    const double* Ls = stage_l(ch & 1);
    const double2* Is = stage_i(ch & 1);
    // k-steps holding at least one node (the last chunk is mostly padding)
    const int ksn = min(MG_K / 4, (n_nodes - k0 + 3) / 4);
    if (warp_cols) {
#pragma unroll
      for (int ks = 0; ks < MG_K / 4; ++ks) {
        if (ks < ksn) {
          const int k = ks * 4 + (lane & 3);
          const double a0 = As[(rg * 16 + (lane >> 2)) * MG_KS + k];
          const double a1 = As[(rg * 16 + 8 + (lane >> 2)) * MG_KS + k];
#pragma unroll
          for (int cf = 0; cf < CF; ++cf) {
            const int col = cgp * 8 * CF + cf * 8 + (lane >> 2);
            const double lv = Ls[col * MG_KS + k];
            const double2 iv = Is[k * MG_NQ * 2 + qi[cf]];
            const double br = iv.x * lv, bi = iv.y * lv;
            dmma(acc[0][cf][0][0], acc[0][cf][0][1], a0, br);
            dmma(acc[0][cf][1][0], acc[0][cf][1][1], a0, bi);
            dmma(acc[1][cf][0][0], acc[1][cf][0][1], a1, br);
            dmma(acc[1][cf][1][0], acc[1][cf][1][1], a1, bi);
          }
        }
      }
    }
    __syncthreads();  // stage ch & 1 is refilled by the issue of chunk ch + 2
  }
#pragma unroll
  for (int rf = 0; rf < 2; ++rf) {
    const int r = rg * 16 + rf * 8 + (lane >> 2);
    if (r >= t.rows) continue;
#pragma unroll
    for (int cf = 0; cf < CF; ++cf)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = cbase + cgp * 8 * CF + cf * 8 + 2 * (lane & 3) + e;
        if (c < NPQ) {
          const int row = t.nat0 + 2 * r;
          // u_group == 0: U[row][c]; else the stage-tiled layout of the warp-specialized
          // coupling kernel: group row / MT, stage block u_base[c], row stride u_str[c]
          const size_t dst = u_group ? (size_t)(row / u_group) * u_gs + u_base[c] +
                                           (size_t)(row % u_group) * u_str[c]
                                     : (size_t)row * NPQ + c;
          U[dst] = make_double2(acc[rf][cf][0][e], -acc[rf][cf][1][e]);
        }
      }
  }
}

// Tiles of at most 16 rows (short order segments: the high-degree shards, the tail of every
// order) take the 16-row variant; the others 32 rows.
__global__ void __launch_bounds__(256) k_modgemm(const MTile* __restrict__ tiles, int n_nodes,
                                                 int ldA, int L_f, int NPQ,
                                                 const double* __restrict__ A,
                                                 const double2* __restrict__ itab,
                                                 const double* __restrict__ lamh,
                                                 const int* __restrict__ pq_q,
                                                 int u_group, long long u_gs,
                                                 const int* __restrict__ u_base,
                                                 const int* __restrict__ u_str,
                                                 double2* __restrict__ U) {
  __shared__ int colq[MG_COLS], colpar[MG_COLS];  // q and the parity of p + q per column
  const int cbase = blockIdx.y * MG_COLS;
  if (threadIdx.x < MG_COLS) {
    const bool in = cbase + (int)threadIdx.x < NPQ;
    const int c = in ? cbase + threadIdx.x : 0;
    colq[threadIdx.x] = in ? pq_q[2 * c] : 0;
    colpar[threadIdx.x] = in ? ((pq_q[2 * c] + pq_q[2 * c + 1]) & 1) : 0;
  }
  __syncthreads();
  const MTile t = tiles[blockIdx.x];
  if (t.rows <= 16)
    modgemm_tile<1>(t, n_nodes, ldA, L_f, NPQ, colq, colpar, A, itab, lamh, u_group, u_gs, u_base,
                    u_str, U);
  else
    modgemm_tile<2>(t, n_nodes, ldA, L_f, NPQ, colq, colpar, A, itab, lamh, u_group, u_gs, u_base,
                    u_str, U);
}

// ---------------------------------------------------------------------------------------------
// Digest of every emitted component from the per-column-tile partials of k_couple: one warp
// per component, lanes stride the tiles in order, then a fixed shuffle tree (bitwise
// deterministic for a given plan). Mirrors (real mode) follow exactly from conjugation.
__global__ void k_digest(const CompRec* __restrict__ comps, int count, int n_col_tiles, int n,
                         const double* __restrict__ partials, int mirror,
                         double* __restrict__ digest) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= count) return;
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int t = lane; t < n_col_tiles; t += 32) {
    const double* r = partials + ((size_t)w * n_col_tiles + t) * 8;
    acc[0] += r[0];
    acc[1] = fmax(acc[1], r[1]);
    acc[2] += r[2];
    acc[3] += r[3];
    acc[4] += r[4];
    acc[5] += r[5];
    acc[6] += r[6];
    acc[7] += r[7];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double o = __shfl_down_sync(0xffffffffu, acc[k], off);
      acc[k] = (k == 1) ? fmax(acc[k], o) : acc[k] + o;
    }
  }
  if (lane != 0) return;
  const CompRec rec = comps[w];
  acc[1] = sqrt(acc[1]);  // partials carry max |g|^2
  const double inv = 1.0 / ((double)n * n * n);
  acc[6] *= inv;
  acc[7] *= inv;
  const int l = rec.l, m = rec.m;
  double* d = digest + (size_t)(l * l + l + m) * 8;
#pragma unroll
  for (int k = 0; k < 8; ++k) d[k] = acc[k];
  if (mirror && m > 0) {
    const double s = (m & 1) ? -1.0 : 1.0;
    double* dm = digest + (size_t)(l * l + l - m) * 8;
    dm[0] = acc[0];
    dm[1] = acc[1];
    dm[2] = s * acc[2];
    dm[3] = -(s * acc[3]);
    dm[4] = s * acc[4];
    dm[5] = -(s * acc[5]);
    dm[6] = s * acc[6];
    dm[7] = -(s * acc[7]);
  }
}

// ---------------------------------------------------------------------------------------------
// Inversion from the digests (transform.cpp:469-544): f_rec(l, m) = integral(l, m) /
// (sqrt(16 pi^3) h00), the integral being digest fields 6-7 (integrate_volume). With
// fill_negative, m < 0 comes from (-1)^m conj of (l, -m) (InverseAccumulator::finish).
__global__ void k_inverse(const double* __restrict__ digest, int L, int fill_negative,
                          double h00_re, double h00_im, double* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (L + 1) * (L + 1)) return;
  int l = (int)sqrt((double)idx);
  while (l * l > idx) --l;
  while ((l + 1) * (l + 1) <= idx) ++l;
  const int m = idx - l * l - l;
  const bool mirror = fill_negative && m < 0;
  const int src = mirror ? l * l + l - m : idx;
  const double ir = digest[(size_t)src * 8 + 6], ii = digest[(size_t)src * 8 + 7];
  // (ir + i ii) / (s h00), s = sqrt(16 pi^3), as complex division
  const double s = sqrt(16.0 * kPi * kPi * kPi);
  const double dr = s * h00_re, di = s * h00_im;
  const double den = dr * dr + di * di;
  double qr = (ir * dr + ii * di) / den, qi = (ii * dr - ir * di) / den;
  if (mirror) {  // (-1)^m conj
    const double sg = (m & 1) ? -1.0 : 1.0;
    qr = sg * qr;
    qi = -(sg * qi);
  }
  out[2 * (size_t)idx] = qr;
  out[2 * (size_t)idx + 1] = qi;
}

}  // namespace slsht_cuda
