// Setup-stage kernels: every table that depends on f, h or the band limits, recomputed on
// each forward call (all inside the timed region of bench.py).
#pragma once

#include "common.cuh"

namespace slsht_cuda {

// ---------------------------------------------------------------------------------------------
// Setup: theta nodes of S_{2L_g}, theta_weights(2L_g) (grids.cpp:76-92), beta_weights(L_h)
// (grids.cpp:54-74). One warp per weight: lanes take the k terms of the quadrature sum
// (only w(0), w(+-1) and even k are nonzero) and a fixed shuffle tree adds them, so the result
// is deterministic (it differs from the reference's serial k order by roundoff only).
__device__ __forceinline__ void quad_weight_sum(int K, double angle, int lane, double& sr,
                                                double& si) {
  sr = 0.0;
  si = 0.0;
  for (int k = -K + lane; k <= K; k += 32) {
    const int mk = -k;
    double wr = 0.0, wi = 0.0;
    if (mk == 0) wr = 2.0;
    else if (mk == 1) wi = kPi / 2.0;
    else if (mk == -1) wi = -kPi / 2.0;
    else if ((mk & 1) == 0) wr = 2.0 / (1.0 - (double)mk * mk);
    if (wr == 0.0 && wi == 0.0) continue;
    const double ck = cos(k * angle);
    sr += wr * ck;
    si += wi * ck;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, off);
    si += __shfl_xor_sync(0xffffffffu, si, off);
  }
}

__global__ void k_nodes(int N, double* __restrict__ ncos, double* __restrict__ nsin,
                        double* __restrict__ weights, int L_h, double* __restrict__ betaw,
                        int* __restrict__ err_flag) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w <= N) {
    const int t = w;
    const double theta = kPi * (2 * t + 1) / (2 * N + 1);
    double sr, si;
    quad_weight_sum(N, theta, lane, sr, si);
    if (lane == 0) {
      double s, c;
      sincos(theta, &s, &c);
      ncos[t] = c;
      nsin[t] = s;
      if (fabs(si) >= 1e-12) atomicExch(err_flag, 1);
      weights[t] = (t < N) ? 2.0 * sr / (2 * N + 1) : sr / (2 * N + 1);
    }
  } else if (w - (N + 1) <= L_h) {
    const int t = w - (N + 1);
    const int L = L_h, n = 2 * L + 1;
    if (t == 0) {
      if (lane == 0) betaw[0] = 4.0 * kPi * kPi / (L / 2 + 0.5);
    } else {
      double sr, si;
      quad_weight_sum(L, 2.0 * kPi * t / n, lane, sr, si);
      if (lane == 0) {
        if (fabs(si) >= 1e-12) atomicExch(err_flag, 2);
        betaw[t] = 8.0 * kPi * kPi * sr;
      }
    }
  }
}

// lambda_p^q(theta_j) for the window band, rows in q-major (p, q) order: row c = qoff[q+L] + p-|q|,
// row stride ld (>= n_nodes; the padding stays zero).
// grid (node blocks, 2L_h+1 orders); dynamic smem 3 (L_h+1) doubles.
__global__ void k_legendre_window(int L_h, int n_nodes, int ld, const double* __restrict__ ncos,
                                  const double* __restrict__ nsin, const int* __restrict__ qoff,
                                  double* __restrict__ lamh) {
  extern __shared__ double coef[];
  double *sf = coef, *ca = coef + (L_h + 1), *cb = coef + 2 * (L_h + 1);
  const int q = (int)blockIdx.y - L_h;
  const int aq = q < 0 ? -q : q;
  legendre_coeffs(aq, L_h, sf, ca, cb);
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_nodes) return;
  LegendreIt r;
  r.seed(q, ncos[j], nsin[j], sf);
  const int base = qoff[q + L_h];
  for (int p = aq; p <= L_h; ++p) {
    if (p > aq) r.next(ca, cb);
    lamh[(size_t)(base + p - aq) * ld + j] = r.cur;
  }
}

// I(theta_j, mu) = 2 pi conj(sum_{l=|mu|}^{L_f} f_l^mu lambda_l^mu(theta_j)) (transform.cpp:158-173)
// grid (node blocks, 2L_f+1 orders); dynamic smem 3 (L_f+1) doubles + (L_f+1) complex (f_l^mu).
__global__ void k_itab(int L_f, int n_nodes, int ld, const double* __restrict__ ncos,
                       const double* __restrict__ nsin, const double* __restrict__ f,
                       double* __restrict__ itab) {
  extern __shared__ double coef[];
  double *sf = coef, *ca = coef + (L_f + 1), *cb = coef + 2 * (L_f + 1);
  double2* fs = reinterpret_cast<double2*>(coef + 3 * (L_f + 1) + ((3 * (L_f + 1)) & 1));
  const int mu = (int)blockIdx.y - L_f;
  const int amu = mu < 0 ? -mu : mu;
  legendre_coeffs(amu, L_f, sf, ca, cb);
  for (int l = amu + threadIdx.x; l <= L_f; l += blockDim.x)
    fs[l] = *reinterpret_cast<const double2*>(f + 2 * (l * l + l + mu));
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_nodes) return;
  LegendreIt r;
  r.seed(mu, ncos[j], nsin[j], sf);
  double ar = 0.0, ai = 0.0;
  for (int l = amu; l <= L_f; ++l) {
    if (l > amu) r.next(ca, cb);
    const double2 fv = fs[l];
    ar += fv.x * r.cur;
    ai += fv.y * r.cur;
  }
  double2 o;
  o.x = 2.0 * kPi * ar;
  o.y = -(2.0 * kPi * ai);
  reinterpret_cast<double2*>(itab)[(size_t)(mu + L_f) * ld + j] = o;
}

// Delta^p = d^p(pi/2) for p <= L (wigner.cpp:28-80), one CTA, level by level. The previous
// level's top row is staged in shared memory; each level's non-negative sector is built in
// shared memory (downward three-term recursion per column, then transpose) and written to
// global through the d-matrix symmetries. Explicit _rn intrinsics keep every operation
// separately rounded (no FMA contraction), so the table is bit-identical to the reference.
// PRE: the recursion coefficients of a level (a square root and a division per (m, m') --
// the slow part) are computed by all threads before the recursion, so the serial chain of a
// column is two multiplies and a subtraction per step. Shared memory: 2 S^2 + 2 S doubles
// (PRE) or S^2 + S, S = L + 1.
template <bool PRE>
__global__ void k_delta(int L, double* __restrict__ delta) {
  extern __shared__ double sm[];
  const int S = L + 1;
  double* sec = sm;           // S x S sector [m][mp], m, mp >= 0
  double* top = sm + S * S;   // previous level's top row Delta^{l-1}_{l-1, mp}
  double* ca = top + S;       // PRE: 2 mp / sqrt((l - m)(l + m + 1)) at [m][mp]
  double* cc = ca + S * S;    // PRE: sqrt((l - m - 1)(l + m + 2)) / sqrt((l - m)(l + m + 1))
  const int tid = threadIdx.x;
  if (tid == 0) {
    delta[0] = 1.0;
    top[0] = 1.0;
  }
  __syncthreads();
  size_t off = 1;
  for (int l = 1; l <= L; ++l) {
    const int w = 2 * l + 1;
    // top row m = l from the previous degree (Trapani seeds)
    for (int mp = tid; mp <= l; mp += blockDim.x) {
      double v;
      if (mp == 0) {
        v = __dmul_rn(-__dsqrt_rn(__ddiv_rn(2.0 * l - 1.0, 2.0 * l)), top[0]);
      } else {
        const double num = __dmul_rn((double)l, 2.0 * l - 1.0);
        const double den = __dmul_rn(2.0 * (l + mp), (double)l + mp - 1.0);
        v = __dmul_rn(__dsqrt_rn(__ddiv_rn(num, den)), top[mp - 1]);
      }
      sec[l * S + mp] = v;
    }
    if constexpr (PRE) {
      for (int idx = tid; idx < l * l; idx += blockDim.x) {
        const int m = idx / l, mp = idx % l;
        if (mp > m) continue;
        const double denom = __dsqrt_rn(__dmul_rn((double)(l - m), l + m + 1.0));
        ca[m * S + mp] = __ddiv_rn(2.0 * mp, denom);
        if (mp == 0 && m + 2 <= l)
          cc[m] = __ddiv_rn(__dsqrt_rn(__dmul_rn(l - m - 1.0, l + m + 2.0)), denom);
      }
    }
    __syncthreads();
    // downward recursion in m over the sector m >= mp >= 0, one column per thread
    for (int mp = tid; mp <= l - 1; mp += blockDim.x) {
      for (int m = l - 1; m >= mp; --m) {
        double value;
        if constexpr (PRE) {
          value = __dmul_rn(ca[m * S + mp], sec[(m + 1) * S + mp]);
          if (m + 2 <= l) value = __dsub_rn(value, __dmul_rn(cc[m], sec[(m + 2) * S + mp]));
        } else {
          const double denom = __dsqrt_rn(__dmul_rn((double)(l - m), l + m + 1.0));
          value = __dmul_rn(__ddiv_rn(2.0 * mp, denom), sec[(m + 1) * S + mp]);
          if (m + 2 <= l) {
            const double c2 = __ddiv_rn(__dsqrt_rn(__dmul_rn(l - m - 1.0, l + m + 2.0)), denom);
            value = __dsub_rn(value, __dmul_rn(c2, sec[(m + 2) * S + mp]));
          }
        }
        sec[m * S + mp] = value;
      }
    }
    __syncthreads();
    // transpose into the upper triangle
    for (int idx = tid; idx < (l + 1) * (l + 1); idx += blockDim.x) {
      const int m = idx / (l + 1), mp = idx % (l + 1);
      if (mp > m) sec[m * S + mp] = (((mp - m) & 1) ? -1.0 : 1.0) * sec[mp * S + m];
    }
    __syncthreads();
    // write the full level through the symmetries
    double* lev = delta + off;
    for (int idx = tid; idx < w * w; idx += blockDim.x) {
      const int q = idx / w - l, qp = idx % w - l;
      const int m = q < 0 ? -q : q, mp = qp < 0 ? -qp : qp;
      const double v = sec[m * S + mp];
      double sgn = 1.0;
      if (q < 0 && qp >= 0) sgn = ((l + mp) & 1) ? -1.0 : 1.0;
      else if (q >= 0 && qp < 0) sgn = ((l + m) & 1) ? -1.0 : 1.0;
      else if (q < 0 && qp < 0) sgn = ((m + mp) & 1) ? -1.0 : 1.0;
      lev[idx] = sgn * v;
    }
    for (int mp = tid; mp <= l; mp += blockDim.x) top[mp] = sec[l * S + mp];
    off += (size_t)w * w;
    __syncthreads();
  }
}

// Launch k_delta for band limit L on stream s (one CTA).
inline cudaError_t launch_delta(int L, double* out, cudaStream_t s) {
  const size_t S = (size_t)L + 1;
  const size_t pre = sizeof(double) * (2 * S * S + 2 * S), plain = sizeof(double) * (S * S + S);
  if (pre <= 227 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_delta<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)pre);
    if (e != cudaSuccess) return e;
    k_delta<true><<<1, 256, pre, s>>>(L, out);
  } else {
    if (plain > 227 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(k_delta<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plain);
    if (e != cudaSuccess) return e;
    k_delta<false><<<1, 256, plain, s>>>(L, out);
  }
  return cudaGetLastError();
}

__device__ __forceinline__ size_t delta_offset(int p) {
  return (size_t)p * (2 * p - 1) * (2 * p + 1) / 3;
}

// d^p_{q,q'}(beta_b) = Re[i^{q-q'} sum_q'' Delta^p_{q''q} Delta^p_{q''q'} e^{-i q'' beta_b}]
// (wigner.hpp:55-60), beta_b = 2 pi b / n for b <= L. Layout [p][q][q'][b].
__global__ void k_dtab(int L, const double* __restrict__ delta, const double2* __restrict__ rou,
                       double* __restrict__ dtab) {
  const int p = blockIdx.y;
  const int w = 2 * p + 1, nb = L + 1, n = 2 * L + 1;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= w * w * nb) return;
  const int b = idx % nb;
  const int qq = idx / nb;
  const int iq = qq / w, iqp = qq % w;  // q + p, q' + p
  const double* lev = delta + delta_offset(p);
  double ar = 0.0, ai = 0.0;
  for (int ipp = 0; ipp < w; ++ipp) {
    const int qpp = ipp - p;
    const double dd = lev[ipp * w + iq] * lev[ipp * w + iqp];
    int e = (qpp * b) % n;
    if (e < 0) e += n;
    const double2 z = rou[e];
    ar += dd * z.x;
    ai += dd * z.y;
  }
  const int k = (((iq - iqp) % 4) + 4) % 4;  // i^{q-q'}
  double v;
  switch (k) {
    case 0: v = ar; break;
    case 1: v = -ai; break;
    case 2: v = -ar; break;
    default: v = ai; break;
  }
  dtab[delta_offset(p) * nb + idx] = v;
}

// Window table of the coupling stage: W[c][col] with c = qoff[q+L] + p-|q| and col = b*n + c_g:
//   W = sum_{q'=-p}^{p} h_p^{q'} d^p_{q q'}(beta_b) e^{-i q' gamma_{c_g}}.
// Then g(l, m)[a][b][c] = sum_q e^{-i q alpha_a} sum_p conj(mod_p^q) W[c(p,q)][b*n+c].
// Layout: tile_nt == 0 -> W[c][col]; tile_nt = NT > 0 -> the column-tiled layout of the
// warp-specialized coupling kernel, W[col / NT][c][swz(c, col % NT)] with the 16-B chunk
// swizzle of wtile_index(), columns of the last tile beyond ncol zero-filled.
__host__ __device__ __forceinline__ size_t wtile_index(int c, int col, int NPQ, int NT) {
  const int cc = col % NT;
  const int sw = (cc & ~7) | ((cc & 7) ^ ((2 * c) & 7));
  return ((size_t)(col / NT) * NPQ + c) * NT + sw;
}

__global__ void k_wtab(int L, const double* __restrict__ h, const double* __restrict__ dtab,
                       const double2* __restrict__ rou, const int* __restrict__ pq_q,
                       int tile_nt, int ncol_pad, double2* __restrict__ W) {
  const int n = 2 * L + 1, nb = L + 1, ncol = n * nb;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  const int NPQ = (L + 1) * (L + 1);
  if (col >= ncol_pad) return;
  if (col >= ncol) {
    W[wtile_index(c, col, NPQ, tile_nt)] = make_double2(0.0, 0.0);
    return;
  }
  const int q = pq_q[2 * c], p = pq_q[2 * c + 1];
  const int b = col / n, cg = col % n;
  const int w = 2 * p + 1;
  const double* drow = dtab + delta_offset(p) * nb + (size_t)(q + p) * w * nb + b;
  double ar = 0.0, ai = 0.0;
  for (int iqp = 0; iqp < w; ++iqp) {
    const int qp = iqp - p;
    const double2 hv = *reinterpret_cast<const double2*>(h + 2 * (p * p + p + qp));
    const double d = drow[(size_t)iqp * nb];
    int e = (qp * cg) % n;
    if (e < 0) e += n;
    const double2 z = rou[e];
    const double tr = hv.x * d, ti = hv.y * d;
    ar += tr * z.x - ti * z.y;
    ai += tr * z.y + ti * z.x;
  }
  const size_t dst = tile_nt ? wtile_index(c, col, NPQ, tile_nt) : (size_t)c * ncol + col;
  W[dst] = make_double2(ar, ai);
}


}  // namespace slsht_cuda
