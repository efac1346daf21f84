// The direct engine, forward_direct (transform.cpp:313-388), on the device: for every rotation
// cell rho = (alpha_a, beta_b, gamma_c) of the So3 grid,
//
//   g(l, m; rho) = sh_analysis( sh_synthesis(f) * sh_synthesis(R_rho h) )_l^m
//
// on the sphere grid of band L = max(lmax, L_g) (harmonics.cpp:99-203, grids.cpp:28-39). It shares
// only the Delta tables and d(beta) with the fast engine (as the reference's direct engine
// does, wigner_d_from_delta), so it is an independent check of the modulated SHT, the coupling
// and the alpha FFT at band limits where the CPU direct engine is infeasible.
//
// Batched over R cells at a time, every transform is a GEMM (cuBLAS) against tables built here:
//   HR[(p,q)][r]   = e^{-i q alpha_a} t1[(p,q)][b,c]   (t1 = the window table W of the fast path)
//   S[t][q][r]     = sum_p lambda_p^q(theta_t) HR        synthesis Legendre step, per q
//   H[t][k][r]     = sum_q e^{+2 pi i q k/n} S            synthesis ring DFT
//   P              = F[t][k] * H                           the product map (F = synthesis of f)
//   FM[t][m][r]    = (1/n) sum_k e^{-2 pi i m k/n} P      analysis ring DFT
//   g[(l,m)][r]    = sum_t Q_m[l][t] FM[t][m][r]          analysis theta step
// Q_m folds the reference's parity extension, trigonometric interpolation to the colatitudes of
// S_{2L} and exact quadrature (theta_weights(2L) against lambda_l^m) into one real matrix:
//   Q_m = Lambda_m diag(2 pi v) B_{m mod 2},
//   B_par[j][t] = (1/n) [ D(theta_j - theta_t) + (-1)^m [t < L] D(theta_j + theta_t) ],
// D(x) = sum_{u=-L}^{L} e^{iux} the Dirichlet kernel (the sum over k of the reference's
// trigonometric coefficients, harmonics.cpp:117-147, in closed form).
#pragma once

#include "common.cuh"

namespace slsht_cuda {

// rows l = |m|..l1 of lambda_l^m at the colatitudes th[0..nt), optionally scaled per column:
// out[(l - |m|) * ld + t]. One thread per colatitude; recursion coefficients in shared memory.
__global__ void k_dir_lrows(int m, int l1, int nt, const double* __restrict__ th,
                            const double* __restrict__ scale, double* __restrict__ out, int ld) {
  extern __shared__ double coef[];
  double *sf = coef, *ca = coef + (l1 + 2), *cb = coef + 2 * (l1 + 2);
  const int am = m < 0 ? -m : m;
  legendre_coeffs(am, l1, sf, ca, cb);
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  double s, c;
  sincos(th[t], &s, &c);
  const double w = scale ? scale[t] : 1.0;
  LegendreIt r;
  r.seed(m, c, s, sf);
  for (int l = am; l <= l1; ++l) {
    if (l > am) r.next(ca, cb);
    out[(size_t)(l - am) * ld + t] = w * r.cur;
  }
}

// Fring[m + L_f][t] = sum_l f_l^m lambda_l^m(theta_t)  (synthesis Legendre step of f)
__global__ void k_dir_fring(int L_f, const double2* __restrict__ f, int nt,
                            const double* __restrict__ th, double2* __restrict__ fring) {
  extern __shared__ double coef[];
  double *sf = coef, *ca = coef + (L_f + 2), *cb = coef + 2 * (L_f + 2);
  const int m = (int)blockIdx.y - L_f, am = m < 0 ? -m : m;
  legendre_coeffs(am, L_f, sf, ca, cb);
  __syncthreads();
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  double s, c;
  sincos(th[t], &s, &c);
  LegendreIt r;
  r.seed(m, c, s, sf);
  double ar = 0.0, ai = 0.0;
  for (int l = am; l <= L_f; ++l) {
    if (l > am) r.next(ca, cb);
    const double2 v = f[l * l + l + m];
    ar = fma(v.x, r.cur, ar);
    ai = fma(v.y, r.cur, ai);
  }
  fring[(size_t)(m + L_f) * nt + t] = make_double2(ar, ai);
}

// e^{sign 2 pi i (r + r0)(c + c0) / n} * scale, row-major rows x cols (exact integer phases)
__global__ void k_dir_dft(int rows, int cols, int r0, int c0, int n, double sign, double scale,
                          double2* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * cols) return;
  const int r = idx / cols + r0, c = idx % cols + c0;
  long long e = ((long long)r * c) % n;
  if (e < 0) e += n;
  double s, co;
  sincospi(2.0 * (double)e / n, &s, &co);
  out[idx] = make_double2(co * scale, sign * s * scale);
}

// F[t][k] = sum_m Fring[m][t] e^{+2 pi i m k / n}
__global__ void k_dir_fmap(int L_f, int nt, int n, const double2* __restrict__ fring,
                           double2* __restrict__ F) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nt * n) return;
  const int t = idx / n, k = idx % n;
  double ar = 0.0, ai = 0.0;
  for (int m = -L_f; m <= L_f; ++m) {
    long long e = ((long long)m * k) % n;
    if (e < 0) e += n;
    double s, c;
    sincospi(2.0 * (double)e / n, &s, &c);
    const double2 v = fring[(size_t)(m + L_f) * nt + t];
    ar += v.x * c - v.y * s;
    ai += v.x * s + v.y * c;
  }
  F[idx] = make_double2(ar, ai);
}

__device__ __forceinline__ double dirichlet(int L, double x) {
  const double s = sin(0.5 * x);
  if (s == 0.0) return 2.0 * L + 1.0;
  return sin((L + 0.5) * x) / s;
}

// B[par][j][t], j < nn = 2L+1 analysis colatitudes (of S_{2L}), t <= L rings
__global__ void k_dir_bpar(int L, int nn, const double* __restrict__ nodes,
                           const double* __restrict__ rings, double* __restrict__ B) {
  const int nt = L + 1, n = 2 * L + 1;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nn * nt) return;
  const int j = idx / nt, t = idx % nt;
  const double d0 = dirichlet(L, nodes[j] - rings[t]);
  const double d1 = (t < L) ? dirichlet(L, nodes[j] + rings[t]) : 0.0;
  B[idx] = (d0 + d1) / n;                    // even m
  B[(size_t)nn * nt + idx] = (d0 - d1) / n;  // odd m
}

// HR[c][r] = e^{-i q alpha_a} W[c][col] for cell r = a * ncol + col (a < nh, col < ncol)
__global__ void k_dir_hr(int R, const long long* __restrict__ cells, int NPQ, int ncol, int nh,
                         const int* __restrict__ pq, const double2* __restrict__ W,
                         double2* __restrict__ HR) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r >= R) return;
  const long long cell = cells[r];
  const int a = (int)(cell / ncol), col = (int)(cell % ncol);
  const int q = pq[2 * c];
  int e = (int)(((long long)q * a) % nh);
  if (e < 0) e += nh;
  double s, co;
  sincospi(2.0 * (double)e / nh, &s, &co);  // e^{-i q alpha_a} = co - i s
  const double2 w = W[(size_t)c * ncol + col];
  HR[(size_t)c * R + r] = make_double2(w.x * co + w.y * s, w.y * co - w.x * s);
}

// H[t][k][r] *= F[t][k]
__global__ void k_dir_product(long long total, int R, const double2* __restrict__ F,
                              double2* __restrict__ H) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const double2 f = F[idx / R];
  const double2 h = H[idx];
  H[idx] = make_double2(f.x * h.x - f.y * h.y, f.x * h.y + f.y * h.x);
}

// result[(l^2 + l + m)][r] = OUT[m + lmax][l - |m|][r]  (OUT rows padded to lmax + 1)
__global__ void k_dir_scatter(int lmax, int R, long long total, const double2* __restrict__ OUT,
                              double2* __restrict__ res) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int row = (int)(idx / R), r = (int)(idx % R);  // coeff index, cell
  int l = (int)sqrt((double)row);
  while (l * l > row) --l;
  while ((l + 1) * (l + 1) <= row) ++l;
  const int m = row - l * l - l, am = m < 0 ? -m : m;
  res[idx] = OUT[((size_t)(m + lmax) * (lmax + 1) + (l - am)) * R + r];
}

}  // namespace slsht_cuda
