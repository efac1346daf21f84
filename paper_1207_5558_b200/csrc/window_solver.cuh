// Slepian window solver on the device: the dominant eigenfunction of the concentration kernel
// of an elliptical region (reference proj/src/window.cpp:44-198).
//
//   1. mask samples of S_{oversample * L} inside the region with weights theta_weights * dphi
//      (host: the same formulas as window.cpp:57-71, so the same samples and weights);
//   2. Y[s][coeff_index(l, m)] = lambda_l^m(theta_s) e^{i m phi_s} on the device
//      (window.cpp:77-88), one thread per (sample, order);
//   3. K = Y^H diag(w) Y with one ZGEMM (cuBLAS: a plain library GEMM), symmetrized
//      (window.cpp:95-123);
//   4. power iteration from e_(0,0) with the reference's Rayleigh-quotient stopping rule
//      (window.cpp:133-157): ZGEMV, ZDOTC, DZNRM2 on the device, the two scalars per step to
//      the host;
//   5. host: north-pole phase, conjugate symmetrization, unit norm, DC check
//      (window.cpp:159-196).
#pragma once


#include <complex>

#include <cmath>
#include <vector>

#include "common.cuh"

namespace slsht_cuda {

// Y rows of the mask samples, row-major [sample][coeff_index], Legendre recursion as
// harmonics.cpp:36-58 (legendre_column).
__global__ void k_window_y(int L, int n_samples, const double* __restrict__ theta,
                           const double* __restrict__ phi, double2* __restrict__ Y) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 2 * L + 1;
  if (idx >= n_samples * n) return;
  const int s = idx / n, m = idx % n - L;
  const int am = m < 0 ? -m : m;
  const double th = theta[s];
  const double x = cos(th), sn = sin(th);
  double sect = 1.0 / sqrt(4.0 * kPi);
  for (int j = 1; j <= am; ++j) sect *= -sn * sqrt((2.0 * j + 1.0) / (2.0 * j));
  if (m < 0 && (am & 1)) sect = -sect;
  double ec, es;
  sincos(m * phi[s], &es, &ec);
  double2* row = Y + (size_t)s * (L + 1) * (L + 1);
  double prev = 0.0, cur = sect;
  for (int l = am; l <= L; ++l) {
    if (l == am + 1) {
      const double v = x * sqrt(2.0 * am + 3.0) * cur;
      prev = cur;
      cur = v;
    } else if (l > am + 1) {
      const double ll = (double)l * l, l1 = (double)(l - 1) * (l - 1);
      const double a = sqrt((4.0 * ll - 1.0) / (ll - (double)am * am));
      const double b = sqrt((l1 - (double)am * am) / (4.0 * l1 - 1.0));
      const double v = a * (x * cur - b * prev);
      prev = cur;
      cur = v;
    }
    row[l * l + l + m] = make_double2(cur * ec, cur * es);
  }
}

// B = Y with sample row s scaled by w_s
__global__ void k_window_scale(int dim, int n_samples, const double* __restrict__ w,
                               const double2* __restrict__ Y, double2* __restrict__ B) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)dim * n_samples) return;
  const double ws = w[i / dim];
  const double2 y = Y[i];
  B[i] = make_double2(ws * y.x, ws * y.y);
}

// K[r][c] <- (K[r][c] + conj(K[c][r])) / 2 (window.cpp:115-123)
__global__ void k_window_symmetrize(int dim, double2* __restrict__ K) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)dim * dim) return;
  const int r = (int)(i / dim), c = (int)(i % dim);
  if (c < r) return;
  const double2 a = K[(size_t)r * dim + c], b = K[(size_t)c * dim + r];
  const double2 avg = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
  K[(size_t)r * dim + c] = avg;
  K[(size_t)c * dim + r] = make_double2(avg.x, -avg.y);
}

}  // namespace slsht_cuda
