// FP64 dense linear algebra of the §8(f) engines (the Slepian window solver and the device
// direct engine): real and complex GEMMs on the FP64 tensor cores (DMMA 8x8x4), a transposed
// complex GEMV and the vector reductions of the power iteration. Column-major operands with
// leading dimensions, cuBLAS conventions (op(X) = X, X^T, or X^H), C = op(A) op(B) (alpha = 1,
// beta = 0: the only form the engines use). Every reduction runs in a fixed order, so results
// are bitwise reproducible.
#pragma once

#include "common.cuh"

namespace slsht_cuda {

enum BlasOp { kOpN = 0, kOpT = 1, kOpC = 2 };

// Tiles: 64 x 64 of C per CTA, K chunks of 16, 8 warps as 2 (rows) x 4 (columns), each warp
// 32 x 16 = 4 x 2 DMMA tiles. Operands are staged in shared memory with plain loads (any op,
// any leading dimension; these GEMMs are not on the hot path).
constexpr int BL_TM = 64, BL_TN = 64, BL_TK = 16;

// element (r, c) of op(X) for a column-major X with leading dimension ld
template <typename T>
__device__ __forceinline__ T bl_op_elem(const T* X, int ld, int op, int r, int c);
template <>
__device__ __forceinline__ double bl_op_elem<double>(const double* X, int ld, int op, int r, int c) {
  return op == kOpN ? X[(size_t)c * ld + r] : X[(size_t)r * ld + c];
}
template <>
__device__ __forceinline__ double2 bl_op_elem<double2>(const double2* X, int ld, int op, int r,
                                                       int c) {
  if (op == kOpN) return X[(size_t)c * ld + r];
  const double2 v = X[(size_t)r * ld + c];
  return op == kOpC ? make_double2(v.x, -v.y) : v;
}

// C (m x n) = op(A) (m x k) op(B) (k x n), real; batch z with element strides sA, sB, sC
__global__ void __launch_bounds__(256) k_dgemm(int opA, int opB, int m, int n, int k,
                                               const double* __restrict__ A, int lda, long long sA,
                                               const double* __restrict__ B, int ldb, long long sB,
                                               double* __restrict__ C, int ldc, long long sC) {
  __shared__ double As[BL_TM][BL_TK + 1];
  __shared__ double Bs[BL_TK][BL_TN + 1];
  const int z = blockIdx.z;
  A += z * sA;
  B += z * sB;
  C += z * sC;
  const int m0 = blockIdx.x * BL_TM, n0 = blockIdx.y * BL_TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // warp tile rows wm*32.., cols wn*16..
  double acc[4][2][2] = {};
  for (int k0 = 0; k0 < k; k0 += BL_TK) {
    for (int e = tid; e < BL_TM * BL_TK; e += 256) {
      const int r = e % BL_TM, kk = e / BL_TM;
      As[r][kk] = (m0 + r < m && k0 + kk < k) ? bl_op_elem(A, lda, opA, m0 + r, k0 + kk) : 0.0;
    }
    for (int e = tid; e < BL_TK * BL_TN; e += 256) {
      const int kk = e % BL_TK, c = e / BL_TK;
      Bs[kk][c] = (k0 + kk < k && n0 + c < n) ? bl_op_elem(B, ldb, opB, k0 + kk, n0 + c) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < BL_TK / 4; ++ks) {
      const int kk = ks * 4 + (lane & 3);
      double a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[wm * 32 + mi * 8 + (lane >> 2)][kk];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = Bs[kk][wn * 16 + ni * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = m0 + wm * 32 + mi * 8 + (lane >> 2);
        const int c = n0 + wn * 16 + ni * 8 + 2 * (lane & 3) + e;
        if (r < m && c < n) C[(size_t)c * ldc + r] = acc[mi][ni][e];
      }
}

// The complex version: Gauss 3-product per complex MAC (K1 += (ar+ai) br, K2 += ar (bi-br),
// K3 += ai (br+bi); re = K1 - K3, im = K1 + K2), the same tiles
__global__ void __launch_bounds__(256) k_zgemm(int opA, int opB, int m, int n, int k,
                                               const double2* __restrict__ A, int lda, long long sA,
                                               const double2* __restrict__ B, int ldb, long long sB,
                                               double2* __restrict__ C, int ldc, long long sC) {
  __shared__ double2 As[BL_TM][BL_TK + 1];
  __shared__ double2 Bs[BL_TK][BL_TN + 1];
  const int z = blockIdx.z;
  A += z * sA;
  B += z * sB;
  C += z * sC;
  const int m0 = blockIdx.x * BL_TM, n0 = blockIdx.y * BL_TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  double c1[4][2][2] = {}, c2[4][2][2] = {}, c3[4][2][2] = {};
  const double2 z0 = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < k; k0 += BL_TK) {
    for (int e = tid; e < BL_TM * BL_TK; e += 256) {
      const int r = e % BL_TM, kk = e / BL_TM;
      As[r][kk] = (m0 + r < m && k0 + kk < k) ? bl_op_elem(A, lda, opA, m0 + r, k0 + kk) : z0;
    }
    for (int e = tid; e < BL_TK * BL_TN; e += 256) {
      const int kk = e % BL_TK, c = e / BL_TK;
      Bs[kk][c] = (k0 + kk < k && n0 + c < n) ? bl_op_elem(B, ldb, opB, k0 + kk, n0 + c) : z0;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < BL_TK / 4; ++ks) {
      const int kk = ks * 4 + (lane & 3);
      double2 a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = As[wm * 32 + mi * 8 + (lane >> 2)][kk];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = Bs[kk][wn * 16 + ni * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) {
          dmma(c1[mi][ni][0], c1[mi][ni][1], a[mi].x + a[mi].y, b[ni].x);
          dmma(c2[mi][ni][0], c2[mi][ni][1], a[mi].x, b[ni].y - b[ni].x);
          dmma(c3[mi][ni][0], c3[mi][ni][1], a[mi].y, b[ni].x + b[ni].y);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = m0 + wm * 32 + mi * 8 + (lane >> 2);
        const int c = n0 + wn * 16 + ni * 8 + 2 * (lane & 3) + e;
        if (r < m && c < n)
          C[(size_t)c * ldc + r] =
              make_double2(c1[mi][ni][e] - c3[mi][ni][e], c1[mi][ni][e] + c2[mi][ni][e]);
      }
}

inline cudaError_t dgemm(int opA, int opB, int m, int n, int k, const double* A, int lda,
                         const double* B, int ldb, double* C, int ldc, cudaStream_t s,
                         int batch = 1, long long sA = 0, long long sB = 0, long long sC = 0) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((m + BL_TM - 1) / BL_TM, (n + BL_TN - 1) / BL_TN, batch);
  k_dgemm<<<grid, 256, 0, s>>>(opA, opB, m, n, k, A, lda, sA, B, ldb, sB, C, ldc, sC);
  return cudaGetLastError();
}

inline cudaError_t zgemm(int opA, int opB, int m, int n, int k, const double2* A, int lda,
                         const double2* B, int ldb, double2* C, int ldc, cudaStream_t s,
                         int batch = 1, long long sA = 0, long long sB = 0, long long sC = 0) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((m + BL_TM - 1) / BL_TM, (n + BL_TN - 1) / BL_TN, batch);
  k_zgemm<<<grid, 256, 0, s>>>(opA, opB, m, n, k, A, lda, sA, B, ldb, sB, C, ldc, sC);
  return cudaGetLastError();
}

// y = A^T x for a column-major complex n x n A (no conjugation: cuBLAS OP_T): one warp per
// output, lanes stride the column, fixed shuffle tree
__global__ void k_zgemv_t(int n, const double2* __restrict__ A, int lda,
                          const double2* __restrict__ x, double2* __restrict__ y) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n) return;
  const double2* col = A + (size_t)row * lda;
  double sr = 0.0, si = 0.0;
  for (int i = lane; i < n; i += 32) {
    const double2 a = col[i], v = x[i];
    sr = fma(a.x, v.x, fma(-a.y, v.y, sr));
    si = fma(a.x, v.y, fma(a.y, v.x, si));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, off);
    si += __shfl_xor_sync(0xffffffffu, si, off);
  }
  if (lane == 0) y[row] = make_double2(sr, si);
}

// out[0] = (v^H x) (complex), out[1] = (||x||_2, 0): one CTA of 1024 threads, fixed tree
// (a scaled sum of squares guards ||x|| against overflow like DZNRM2)
__global__ void __launch_bounds__(1024) k_zdot_nrm(int n, const double2* __restrict__ v,
                                                   const double2* __restrict__ x,
                                                   double2* __restrict__ out) {
  __shared__ double red[3][32];
  __shared__ double xmax_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double mx = 0.0;
  for (int i = tid; i < n; i += 1024) mx = fmax(mx, fmax(fabs(x[i].x), fabs(x[i].y)));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) red[0][warp] = mx;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < 32; ++w) m = fmax(m, red[0][w]);
    xmax_s = m;
  }
  __syncthreads();
  const double scale = xmax_s > 0.0 ? 1.0 / xmax_s : 0.0;
  double dr = 0.0, di = 0.0, ss = 0.0;
  for (int i = tid; i < n; i += 1024) {
    const double2 a = v[i], b = x[i];
    dr = fma(a.x, b.x, fma(a.y, b.y, dr));  // conj(a) b
    di = fma(a.x, b.y, fma(-a.y, b.x, di));
    const double bx = b.x * scale, by = b.y * scale;
    ss = fma(bx, bx, fma(by, by, ss));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dr += __shfl_xor_sync(0xffffffffu, dr, off);
    di += __shfl_xor_sync(0xffffffffu, di, off);
    ss += __shfl_xor_sync(0xffffffffu, ss, off);
  }
  __syncthreads();
  if (lane == 0) {
    red[0][warp] = dr;
    red[1][warp] = di;
    red[2][warp] = ss;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0, c = 0.0;
    for (int w = 0; w < 32; ++w) {
      a += red[0][w];
      b += red[1][w];
      c += red[2][w];
    }
    out[0] = make_double2(a, b);
    out[1] = make_double2(xmax_s * sqrt(c), 0.0);
  }
}

// x *= 1 / ||x|| with the norm from k_zdot_nrm's out[1] (on the device: no host round trip)
__global__ void k_zscale_inv(int n, const double2* __restrict__ nrm, double2* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double inv = 1.0 / nrm[1].x;
  x[i] = make_double2(x[i].x * inv, x[i].y * inv);
}

}  // namespace slsht_cuda
