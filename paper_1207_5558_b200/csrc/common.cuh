// Shared definitions of the sm_100a directional-SLSHT kernels (FP64 throughout).
#pragma once

#include <cstdint>

namespace slsht_cuda {

constexpr double kPi = 3.14159265358979323846;

// FP64 tensor-core MMA (DMMA.8x8x4): D(8x8) += A(8x4) * B(4x8); one double per lane for A and
// B, two for D.  A: row = lane/4, k = lane%4;  B: k = lane%4, col = lane/4;
// D: row = lane/4, col = 2*(lane%4) + e.  Measured 37.1 TFLOP/s on B200 vs 34.2 for DFMA
// (profiles/fp64_peak.txt), and it takes operands from registers at 1 double per lane.
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Same MMA as a non-volatile asm: the compiler may schedule fragment loads and other MMAs
// around it (the result is only consumed through its outputs).
__device__ __forceinline__ void dmma_nv(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

struct CompRec {
  int l, m;
  long long slot;   // output volume slot of (l, m)
  long long mslot;  // output slot of the mirrored (l, -m) volume, -1 when not emitted
};

struct FftPlan {
  int nstages;
  int radix[8];
  int span[8];
};

// Coefficients of the normalized associated-Legendre recursion of harmonics.cpp:60-89 for
// order |m| = am, degrees lo..hi, written to shared memory once per CTA so the per-node
// recursion is pure FMA work:
//   sf[k] = sqrt((2k+1)/(2k)) (sectoral seed factors, k = 1..am)
//   ca[l] = sqrt((4l^2-1)/(l^2-am^2)), cb[l] = sqrt(((l-1)^2-am^2)/(4(l-1)^2-1)), l >= am+2
//   c1    = sqrt(2 am + 3)
__device__ __forceinline__ void legendre_coeffs(int am, int hi, double* sf, double* ca,
                                                double* cb) {
  for (int k = 1 + threadIdx.x; k <= am; k += blockDim.x) sf[k] = sqrt((2.0 * k + 1.0) / (2.0 * k));
  const double am2 = (double)am * am;
  for (int l = am + 2 + threadIdx.x; l <= hi; l += blockDim.x) {
    const double ll = (double)l * l;
    const double l1 = (double)(l - 1) * (l - 1);
    ca[l] = sqrt((4.0 * ll - 1.0) / (ll - am2));
    cb[l] = sqrt((l1 - am2) / (4.0 * l1 - 1.0));
  }
}

// lambda_l^m(theta) recursion state for one node, driven by the shared coefficient tables.
struct LegendreIt {
  double x, prev, cur;
  int am, l;
  __device__ __forceinline__ void seed(int m, double c, double s, const double* sf) {
    am = m < 0 ? -m : m;
    double sect = 0.28209479177387814;  // 1/sqrt(4 pi)
    for (int k = 1; k <= am; ++k) sect *= -s * sf[k];
    if (m < 0 && (am & 1)) sect = -sect;
    x = c;
    l = am;
    prev = 0.0;
    cur = sect;
  }
  __device__ __forceinline__ void next(const double* ca, const double* cb) {
    ++l;
    double v;
    if (l == am + 1) v = x * sqrt(2.0 * am + 3.0) * cur;
    else v = ca[l] * (x * cur - cb[l] * prev);
    prev = cur;
    cur = v;
  }
};

}  // namespace slsht_cuda
