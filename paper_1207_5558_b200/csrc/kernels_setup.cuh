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

// ---------------------------------------------------------------------------------------------
// The theta quadrature of the modulated SHT. The reference integrates over theta with the
// exact rule of S_{2L_g} (theta_weights(2L_g) on N_theta = 2L_g + 1 nodes, transform.cpp:
// 151-156, 206-219). The integrand lambda_{l'}^{m-q} lambda_l^m lambda_p^q (l' <= L_f, l <= L_g,
// p <= L_h) is sin(theta) times a polynomial in x = cos(theta) of degree <= l' + l + p <=
// 2 L_g (the three orders sum to zero, so the sin powers pair up), so the (L_g + 1)-point
// Gauss-Legendre rule in x is exact for it too: the same integral, on fewer nodes, equal to
// the reference's up to roundoff (~1e-13 relative; tests/test_gpu.py). The GL nodes are
// symmetric, x <-> -x, and lambda_l^m(-x) = (-1)^(l+m) lambda_l^m(x), so the engine keeps only
// the nodes with x >= 0 and folds the mirrored node into the I-table:
//   mod_p^q(l, m) = sum_{x_j >= 0} w_j lambda_l^m lambda_p^q I_s(x_j, m - q),
//   s = (l + m + p + q) mod 2, I_0 = I(x) + I(-x), I_1 = I(x) - I(-x)
// (the x = 0 node of an odd rule enters with half its weight; there I_1 = 0 and I_0 = 2 I).
// Half the nodes again, so the modulated-SHT GEMM does a quarter of the reference rule's work.
//
// k_glnodes: node j < K (the j-th root of P_NG from theta = 0) by Newton's method in theta,
// from Tricomi's asymptotic guess x = (1 - 1/(8 NG^2) + 1/(8 NG^3)) cos(pi (j + 3/4) /
// (NG + 1/2)) (error O(NG^-4): one or two steps reach full precision). Near the pole x = cos
// theta carries theta only to eps / sin(theta), so P_NG is evaluated through y = 1 - x =
// 2 sin^2(theta / 2), exact to an ulp at every theta, with the recursion on the differences
//   D_k = P_k - P_{k-1} = b_k D_{k-1} - a_k y P_{k-1},   a_k = (2k - 1)/k, b_k = (k - 1)/k
// (shared tables, no division in the dependent chain). A node from x-space Newton steps is off
// by up to ~1e-14 rad near the pole, which at l = L_g costs ~1e-13 relative in the modulated
// SHT (measured in long double at config 5, (l, m) = (1088, 0)). dP_NG/dtheta = NG (D_NG -
// y P_NG) / sin(theta). The weight w = 2 sin^2(theta) / (NG (D_NG - y P_NG))^2 needs the
// recursion to full precision (double loses ~NG ulps: 6e-13 rms at NG = 1089): for large NG
// the last evaluation runs in double-double arithmetic (a_k, b_k as double-double pairs). One thread
// per node; dynamic smem 4 (NG + 1) doubles.
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_fast2sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return DD{s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  const double s = __dadd_rn(a.hi, b.hi), v = __dsub_rn(s, a.hi);
  double e = __dadd_rn(__dsub_rn(a.hi, __dsub_rn(s, v)), __dsub_rn(b.hi, v));
  e = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
  return dd_fast2sum(s, e);
}
__device__ __forceinline__ DD dd_mul(DD a, DD b) {
  const double p = __dmul_rn(a.hi, b.hi);
  double e = fma(a.hi, b.hi, -p);
  e = fma(a.hi, b.lo, e);
  e = fma(a.lo, b.hi, e);
  return dd_fast2sum(p, e);
}
__device__ __forceinline__ DD dd_mul_d(DD a, double b) {
  const double p = __dmul_rn(a.hi, b);
  double e = fma(a.hi, b, -p);
  e = fma(a.lo, b, e);
  return dd_fast2sum(p, e);
}

__global__ void k_glnodes(int NG, int K, double* __restrict__ ncos, double* __restrict__ nsin,
                          double* __restrict__ weights) {
  extern __shared__ double tb[];  // [k][4]: a_k, its residual, b_k, its residual
  for (int k = 2 + threadIdx.x; k <= NG; k += blockDim.x) {
    const double a = (double)(2 * k - 1) / k, b = (double)(k - 1) / k;
    tb[4 * k] = a;
    tb[4 * k + 1] = fma(-a, (double)k, (double)(2 * k - 1)) / k;
    tb[4 * k + 2] = b;
    tb[4 * k + 3] = fma(-b, (double)k, (double)(k - 1)) / k;
  }
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= K) return;
  // P_NG and D_NG at y (double)
  auto eval = [&](double y, double& pn, double& dn) {
    double p = 1.0 - y, d = -y;  // P_1, D_1
    for (int k = 2; k <= NG; ++k) {
      d = fma(tb[4 * k + 2], d, -(tb[4 * k] * y) * p);
      p += d;
    }
    pn = p;
    dn = d;
  };
  const double g = (double)NG;
  const bool mid = 2 * j + 1 == NG;  // the middle node of an odd rule: x = 0 exactly
  double th = 0.5 * kPi;
  if (!mid) {
    th = acos((1.0 - 1.0 / (8.0 * g * g) + 1.0 / (8.0 * g * g * g)) *
              cos(kPi * (j + 0.75) / (g + 0.5)));
    for (int it = 0; it < 10; ++it) {
      const double sh = sin(0.5 * th), y = 2.0 * sh * sh;
      double pn, dn;
      eval(y, pn, dn);
      const double d = pn * sin(th) / (g * (dn - y * pn));  // P_NG / (dP_NG / dtheta)
      th -= d;
      if (fabs(d) < 1e-14) break;
    }
  }
  double c, s;
  sincos(th, &s, &c);
  double y;
  if (mid) {
    c = 0.0;
    s = 1.0;
    y = 1.0;
  } else {
    const double sh = sin(0.5 * th);
    y = 2.0 * sh * sh;
  }
  // the weight's P_NG, D_NG: in double-double above NG = 256 (below, the double recursion's
  // ~NG ulps stay under the other roundoff of the modulated SHT: 1.5e-14 rms at NG = 145)
  double dv;
  if (NG > 256) {
    DD p{1.0, 0.0}, d{-y, 0.0};
    p = dd_add(p, d);
    for (int k = 2; k <= NG; ++k) {
      const DD ay = dd_mul_d(DD{tb[4 * k], tb[4 * k + 1]}, y);
      const DD t = dd_mul(ay, p);
      d = dd_add(dd_mul(DD{tb[4 * k + 2], tb[4 * k + 3]}, d), DD{-t.hi, -t.lo});
      p = dd_add(p, d);
    }
    const DD yp = dd_mul_d(p, y);
    const DD den = dd_add(d, DD{-yp.hi, -yp.lo});  // D_NG - y P_NG = x P_NG - P_{NG-1}
    dv = g * (den.hi + den.lo);
  } else {
    double pn, dn;
    eval(y, pn, dn);
    dv = g * (dn - y * pn);
  }
  double w = 2.0 * s * s / (dv * dv);
  if (mid) w *= 0.5;
  ncos[j] = c;
  nsin[j] = s;
  weights[j] = w;
}

// The main-stream setup in one launch. Three independent parts run side by side:
//   blocks [0, ni): the I-table per (node block, order mu), recursion coefficients and f_l^mu
//     staged in shared memory: I_0 and I_1 (above) of I(theta_j, mu) = 2 pi conj(sum_l f_l^mu
//     lambda_l^mu(theta_j)) (transform.cpp:158-173), rows 2 (mu + L_f) + s;
//   blocks [ni, ni + nw): the window rows lambda_p^q(theta_j), q-major (p, q) rows
//     c = qoff[q+L] + p-|q| (transform.cpp:175-186), per (node block, order q);
//   the rest: theta_weights(2 L_g) of the reference rule, for its imaginary-residue check
//     (grids.cpp:86-89: NumericError), and beta weights (4 warps = 4 weights per block).
// The GL nodes come from k_glnodes. Row strides are ld (>= n_nodes, the padding stays zero).
struct SetupMainParams {
  int N, L_h, L_f, n_nodes, ld, nbx, ni, nw;
  const double* f;
  const int* qoff;
  const double *ncos, *nsin;
  double *betaw, *lamh, *itab;
  int* err;
};

__global__ void __launch_bounds__(128) k_setup_main(const SetupMainParams P) {
  extern __shared__ double coef[];
  int b = blockIdx.x;
  if (b < P.ni) {  // ---- I-table block (transform.cpp:158-173)
    const int L_f = P.L_f;
    double *sf = coef, *ca = coef + (L_f + 1), *cb = coef + 2 * (L_f + 1);
    double2* fs = reinterpret_cast<double2*>(coef + 3 * (L_f + 1) + ((3 * (L_f + 1)) & 1));
    const int mu = b / P.nbx - L_f;
    const int amu = mu < 0 ? -mu : mu;
    legendre_coeffs(amu, L_f, sf, ca, cb);
    for (int l = amu + threadIdx.x; l <= L_f; l += blockDim.x)
      fs[l] = *reinterpret_cast<const double2*>(P.f + 2 * (l * l + l + mu));
    __syncthreads();
    const int j = (b % P.nbx) * blockDim.x + threadIdx.x;
    if (j >= P.n_nodes) return;
    LegendreIt r;
    r.seed(mu, P.ncos[j], P.nsin[j], sf);
    // [parity of l + mu][re, im]: the even terms make I_0 / 2, the odd ones I_1 / 2
    double a[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int l = amu; l <= L_f; ++l) {
      if (l > amu) r.next(ca, cb);
      const double2 fv = fs[l];
      const int s = (l + amu) & 1;
      a[s][0] += fv.x * r.cur;
      a[s][1] += fv.y * r.cur;
    }
    double2* it = reinterpret_cast<double2*>(P.itab);
#pragma unroll
    for (int s = 0; s < 2; ++s)
      it[(size_t)(2 * (mu + L_f) + s) * P.ld + j] =
          make_double2(4.0 * kPi * a[s][0], -(4.0 * kPi * a[s][1]));
    return;
  }
  b -= P.ni;
  if (b < P.nw) {  // ---- window Legendre rows lambda_p^q(theta_j) (transform.cpp:175-186)
    const int L_h = P.L_h;
    double *sf = coef, *ca = coef + (L_h + 1), *cb = coef + 2 * (L_h + 1);
    const int q = b / P.nbx - L_h;
    const int aq = q < 0 ? -q : q;
    legendre_coeffs(aq, L_h, sf, ca, cb);
    __syncthreads();
    const int j = (b % P.nbx) * blockDim.x + threadIdx.x;
    if (j >= P.n_nodes) return;
    LegendreIt r;
    r.seed(q, P.ncos[j], P.nsin[j], sf);
    const int base = P.qoff[q + L_h];
    for (int p = aq; p <= L_h; ++p) {
      if (p > aq) r.next(ca, cb);
      P.lamh[(size_t)(base + p - aq) * P.ld + j] = r.cur;
    }
    return;
  }
  b -= P.nw;
  // ---- the reference rule's theta weights (only their residue check is used) and the beta
  // weights: one warp per weight
  const int N = P.N, L_h = P.L_h;
  const int w = (b * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w <= N) {
    const double theta = kPi * (2 * w + 1) / (2 * N + 1);
    double sr, si;
    quad_weight_sum(N, theta, lane, sr, si);
    if (lane == 0 && fabs(si) >= 1e-12) atomicExch(P.err, 1);
  } else if (w - (N + 1) <= L_h) {
    const int t = w - (N + 1);
    const int L = L_h, n = 2 * L + 1;
    if (t == 0) {
      if (lane == 0) P.betaw[0] = 4.0 * kPi * kPi / (L / 2 + 0.5);
    } else {
      double sr, si;
      quad_weight_sum(L, 2.0 * kPi * t / n, lane, sr, si);
      if (lane == 0) {
        if (fabs(si) >= 1e-12) atomicExch(P.err, 2);
        P.betaw[t] = 8.0 * kPi * kPi * sr;
      }
    }
  }
}

// Component-level entry points of the grid functions (slsht_cuda_theta_weights,
// slsht_cuda_beta_weights, slsht_cuda_legendre_rows): the same device code as the setup
// launch, one warp per weight / one thread per angle.
__global__ void k_theta_weights(int N, double* __restrict__ out, int* __restrict__ err) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t > N) return;
  const double theta = kPi * (2 * t + 1) / (2 * N + 1);  // grids.cpp:79-80
  double sr, si;
  quad_weight_sum(N, theta, lane, sr, si);
  if (lane == 0) {
    if (fabs(si) >= 1e-12) atomicExch(err, 1);
    out[t] = (t < N) ? 2.0 * sr / (2 * N + 1) : sr / (2 * N + 1);
  }
}

__global__ void k_beta_weights(int L, double* __restrict__ out, int* __restrict__ err) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t > L) return;
  const int n = 2 * L + 1;
  if (t == 0) {
    if (lane == 0) out[0] = 4.0 * kPi * kPi / (L / 2 + 0.5);
    return;
  }
  double sr, si;
  quad_weight_sum(L, 2.0 * kPi * t / n, lane, sr, si);
  if (lane == 0) {
    if (fabs(si) >= 1e-12) atomicExch(err, 2);
    out[t] = 8.0 * kPi * kPi * sr;
  }
}

// rows[(l - |m|) n + j] = lambda_l^m(theta_j), |m| <= l <= lmax (harmonics.cpp:60-89)
__global__ void k_legendre_rows(int m, int lmax, const double* __restrict__ thetas, int n,
                                double* __restrict__ rows) {
  extern __shared__ double coef[];
  double *sf = coef, *ca = coef + (lmax + 1), *cb = coef + 2 * (lmax + 1);
  const int am = m < 0 ? -m : m;
  legendre_coeffs(am, lmax, sf, ca, cb);
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double c, s;
  sincos(thetas[j], &s, &c);
  LegendreIt r;
  r.seed(m, c, s, sf);
  for (int l = am; l <= lmax; ++l) {
    if (l > am) r.next(ca, cb);
    rows[(size_t)(l - am) * n + j] = r.cur;
  }
}

__device__ __forceinline__ size_t delta_offset(int p) {
  return (size_t)p * (2 * p - 1) * (2 * p + 1) / 3;
}

// Delta^p = d^p(pi/2) for p <= L (wigner.cpp:28-80). The reference builds level l from level
// l-1 only through its top row, so the levels decouple once the top rows are known:
//   1. every top-row factor (a square root and a division each) in parallel;
//   2. the top rows: Delta^l_{l,0} chains down the levels, then Delta^l_{l,m'} for m' >= 1
//      chains along the diagonal l - m' (one multiply per step);
//   3. every column (l, m') of every level's m >= m' sector in parallel: the downward
//      three-term recursion in m with the values in registers, each value written straight to
//      all its symmetric positions (transpose with (-1)^(m-m'), then the four quadrants).
// Explicit _rn intrinsics keep every operation of the reference separately rounded (no FMA
// contraction), so the table is bit-identical to the reference. One CTA; its (L+1)(L+2)
// doubles of top-row factors and values live in shared memory, or (large L, gws != nullptr)
// in a global-memory workspace.
__device__ __forceinline__ int tri_index(int l, int mp) { return l * (l + 1) / 2 + mp; }

__device__ __forceinline__ void delta_put(double* lev, int l, int m, int mp, double v) {
  // v = sector value at (m, mp), m >= mp >= 0 (and its transpose when m != mp)
  const int w = 2 * l + 1;
#pragma unroll
  for (int tr = 0; tr < 2; ++tr) {
    if (tr == 1 && m == mp) break;
    const int a = tr ? mp : m, b = tr ? m : mp;  // sector position (a, b)
    const double sv = tr ? (((m - mp) & 1) ? -1.0 : 1.0) * v : v;
#pragma unroll
    for (int sq = 0; sq < 2; ++sq) {
      if (sq == 1 && a == 0) break;
      const int q = sq ? -a : a;
#pragma unroll
      for (int sqp = 0; sqp < 2; ++sqp) {
        if (sqp == 1 && b == 0) break;
        const int qp = sqp ? -b : b;
        double sgn = 1.0;
        if (q < 0 && qp >= 0) sgn = ((l + b) & 1) ? -1.0 : 1.0;
        else if (q >= 0 && qp < 0) sgn = ((l + a) & 1) ? -1.0 : 1.0;
        else if (q < 0 && qp < 0) sgn = ((a + b) & 1) ? -1.0 : 1.0;
        lev[(q + l) * w + qp + l] = sgn * sv;
      }
    }
  }
}

__global__ void __launch_bounds__(1024) k_delta(int L, double* __restrict__ delta,
                                                double* __restrict__ gws) {
  extern __shared__ double smem_d[];
  double* sm = gws ? gws : smem_d;
  const int T = (L + 1) * (L + 2) / 2;
  double* fac = sm;      // [tri(l, mp)] top-row factor of level l
  double* top = sm + T;  // [tri(l, mp)] Delta^l_{l, mp}
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < T; i += nt) {
    int l = (int)((sqrt(8.0 * i + 1.0) - 1.0) * 0.5);
    while (tri_index(l + 1, 0) <= i) ++l;
    while (tri_index(l, 0) > i) --l;
    const int mp = i - tri_index(l, 0);
    double f = 1.0;
    if (l > 0) {
      if (mp == 0) {
        f = -__dsqrt_rn(__ddiv_rn(2.0 * l - 1.0, 2.0 * l));
      } else {
        const double num = __dmul_rn((double)l, 2.0 * l - 1.0);
        const double den = __dmul_rn(2.0 * (l + mp), (double)l + mp - 1.0);
        f = __dsqrt_rn(__ddiv_rn(num, den));
      }
    }
    fac[i] = f;
  }
  __syncthreads();
  if (tid == 0) {
    double v = 1.0;
    top[0] = 1.0;
    for (int l = 1; l <= L; ++l) {
      v = __dmul_rn(fac[tri_index(l, 0)], v);
      top[tri_index(l, 0)] = v;
    }
  }
  __syncthreads();
  for (int d = tid; d < L; d += nt) {  // diagonal l - mp = d, mp >= 1
    double v = top[tri_index(d, 0)];
    for (int mp = 1; d + mp <= L; ++mp) {
      const int l = d + mp;
      v = __dmul_rn(fac[tri_index(l, mp)], v);
      top[tri_index(l, mp)] = v;
    }
  }
  __syncthreads();
  // columns: item = tri(l, mp) over all levels (top-row entries included)
  for (int i = tid; i < T; i += nt) {
    int l = (int)((sqrt(8.0 * i + 1.0) - 1.0) * 0.5);
    while (tri_index(l + 1, 0) <= i) ++l;
    while (tri_index(l, 0) > i) --l;
    const int mp = i - tri_index(l, 0);
    double* lev = delta + delta_offset(l);
    double v1 = top[i];  // (m + 1, mp) as m runs down; starts at m = l
    delta_put(lev, l, l, mp, v1);
    double v2 = 0.0;     // (m + 2, mp)
    for (int m = l - 1; m >= mp; --m) {
      const double denom = __dsqrt_rn(__dmul_rn((double)(l - m), l + m + 1.0));
      double value = __dmul_rn(__ddiv_rn(2.0 * mp, denom), v1);
      if (m + 2 <= l) {
        const double c2 = __ddiv_rn(__dsqrt_rn(__dmul_rn(l - m - 1.0, l + m + 2.0)), denom);
        value = __dsub_rn(value, __dmul_rn(c2, v2));
      }
      delta_put(lev, l, m, mp, value);
      v2 = v1;
      v1 = value;
    }
  }
}

// Workspace of k_delta for band limit L: shared memory up to L = 166, above that a global
// buffer of delta_ws_doubles(L) doubles (delta_needs_gws). The opt-in attribute is set by
// configure_delta, outside any stream capture.
inline size_t delta_smem(int L) { return sizeof(double) * (size_t)(L + 1) * (L + 2); }
inline bool delta_needs_gws(int L) { return delta_smem(L) > 227 * 1024; }
inline size_t delta_ws_doubles(int L) { return (size_t)(L + 1) * (L + 2); }
inline cudaError_t configure_delta(int L) {
  if (delta_needs_gws(L)) return cudaSuccess;
  return cudaFuncSetAttribute(k_delta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)delta_smem(L));
}
// Launch k_delta for band limit L on stream s (one CTA); gws: the workspace when
// delta_needs_gws(L).
inline cudaError_t launch_delta(int L, double* out, cudaStream_t s, double* gws = nullptr) {
  if (delta_needs_gws(L)) {
    if (!gws) return cudaErrorInvalidValue;
    k_delta<<<1, 1024, 0, s>>>(L, out, gws);
  } else {
    k_delta<<<1, 1024, delta_smem(L), s>>>(L, out, nullptr);
  }
  return cudaGetLastError();
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
                       int tile_nt, int ncol_pad, const int* __restrict__ wrow,
                       double2* __restrict__ W, int fu_kp = 0) {
  const int n = 2 * L + 1, nb = L + 1, ncol = n * nb;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int NPQ = (L + 1) * (L + 1);
  if (col >= ncol_pad) return;
  for (int c = blockIdx.y; c < NPQ; c += gridDim.y) {  // gridDim.y <= 65535
    // fu_kp > 0: the fused kernel's column-tile-major layout [col / 8][KR][8] with the K row
    // wrow[c] of the interleaved row-group layout and XOR-swizzled columns (kernels_fused.cuh)
    auto fused_index = [&](int cl) {
      const int kr = wrow[c];
      return ((size_t)(cl / 8) * fu_kp + kr) * 8 + ((cl & 7) ^ ((2 * kr) & 7));
    };
    if (col >= ncol) {
      W[fu_kp ? fused_index(col)
              : wrow ? (size_t)wrow[c] * ncol_pad + col : wtile_index(c, col, NPQ, tile_nt)] =
          make_double2(0.0, 0.0);
      continue;
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
    // wrow: the two-pass GEMM's q-padded row layout with row stride ncol_pad
    const size_t dst = fu_kp     ? fused_index(col)
                       : wrow    ? (size_t)wrow[c] * ncol_pad + col
                       : tile_nt ? wtile_index(c, col, NPQ, tile_nt)
                                 : (size_t)c * ncol + col;
    W[dst] = make_double2(ar, ai);
  }
}


}  // namespace slsht_cuda
