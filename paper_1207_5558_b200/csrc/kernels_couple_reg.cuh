// k_couple_reg<N>: the coupling stage for a short prime alpha length (N = 17, L_h = 8: config 1),
// one thread per (component, grid column), everything in registers.
//
// With L_h = 8 a T row has 1..9 coupling terms (4.8 on average): on the tensor-core paths almost
// every k-step ends a row, and the per-row bookkeeping (fragment loads, the Gauss sums, the T
// tile in shared memory, the barriers around the FFT) costs far more than the products
// (k_couple_ws<17>: 47.5 us for 70 MB of volumes, its MMA phase 8000 cycles per tile for 600
// cycles of DMMA work). Here a thread owns one column of one component: it accumulates the N
// rows T_q = sum_p U[(p,q)] W[(p,q)][col] straight into the registers of its length-N transform
// (row q mod N, so the DFT needs no phase), runs the generated radix-N butterfly in place, and
// writes its N samples (a warp writes 32 consecutive samples of a row), the mirror volume and
// the digest partials. The W tile of the CTA's 32 columns is staged once in shared memory and
// reused for all its components; a warp's U rows are copied one component ahead into its own
// two buffers (cp.async) and read as broadcasts. No barrier after the W stage, no T in shared
// memory.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "fft_radix.cuh"
#include "kernels_chunk.cuh"
#include "kernels_couple.cuh"

namespace slsht_cuda {

struct RegParams {
  CoupleParams c;  // U [comp][NPQ] (q-major rows), W [NPQ][ncol], out, partials [comp][tile][8]
  int n_tiles;     // column tiles of 32
  int cpb;         // components per CTA
};

constexpr int RG_NT = 32, RG_WARPS = 8, RG_THREADS = RG_NT * RG_WARPS;
__host__ __device__ constexpr size_t couple_reg_smem_bytes(int n) {
  const int L = (n - 1) / 2;
  return (size_t)(L + 1) * (L + 1) * (RG_NT + 2 * RG_WARPS) * 16 + (size_t)(L + 1) * 8 + 16;
}

template <int N>
__global__ void __launch_bounds__(RG_THREADS, 2) k_couple_reg(const RegParams R) {
  constexpr int L = (N - 1) / 2, NPQ = (L + 1) * (L + 1);
  static_assert(smallest_prime_factor(N) == N, "one radix-N butterfly: N must be prime");
  const CoupleParams& P = R.c;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* Ws = reinterpret_cast<double2*>(smem_raw);          // [NPQ][32]
  double2* Us = Ws + NPQ * RG_NT;                              // [warp][2][NPQ]: the warp's U rows
  double* betaw_s = reinterpret_cast<double*>(Us + 2 * RG_WARPS * NPQ);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ct = blockIdx.x, col0 = ct * RG_NT, col = col0 + lane;
  const bool ok = col < P.ncol;
  // the W tile: asynchronous copies (zero fill past the last column), all in flight at once
  for (int e = tid; e < NPQ * RG_NT; e += RG_THREADS) {
    const int c = e / RG_NT, k = e % RG_NT;
    const bool in = col0 + k < P.ncol;
    cp_async16(Ws + e, P.W + (in ? (size_t)c * P.ncol + col0 + k : 0), in);
  }
  cp_async_commit();
  for (int i = tid; i <= L; i += RG_THREADS) betaw_s[i] = P.betaw[i];
  const long long sbit = (long long)0x8000000000000000ULL;
  const int comp_end = min(P.count, (int)(blockIdx.y + 1) * R.cpb);
  // the warp's U rows: copied asynchronously one component ahead (two buffers per warp)
  double2* Uw = Us + warp * 2 * NPQ;
  auto load_u = [&](int comp, int buf) {
    if (comp < comp_end)
      for (int i = lane; i < NPQ; i += 32) cp_async16(Uw + buf * NPQ + i, P.U + (size_t)comp * NPQ + i, true);
    cp_async_commit();
  };
  load_u(blockIdx.y * R.cpb + warp, 0);
  cp_async_wait<1>();  // this thread's part of the W tile
  __syncthreads();
  const double qb = ok ? betaw_s[col / N] : 0.0;
  int buf = 0;
  for (int comp = blockIdx.y * R.cpb + warp; comp < comp_end; comp += RG_WARPS, buf ^= 1) {
    load_u(comp + RG_WARPS, buf ^ 1);
    cp_async_wait<1>();
    __syncwarp();
    const double2* Uc = Uw + buf * NPQ;
    // T rows into the transform's registers: x[q mod N] = sum_{p >= |q|} U[(p,q)] W[(p,q)][col]
    double xr[N], xi[N];
    {
      int c = 0;
#pragma unroll
      for (int jq = 0; jq < N; ++jq) {
        const int q = jq - L, K = L + 1 - (q < 0 ? -q : q);
        double arx = 0.0, ary = 0.0, aix = 0.0, aiy = 0.0;  // four independent chains per row
#pragma unroll
        for (int k = 0; k < K; ++k, ++c) {
          const double2 u = Uc[c];  // broadcast
          const double2 w = Ws[c * RG_NT + lane];
          arx = fma(u.x, w.x, arx);
          ary = fma(u.y, w.y, ary);
          aix = fma(u.x, w.y, aix);
          aiy = fma(u.y, w.x, aiy);
        }
        xr[q < 0 ? q + N : q] = arx - ary;
        xi[q < 0 ? q + N : q] = aix + aiy;
      }
    }
    Radix<N>::dft(xr, xi);  // a prime length: outputs in natural order (the identity permutation)

    const CompRec rec = P.comps[comp];
    double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
    long long mx2 = 0;
    if (ok) {
      double2* o = P.out + rec.slot * P.vol + col;
      double2* om = (P.mirror && rec.m > 0) ? P.out + rec.mslot * P.vol + col : nullptr;
      const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
      uint32_t hsh = (uint32_t)col * 0x9E3779B1u;
      const uint32_t hstep = (uint32_t)P.ncol * 0x9E3779B1u;
      auto rows = [&](auto mirror_tag) {
        constexpr bool MIR = decltype(mirror_tag)::value;
#pragma unroll
        for (int a = 0; a < N; ++a, hsh += hstep) {
          const double vr = xr[a], vi = xi[a];
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
      if (col == 0) {
        g0r = xr[0];
        g0i = xi[0];
      }
    }
    // one digest partial per (component, column tile): a fixed shuffle tree over the warp
    double v[8] = {s2, __longlong_as_double(mx2), pr, pi, g0r, g0i, ir, ii};
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double x = __shfl_down_sync(0xffffffffu, v[k], off);
        v[k] = (k == 1) ? fmax(v[k], x) : v[k] + x;
      }
    if (lane == 0) {
      double* part = P.partials + ((size_t)comp * R.n_tiles + ct) * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) part[k] = v[k];
    }
    __syncwarp();  // every lane is done with this U buffer before it is refilled
  }
  cp_async_wait<0>();
}

}  // namespace slsht_cuda
