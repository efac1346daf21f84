// k_tpipe: the two-pass coupling (kernels_twopass.cuh) as ONE persistent kernel whose T stays in
// L2 (n = 49, 65).
//
// k_tgemm + k_qfft write and re-read the whole chunk's T through HBM (config 4: 281 GB written
// and 283 GB read per step, on top of the 277 GB of volumes). Here the same two bodies run as
// work items of one persistent kernel over a small ring of T slots, so a T tile is written by
// the GEMM items, read back by the FFT items a few tens of microseconds later, and overwritten
// by the next sub-block before L2 ever evicts it:
//
//   sub-block s = (64-component block, group of CT 32-column tiles); its T is one ring slot
//   GEMM item   = (column tile of the group, q group): the k-steps [qg[g], qg[g+1]) of k_tgemm's
//                 64 x 32 tile (the T rows of different q are independent GEMMs, so splitting
//                 the sweep by q keeps the operand reuse of the tile and gives CT x NQG items
//                 per sub-block)
//   FFT item    = (column tile, FB consecutive components): k_qfft's tile body per component,
//                 the next component's tile prefetched (cp.async) while the current one runs
//
// Items are handed out by one atomic ticket in the order G(0), G(1), F(0), G(2), F(1), ... A
// GEMM item of sub-block s first waits until every FFT item of sub-block s - NSLOT (the slot's
// previous user) is done; an FFT item waits until the NQG GEMM items of its column tile are
// done. An item only ever waits for items with smaller tickets, which are running or finished,
// so the schedule cannot deadlock whatever the number of resident CTAs. Every value and every
// digest partial is computed by the same instruction sequence as in k_tgemm / k_qfft: results
// are bitwise equal to the two-pass kernels.
#pragma once

#include "kernels_twopass.cuh"

namespace slsht_cuda {

struct TpParams {
  // GEMM operands (as TgParams)
  const double2* U;   // [comp][KP]
  const double2* W;   // [KP][wpitch]
  double2* T;         // ring: nslot slots of slot_elems; slot layout [64 comps][n][tpitch]
  const short* qend;  // per k-step: T row completed by it, or -1
  int count, KP, wpitch, n;
  // pipeline shape
  int* sync;          // [0] ticket; [1, 1 + nsub) FFT items done; then [s CT + tile] GEMM items done
  const int* qg;      // [nqg + 1] k-step bounds of the q groups
  int nblk, ncg, CT, nct, nqg, nslot, fb;
  int lag;            // FFT items of sub-block r - lag follow the GEMM items of sub-block r (>= 1, < nslot)
  int exp;            // timing experiments (wrong results): 1 no waits, 2 no GEMM items, 4 no FFT items
  long long slot_elems;
  int tpitch;         // CT * 32
  // alpha pass and epilogue (as QfParams)
  double2* out;
  double* partials;
  const CompRec* comps;
  int ncol, n_tiles;
  long long vol;
  int rpitch, mirror;
  const double2* rou;
  const int* perm;
  const double* betaw;
};

constexpr int TP_THREADS = 128, TP_BN = 32, TP_NT = 32;
__host__ __device__ constexpr size_t tpipe_union_bytes(int n) {
  const size_t g = (size_t)2 * (TG_BM * TG_ASTR + TG_KS * (TP_BN + 2)) * 16;
  const size_t f = (size_t)2 * n * TP_NT * 16;
  return g > f ? g : f;
}
__host__ __device__ constexpr size_t tpipe_smem_bytes(int n, int KP) {
  return tpipe_union_bytes(n) + (size_t)n * 16 + (size_t)((n + 1) / 2) * 8 + (size_t)n * 4 +
         (size_t)(KP / 4 + 4) * 2 + 64;
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// thread 0 waits until *p >= want; the CTA barrier publishes the acquired state to every thread
__device__ __forceinline__ void cta_wait_counter(const int* p, int want, int tid) {
  if (tid == 0) {
    while (ld_acquire_gpu(p) < want) __nanosleep(64);
  }
  __syncthreads();
}
// every thread's global writes (or smem-completed reads) first, then one release increment
__device__ __forceinline__ void cta_signal_counter(int* p, int tid) {
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    atomicAdd(p, 1);
  }
}

// FV = 0: k_qfft's tile body (cp.async tile, FftDif in shared memory, epilogue pass): digests
// bitwise equal to k_qfft's. FV = 1: the lean alpha pass for N = R1 R2: the first DIF stage reads
// its rows straight from L2 into registers and writes the tile once; the last stage's outputs go
// from registers to the volume rows (and the digest), per-warp digest partials (4 per tile).
template <int N, int FV>
__global__ void __launch_bounds__(TP_THREADS, 3) k_tpipe(const TpParams P) {
  constexpr int NTHR = TP_THREADS, BN = TP_BN, WNF = 2, NST = 2, BM = TG_BM, NT = TP_NT;
  constexpr int BSTR = BN + 2, L = (N - 1) / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* As = reinterpret_cast<double2*>(smem_raw);
  double2* Bs = As + NST * BM * TG_ASTR;
  double2* rou_s = reinterpret_cast<double2*>(smem_raw + tpipe_union_bytes(N));
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  int* perm_s = reinterpret_cast<int*>(betaw_s + (L + 1));
  int* s_ticket = perm_s + N;
  short* qend_s = reinterpret_cast<short*>(s_ticket + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nks = P.KP / 4;
  for (int i = tid; i < nks; i += NTHR) qend_s[i] = P.qend[i];
  for (int i = tid; i < N; i += NTHR) {
    rou_s[i] = P.rou[i];
    perm_s[i] = P.perm[i];
  }
  for (int i = tid; i <= L; i += NTHR) betaw_s[i] = P.betaw[i];

  const int nsub = P.nblk * P.ncg;
  const int ncgrp = BM / P.fb;  // FFT component groups per block
  const int NG = P.CT * P.nqg, NF = P.CT * ncgrp, per_round = NG + NF;
  const long long total = (long long)(nsub + P.lag) * per_round;
  int* fft_done = P.sync + 1;
  int* gemm_done = P.sync + 1 + nsub;

  for (;;) {
    __syncthreads();  // the previous item is finished with shared memory and s_ticket
    if (tid == 0) *s_ticket = atomicAdd(P.sync, 1);
    __syncthreads();
    const long long t = *s_ticket;
    if (t >= total) break;
    const int r = (int)(t / per_round), i = (int)(t % per_round);

    if (i < NG) {
      // ---------------- GEMM item: sub-block r, column tile ctl of its group, q group g
      const int s = r;
      if (s >= nsub) continue;
      const int blk = s / P.ncg, cg = s % P.ncg;
      const int ctl = i / P.nqg, g = i % P.nqg;
      const int ct = cg * P.CT + ctl;
      if (ctl >= P.CT || ct >= P.nct) continue;
      if (P.exp & 2) continue;
      if (s >= P.nslot && !(P.exp & 1)) {  // the slot's previous sub-block must have been read completely
        const int sp = s - P.nslot, bp = sp / P.ncg, cgp = sp % P.ncg;
        const int tiles = min(P.CT, P.nct - cgp * P.CT);
        const int comps_p = min(BM, P.count - bp * BM);
        cta_wait_counter(fft_done + sp, tiles * ((comps_p + P.fb - 1) / P.fb), tid);
      }
      const int comp0 = blk * BM, col0 = ct * BN;
      const int ks0 = P.qg[g], ks1 = P.qg[g + 1];
      const int nst = (ks1 - ks0 + TG_KS / 4 - 1) / (TG_KS / 4);
      double2* Tslot = P.T + (size_t)(s % P.nslot) * P.slot_elems;

      auto load_stage = [&](int st) {
        if (st < nst) {
          const int kb = ks0 * 4 + st * TG_KS;
          double2* Ad = As + (st % NST) * BM * TG_ASTR;
          double2* Bd = Bs + (st % NST) * TG_KS * BSTR;
#pragma unroll
          for (int j = 0; j < BM * TG_KS / NTHR; ++j) {
            const int e = tid + j * NTHR;
            const int c = e / TG_KS, k = e % TG_KS;
            const bool ok = comp0 + c < P.count && kb + k < P.KP;
            cp_async16(Ad + c * TG_ASTR + k, P.U + (ok ? (size_t)(comp0 + c) * P.KP + kb + k : 0), ok);
          }
#pragma unroll
          for (int j = 0; j < TG_KS * BN / NTHR; ++j) {
            const int e = tid + j * NTHR;
            const int k = e / BN, c = e % BN;
            const bool ok = kb + k < P.KP;
            cp_async16(Bd + k * BSTR + c, P.W + (ok ? (size_t)(kb + k) * P.wpitch + col0 + c : 0), ok);
          }
        }
        cp_async_commit();
      };
#pragma unroll
      for (int st = 0; st < NST - 1; ++st) load_stage(st);

      constexpr int WN = BN / (8 * WNF);
      const int wm = warp / WN, wn = warp % WN;
      const int arow = wm * 32 + (lane >> 2), acol = lane & 3;
      const int brow = lane & 3, bcol = wn * 8 * WNF + (lane >> 2);
      double c1[4][WNF][2], c2[4][WNF][2], c3[4][WNF][2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < WNF; ++ni)
#pragma unroll
          for (int e = 0; e < 2; ++e) c1[mi][ni][e] = c2[mi][ni][e] = c3[mi][ni][e] = 0.0;
      const int scl = wm * 32 + (lane >> 2);                         // component within the block
      const int scol = ctl * BN + wn * 8 * WNF + 2 * (lane & 3);     // column within the slot

      for (int st = 0; st < nst; ++st) {
        cp_async_wait<NST - 2>();
        __syncthreads();
        load_stage(st + NST - 1);
        const double2* Ab = As + (st % NST) * BM * TG_ASTR;
        const double2* Bb = Bs + (st % NST) * TG_KS * BSTR;
#pragma unroll
        for (int kk = 0; kk < TG_KS / 4; ++kk) {
          const int ks = ks0 + st * (TG_KS / 4) + kk;
          double2 a[4], b[WNF];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) a[mi] = Ab[(arow + mi * 8) * TG_ASTR + kk * 4 + acol];
#pragma unroll
          for (int ni = 0; ni < WNF; ++ni) b[ni] = Bb[(kk * 4 + brow) * BSTR + bcol + ni * 8];
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
          // k-steps past the group's end (the tail of its last stage) belong to the next group
          const int row = ks < ks1 ? qend_s[ks] : -1;
          if (row >= 0) {
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
              const int cl = scl + mi * 8;
              if (comp0 + cl < P.count) {
                double2* dst = Tslot + ((size_t)cl * N + row) * P.tpitch + scol;
#pragma unroll
                for (int ni = 0; ni < WNF; ++ni)
                  st_global_v4(dst + ni * 8, c1[mi][ni][0] - c3[mi][ni][0],
                               c1[mi][ni][0] + c2[mi][ni][0], c1[mi][ni][1] - c3[mi][ni][1],
                               c1[mi][ni][1] + c2[mi][ni][1]);
              }
            }
          }
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
      cta_signal_counter(gemm_done + (size_t)s * P.CT + ctl, tid);
    } else {
      // ---------------- FFT item: sub-block r - lag, column tile ctl, FB components
      if (r < P.lag) continue;
      const int s = r - P.lag;
      const int blk = s / P.ncg, cg = s % P.ncg;
      const int j = i - NG;
      const int cgi = j / P.CT, ctl = j % P.CT;
      const int ct = cg * P.CT + ctl;
      const int cl0 = cgi * P.fb;
      if (ct >= P.nct || blk * BM + cl0 >= P.count) continue;
      const int ncomp = min(P.fb, P.count - (blk * BM + cl0));
      if (P.exp & 4) continue;
      if (!(P.exp & 1)) cta_wait_counter(gemm_done + (size_t)s * P.CT + ctl, P.nqg, tid);
      const double2* Tslot = P.T + (size_t)(s % P.nslot) * P.slot_elems + ctl * NT;
      if constexpr (FV == 1) {
        constexpr int R1 = smallest_prime_factor(N), R2 = N / R1;
        static_assert(R1 * R2 == N && smallest_prime_factor(R2) == R2, "N must be a product of two primes");
        double2* Ts = reinterpret_cast<double2*>(smem_raw);
        const int col0 = ct * NT;
        for (int k = 0; k < ncomp; ++k) {
          const double2* src = Tslot + (size_t)(cl0 + k) * N * P.tpitch;
          // first DIF stage (radix R1, twiddles) from L2 to shared memory
          for (int item = tid; item < NT * R2; item += NTHR) {
            const int c = item % NT, t = item / NT;
            double xr[R1], xi[R1];
#pragma unroll
            for (int jj = 0; jj < R1; ++jj) {
              const double2 v = __ldcg(src + (size_t)(t + jj * R2) * P.tpitch + c);
              xr[jj] = v.x;
              xi[jj] = v.y;
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
          __syncthreads();
          if (k + 1 == ncomp && tid == 0) {  // every T tile of the item has been read
            __threadfence();
            atomicAdd(fft_done + s, 1);
          }
          // last stage (radix R2) from shared memory to the volume rows, with the digest
          const int comp = blk * BM + cl0 + k;
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
          if (lane == 0) {  // one partial per warp: k_digest adds them in a fixed order
            double* part = P.partials + (((size_t)comp * P.n_tiles + ct) * (NTHR / 32) + warp) * 8;
#pragma unroll
            for (int q = 0; q < 8; ++q) part[q] = v[q];
          }
          __syncthreads();  // the tile is rewritten by the next component's first stage
        }
        continue;
      }
      double2* Tbuf = reinterpret_cast<double2*>(smem_raw);
      auto load_tile = [&](int k) {
        if (k < ncomp) {
          const double2* src = Tslot + (size_t)(cl0 + k) * N * P.tpitch;
          double2* dst = Tbuf + (k & 1) * (N * NT);
          for (int e = tid; e < N * NT; e += NTHR) {
            const int row = e / NT, c = e % NT;
            cp_async16(dst + row * NT + c, src + (size_t)row * P.tpitch + c, true);
          }
        }
        cp_async_commit();
      };
      load_tile(0);
      const int col0 = ct * NT;
      const int cc = tid % NT, col = col0 + cc;
      const bool ok = col < P.ncol;
      for (int k = 0; k < ncomp; ++k) {
        load_tile(k + 1);
        cp_async_wait<1>();
        __syncthreads();
        if (k + 1 == ncomp && tid == 0) {  // every T tile of the item is on chip: release the slot share
          __threadfence();
          atomicAdd(fft_done + s, 1);
        }
        double2* Ts = Tbuf + (k & 1) * (N * NT);
        const int comp = blk * BM + cl0 + k;
        FftDif<N, N, NT, NT, NTHR, true>::run(Ts, rou_s, tid, 0);

        // epilogue: as k_qfft
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
            const double2 t0 = Tp[(size_t)perm_s[0] * NT];
            g0r = t0.x;
            g0i = t0.y;
          }
          auto rows = [&](auto mirror_tag) {
            constexpr bool MIR = decltype(mirror_tag)::value;
#pragma unroll 4
            for (int a = a_first; a < N; a += A_STEP, hsh += hstep) {
              const double2 tv = Tp[(size_t)perm_s[a] * NT];
              const double vr = tv.x, vi = tv.y;
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
        double v[6] = {s2, __longlong_as_double(mx2), pr, pi, ir, ii};
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int q = 0; q < 6; ++q) {
            const double x = __shfl_down_sync(0xffffffffu, v[q], off);
            v[q] = (q == 1) ? fmax(v[q], x) : v[q] + x;
          }
        __syncthreads();  // the tile is reused as the reduction scratch
        double* red = reinterpret_cast<double*>(Ts);
        if ((tid & 31) == 0)
#pragma unroll
          for (int q = 0; q < 6; ++q) red[(tid >> 5) * 6 + q] = v[q];
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
        __syncthreads();  // red is read before the tile buffer is refilled (load_tile(k + 2))
      }
      cp_async_wait<0>();
    }
  }
}

}  // namespace slsht_cuda
