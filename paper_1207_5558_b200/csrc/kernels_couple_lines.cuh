// Line-aligned persistent coupling kernel for the small transform lengths (n <= 33), where the
// output stream dominates ("store path").
//
// Why: every BASELINE volume row holds ncol = n (L_h+1) complex, an odd count, so the rows of an
// So3Volume start at alternating (and generally unaligned) 16-B offsets. A kernel that stores
// column strips writes every row as a misaligned 128-B segment, i.e. two partial L2 lines, and
// the B200 write path then saturates at ~2.3 TB/s whatever the store instruction (STG, TMA
// tensor store, cache policy: profiles/store_microbench.txt). Full aligned lines reach 4.3+.
//
// How: a CTA owns one group of MT = 8 components at a time and walks its column tiles
// ct = 0, 1, ... in order. U of the group stays resident in shared memory (one bulk copy);
// the W column tile streams through a 2-deep ring (one bulk copy per tile). After the DMMA
// coupling and the in-place alpha FFT of tile ct, the epilogue writes, for every
// (component, row a), exactly the one 128-B line whose last element falls inside the tile's
// columns of that row; the first part of that line comes from tile ct-1 (still resident in
// the other T buffer). Lines that cross a row boundary are written when the last tile of the
// row is done, from a kept copy of tile 0. Only the two lines at each volume's ends can be
// partial. The mirror volume (real mode) has its own line phase and is written the same way.
// The digest of each component accumulates over its tiles in registers (one warp per
// component, fixed order) and is written once per group, so no partials pass is needed.
#pragma once

#include "common.cuh"
#include "fft_radix.cuh"
#include "kernels_couple.cuh"
#include "kernels_couple_ws.cuh"

namespace slsht_cuda {

struct LnParams {
  CoupleParams c;
  long long group_elems;  // U elements per group (stage-tiled layout, zero-padded q blocks)
  int urb[136];           // per q row jq: offset of its padded row block in the group's U
  int n_groups;
  double* digest;         // [coeff_count(lmax)][8], rows coeff_index(l, m) (and the mirror)
  long long* trace;       // debug (SLSHT_WS_TRACE builds): phase timestamps of CTA 0
};

template <int N, int NWARP>
struct LnCfg {
  static constexpr int L = (N - 1) / 2;
  static constexpr int NPQ = (L + 1) * (L + 1);
  static constexpr int MT = 8, NT = 8;
  static constexpr int NC = NWARP * 32;            // consumer threads
  static constexpr int NTHREADS = NC + 32;         // + producer warp
  static constexpr int UPAD = (NPQ + 3 * N + 8);   // >= padded rows of a group (per component)
  static constexpr size_t U_BYTES = (size_t)MT * UPAD * 16;
  static constexpr size_t W_BYTES = (size_t)(NPQ + 8) * NT * 16;
  static constexpr size_t T_BYTES = (size_t)MT * N * NT * 16;
  static constexpr size_t OFF_W = U_BYTES;
  static constexpr size_t OFF_T = OFF_W + 2 * W_BYTES;
  static constexpr size_t OFF_TAB = OFF_T + 3 * T_BYTES;
  static constexpr size_t TAB_BYTES =
      (size_t)N * 16 + (size_t)(L + 1) * 8 + (size_t)(2 * N + 2) * 4 + (size_t)N * 4 + 16 + MT * 24;
  static constexpr size_t OFF_BAR = (OFF_TAB + TAB_BYTES + 15) / 16 * 16;
  static constexpr size_t SMEM = OFF_BAR + 6 * 8;
  static_assert(UPAD % 8 == 4, "U row stride must be 4 mod 8 (16-B units) for conflict-free A loads");
};

template <int N, int NWARP>
__global__ void __launch_bounds__(LnCfg<N, NWARP>::NTHREADS, 1) k_couple_lines(const LnParams LP) {
  using Cfg = LnCfg<N, NWARP>;
  constexpr int L = Cfg::L, MT = Cfg::MT, NT = Cfg::NT, NC = Cfg::NC, NPQ = Cfg::NPQ;
  const CoupleParams& P = LP.c;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* Us = reinterpret_cast<double2*>(smem);
  double2* Wsb = reinterpret_cast<double2*>(smem + Cfg::OFF_W);
  double2* Tb = reinterpret_cast<double2*>(smem + Cfg::OFF_T);
  double2* rou_s = reinterpret_cast<double2*>(smem + Cfg::OFF_TAB);
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  int* perm_s = reinterpret_cast<int*>(betaw_s + (L + 1));
  int* qoff_s = perm_s + N;
  int* urb_s = qoff_s + (N + 1) + 1;
  CompRec* rec_s = reinterpret_cast<CompRec*>(
      (reinterpret_cast<uintptr_t>(urb_s + N) + 15) & ~static_cast<uintptr_t>(15));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* ufull = bars + 0;
  uint64_t* uempty = bars + 1;
  uint64_t* wfull = bars + 2;   // [2]
  uint64_t* wempty = bars + 4;  // [2]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nct = P.n_col_tiles;

  for (int i = tid; i < N; i += Cfg::NTHREADS) {
    rou_s[i] = P.rou[i];
    perm_s[i] = P.perm[i];
    urb_s[i] = LP.urb[i];
  }
  for (int i = tid; i <= N; i += Cfg::NTHREADS) qoff_s[i] = P.qoff[i];
  for (int i = tid; i <= L; i += Cfg::NTHREADS) betaw_s[i] = P.betaw[i];
  {
    // W rows past NPQ are read (times a zero U pad) by partial k-steps: keep them finite
    double4* w4 = reinterpret_cast<double4*>(smem + Cfg::OFF_W);
    for (size_t i = tid; i < 2 * Cfg::W_BYTES / 32; i += Cfg::NTHREADS)
      w4[i] = make_double4(0.0, 0.0, 0.0, 0.0);
  }
  if (tid == 0) {
    mbar_init(ufull, 1);
    mbar_init(uempty, NWARP);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&wfull[b], 1);
      mbar_init(&wempty[b], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == NWARP) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t uphase = 0;
      int wslot = 0;
      uint32_t wphase = 0;
      for (int g = blockIdx.x; g < LP.n_groups; g += gridDim.x) {
        mbar_wait(uempty, uphase ^ 1);
        const uint32_t ub = (uint32_t)(LP.group_elems * 16);
        mbar_arrive_expect_tx(ufull, ub);
        bulk_g2s(Us, P.U + (size_t)g * LP.group_elems, ub, ufull);
        uphase ^= 1;
        for (int ct = 0; ct < nct; ++ct) {
          mbar_wait(&wempty[wslot], wphase ^ 1);
          const uint32_t wb = (uint32_t)(NPQ * NT * 16);
          mbar_arrive_expect_tx(&wfull[wslot], wb);
          bulk_g2s(Wsb + (size_t)wslot * (Cfg::W_BYTES / 16), P.W + (size_t)ct * NPQ * NT, wb,
                   &wfull[wslot]);
          if (++wslot == 2) {
            wslot = 0;
            wphase ^= 1;
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumers
  const int kl = lane & 3;
  uint32_t uphase = 0;
  int wslot = 0;
  uint32_t wphase = 0;
  const long long vol = P.vol;
  const int ncol = P.ncol;
  for (int g = blockIdx.x; g < LP.n_groups; g += gridDim.x) {
    const int comp0 = g * MT;
    const int ncomp = min(MT, P.count - comp0);
    if (tid < MT) rec_s[tid] = (tid < ncomp) ? P.comps[comp0 + tid] : CompRec{0, 0, -1, -1};
    mbar_wait(ufull, uphase);
    uphase ^= 1;
    // digest accumulators: warp c < MT owns component c for the whole group
    double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
    long long mx2 = 0;
    named_sync(1, NC);  // rec_s visible
    for (int ct = 0; ct < nct; ++ct) {
      const int C = ct * NT;
      const int tb = ct == 0 ? 2 : (ct & 1);
      const int tprev = ct == 1 ? 2 : ((ct - 1) & 1);
      double2* T = Tb + (size_t)tb * (Cfg::T_BYTES / 16);
#ifdef SLSHT_WS_TRACE
      const bool tr = LP.trace && blockIdx.x == 0 && tid == 0 && g == 0 && ct < 64;
      if (tr) LP.trace[ct * 6 + 0] = clock64();
#endif
      // ---------------- MMA: one item per q row, NWARP warps
      mbar_wait(&wfull[wslot], wphase);
#ifdef SLSHT_WS_TRACE
      if (tr) LP.trace[ct * 6 + 1] = clock64();
#endif
      const double2* Ws = Wsb + (size_t)wslot * (Cfg::W_BYTES / 16);
      for (int jq = warp; jq < N; jq += NWARP) {
        const int np = L + 1 - abs(jq - L);
        const int nks = (np + 3) >> 2;
        const int wrb = qoff_s[jq];
        const int ar = lane >> 2;
        const int blo = lane >> 2;
        const double2* ap = Us + ar * Cfg::UPAD + urb_s[jq] + kl;
        const double2* bp = Ws + (wrb + kl) * NT + (blo ^ ((2 * (wrb + kl)) & 7));
        double c1[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0}, c3[2] = {0.0, 0.0};
        double2 a = ap[0], b = bp[0];
        for (int ks = 0; ks < nks; ++ks) {
          const int kn = min(ks + 1, nks - 1);
          const double2 na = ap[4 * kn], nb = bp[4 * kn * NT];
          dmma(c1[0], c1[1], a.x + a.y, b.x);
          dmma(c2[0], c2[1], a.x, b.y - b.x);
          dmma(c3[0], c3[1], a.y, b.x + b.y);
          a = na;
          b = nb;
        }
        const int row = jq >= L ? jq - L : jq + L + 1;  // q mod n
        double2* dst = T + (size_t)(ar * N + row) * NT + 2 * kl;
        dst[0] = make_double2(c1[0] - c3[0], c1[0] + c2[0]);
        dst[1] = make_double2(c1[1] - c3[1], c1[1] + c2[1]);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&wempty[wslot]);
        if (ct == nct - 1) mbar_arrive(uempty);
      }
      if (++wslot == 2) {
        wslot = 0;
        wphase ^= 1;
      }
      named_sync(1, NC);
#ifdef SLSHT_WS_TRACE
      if (tr) LP.trace[ct * 6 + 2] = clock64();
#endif
      // ---------------- alpha FFT of the tile, in place
      FftDif<N, N, NT, MT * NT, NC>::run(T, rou_s, tid, 1);
#ifdef SLSHT_WS_TRACE
      if (tr) LP.trace[ct * 6 + 3] = clock64();
#endif
      // ---------------- digest of the tile's own samples (warp c: component c)
      if (warp < ncomp) {
        const int c = warp;
        const double2* Tc = T + (size_t)c * N * NT;
        for (int v = lane; v < N * NT; v += 32) {
          const int a = v / NT, j = v % NT, col = C + j;
          if (col >= ncol) continue;
          const double2 x = Tc[perm_s[a] * NT + j];
          const double a2 = fma(x.x, x.x, x.y * x.y);
          s2 += a2;
          mx2 = max(mx2, __double_as_longlong(a2));
          const uint32_t hsh = (uint32_t)((size_t)a * ncol + col) * 0x9E3779B1u;
          const double wgt = digest_weight(hsh);
          pr = fma(wgt, x.x, pr);
          pi = fma(wgt, x.y, pi);
          const double qb = betaw_s[col / N];
          ir = fma(qb, x.x, ir);
          ii = fma(qb, x.y, ii);
          if (a == 0 && col == 0) {
            g0r = x.x;
            g0i = x.y;
          }
        }
      }
#ifdef SLSHT_WS_TRACE
      if (tr) LP.trace[ct * 6 + 4] = clock64();
#endif
      // ---------------- aligned line stores: job = (component, row, volume) -> one 128-B line
      const double2* Tcur = T;
      const double2* Tprv = Tb + (size_t)tprev * (Cfg::T_BYTES / 16);
      const double2* T0 = Tb + (size_t)2 * (Cfg::T_BYTES / 16);
      const bool last = ct == nct - 1;
      const int n_jobs = MT * N * (P.mirror ? 2 : 1);
      for (int job = (tid >> 3); job < n_jobs; job += NC / 8) {
        const int j = tid & 7;
        const int which = job / (MT * N);  // 0: the component, 1: its conjugate mirror
        const int r = job % (MT * N);
        const int c = r / N, a = r % N;
        if (c >= ncomp) continue;
        const CompRec rec = rec_s[c];
        if (which == 1 && !(rec.m > 0)) continue;
        const long long base = (which ? rec.mslot : rec.slot) * vol;  // volume start
        const long long rowp = base + (long long)a * ncol;            // row start
        const long long p0 = rowp + C;
        const long long e = p0 + ((7 - (p0 & 7)) & 7);  // the line's last element
        const long long s = e - 7;
        if (ct == 0 && s < rowp && a > 0) continue;  // written with row a-1's last tile
        const long long x = s + j;                    // this lane's element
        if (x < base || x >= base + vol) continue;    // partial line at a volume end
        const int d = (int)(x - rowp);                // column within row a (may run past it)
        double2 v;
        if (d >= ncol) {
          v = T0[(size_t)(c * N + perm_s[a + 1]) * NT + (d - ncol)];  // next row's head (tile 0)
        } else if (d >= C) {
          v = Tcur[(size_t)(c * N + perm_s[a]) * NT + (d - C)];
        } else {
          v = Tprv[(size_t)(c * N + perm_s[a]) * NT + (d - (C - NT))];
        }
        if (which) {
          const long long sbit = (long long)0x8000000000000000ULL;
          const long long fr = (rec.m & 1) ? sbit : 0, fi = (rec.m & 1) ? 0 : sbit;
          v = make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ fr),
                           __longlong_as_double(__double_as_longlong(v.y) ^ fi));
        }
        P.out[x] = v;
        (void)last;
      }
      named_sync(1, NC);  // T buffers reused by the next tiles
#ifdef SLSHT_WS_TRACE
      if (tr) LP.trace[ct * 6 + 5] = clock64();
#endif
    }
    // ---------------- digest rows of the group
    if (warp < ncomp) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        s2 += __shfl_down_sync(0xffffffffu, s2, off);
        mx2 = max(mx2, (long long)__shfl_down_sync(0xffffffffu, (unsigned long long)mx2, off));
        pr += __shfl_down_sync(0xffffffffu, pr, off);
        pi += __shfl_down_sync(0xffffffffu, pi, off);
        ir += __shfl_down_sync(0xffffffffu, ir, off);
        ii += __shfl_down_sync(0xffffffffu, ii, off);
        g0r += __shfl_down_sync(0xffffffffu, g0r, off);
        g0i += __shfl_down_sync(0xffffffffu, g0i, off);
      }
      if (lane == 0) {
        const CompRec rec = rec_s[warp];
        const double inv = 1.0 / ((double)N * N * N);
        double d[8] = {s2, sqrt(__longlong_as_double(mx2)), pr, pi, g0r, g0i, ir * inv, ii * inv};
        double* dst = LP.digest + (size_t)(rec.l * rec.l + rec.l + rec.m) * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) dst[k] = d[k];
        if (P.mirror && rec.m > 0) {
          const double sg = (rec.m & 1) ? -1.0 : 1.0;
          double* dm = LP.digest + (size_t)(rec.l * rec.l + rec.l - rec.m) * 8;
          dm[0] = d[0];
          dm[1] = d[1];
          dm[2] = sg * d[2];
          dm[3] = -(sg * d[3]);
          dm[4] = sg * d[4];
          dm[5] = -(sg * d[5]);
          dm[6] = sg * d[6];
          dm[7] = -(sg * d[7]);
        }
      }
    }
    named_sync(1, NC);  // rec_s reused by the next group
  }
}

}  // namespace slsht_cuda
