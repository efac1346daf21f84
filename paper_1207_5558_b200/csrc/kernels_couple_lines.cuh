// Line-aligned persistent coupling kernel for the small transform lengths (n = 17, 33), where
// the output stream dominates ("store path").
//
// Why: every BASELINE volume row holds ncol = n (L_h+1) complex, an odd count, so the rows of an
// So3Volume start at unaligned 16-B offsets. A kernel that stores column strips writes every
// row as a misaligned 128-B segment, i.e. two partial L2 lines, and the B200 write path then
// saturates at ~2.3 TB/s whatever the store instruction (STG, TMA tensor store, cache policy:
// profiles/microbench_store_*.txt). Whole aligned 128-B lines reach 4.3+ TB/s.
//
// How: a CTA owns one group of MT = 8 components at a time and walks its column tiles
// ct = 0, 1, ... in order (8 columns each).
//   producer warp : the group's U block (resident for the whole group, one bulk copy) and the
//                   whole W column tile through two slots (mbarriers);
//   compute warps : one warp per first-stage DIF butterfly row group (n = R1 * MP: rows
//                   r + k MP, k < R1). The warp runs the R1 DMMA chains of its rows (Gauss
//                   3-product complex MMA), applies the radix-R1 butterfly and twiddles to the
//                   accumulators in registers and writes T; the remaining DIF stages run in
//                   shared memory, the last one also accumulating the digest of its outputs;
//   store warps   : 16 line groups = (component, volume). For every row of the tile the one
//                   aligned 128-B line that starts in (p0 - 8, p0], p0 = the row's first
//                   element in the tile, read from the tile's T buffer and the previous tile's
//                   (3 rolling buffers). The few lines that cross a row end are written as two
//                   partial lines (tail by the row's last tile, head by the next row's first).
// Compute runs one tile ahead of the stores (buffer reuse waits for the stores of tile t-2), so
// the FP64 work overlaps the store stream.
#pragma once

#include "common.cuh"
#include "fft_radix.cuh"
#include "kernels_couple.cuh"
#include "kernels_couple_ws.cuh"

namespace slsht_cuda {

struct LnParams {
  CoupleParams c;
  long long group_elems;  // U elements per group: MT rows of UPAD (zero-padded q blocks)
  int urb[136];           // per q row jq: offset of its padded row block in a U row
  int n_groups;
  int nseg;               // column segments per group: a work unit is (group, segment)
  int nseg_dig;           // digest segments per group (a fixed split; nseg divides it)
  double* partials;       // [component][digest segment][8] partials (k_digest reduces them)
  long long* trace;       // debug (SLSHT_WS_TRACE builds)
};

// compile-time q-row layout: rows of q row jq start at qoff(jq); the W halves split at the
// first jq whose rows start at or past NPQ / 2
template <int N>
struct LnRows {
  static constexpr int L = (N - 1) / 2;
  static constexpr int NPQ = (L + 1) * (L + 1);
  static constexpr int np(int jq) { return L + 1 - (jq > L ? jq - L : L - jq); }
  // U rows of one component: each q row zero-padded to whole k-steps of 4, the total == 4 mod 8
  // (16-B units) so the 8 component rows of an A fragment hit distinct bank groups
  static constexpr int urows() {
    int s = 0;
    for (int jq = 0; jq < N; ++jq) s += (np(jq) + 3) / 4 * 4;
    return s;
  }
  static constexpr int UPAD = urows() + ((4 - urows()) % 8 + 8) % 8;
  static constexpr int qoff(int jq) {
    int s = 0;
    for (int j = 0; j < jq; ++j) s += np(j);
    return s;
  }
  static constexpr int urb(int jq) {  // start of q row jq's padded block in a U row
    int s = 0;
    for (int j = 0; j < jq; ++j) s += (np(j) + 3) / 4 * 4;
    return s;
  }
  static constexpr int jq_of_row(int x) { return x <= L ? x + L : x - L - 1; }  // T row = q mod n
};

template <int N>
struct LnCfg {
  using Rows = LnRows<N>;
  static constexpr int L = (N - 1) / 2;
  static constexpr int NPQ = Rows::NPQ;
  static constexpr int MT = 8, NT = 8;
  static constexpr int R1 = smallest_prime_factor(N);  // first DIF radix: fused into the MMA
  static constexpr int MP = N / R1;                     // row groups = compute warps
  static constexpr int NCW = MP;
  static constexpr int NSW = 4;                         // store warps: 16 (component, volume) lines
  static constexpr int NC = NCW * 32;
  static constexpr int NTHREADS = 32 + NC + NSW * 32;
  static constexpr int UPAD = Rows::UPAD;
  static constexpr int KSMAX = (L + 1 + 3) / 4;
  static constexpr size_t U_BYTES = (size_t)MT * UPAD * 16;
  static constexpr size_t WS_BYTES = (size_t)(NPQ + 4) * NT * 16;  // + rows read by k-step tails
  static constexpr size_t T_BYTES = (size_t)MT * N * NT * 16;
  static constexpr size_t OFF_W = U_BYTES;
  static constexpr size_t OFF_T = OFF_W + 2 * WS_BYTES;
  static constexpr size_t OFF_TAB = OFF_T + 3 * T_BYTES;
  static constexpr int RLAST = []() constexpr {  // radix of the last DIF stage
    int x = N, r = N;
    for (int p = 3; x > 1; p += 2)
      while (x % p == 0) {
        r = p;
        x /= p;
      }
    return r;
  }();
  static constexpr int LAST_ITEMS = MT * NT * (N / RLAST);  // butterflies of the last stage
  // the last stage runs on the first NFW compute warps only (one butterfly per thread); the
  // other compute warps go on to the next tile's DMMA meanwhile
  static constexpr int NFW = LAST_ITEMS / 32;
  static constexpr int NF = NFW * 32;
  static constexpr int NPART = LAST_ITEMS / (MT * NT);       // digest partials per component
  static constexpr size_t TAB_BYTES = (size_t)N * 16 + (size_t)(L + 1) * 8 + (size_t)(N + 2) * 4 +
                                      (size_t)N * 4 + 16 + MT * 24 + (size_t)NPART * MT * 8 * 8;
  static constexpr size_t OFF_BAR = (OFF_TAB + TAB_BYTES + 15) / 16 * 16;
  static constexpr int NBAR = 2 + 4 + 4;  // ufull uempty | wfull[2] wempty[2] | tready[2] tfree[2]
  static constexpr size_t SMEM = OFF_BAR + NBAR * 8;
  static_assert(R1 < N, "the fused first stage needs a composite length");
  static_assert(LAST_ITEMS <= NC && LAST_ITEMS % 32 == 0, "one butterfly per FFT thread");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// Digest state of one compute thread: its last-stage butterfly always covers the same
// (component, column-in-tile) pair, so the 8 sums are accumulated in registers across tiles.
struct DigestAcc {
  double s2, pr, pi, g0r, g0i, ir, ii;
  long long mx2;
};

// Last DIF stage (span R, no twiddles) with the digest of every produced output.
// Frequency held at position blk * R of the DIF output (R = the last radix): position
// blk * R + k holds a0 + k (N / R), the last DIF digit being the most significant of the
// frequency. Thread-constant: computed once, outside the tile loop.
template <int N, int R>
__device__ __forceinline__ int dif_last_freq0(int blk) {
  int a0 = 0, rem = blk * R, mult = 1, mm = N, x = N;
#pragma unroll
  for (int p = 3; p <= N; p += 2)
    if (x > 1)
      while (x % p == 0) {
        const int mp = mm / p, d = rem / mp;
        rem %= mp;
        a0 += d * mult;
        mult *= p;
        mm = mp;
        x /= p;
      }
  return a0;
}

template <int N, int R, int NT, int PAIRS>
__device__ __forceinline__ void fft_last_digest(double2* T, int tid, int C, int ncol, int ncomp,
                                                const double* betaw_s, int a0, DigestAcc& D) {
  constexpr int TOTAL = PAIRS * (N / R);
  if (tid >= TOTAL) return;
  const int pair = tid % PAIRS;
  const int blk = tid / PAIRS;
  const int comp = pair / NT, cc = pair % NT;
  double2* base = T + (size_t)(comp * N + blk * R) * NT + cc;
  double xr[R], xi[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const double2 v = base[k * NT];
    xr[k] = v.x;
    xi[k] = v.y;
  }
  Radix<R>::dft(xr, xi);
#pragma unroll
  for (int k = 0; k < R; ++k) base[k * NT] = make_double2(xr[k], xi[k]);
  const int col = C + cc;
  if (comp >= ncomp || col >= ncol) return;
  const double qb = betaw_s[col / N];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int a = a0 + k * (N / R);
    const double vx = xr[k], vy = xi[k];
    const double a2 = fma(vx, vx, vy * vy);
    D.s2 += a2;
    D.mx2 = max(D.mx2, __double_as_longlong(a2));
    const uint32_t hsh = (uint32_t)((size_t)a * ncol + col) * 0x9E3779B1u;
    const double wgt = digest_weight(hsh);
    D.pr = fma(wgt, vx, D.pr);
    D.pi = fma(wgt, vy, D.pi);
    D.ir = fma(qb, vx, D.ir);
    D.ii = fma(qb, vy, D.ii);
    if (a == 0 && col == 0) {
      D.g0r = vx;
      D.g0i = vy;
    }
  }
}

template <int N, int S, int NT, int PAIRS, int NTHR>
struct FftDifDigest {
  __device__ __forceinline__ static void run(double2* T, const double2* rou_s, int tid, int bar,
                                             int C, int ncol, int ncomp, const double* betaw_s,
                                             int a0, DigestAcc& D) {
    constexpr int R = smallest_prime_factor(S);
    if constexpr (R == S) {
      fft_last_digest<N, R, NT, PAIRS>(T, tid, C, ncol, ncomp, betaw_s, a0, D);
      stage_sync(bar, NTHR);
    } else {
      fft_stage_ct<N, R, S, NT, PAIRS, NTHR>(T, rou_s, tid);
      stage_sync(bar, NTHR);
      FftDifDigest<N, S / R, NT, PAIRS, NTHR>::run(T, rou_s, tid, bar, C, ncol, ncomp, betaw_s, a0,
                                                     D);
    }
  }
};

// Warp -> first-stage row group: the FFT warps (the first NFW) take the groups with the fewest
// k-steps, since they also run the last stage.
template <int N>
struct LnGroupMap {
  int v[LnCfg<N>::MP];
  constexpr LnGroupMap() : v() {
    using Rows = LnRows<N>;
    constexpr int MP = LnCfg<N>::MP, R1 = LnCfg<N>::R1;
    int ks[MP] = {};
    for (int r = 0; r < MP; ++r)
      for (int k = 0; k < R1; ++k) ks[r] += (Rows::np(Rows::jq_of_row(r + k * MP)) + 3) / 4;
    bool used[MP] = {};
    for (int i = 0; i < MP; ++i) {  // stable selection by ascending k-step count
      int best = -1;
      for (int r = 0; r < MP; ++r)
        if (!used[r] && (best < 0 || ks[r] < ks[best])) best = r;
      used[best] = true;
      v[i] = best;
    }
  }
};

// DMMA chains of first-stage row group CW (T rows CW + k MP, k < R1): Gauss 3-product complex
// MMA over the k-steps of each row's q block. Every row offset and k-step count is a
// compile-time constant (the warp dispatches on its group once per tile), so the loop has no
// guards and the operand addresses are immediates.
template <int N, int CW>
struct LnRowGroup {
  using Cfg = LnCfg<N>;
  using Rows = typename Cfg::Rows;
  static constexpr int R1 = Cfg::R1, MP = Cfg::MP, NT = Cfg::NT;
  __device__ __forceinline__ static void mma(int cw, const double2* Us, const double2* Ws,
                                             int lane, double (&c1)[R1][2], double (&c2)[R1][2],
                                             double (&c3)[R1][2]) {
    if constexpr (CW + 1 < MP) {
      if (cw != CW) {
        LnRowGroup<N, CW + 1>::mma(cw, Us, Ws, lane, c1, c2, c3);
        return;
      }
    }
    const int kl = lane & 3, ar = lane >> 2;
    const double2* Ua = Us + ar * Cfg::UPAD + kl;
#pragma unroll
    for (int k = 0; k < R1; ++k) c1[k][0] = c1[k][1] = c2[k][0] = c2[k][1] = c3[k][0] = c3[k][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < Cfg::KSMAX; ++ks)
#pragma unroll
      for (int k = 0; k < R1; ++k) {
        const int jq = Rows::jq_of_row(CW + k * MP);
        if (ks < (Rows::np(jq) + 3) / 4) {
          const int wr = Rows::qoff(jq) + 4 * ks + kl;
          const double2 a = Ua[Rows::urb(jq) + 4 * ks];
          const double2 b = Ws[wr * NT + (ar ^ ((2 * wr) & 7))];
          dmma(c1[k][0], c1[k][1], a.x + a.y, b.x);
          dmma(c2[k][0], c2[k][1], a.x, b.y - b.x);
          dmma(c3[k][0], c3[k][1], a.y, b.x + b.y);
        }
      }
  }
};

template <int N>
__global__ void __launch_bounds__(LnCfg<N>::NTHREADS, 1) k_couple_lines(const LnParams LP) {
  using Cfg = LnCfg<N>;
  constexpr int L = Cfg::L, MT = Cfg::MT, NT = Cfg::NT, NC = Cfg::NC, NPQ = Cfg::NPQ;
  constexpr int NCW = Cfg::NCW, R1 = Cfg::R1, MP = Cfg::MP;
  const CoupleParams& P = LP.c;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* Us = reinterpret_cast<double2*>(smem);
  double2* Wsb = reinterpret_cast<double2*>(smem + Cfg::OFF_W);
  double2* Tb = reinterpret_cast<double2*>(smem + Cfg::OFF_T);
  double2* rou_s = reinterpret_cast<double2*>(smem + Cfg::OFF_TAB);
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  int* qoff_s = reinterpret_cast<int*>(betaw_s + (L + 1));
  int* urb_s = qoff_s + (N + 2);
  CompRec* rec_s = reinterpret_cast<CompRec*>(
      (reinterpret_cast<uintptr_t>(urb_s + N) + 15) & ~static_cast<uintptr_t>(15));
  double* dpart = reinterpret_cast<double*>(rec_s + MT);  // [NPART][MT][8] digest partials
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* ufull = bars + 0;
  uint64_t* uempty = bars + 1;
  uint64_t* wfull = bars + 2;   // [2] W tile slots
  uint64_t* wempty = bars + 4;  // [2]
  uint64_t* tready = bars + 6;  // [2] per tile parity: FFT of the tile done
  uint64_t* tfree = bars + 8;   // [2] per tile parity: stores of the tile done
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nct = P.n_col_tiles;
  constexpr size_t TE = Cfg::T_BYTES / 16;  // complex per T buffer
  constexpr size_t WE = Cfg::WS_BYTES / 16;

  for (int i = tid; i < N; i += Cfg::NTHREADS) {
    rou_s[i] = P.rou[i];
    urb_s[i] = LP.urb[i];
  }
  for (int i = tid; i <= N; i += Cfg::NTHREADS) qoff_s[i] = P.qoff[i];
  for (int i = tid; i <= L; i += Cfg::NTHREADS) betaw_s[i] = P.betaw[i];
  // W rows past NPQ are read (times a zero U pad) by partial k-steps: keep them finite
  for (int i = tid; i < 2 * 4 * NT; i += Cfg::NTHREADS)
    Wsb[(i / (4 * NT)) * WE + (size_t)NPQ * NT + i % (4 * NT)] = make_double2(0.0, 0.0);
  if (tid == 0) {
    mbar_init(ufull, 1);
    mbar_init(uempty, NCW);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&wfull[b], 1);
      mbar_init(&wempty[b], NCW);
      mbar_init(&tready[b], Cfg::NFW);
      mbar_init(&tfree[b], Cfg::NSW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // work units: (group g, column segment sg) storing tiles [seg_lo(sg), seg_lo(sg + 1)). A
  // unit after the first also computes the tile before its range (no stores, no digest), so
  // its first lines have their previous tile: every line is written whole by one unit.
  const int n_units = LP.n_groups * LP.nseg;
  auto seg_lo = [&](int sg) { return (int)(((long long)sg * nct) / LP.nseg); };
  auto seg_c0 = [&](int sg) { return sg > 0 ? seg_lo(sg) - 1 : 0; };
  // digest segments: a fixed split of every group's tiles, refined by the execution split, so
  // the digest partials (and their sums) do not depend on how the work is cut into units
  auto dig_lo = [&](int k) { return (int)(((long long)k * nct) / LP.nseg_dig); };

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t uphase = 0;
      long long t = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int g = u / LP.nseg, sg = u % LP.nseg;
        mbar_wait(uempty, uphase ^ 1);
        const uint32_t ub = (uint32_t)(LP.group_elems * 16);
        mbar_arrive_expect_tx(ufull, ub);
        bulk_g2s(Us, P.U + (size_t)g * LP.group_elems, ub, ufull);
        uphase ^= 1;
        for (int ct = seg_c0(sg); ct < seg_lo(sg + 1); ++ct, ++t) {
          const int sl = (int)(t & 1);
          mbar_wait(&wempty[sl], (uint32_t)(((t >> 1) & 1) ^ 1));
          constexpr uint32_t wb = (uint32_t)(NPQ * NT * 16);
          mbar_arrive_expect_tx(&wfull[sl], wb);
          bulk_g2s(Wsb + sl * WE, P.W + (size_t)ct * NPQ * NT, wb, &wfull[sl]);
        }
      }
    }
    return;
  }

  if (warp <= NCW) {
    // ------------------------------------------------------------------ compute warps
    constexpr LnGroupMap<N> kMap{};
    constexpr int NF = Cfg::NF;
    const int cw = kMap.v[warp - 1];  // row group: T rows cw + k MP, k < R1
    const bool fft = warp - 1 < Cfg::NFW;
    const int c_tid = tid - 32;
    const int kl = lane & 3, ar = lane >> 2;
    const int a0 = dif_last_freq0<N, Cfg::RLAST>(c_tid / (MT * NT));
    uint32_t uphase = 0;
    long long t = 0;  // global tile counter of this CTA
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const int g = u / LP.nseg, sg = u % LP.nseg;
      const int s0 = seg_lo(sg), s1 = seg_lo(sg + 1);
      const int ncomp = min(MT, P.count - g * MT);
      DigestAcc D{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0};
      int kd = sg * (LP.nseg_dig / LP.nseg);  // digest segment of tile s0
      int kd_end = dig_lo(kd + 1);
      mbar_wait(ufull, uphase);
      uphase ^= 1;
      for (int ct = seg_c0(sg); ct < s1; ++ct, ++t) {
        double2* T = Tb + (size_t)(t % 3) * TE;
#ifdef SLSHT_WS_TRACE
        const bool tr = LP.trace && blockIdx.x == 0 && c_tid == 0 && t < 128;
        if (tr) LP.trace[t * 8 + 0] = clock64();
#endif
        // buffer t % 3 was last read by the stores of tile t-2 (as their previous tile)
        if (t >= 2) mbar_wait(&tfree[t & 1], (uint32_t)(((t - 2) >> 1) & 1));
#ifdef SLSHT_WS_TRACE
        if (tr) LP.trace[t * 8 + 1] = clock64();
#endif
        const int sl = (int)(t & 1);
        mbar_wait(&wfull[sl], (uint32_t)((t >> 1) & 1));
#ifdef SLSHT_WS_TRACE
        if (tr) LP.trace[t * 8 + 2] = clock64();
#endif
        const double2* Ws = Wsb + sl * WE;
        double c1[R1][2], c2[R1][2], c3[R1][2];
        LnRowGroup<N, 0>::mma(cw, Us, Ws, lane, c1, c2, c3);
#ifdef SLSHT_WS_TRACE
        if (tr) LP.trace[t * 8 + 3] = clock64();
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&wempty[sl]);
        if (ct == s1 - 1 && lane == 0) mbar_arrive(uempty);
        // first DIF stage (radix R1, span N) on the accumulators: rows cw + k MP, twiddle
        // rou^(cw k)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double xr[R1], xi[R1];
#pragma unroll
          for (int k = 0; k < R1; ++k) {
            xr[k] = c1[k][e] - c3[k][e];
            xi[k] = c1[k][e] + c2[k][e];
          }
          Radix<R1>::dft(xr, xi);
          double2* dst = T + (size_t)(ar * N + cw) * NT + 2 * kl + e;
          dst[0] = make_double2(xr[0], xi[0]);
#pragma unroll
          for (int k = 1; k < R1; ++k) {
            const double2 w = rou_s[cw * k];
            dst[(size_t)k * MP * NT] =
                make_double2(xr[k] * w.x - xi[k] * w.y, xr[k] * w.y + xi[k] * w.x);
          }
        }
#ifdef SLSHT_WS_TRACE
        if (tr) LP.trace[t * 8 + 4] = clock64();
#endif
        named_sync(1, NC);
#ifdef SLSHT_WS_TRACE
        if (tr) LP.trace[t * 8 + 5] = clock64();
#endif
        if (!fft) continue;  // on to the next tile's DMMA
        // the warm-up tile before the unit's range adds nothing to the digest
        FftDifDigest<N, MP, NT, MT * NT, NF>::run(T, rou_s, c_tid, 2, ct * NT, P.ncol,
                                                  ct < s0 ? 0 : ncomp, betaw_s, a0, D);
#ifdef SLSHT_WS_TRACE
        if (tr) LP.trace[t * 8 + 6] = clock64();
#endif
        if (lane == 0) mbar_arrive(&tready[t & 1]);
        if (ct < s0) continue;
        // end of a digest segment: its partial (8-lane shuffle trees, then the NPART partial
        // blocks in order; max |g|^2 and unscaled integrals, k_digest finishes the row)
        if (ct + 1 == kd_end) {
          constexpr int LI = Cfg::LAST_ITEMS;  // thread c_tid < LI holds pair c_tid % 64
          const unsigned m8 = 0xffu << (lane & ~7);
          double v[8] = {D.s2, __longlong_as_double(D.mx2), D.pr, D.pi, D.g0r, D.g0i, D.ir, D.ii};
#pragma unroll
          for (int off = 4; off > 0; off >>= 1)
#pragma unroll
            for (int f = 0; f < 8; ++f) {
              const double o = __shfl_down_sync(m8, v[f], off, 8);
              v[f] = (f == 1) ? fmax(v[f], o) : v[f] + o;
            }
          if ((lane & 7) == 0 && c_tid < LI) {
            const int c = (c_tid % (MT * NT)) / NT, ip = c_tid / (MT * NT);
#pragma unroll
            for (int f = 0; f < 8; ++f) dpart[(ip * MT + c) * 8 + f] = v[f];
          }
          named_sync(2, NF);
          if (c_tid < ncomp * 8) {
            const int c = c_tid >> 3, f = c_tid & 7;
            double sacc = 0.0;
#pragma unroll
            for (int ip = 0; ip < Cfg::NPART; ++ip) {
              const double x = dpart[(ip * MT + c) * 8 + f];
              sacc = (f == 1) ? fmax(sacc, x) : sacc + x;
            }
            LP.partials[((size_t)(g * MT + c) * LP.nseg_dig + kd) * 8 + f] = sacc;
          }
          named_sync(2, NF);  // dpart reused by the next flush
          D = DigestAcc{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0};
          ++kd;
          kd_end = dig_lo(kd + 1);
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ store warps
  // line group g8 = (component c, volume w): for every row a of tile ct the aligned 128-B line
  // that starts in (p0 - 8, p0], p0 = the row's first element in the tile. Row a starts at
  // base + a ncol, ncol == 1 (mod 8), so the line phase of row a is (base + a) & 7.
  constexpr DifPerm<N> kPerm{};
  const int st = tid - 32 - NC;  // 0 .. NSW*32-1
  const int j = st & 7;          // element of the line
  const int g8 = st >> 3;
  const int c = g8 & 7, w = g8 >> 3;
  const int ncol = P.ncol;
  const long long sbit = (long long)0x8000000000000000ULL;
  long long t = 0;
  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    const int g = u / LP.nseg, sg = u % LP.nseg;
    const int s0 = seg_lo(sg), s1 = seg_lo(sg + 1);
    const int ncomp = min(MT, P.count - g * MT);
    bool act = c < ncomp;
    long long base = 0;
    long long fr = 0, fi = 0;
    if (act) {
      const CompRec rec = P.comps[g * MT + c];
      act = (w == 0) || (P.mirror && rec.m > 0);
      base = (w ? rec.mslot : rec.slot) * P.vol;
      if (w) {  // (-1)^m conj
        fr = (rec.m & 1) ? sbit : 0;
        fi = (rec.m & 1) ? 0 : sbit;
      }
    }
    const int ksh0 = (int)(base & 7);
    double2* outp = P.out + base;
    for (int ct = seg_c0(sg); ct < s1; ++ct, ++t) {
      const int C = ct * NT;
      mbar_wait(&tready[t & 1], (uint32_t)((t >> 1) & 1));
#ifdef SLSHT_WS_TRACE
      const bool tr = LP.trace && blockIdx.x == 0 && st == 0 && t < 128;
#endif
#ifndef LN_NO_STORE
      if (act && ct >= s0) {
        const double2* Tc = Tb + (size_t)(t % 3) * TE + (size_t)c * N * NT;
        const double2* Tp = Tb + (size_t)((t + 2) % 3) * TE + (size_t)c * N * NT + 8;
        double2* orow = outp + C;  // row a: orow + a ncol
        if (ct > 0 && ct < nct - 1) {
          // interior tile: every element of every line exists (the previous tile is resident,
          // also at a unit's first tile: the unit computed it)
#pragma unroll
          for (int a = 0; a < N; ++a) {
            const int d = j - ((ksh0 + a) & 7);  // column offset from C (< 0: previous tile)
            const double2* src = (d < 0 ? Tp : Tc) + kPerm.v[a] * NT + d;
            double2 v = *src;
            v = make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ fr),
                             __longlong_as_double(__double_as_longlong(v.y) ^ fi));
            orow[a * ncol + d] = v;
          }
        } else {
          // the row's first tile (the line's head is in row a - 1: written with that row's last
          // tile) and last tile (one column); stores predicated, loads always in range
          const int cmax = ncol - C;  // columns of this tile in the row
#pragma unroll
          for (int a = 0; a < N; ++a) {
            const int d = j - ((ksh0 + a) & 7);
            const bool ok = d >= 0 ? d < cmax : ct > 0;
            const double2* src = (d < 0 ? Tp : Tc) + kPerm.v[a] * NT + d;
            double2 v = *src;
            v = make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ fr),
                             __longlong_as_double(__double_as_longlong(v.y) ^ fi));
            if (ok) orow[a * ncol + d] = v;
          }
        }
      }
#endif
#ifdef SLSHT_WS_TRACE
      if (tr) LP.trace[t * 8 + 7] = clock64();
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&tfree[t & 1]);
    }
  }
}

}  // namespace slsht_cuda
