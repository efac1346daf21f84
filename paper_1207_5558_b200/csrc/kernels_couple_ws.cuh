// Warp-specialized persistent coupling kernel, used for the compile-time
// transform lengths. One CTA per SM loops over (component group, column tile) tiles:
//
//   producer warp  : cp.async.bulk (TMA bulk-copy engine) of the operand rows of one q-group
//                    per stage -- U[comp][rows] (contiguous per component) and
//                    W[row][col0 : col0+NT] -- into an NSTAGE-deep shared-memory ring guarded
//                    by mbarriers (full: complete_tx bytes, empty: consumer arrivals);
//   MMA warps      : T[comp][q mod n][col] = sum_p U W on the FP64 tensor cores (DMMA 8x8x4,
//                    complex product as 3 real MMAs), operands read from the ring, results
//                    into one of NTBUF T buffers;
//   epilogue warps : alpha FFT in place (compile-time DIF plan), streaming stores of the
//                    volume (and its conjugate mirror), digest partials -- on the previous
//                    tile's T buffer while the MMA warps fill the next one.
#pragma once

#include "common.cuh"
#include "fft_radix.cuh"
#include "kernels_couple.cuh"

namespace slsht_cuda {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Bulk copy global -> shared through the TMA unit; completion counted on `bar` in bytes.
// The same wait with a suspend-time hint: a thread whose phase is not complete sleeps
// (NANOSLEEP.SYNCS, woken by the barrier) instead of spinning on try_wait, so waiting warps do
// not take issue slots from the working warps of their SM sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// Host-computed stage table: stage s covers q rows jq in [js[s], js[s+1]); its U block sits at
// uoff[s] inside a component group's U region with row stride ustr[s] (== 4 mod 8 16-B units).
struct WsStages {
  int count;
  int js[136];    // n + 1 entries at most (n <= 129 for the compile-time lengths)
  int uoff[136];
  int ustr[136];
  int urb[136];           // per q row jq: offset of its zero-padded row block in its U stage
  long long group_elems;  // U elements per component group
};

struct WsParams {
  CoupleParams c;
  long long* trace;  // debug: per-tile phase timestamps of CTA 0 (SLSHT_WS_TRACE builds)
  WsStages st;
  int n_groups;  // component groups of MT in this chunk
  int n_tiles;   // n_groups * n_col_tiles
  int ct_fast;   // tile order: 1 -> column tile fastest (small W), 0 -> group fastest
};

template <int N, int MG, int NG, int RS, int NSTAGE, int GW>
struct WsCfg {
  static constexpr int L = (N - 1) / 2;
  static constexpr int MT = 8 * MG, NT = 8 * NG, WT = MG * NG;
  static constexpr int GW_ = GW;                     // warps per consumer group
  static constexpr int GT = GW * 32;                 // threads per consumer group
  static constexpr int NTHREADS = 32 + 2 * GT;       // producer warp + two groups
  static constexpr int PAIRS = MT * NT;
  static constexpr int USTR = RS + 8;                // max 16-B units per staged U row
  static constexpr size_t T_BYTES = (size_t)MT * N * NT * 16;
  static constexpr size_t U_BYTES = (size_t)MT * USTR * 16;
  static constexpr size_t W_BYTES = (size_t)(RS + 4) * NT * 16;  // +4 spare rows read by partial k-steps
  static constexpr size_t STAGE_BYTES = U_BYTES + W_BYTES;
  static constexpr size_t OFF_STAGE = 2 * T_BYTES;
  static constexpr size_t OFF_TAB = OFF_STAGE + NSTAGE * STAGE_BYTES;
  static constexpr size_t TAB_BYTES = (size_t)N * 16 + (size_t)(L + 1) * 8 + (size_t)(2 * N + 2) * 4;
  static constexpr size_t OFF_BAR = (OFF_TAB + TAB_BYTES + 15) / 16 * 16;
  static constexpr size_t SMEM = OFF_BAR + (2 * NSTAGE + 1) * 8;
  static_assert(GT % PAIRS == 0, "group threads must cover the pairs");
  static_assert(T_BYTES >= (size_t)GT * 8 * 8, "T buffer doubles as reduction scratch");
  static_assert(RS % 4 == 0, "stage rows in k-steps");
};

// Output rows a = A0, A0 + A_STEP, ... of one (component, column) transform: the permutation is
// a compile-time table, so every T read is a constant offset.
template <int N>
struct DifPerm {
  int v[N];
  constexpr DifPerm() : v() {
    int fac[16] = {}, nf = 0, x = N;
    for (int p = 3; x > 1; p += 2)
      while (x % p == 0) {
        fac[nf++] = p;
        x /= p;
      }
    for (int pos = 0; pos < N; ++pos) {
      int rem = pos, freq = 0, mult = 1, mm = N;
      for (int i = 0; i < nf; ++i) {
        const int mp = mm / fac[i], k = rem / mp;
        rem %= mp;
        freq += k * mult;
        mult *= fac[i];
        mm = mp;
      }
      v[freq] = pos;
    }
  }
};

template <int N, int NT, int PAIRS, int A_STEP, int A0>
__device__ __forceinline__ void ws_epilogue(const double2* T, const int* perm_s,
                                            const CoupleParams& P, const CompRec& rec, int cl,
                                            int cc, int col, double& s2, long long& mx2,
                                            double& pr, double& pi, double& ir, double& ii,
                                            double& g0r, double& g0i) {
  constexpr DifPerm<N> kPerm{};
  (void)perm_s;
  double2* o = P.out + rec.slot * P.vol + col + (size_t)A0 * P.ncol;
  double2* om = (P.mirror && rec.m > 0) ? P.out + rec.mslot * P.vol + col + (size_t)A0 * P.ncol
                                        : nullptr;
  const long long sbit = (long long)0x8000000000000000ULL;
  const long long fr = (rec.m & 1) ? sbit : 0, fi = (rec.m & 1) ? 0 : sbit;
  const double2* Tp = T + (size_t)cl * N * NT + cc;
  const size_t ostep = (size_t)A_STEP * P.ncol;
  uint32_t hsh = (uint32_t)((size_t)A0 * P.ncol + col) * 0x9E3779B1u;
  const uint32_t hstep = (uint32_t)ostep * 0x9E3779B1u;
  if (A0 == 0 && col == 0) {
    const double2 v = Tp[kPerm.v[0] * NT];
    g0r = v.x;
    g0i = v.y;
  }
#pragma unroll
  for (int a = A0; a < N; a += A_STEP) {
    const double2 v = Tp[kPerm.v[a] * NT];
    *o = v;
    o += ostep;
    if (om) {
      *om = make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ fr),
                         __longlong_as_double(__double_as_longlong(v.y) ^ fi));
      om += ostep;
    }
    const double a2 = fma(v.x, v.x, v.y * v.y);
    s2 += a2;
    mx2 = max(mx2, __double_as_longlong(a2));
    const double wgt = digest_weight(hsh);
    hsh += hstep;
    pr = fma(wgt, v.x, pr);
    pi = fma(wgt, v.y, pi);
    ir += v.x;
    ii += v.y;
  }
}

// Ping-pong persistent kernel: a producer warp streams the operand stages of the CTA's tiles in
// order through the ring; consumer group k (GW warps) owns every other tile and its own T
// buffer and runs MMA -> FFT -> epilogue on it, so one group's tensor-core phase overlaps the
// other group's FFT and store phase.
template <int N, int MG, int NG, int RS, int NSTAGE, int GW>
__global__ void __launch_bounds__(WsCfg<N, MG, NG, RS, NSTAGE, GW>::NTHREADS, 1)
    k_couple_ws(const WsParams WP) {
  using Cfg = WsCfg<N, MG, NG, RS, NSTAGE, GW>;
  constexpr int L = Cfg::L, MT = Cfg::MT, NT = Cfg::NT, WT = Cfg::WT;
  constexpr int GT = Cfg::GT, PAIRS = Cfg::PAIRS, USTR = Cfg::USTR;
  const CoupleParams& P = WP.c;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* rou_s = reinterpret_cast<double2*>(smem + Cfg::OFF_TAB);
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  int* perm_s = reinterpret_cast<int*>(betaw_s + (L + 1));
  int* qoff_s = perm_s + N;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* full = bars;
  uint64_t* empty = bars + NSTAGE;
  // turn: completion j = the MMA phase of the CTA's j-th tile has released its stages. A group
  // starts tile k's stages only after completion k-1, so ring waits never see a stale phase.
  uint64_t* turn = bars + 2 * NSTAGE;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < N; i += Cfg::NTHREADS) {
    rou_s[i] = P.rou[i];
    perm_s[i] = P.perm[i];
  }
  for (int i = tid; i <= N; i += Cfg::NTHREADS) qoff_s[i] = P.qoff[i];
  for (int i = tid; i <= L; i += Cfg::NTHREADS) betaw_s[i] = P.betaw[i];
  {
    // W rows past a stage's rows are read (times a zero U pad) by partial k-steps: keep the
    // ring finite from the start
    double4* ring = reinterpret_cast<double4*>(smem + Cfg::OFF_STAGE);
    for (size_t i = tid; i < NSTAGE * Cfg::STAGE_BYTES / 32; i += Cfg::NTHREADS)
      ring[i] = make_double4(0.0, 0.0, 0.0, 0.0);
  }
  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], GW);
    }
    mbar_init(turn, GW);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int nst = WP.st.count;
  auto tile_of = [&](int t, int& g, int& ct) {
    g = WP.ct_fast ? t / P.n_col_tiles : t % WP.n_groups;
    ct = WP.ct_fast ? t % P.n_col_tiles : t / WP.n_groups;
  };
  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    int stage = 0;
    uint32_t phase = 0;
    for (int t = blockIdx.x; t < WP.n_tiles; t += gridDim.x) {
      int g, ct;
      tile_of(t, g, ct);
      for (int s = 0; s < nst; ++s) {
        mbar_wait(&empty[stage], phase ^ 1);
        if (lane == 0) {
          const int r0 = qoff_s[WP.st.js[s]], rows = qoff_s[WP.st.js[s + 1]] - r0;
          double2* Us = reinterpret_cast<double2*>(smem + Cfg::OFF_STAGE + stage * Cfg::STAGE_BYTES);
          double2* Ws = Us + MT * USTR;
          const uint32_t ub = (uint32_t)(MT * WP.st.ustr[s]) * 16u;
          const uint32_t wb = (uint32_t)(rows * NT) * 16u;
          mbar_arrive_expect_tx(&full[stage], ub + wb);
          bulk_g2s(Us, P.U + (size_t)g * WP.st.group_elems + WP.st.uoff[s], ub, &full[stage]);
          bulk_g2s(Ws, P.W + ((size_t)ct * P.NPQ + r0) * NT, wb, &full[stage]);
        }
        __syncwarp();
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------------ consumer groups
  const int grp = (warp - 1) / GW;          // 0 or 1
  const int gw = (warp - 1) % GW;           // warp within the group
  const int gt = tid - 32 - grp * GT;       // thread within the group
  const int bar_id = 1 + grp;
  double2* T = reinterpret_cast<double2*>(smem + grp * Cfg::T_BYTES);
  const int kl = lane & 3;
  // the group's first stage slot: group 1 starts after the first tile's stages
  int stage = 0;
  uint32_t phase = 0;
  auto advance = [&](int k) {
    for (int i = 0; i < k; ++i)
      if (++stage == NSTAGE) {
        stage = 0;
        phase ^= 1;
      }
  };
  int k_local = 0;  // index of the tile within this CTA's sequence
  for (int t = blockIdx.x; t < WP.n_tiles; t += gridDim.x, ++k_local) {
    if ((k_local & 1) != grp) {
      advance(nst);  // the other group's tile: skip its stages in the ring
      continue;
    }
    int g, ct;
    tile_of(t, g, ct);
    const int comp0 = g * MT, col0 = ct * NT;
    constexpr int A_STEP = GT / PAIRS;
    const int pair = gt % PAIRS;
    const int cl = pair / NT, cc = pair % NT;
    const int a_first = gt / PAIRS;  // warp-uniform
    const int comp = comp0 + cl, col = col0 + cc;
    const bool ok = comp < P.count && col < P.ncol;
    CompRec rec{0, 0, 0, -1};
    if (ok) rec = P.comps[comp];  // in flight during the MMA phase
    // ---------------- MMA phase: items (q, warp tile), q-major, one per warp per round
#ifdef SLSHT_WS_TRACE
    const bool tr = WP.trace && blockIdx.x == 0 && gt == 0 && k_local < 64;
    if (tr) WP.trace[k_local * 6 + 0] = clock64();
#endif
    if (k_local > 0) mbar_wait(turn, (uint32_t)((k_local - 1) & 1));
#ifdef SLSHT_WS_TRACE
    if (tr) WP.trace[k_local * 6 + 1] = clock64();
#endif
    for (int s = 0; s < nst; ++s) {
#ifdef SLSHT_WS_TRACE
      long long tw0 = clock64();
#endif
      mbar_wait(&full[stage], phase);
#ifdef SLSHT_WS_TRACE
      if (tr && s < 8) WP.trace[384 + k_local * 16 + 2 * s] = clock64() - tw0;
      tw0 = clock64();
#endif
      const double2* Us =
          reinterpret_cast<const double2*>(smem + Cfg::OFF_STAGE + stage * Cfg::STAGE_BYTES);
      const double2* Ws = Us + MT * USTR;
      const int j0 = WP.st.js[s], j1 = WP.st.js[s + 1];
      const int r0 = qoff_s[j0];
      const int ustr = WP.st.ustr[s];
      const int n_items = (j1 - j0) * WT;
#ifdef SLSHT_WS_NO_MMA
      if (false)
#endif
      for (int it = gw; it < n_items; it += GW) {
        const int jq = j0 + it / WT, wt = it % WT;
        const int np = L + 1 - abs(jq - L);
        const int nks = (np + 3) >> 2;
        const int wrb = qoff_s[jq] - r0;  // W rows of q in the stage
        const int ar = (wt / NG) * 8 + (lane >> 2);
        const int bhi = (wt % NG) * 8, blo = lane >> 2;
        // U rows of q are zero-padded to whole k-steps, so no masking; the W swizzle of a lane
        // is the same in every k-step (rows advance by 4, 2*4 == 0 mod 8)
        const double2* ap = Us + ar * ustr + WP.st.urb[jq] + kl;
        const double2* bp = Ws + (wrb + kl) * NT + (bhi | (blo ^ ((2 * (r0 + wrb + kl)) & 7)));
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
        double2* dst = T + (size_t)(ar * N + row) * NT + bhi + 2 * kl;
        dst[0] = make_double2(c1[0] - c3[0], c1[0] + c2[0]);
        dst[1] = make_double2(c1[1] - c3[1], c1[1] + c2[1]);
      }
      __syncwarp();
#ifdef SLSHT_WS_TRACE
      if (tr && s < 8) WP.trace[384 + k_local * 16 + 2 * s + 1] = clock64() - tw0;
#endif
      if (lane == 0) mbar_arrive(&empty[stage]);
      advance(1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(turn);
#ifdef SLSHT_WS_TRACE
    if (tr) WP.trace[k_local * 6 + 2] = clock64();
#endif
    named_sync(bar_id, GT);
#ifdef SLSHT_WS_TRACE
    if (tr) WP.trace[k_local * 6 + 3] = clock64();
#endif
#ifdef SLSHT_WS_NO_EPI
    continue;
#endif
    // ---------------- alpha FFT in place
    FftDif<N, N, NT, PAIRS, GT>::run(T, rou_s, gt, bar_id);
    // ---------------- epilogue: stores, mirror, digest partials
#ifdef SLSHT_WS_TRACE
    if (tr) WP.trace[k_local * 6 + 4] = clock64();
#endif
    double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
    long long mx2 = 0;
    if (ok) {
      if (a_first == 0)
        ws_epilogue<N, NT, PAIRS, A_STEP, 0>(T, perm_s, P, rec, cl, cc, col, s2, mx2, pr, pi, ir, ii,
                                             g0r, g0i);
      else if constexpr (A_STEP > 1)
        ws_epilogue<N, NT, PAIRS, A_STEP, 1>(T, perm_s, P, rec, cl, cc, col, s2, mx2, pr, pi, ir, ii,
                                             g0r, g0i);
      const double qb = betaw_s[col / N];
      ir *= qb;
      ii *= qb;
    }
    named_sync(bar_id, GT);  // all reads of T done: reuse it as the reduction scratch
    double* red = reinterpret_cast<double*>(T);
    red[gt * 8 + 0] = s2;
    red[gt * 8 + 1] = __longlong_as_double(mx2);
    red[gt * 8 + 2] = pr;
    red[gt * 8 + 3] = pi;
    red[gt * 8 + 4] = g0r;
    red[gt * 8 + 5] = g0i;
    red[gt * 8 + 6] = ir;
    red[gt * 8 + 7] = ii;
    named_sync(bar_id, GT);
    if (gt < MT * 8) {
      const int c = gt >> 3, k = gt & 7;
      if (comp0 + c < P.count) {
        double acc = 0.0;
        for (int t2 = c * NT; t2 < GT; t2 += PAIRS)
          for (int u = 0; u < NT; ++u) {
            const double v = red[(t2 + u) * 8 + k];
            acc = (k == 1) ? fmax(acc, v) : acc + v;
          }
        P.partials[((size_t)(comp0 + c) * P.n_col_tiles + ct) * 8 + k] = acc;
      }
    }
    named_sync(bar_id, GT);  // scratch read before the next tile's MMA writes T
#ifdef SLSHT_WS_TRACE
    if (tr) WP.trace[k_local * 6 + 5] = clock64();
#endif
  }
}

}  // namespace slsht_cuda
