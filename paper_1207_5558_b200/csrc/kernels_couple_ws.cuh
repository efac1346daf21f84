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
  long long group_elems;  // U elements per component group
};

struct WsParams {
  CoupleParams c;
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
  static constexpr size_t W_BYTES = (size_t)RS * NT * 16;
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
    // ---------------- MMA phase: items (q, warp tile), q-major, one per warp per round
    if (k_local > 0) mbar_wait(turn, (uint32_t)((k_local - 1) & 1));
    for (int s = 0; s < nst; ++s) {
      mbar_wait(&full[stage], phase);
      const double2* Us =
          reinterpret_cast<const double2*>(smem + Cfg::OFF_STAGE + stage * Cfg::STAGE_BYTES);
      const double2* Ws = Us + MT * USTR;
      const int j0 = WP.st.js[s], j1 = WP.st.js[s + 1];
      const int r0 = qoff_s[j0];
      const int ustr = WP.st.ustr[s];
      const int n_items = (j1 - j0) * WT;
      for (int it = gw; it < n_items; it += GW) {
        const int jq = j0 + it / WT, wt = it % WT;
        const int np = L + 1 - abs(jq - L);
        const int rb = qoff_s[jq] - r0;
        const int ar = (wt / NG) * 8 + (lane >> 2);
        const int bc = (wt % NG) * 8 + (lane >> 2);
        const int bsw_hi = bc & ~7, bsw_lo = bc & 7;
        // branch-free fragments: rows clamped into the q's range, A zeroed past np (B x 0 = 0)
        auto frag = [&](int ks, double& s_, double& ax, double& ay, double& bx, double& d_, double& e_) {
          const int k = 4 * ks + kl;
          const int r = rb + min(k, np - 1);
          const double2 a = Us[ar * ustr + r];
          const double2 b = Ws[r * NT + (bsw_hi | (bsw_lo ^ ((2 * (r0 + r)) & 7)))];
          const bool keep = k < np;
          ax = keep ? a.x : 0.0;
          ay = keep ? a.y : 0.0;
          s_ = ax + ay;
          bx = b.x;
          d_ = b.y - b.x;
          e_ = b.x + b.y;
        };
        double c1[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0}, c3[2] = {0.0, 0.0};
        const int ks_n = (np + 3) / 4;
        double s_, ax, ay, bx, d_, e_;
        frag(0, s_, ax, ay, bx, d_, e_);
        for (int ks = 0; ks < ks_n; ++ks) {
          double ns_, nax, nay, nbx, nd_, ne_;
          frag(min(ks + 1, ks_n - 1), ns_, nax, nay, nbx, nd_, ne_);
          dmma(c1[0], c1[1], s_, bx);
          dmma(c2[0], c2[1], ax, d_);
          dmma(c3[0], c3[1], ay, e_);
          s_ = ns_; ax = nax; ay = nay; bx = nbx; d_ = nd_; e_ = ne_;
        }
        const int row = jq >= L ? jq - L : jq + L + 1;  // q mod n
        double2* dst = T + (size_t)(ar * N + row) * NT + bsw_hi + 2 * kl;
        dst[0] = make_double2(c1[0] - c3[0], c1[0] + c2[0]);
        dst[1] = make_double2(c1[1] - c3[1], c1[1] + c2[1]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      advance(1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(turn);
    named_sync(bar_id, GT);
    // ---------------- alpha FFT in place
    FftDif<N, N, NT, PAIRS, GT>::run(T, rou_s, gt, bar_id);
    // ---------------- epilogue: stores, mirror, digest partials
    const int pair = gt % PAIRS;
    const int cl = pair / NT, cc = pair % NT;
    constexpr int A_STEP = GT / PAIRS;
    const int comp = comp0 + cl, col = col0 + cc;
    const bool ok = comp < P.count && col < P.ncol;
    double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
    long long mx2 = 0;
    if (ok) {
      const CompRec rec = P.comps[comp];
      double2* o = P.out + rec.slot * P.vol + col;
      double2* om = (P.mirror && rec.m > 0) ? P.out + rec.mslot * P.vol + col : nullptr;
      const long long sbit = (long long)0x8000000000000000ULL;
      const long long fr = (rec.m & 1) ? sbit : 0, fi = (rec.m & 1) ? 0 : sbit;
      const double qb = betaw_s[col / N];
      const double2* Tp = T + (size_t)cl * N * NT + cc;
      const int a_first = gt / PAIRS;
      uint32_t hsh = (uint32_t)((size_t)a_first * P.ncol + col) * 0x9E3779B1u;
      const uint32_t hstep = (uint32_t)((size_t)A_STEP * P.ncol) * 0x9E3779B1u;
#pragma unroll 4
      for (int a = a_first; a < N; a += A_STEP, hsh += hstep) {
        const double2 v = Tp[(size_t)perm_s[a] * NT];
        const size_t idx = (size_t)a * P.ncol;
        o[idx] = v;
        if (om)
          om[idx] = make_double2(__longlong_as_double(__double_as_longlong(v.x) ^ fr),
                                 __longlong_as_double(__double_as_longlong(v.y) ^ fi));
        const double a2 = fma(v.x, v.x, v.y * v.y);
        s2 += a2;
        mx2 = max(mx2, __double_as_longlong(a2));
        const double wgt = digest_weight(hsh);
        pr = fma(wgt, v.x, pr);
        pi = fma(wgt, v.y, pi);
        ir += v.x;
        ii += v.y;
        if (a == 0 && col == 0) {
          g0r = v.x;
          g0i = v.y;
        }
      }
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
  }
}

}  // namespace slsht_cuda
