// Fused coupling for n = 49 (config 4): the k_tgemm GEMM, the alpha FFT and the store/digest
// epilogue of the two-pass path (kernels_twopass.cuh) in ONE kernel, so T never leaves the SM.
//
// Why: the two-pass path writes T (16 B per sample) to HBM and reads it back, 2 x 277 GB per
// config-4 step on top of the 277 GB of volumes. Keeping T in shared memory leaves only the
// volume stream on HBM.
//
// Shape (persistent CTA, one per SM, 227 KB of shared memory):
//   * a work unit is one group of MT = 8 components; the CTA walks ALL column tiles
//     (NT = 16 columns) of its group, so the group's U block (8 x KR complex) is loaded once
//     and stays resident;
//   * the T rows (q mod n) are split into G = 7 row groups of 7 rows (rows j + 7 k), whose
//     k-step counts are equal (25 each); the K layout INTERLEAVES them: stage s (28 K rows)
//     holds k-step s of every row group. So every stage gives every MMA warp exactly one
//     k-step (no warp gates the ring with a long q), and consecutive k-steps of one warp are a
//     whole stage apart (no DMMA latency chain);
//   * the window table W ([ct][KR][16], columns XOR-swizzled by the K row: conflict-free B
//     fragments without padding) streams through an R-slot ring, one cp.async.bulk per stage,
//     mbarrier full/empty pairs. The producer is lane 0 of the last warp, which has no MMA
//     work: during the MMA phase it issues the tile's remaining stages, then the next tile's
//     first R stages (and at a group's end the next group's U block), which land during this
//     tile's FFT (16 warps in all: 128 registers per thread);
//   * 14 MMA warps = (row group j, 8-column subtile); Gauss 3-product DMMA chains as k_tgemm;
//     a completed row goes to the shared T tile [8][n][NT];
//   * then the first DIF stage (radix 7) in shared memory, and the last stage fused with the
//     epilogue: each butterfly's 7 outputs are stored straight to the So3Volume rows (two
//     256-B row segments per warp store), the real-mode mirror, and the digest partials of
//     (component, tile, half) by a fixed shuffle tree, reduced over the tiles in order by
//     k_digest: bitwise independent of the traversal order, the chunking and the sharding;
//   * each group starts at its own column tile (ct0 = 5 g mod nct) and wraps around, so the
//     CTAs in flight read different W tiles.
#pragma once

#include "common.cuh"
#include "fft_radix.cuh"
#include "kernels_couple.cuh"
#include "kernels_couple_lines.cuh"
#include "kernels_couple_ws.cuh"

namespace slsht_cuda {

template <int N>
struct FuCfg {
  static constexpr int L = (N - 1) / 2;
  static constexpr int MT = 8, NT = 16;
  static constexpr int R1 = smallest_prime_factor(N);  // first DIF radix
  static constexpr int G = N / R1;                      // row groups (rows j + G k)
  static constexpr int KSR = 4 * G;                     // K rows per stage
  static constexpr int NCW = 16;                        // warps (2 G of them do MMA)
  static constexpr int NMW = 2 * G;
  static constexpr int NTHREADS = NCW * 32;
  static constexpr int EPW = NCW / MT;                  // epilogue warps per component
  static constexpr int RLAST = N / R1;                  // last DIF radix (N = R1 x RLAST)
  static constexpr int np(int r) {                      // (p, q) rows of T row r = q mod N
    const int q = r <= L ? r : r - N;
    return L + 1 - (q < 0 ? -q : q);
  }
  static constexpr int ksteps(int j) {
    int s = 0;
    for (int k = 0; k < R1; ++k) s += (np(j + G * k) + 3) / 4;
    return s;
  }
  static constexpr int NST = []() constexpr {  // stages per tile: the longest row group
    int m = 0;
    for (int j = 0; j < G; ++j) m = ksteps(j) > m ? ksteps(j) : m;
    return m;
  }();
  static constexpr int KR = NST * KSR;                           // K rows
  static constexpr int UPAD = KR + ((4 - KR) % 8 + 8) % 8;       // == 4 mod 8
  static constexpr int R = 5;                                    // W ring slots
  static constexpr size_t U_BYTES = (size_t)MT * UPAD * 16;
  static constexpr size_t T_BYTES = (size_t)MT * N * NT * 16;
  static constexpr size_t WS_BYTES = (size_t)KSR * NT * 16;
  static constexpr size_t OFF_T = U_BYTES;
  static constexpr size_t OFF_W = OFF_T + T_BYTES;
  static constexpr size_t OFF_TAB = OFF_W + R * WS_BYTES;
  // rou[N] double2 | betaw[L+1] double | kend[NST][G] signed char (T row completed, -1) |
  // kval[NST][G] unsigned char
  static constexpr size_t TAB_BYTES = (size_t)N * 16 + (size_t)(L + 1) * 8 + (size_t)NST * G * 2;
  static constexpr size_t OFF_BAR = (OFF_TAB + TAB_BYTES + 15) / 16 * 16;
  static constexpr int NBAR = 2 + 2 * R;
  static constexpr size_t SMEM = OFF_BAR + NBAR * 8;
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(NMW < NCW, "MMA warps, and a warp without MMA work for the producer");
  static_assert(RLAST * R1 == N, "two DIF stages");
  static_assert(NST <= 32, "per-warp stage masks");
};

// W column swizzle inside a 16-column tile: the 8 lanes of a B-fragment quarter-warp
// (k = lane % 4, column = lane / 4) hit 8 distinct 16-B bank groups.
__host__ __device__ __forceinline__ int fu_wswz(int col, int krow) {
  return (col & 8) | ((col & 7) ^ ((2 * krow) & 7));
}

struct FuParams {
  const double2* U;     // [group][MT][UPAD] (k_modgemm group layout, zero padding)
  const double2* W;     // [ct][KR][16] (fu_wswz columns)
  double2* out;
  double* partials;     // [comp][column tile][EPW][8] digest partials (k_digest)
  const CompRec* comps;
  int count, n_groups, n_col_tiles, ncol;
  long long vol;
  int mirror;
  const double2* rou;
  const double* betaw;
  const signed char* kend;       // [stage][row group]: T row completed by the k-step, or -1
  const unsigned char* kval;     // [stage][row group]: 1 if the k-step exists
};

template <int N>
__global__ void __launch_bounds__(FuCfg<N>::NTHREADS, 1) k_fused(const FuParams P) {
  using Cfg = FuCfg<N>;
  constexpr int L = Cfg::L, MT = Cfg::MT, NT = Cfg::NT, KSR = Cfg::KSR, G = Cfg::G;
  constexpr int NST = Cfg::NST, UPAD = Cfg::UPAD, R = Cfg::R, NCW = Cfg::NCW;
  constexpr int NMW = Cfg::NMW, EPW = Cfg::EPW, R1 = Cfg::R1, RL = Cfg::RLAST;
  constexpr int NC = NCW * 32;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* Us = reinterpret_cast<double2*>(smem);
  double2* T = reinterpret_cast<double2*>(smem + Cfg::OFF_T);
  double2* Wr = reinterpret_cast<double2*>(smem + Cfg::OFF_W);
  double2* rou_s = reinterpret_cast<double2*>(smem + Cfg::OFF_TAB);
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  signed char* kend_s = reinterpret_cast<signed char*>(betaw_s + (L + 1));
  unsigned char* kval_s = reinterpret_cast<unsigned char*>(kend_s + NST * G);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* ufull = bars + 0;
  uint64_t* uempty = bars + 1;
  uint64_t* wfull = bars + 2;       // [R]
  uint64_t* wempty = bars + 2 + R;  // [R]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nct = P.n_col_tiles;
  constexpr size_t WE = Cfg::WS_BYTES / 16;

  for (int i = tid; i < N; i += Cfg::NTHREADS) rou_s[i] = P.rou[i];
  for (int i = tid; i <= L; i += Cfg::NTHREADS) betaw_s[i] = P.betaw[i];
  for (int i = tid; i < NST * G; i += Cfg::NTHREADS) {
    kend_s[i] = P.kend[i];
    kval_s[i] = P.kval[i];
  }
  if (tid == 0) {
    mbar_init(ufull, 1);
    mbar_init(uempty, NMW);
    for (int s = 0; s < R; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], NMW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // ---------------------------------------------------------------- producer (one thread)
  const bool producer = warp == NCW - 1 && lane == 0;
  int psl = 0;        // producer ring position: slot and phase parity
  uint32_t pph = 0;
  auto issue_w = [&](int ct, int s0) {
    mbar_wait(&wempty[psl], pph ^ 1);
    constexpr uint32_t wb = (uint32_t)Cfg::WS_BYTES;
    mbar_arrive_expect_tx(&wfull[psl], wb);
    bulk_g2s(Wr + psl * WE, P.W + ((size_t)ct * Cfg::KR + (size_t)s0 * KSR) * NT, wb, &wfull[psl]);
    if (++psl == R) {
      psl = 0;
      pph ^= 1;
    }
  };
  uint32_t pu_phase = 0;
  auto issue_u = [&](int g) {
    mbar_wait(uempty, pu_phase ^ 1);
    constexpr uint32_t ub = (uint32_t)Cfg::U_BYTES;
    mbar_arrive_expect_tx(ufull, ub);
    bulk_g2s(Us, P.U + (size_t)g * MT * UPAD, ub, ufull);
    pu_phase ^= 1;
  };
  constexpr int PRE = R < NST ? R : NST;  // stages of a tile issued before its MMA phase
  if (producer && (int)blockIdx.x < P.n_groups) {
    issue_u(blockIdx.x);
    for (int s0 = 0; s0 < PRE; ++s0) issue_w((5 * blockIdx.x) % nct, s0);
  }
  __syncwarp();

  // -------------------------------------------------------------------- compute warps
  const int c_tid = tid, cw = warp;
  const bool mma_warp = cw < NMW;
  const int jg = cw >> 1, st = cw & 1;  // MMA: row group, 8-column subtile
  const int kl = lane & 3, ar = lane >> 2;
  // B fragment: stage row jg*4 + kl (== global K row mod 8), swizzled column st*8 + ar
  const int boff = (jg * 4 + kl) * NT + fu_wswz(st * 8 + ar, jg * 4 + kl);
  // epilogue (last DIF stage): warp cw = (component ec, half eh); lane = (column cc, sub)
  const int ec = cw / EPW, eh = cw % EPW;
  const int cc = lane & 15, sub = lane >> 4;
  uint32_t uphase = 0;
  int sl = 0;  // consumer ring position: slot and phase parity
  uint32_t ph = 0;
  auto advance = [&]() {
    if (++sl == R) {
      sl = 0;
      ph ^= 1;
    }
  };
  // this warp's row group as bit masks over the stages: k-step present, row completed (the
  // group's rows complete in order jg, jg + G, ..., so the e-th completion is row jg + G e)
  uint32_t vmask = 0, emask = 0;
  if (mma_warp)
    for (int s0 = 0; s0 < NST; ++s0) {
      vmask |= (uint32_t)(kval_s[s0 * G + jg] != 0) << s0;
      emask |= (uint32_t)(kend_s[s0 * G + jg] >= 0) << s0;
    }
  const long long sbit = (long long)0x8000000000000000ULL;
  for (int g = blockIdx.x; g < P.n_groups; g += gridDim.x) {
    const int ncomp = min(MT, P.count - g * MT);
    const bool cact = ec < ncomp;
    CompRec rec{0, 0, 0, -1};
    if (cact) rec = P.comps[g * MT + ec];
    double2* o = P.out + rec.slot * P.vol;
    const bool mir = cact && P.mirror && rec.m > 0;
    double2* om = mir ? P.out + rec.mslot * P.vol : nullptr;
    const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
    if (mma_warp) {
      mbar_wait(ufull, uphase);
      uphase ^= 1;
    }
    const double2* Ua = Us + ar * UPAD + jg * 4 + kl;
    for (int i = 0, ct = (5 * g) % nct; i < nct; ++i, ct = (ct + 1 == nct) ? 0 : ct + 1) {
      if (mma_warp) {
        // ---- MMA: one k-step of row group jg per stage, stages taken in pairs with one
        // accumulator set per stage parity (independent DMMA chains), summed at a row's end
        double c1[2][2] = {}, c2[2][2] = {}, c3[2][2] = {};
        int e = 0;  // rows completed
        auto row_end = [&]() {
          double2* dst = T + ((size_t)ar * N + jg + G * e) * NT + st * 8 + 2 * kl;
#pragma unroll
          for (int x = 0; x < 2; ++x) {
            const double k1 = c1[0][x] + c1[1][x], k2 = c2[0][x] + c2[1][x];
            const double k3 = c3[0][x] + c3[1][x];
            dst[x] = make_double2(k1 - k3, k1 + k2);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
            c1[h][0] = c1[h][1] = c2[h][0] = c2[h][1] = c3[h][0] = c3[h][1] = 0.0;
          ++e;
        };
        for (int s0 = 0; s0 < NST; s0 += 2) {
          const bool two = s0 + 1 < NST;
          const int sl0 = sl;
          const uint32_t ph0 = ph;
          advance();
          const int sl1 = sl;
          const uint32_t ph1 = ph;
          if (two) advance();
          mbar_wait(&wfull[sl0], ph0);
          if (two) mbar_wait(&wfull[sl1], ph1);
          const bool v0 = (vmask >> s0) & 1u, v1 = two && ((vmask >> (s0 + 1)) & 1u);
          double2 a0 = make_double2(0.0, 0.0), b0 = a0, a1 = a0, b1 = a0;
          if (v0) {
            a0 = Ua[s0 * KSR];
            b0 = Wr[sl0 * WE + boff];
          }
          if (v1) {
            a1 = Ua[(s0 + 1) * KSR];
            b1 = Wr[sl1 * WE + boff];
          }
          if (v0) {
            dmma(c1[0][0], c1[0][1], a0.x + a0.y, b0.x);
            dmma(c2[0][0], c2[0][1], a0.x, b0.y - b0.x);
            dmma(c3[0][0], c3[0][1], a0.y, b0.x + b0.y);
            if ((emask >> s0) & 1u) row_end();
          }
          if (v1) {
            dmma(c1[1][0], c1[1][1], a1.x + a1.y, b1.x);
            dmma(c2[1][0], c2[1][1], a1.x, b1.y - b1.x);
            dmma(c3[1][0], c3[1][1], a1.y, b1.x + b1.y);
            if ((emask >> (s0 + 1)) & 1u) row_end();
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&wempty[sl0]);
            if (two) mbar_arrive(&wempty[sl1]);
          }
        }
        if (i == nct - 1 && lane == 0) mbar_arrive(uempty);  // the group's last MMA is done
      } else if (producer) {
        // the rest of this tile's stages, then the next tile's first ones (at the group's end:
        // the next group's U block first, once every MMA warp is done with this one)
        for (int s0 = PRE; s0 < NST; ++s0) issue_w(ct, s0);
        if (i + 1 < nct) {
          const int nx = (ct + 1 == nct) ? 0 : ct + 1;
          for (int s0 = 0; s0 < PRE; ++s0) issue_w(nx, s0);
        } else if (g + (int)gridDim.x < P.n_groups) {
          const int g2 = g + gridDim.x;
          issue_u(g2);
          for (int s0 = 0; s0 < PRE; ++s0) issue_w((5 * g2) % nct, s0);
        }
      }
      __syncwarp();  // the producer lane rejoins its warp before the aligned barrier
      named_sync(1, NC);
      // ---- first DIF stage (radix R1, span N) in shared memory
      fft_stage_ct<N, R1, N, NT, MT * NT, NC>(T, rou_s, c_tid);
      named_sync(1, NC);
      // ---- last DIF stage (radix RL, no twiddles) fused with the epilogue: block b holds
      // frequencies a0(b) + k N/RL; warp (ec, eh), lane (cc, sub): blocks b = 2 eh + sub + 4 i
      const int col = ct * NT + cc;
      double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
      long long mx2 = 0;
      const bool ok = cact && col < P.ncol;
      const double qb = ok ? betaw_s[col / N] : 0.0;
#pragma unroll
      for (int bi = 0; bi < (R1 + 3) / 4; ++bi) {
        const int b = 2 * eh + sub + 4 * bi;
        if (b >= R1) continue;
        double2* base = T + ((size_t)ec * N + b * RL) * NT + cc;
        double xr[RL], xi[RL];
#pragma unroll
        for (int k = 0; k < RL; ++k) {
          const double2 v = base[k * NT];
          xr[k] = v.x;
          xi[k] = v.y;
        }
        Radix<RL>::dft(xr, xi);
        if (!ok) continue;
        const int a0 = dif_last_freq0<N, RL>(b);
#pragma unroll
        for (int k = 0; k < RL; ++k) {
          const int a = a0 + k * (N / RL);
          const double vx = xr[k], vy = xi[k];
          const size_t idx = (size_t)a * P.ncol + col;
          __stcs(o + idx, make_double2(vx, vy));
          if (mir) {
            const long long br = __double_as_longlong(vx) ^ mflip_r;
            const long long bim = __double_as_longlong(vy) ^ mflip_i;
            __stcs(om + idx, make_double2(__longlong_as_double(br), __longlong_as_double(bim)));
          }
          const double a2 = fma(vx, vx, vy * vy);
          s2 += a2;
          mx2 = max(mx2, __double_as_longlong(a2));
          const double wgt = digest_weight((uint32_t)idx * 0x9E3779B1u);
          pr = fma(wgt, vx, pr);
          pi = fma(wgt, vy, pi);
          ir = fma(qb, vx, ir);
          ii = fma(qb, vy, ii);
          if (a == 0 && col == 0) {
            g0r = vx;
            g0i = vy;
          }
        }
      }
      // digest partial of (component ec, tile ct, half eh): fixed shuffle tree
      double v[8] = {s2, __longlong_as_double(mx2), pr, pi, g0r, g0i, ir, ii};
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const double x = __shfl_down_sync(0xffffffffu, v[f], off);
          v[f] = (f == 1) ? fmax(v[f], x) : v[f] + x;
        }
      if (lane == 0 && cact) {
        double* part = P.partials + (((size_t)(g * MT + ec) * nct + ct) * EPW + eh) * 8;
#pragma unroll
        for (int f = 0; f < 8; ++f) part[f] = v[f];
      }
      named_sync(1, NC);  // T is rewritten by the next tile's MMA
    }
  }
}

}  // namespace slsht_cuda
