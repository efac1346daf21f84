// Fused coupling for n = 49 (config 4): the k_tgemm GEMM, the alpha FFT and the store/digest
// epilogue of the two-pass path (kernels_twopass.cuh) in ONE persistent kernel, so T never
// leaves the SM. The two-pass path writes T (16 B per sample) to HBM and reads it back,
// 2 x 277 GB per config-4 step on top of the 277 GB of volumes; here only the volume stream
// reaches HBM, and the kernel is bound by the FP64 pipe (DMMA and DFMA share it) and the L2
// (the window table streams through every SM).
//
// One CTA per SM, 16 warps, three roles that overlap through mbarriers:
//   * producer (warp 15, one lane): the group's U block (8 components x KR complex, resident
//     for all its column tiles) and, per tile, the NST stages of the window table W ([ct][KR]
//     [8], columns XOR-swizzled by the K row: conflict-free B fragments) through an R-slot
//     ring of cp.async.bulk copies (full/empty mbarrier pairs);
//   * 7 MMA warps, one per row group j of a tile of 8 components x 8 columns. The T rows
//     r = q mod n split into G = 7 row groups of 7 rows (rows j + 7 e); the K layout
//     interleaves the groups (stage s holds k-step s of every group), so each stage gives each
//     warp one k-step (three Gauss DMMA chains). A warp's finished rows stay in registers, and
//     the FIRST DIF STAGE of the alpha FFT (the radix-7 butterfly over rows j + 7 e, twiddled
//     by w^(j k)) runs there: the warp writes only its 7 butterfly outputs (rows j + 7 k) to
//     the T tile, then goes on to the next tile;
//   * 8 epilogue warps, one per component: the last DIF stage (radix 7 over rows 7 b ..
//     7 b + 6, frequencies b + 7 k), the stores of the So3Volume rows (in the pitched ring
//     every row starts on a 128-B line, and the 8 lanes of a block write one whole line), the
//     real-mode mirror, and the digest partial of (component, column tile) by a fixed shuffle
//     tree, reduced over the tiles in order by k_digest: bitwise independent of the traversal
//     order, the chunking and the sharding.
// The T tile is double-buffered, so the epilogue of tile i runs under the MMA of tile i + 1.
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
  static constexpr int MT = 8, NT = 8;
  static constexpr int R1 = smallest_prime_factor(N);  // first DIF radix
  static constexpr int G = N / R1;                      // row groups (rows j + G e)
  static constexpr int RLAST = N / R1;                  // last DIF radix (N = R1 x RLAST)
  static constexpr int KSR = 4 * G;                     // K rows per stage
  static constexpr int NMW = G;                         // MMA warps
  static constexpr int NEW = MT;                        // epilogue warps (one per component)
  static constexpr int NWARPS = NMW + NEW + 1;          // + the producer warp
  static constexpr int NTHREADS = NWARPS * 32;
  static constexpr int EPW = 1;                         // digest partials per (comp, tile)
  static constexpr int np(int r) {                      // (p, q) rows of T row r = q mod N
    const int q = r <= L ? r : r - N;
    return L + 1 - (q < 0 ? -q : q);
  }
  static constexpr int nks(int j, int e) { return (np(j + G * e) + 3) / 4; }
  static constexpr int ksteps(int j) {
    int s = 0;
    for (int e = 0; e < R1; ++e) s += nks(j, e);
    return s;
  }
  static constexpr int NST = []() constexpr {  // stages per tile: the longest row group
    int m = 0;
    for (int j = 0; j < G; ++j) m = ksteps(j) > m ? ksteps(j) : m;
    return m;
  }();
  static constexpr int KR = NST * KSR;                           // K rows
  static constexpr int UPAD = KR + ((4 - KR) % 8 + 8) % 8;       // == 4 mod 8
  static constexpr int NTB = 1;                                  // T buffers
  static constexpr int R = 20;                                   // W ring slots
  static constexpr size_t U_BYTES = (size_t)MT * UPAD * 16;
  // T tile [component][row][NT], component stride N NT + 1 (16-B units): the MMA warps' stores
  // (8 components x 4 column pairs per warp) and the epilogue loads hit 8 distinct bank groups
  static constexpr int TCS = N * NT + 1;
  static constexpr size_t T_BYTES = ((size_t)MT * TCS * 16 + 127) / 128 * 128;  // per buffer
  static constexpr size_t WS_BYTES = (size_t)KSR * NT * 16;
  static constexpr size_t OFF_T = U_BYTES;
  static constexpr size_t OFF_W = OFF_T + NTB * T_BYTES;
  static constexpr size_t OFF_TAB = OFF_W + R * WS_BYTES;
  // rou[N] double2 | betaw[L+1] double
  static constexpr size_t TAB_BYTES = (size_t)N * 16 + (size_t)(L + 1) * 8;
  static constexpr size_t OFF_BAR = (OFF_TAB + TAB_BYTES + 15) / 16 * 16;
  static constexpr int NBAR = 6 + 2 * R;
  static constexpr size_t SMEM = OFF_BAR + NBAR * 8;
  static_assert(SMEM <= 232448, "shared memory budget");
  static_assert(RLAST * R1 == N && RLAST == G, "two DIF stages of the same radix");
  static_assert(RLAST <= 8 && 4 * NT == 32, "epilogue lanes: 8 columns x 4 first blocks");
};

// W column swizzle inside an 8-column tile: the 8 lanes of a B-fragment quarter-warp
// (k = lane % 4, column = lane / 4) hit 8 distinct 16-B bank groups.
__host__ __device__ __forceinline__ int fu_wswz(int col, int krow) {
  return (col & 7) ^ ((2 * krow) & 7);
}

struct FuParams {
  const double2* U;     // [group][MT][UPAD] (k_modgemm group layout, zero padding)
  const double2* W;     // [ct][KR][NT] (fu_wswz columns)
  double2* out;
  double* partials;     // [comp][column tile][8] digest partials (k_digest)
  const CompRec* comps;
  int count, n_groups, n_col_tiles, ncol;
  long long vol;        // slot stride of out (complex elements)
  int rpitch;           // row stride of out (ncol, or ncol rounded to whole lines in the ring)
  int mirror;
  const double2* rou;
  const double* betaw;
  int exp;  // experiments (SLSHT_CUDA_FU_EXP): 1 = epilogue only releases T, 2 = no DMMA
};

// The MMA of one tile for the warp's row group: every stage s < NST waits for W slot
// (sl, ph), reads its k-step's A (resident U) and B (ring) fragments and issues the three
// Gauss DMMA chains, stages taken in pairs. Rows finish in order e = 0..R1-1 (nks: 4 bits of
// k-steps each); each
// finished row is shifted into res[R1 - 1] (the older rows move down), so after the last row
// res[e] holds row e with static register indexing and a compact (not unrolled) stage loop.
// res[e][x]: the lane's component lane / 4, column 2 (lane % 4) + x.
template <int N>
__device__ __forceinline__ void fu_mma_rows(const double2* __restrict__ Ua,
                                            const double2* __restrict__ Wb, uint64_t* wfull,
                                            uint64_t* wempty, int& sl, uint32_t& ph, int lane,
                                            uint32_t nks, int nst_own,
                                            double2 (&res)[FuCfg<N>::R1][2], bool nomma) {
  using Cfg = FuCfg<N>;
  constexpr int KSR = Cfg::KSR, R = Cfg::R, R1 = Cfg::R1;
  constexpr size_t WE = Cfg::WS_BYTES / 16;
  const double2* ua = Ua;
  auto next = [&]() {
    if (++sl == R) {
      sl = 0;
      ph ^= 1;
    }
  };
#pragma unroll 1
  for (int e = 0; e < R1; ++e) {
    // two accumulator sets (k-steps of even / odd position in the row): six independent DMMA
    // chains per pair of stages, summed at the row's end in a fixed order
    double c1[2][2] = {}, c2[2][2] = {}, c3[2][2] = {};
    const int nk = (nks >> (4 * e)) & 15;
    int k = 0;
#pragma unroll 1
    for (; k + 1 < nk; k += 2, ua += 2 * KSR) {
      const int sl0 = sl;
      const uint32_t ph0 = ph;
      next();
      const int sl1 = sl;
      const uint32_t ph1 = ph;
      next();
      mbar_wait(&wfull[sl0], ph0);
      mbar_wait(&wfull[sl1], ph1);
      const double2 a0 = ua[0], a1 = ua[KSR];
      const double2 b0 = Wb[sl0 * WE], b1 = Wb[sl1 * WE];
      if (!nomma) {
      dmma(c1[0][0], c1[0][1], a0.x + a0.y, b0.x);
      dmma(c2[0][0], c2[0][1], a0.x, b0.y - b0.x);
      dmma(c3[0][0], c3[0][1], a0.y, b0.x + b0.y);
      dmma(c1[1][0], c1[1][1], a1.x + a1.y, b1.x);
      dmma(c2[1][0], c2[1][1], a1.x, b1.y - b1.x);
      dmma(c3[1][0], c3[1][1], a1.y, b1.x + b1.y);
      } else {
        c1[0][0] += a0.x * b0.x + a1.x * b1.y;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&wempty[sl0]);
        mbar_arrive(&wempty[sl1]);
      }
    }
    if (k < nk) {
      mbar_wait(&wfull[sl], ph);
      const double2 a = ua[0];
      const double2 b = Wb[sl * WE];
      dmma(c1[0][0], c1[0][1], a.x + a.y, b.x);
      dmma(c2[0][0], c2[0][1], a.x, b.y - b.x);
      dmma(c3[0][0], c3[0][1], a.y, b.x + b.y);
      __syncwarp();
      if (lane == 0) mbar_arrive(&wempty[sl]);
      next();
      ua += KSR;
    }
#pragma unroll
    for (int r = 0; r < R1 - 1; ++r) {
      res[r][0] = res[r + 1][0];
      res[r][1] = res[r + 1][1];
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const double k1 = c1[0][x] + c1[1][x], k2 = c2[0][x] + c2[1][x], k3 = c3[0][x] + c3[1][x];
      res[R1 - 1][x] = make_double2(k1 - k3, k1 + k2);
    }
  }
  // stages past this group's k-steps (none at n = 49): release the slots
#pragma unroll 1
  for (int s = nst_own; s < Cfg::NST; ++s) {
    mbar_wait(&wfull[sl], ph);
    __syncwarp();
    if (lane == 0) mbar_arrive(&wempty[sl]);
    if (++sl == R) {
      sl = 0;
      ph ^= 1;
    }
  }
}

template <int N>
__global__ void __launch_bounds__(FuCfg<N>::NTHREADS, 1) k_fused(const FuParams P) {
  using Cfg = FuCfg<N>;
  constexpr int L = Cfg::L, MT = Cfg::MT, NT = Cfg::NT, KSR = Cfg::KSR, G = Cfg::G;
  constexpr int NST = Cfg::NST, UPAD = Cfg::UPAD, R = Cfg::R, R1 = Cfg::R1;
  constexpr int NMW = Cfg::NMW, NEW = Cfg::NEW, RL = Cfg::RLAST, TCS = Cfg::TCS;
  extern __shared__ __align__(128) unsigned char smem[];
  double2* Us = reinterpret_cast<double2*>(smem);
  double2* Tb = reinterpret_cast<double2*>(smem + Cfg::OFF_T);  // [2][T_BYTES / 16]
  double2* Wr = reinterpret_cast<double2*>(smem + Cfg::OFF_W);
  double2* rou_s = reinterpret_cast<double2*>(smem + Cfg::OFF_TAB);
  double* betaw_s = reinterpret_cast<double*>(rou_s + N);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint64_t* ufull = bars + 0;
  uint64_t* uempty = bars + 1;
  uint64_t* tfull = bars + 2;       // [2]
  uint64_t* tempty = bars + 4;      // [2]
  uint64_t* wfull = bars + 6;       // [R]
  uint64_t* wempty = bars + 6 + R;  // [R]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nct = P.n_col_tiles;
  constexpr size_t WE = Cfg::WS_BYTES / 16;
  constexpr size_t TE = Cfg::T_BYTES / 16;

  for (int i = tid; i < N; i += Cfg::NTHREADS) rou_s[i] = P.rou[i];
  for (int i = tid; i <= L; i += Cfg::NTHREADS) betaw_s[i] = P.betaw[i];
  if (tid == 0) {
    mbar_init(ufull, 1);
    mbar_init(uempty, NMW);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], NMW);
      mbar_init(&tempty[b], NEW);
    }
    for (int s = 0; s < R; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], NMW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto ct_first = [&](int g) { return (5 * g) % nct; };

  if (warp == NMW + NEW) {
    // ------------------------------------------------------------------ producer (one lane)
    if (lane != 0) return;
    int sl = 0;
    uint32_t ph = 0, uph = 0;
    for (int g = blockIdx.x; g < P.n_groups; g += gridDim.x) {
      mbar_wait(uempty, uph ^ 1);
      uph ^= 1;
      mbar_arrive_expect_tx(ufull, (uint32_t)Cfg::U_BYTES);
      bulk_g2s(Us, P.U + (size_t)g * MT * UPAD, (uint32_t)Cfg::U_BYTES, ufull);
      for (int i = 0, ct = ct_first(g); i < nct; ++i, ct = (ct + 1 == nct) ? 0 : ct + 1) {
        for (int s = 0; s < NST; ++s) {
          mbar_wait(&wempty[sl], ph ^ 1);
          mbar_arrive_expect_tx(&wfull[sl], (uint32_t)Cfg::WS_BYTES);
          bulk_g2s(Wr + sl * WE, P.W + ((size_t)ct * Cfg::KR + (size_t)s * KSR) * NT,
                   (uint32_t)Cfg::WS_BYTES, &wfull[sl]);
          if (++sl == R) {
            sl = 0;
            ph ^= 1;
          }
        }
      }
    }
    return;
  }

  if (warp < NMW) {
    // ------------------------------------------------------------------ MMA warps
    const int jg = warp;
    const int kl = lane & 3, ar = lane >> 2;
    // A fragment: U row (stage s, group jg, k = kl) of component ar; B fragment: stage row
    // jg*4 + kl, swizzled column ar
    const double2* Ua = Us + ar * UPAD + jg * 4 + kl;
    const double2* Wb = Wr + (jg * 4 + kl) * NT + fu_wswz(ar, jg * 4 + kl);
    uint32_t nks = 0;  // this row group's k-steps per row, 4 bits each
    int nst_own = 0;
#pragma unroll
    for (int e = 0; e < R1; ++e) {
      const int k = (Cfg::np(jg + G * e) + 3) / 4;
      nks |= (uint32_t)k << (4 * e);
      nst_own += k;
    }
    int sl = 0;
    uint32_t ph = 0, uph = 0, tph[2] = {0, 0};
    int tb = 0;  // T buffer of the tile
    for (int g = blockIdx.x; g < P.n_groups; g += gridDim.x) {
      mbar_wait(ufull, uph);
      uph ^= 1;
      for (int i = 0; i < nct; ++i) {
        double2 res[R1][2];
        fu_mma_rows<N>(Ua, Wb, wfull, wempty, sl, ph, lane, nks, nst_own, res, P.exp & 2);
        if (i == nct - 1 && lane == 0) mbar_arrive(uempty);  // the group's last MMA is done
        // first DIF stage (radix R1, span N) on the warp's rows jg + G e: y_k = sum_e x_e
        // w_R1^(e k), twiddled by w_N^(jg k), to row jg + G k of T buffer tb once it is free
        mbar_wait(&tempty[tb], tph[tb] ^ 1);
        tph[tb] ^= 1;
        double2* Tl = Tb + tb * TE + (size_t)ar * TCS + 2 * kl;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          double xr[R1], xi[R1];
#pragma unroll
          for (int e = 0; e < R1; ++e) {
            xr[e] = res[e][x].x;
            xi[e] = res[e][x].y;
          }
          Radix<R1>::dft(xr, xi);
          Tl[(size_t)jg * NT + x] = make_double2(xr[0], xi[0]);
#pragma unroll
          for (int k = 1; k < R1; ++k) {
            const double2 w = rou_s[jg * k];
            Tl[(size_t)(jg + G * k) * NT + x] =
                make_double2(xr[k] * w.x - xi[k] * w.y, xr[k] * w.y + xi[k] * w.x);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&tfull[tb]);
        tb = (tb + 1 == Cfg::NTB) ? 0 : tb + 1;
      }
    }
    return;
  }

  // -------------------------------------------------------------------- epilogue warps
  // warp = component ec; lane = (column cc = lane % 8, first block b0 = lane / 8): blocks b0
  // and b0 + 4 (when < RL) of the last DIF stage of its column
  const int ec = warp - NMW;
  const int cc = lane & 7, b0 = lane >> 3;
  const bool two = b0 + 4 < RL;
  const long long sbit = (long long)0x8000000000000000ULL;
  uint32_t tph[2] = {0, 0};
  int tb = 0;
  for (int g = blockIdx.x; g < P.n_groups; g += gridDim.x) {
    const int ncomp = min(MT, P.count - g * MT);
    const bool cact = ec < ncomp;
    CompRec rec{0, 0, 0, -1};
    if (cact) rec = P.comps[g * MT + ec];
    double2* o = P.out + rec.slot * P.vol;
    const bool mir = cact && P.mirror && rec.m > 0;
    double2* om = mir ? P.out + rec.mslot * P.vol : nullptr;
    const long long mflip_r = (rec.m & 1) ? sbit : 0, mflip_i = (rec.m & 1) ? 0 : sbit;
    for (int i = 0, ct = ct_first(g); i < nct; ++i, ct = (ct + 1 == nct) ? 0 : ct + 1) {
      mbar_wait(&tfull[tb], tph[tb]);
      tph[tb] ^= 1;
      // both blocks' inputs to registers, then the buffer goes back to the MMA warps
      const double2* base = Tb + tb * TE + (size_t)ec * TCS + cc;
      double xr[2][RL], xi[2][RL];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int k = 0; k < RL; ++k) {
          const int b = b0 + 4 * u;
          double2 v = make_double2(0.0, 0.0);
          if (u == 0 || two) v = base[(size_t)(b * RL + k) * NT];
          xr[u][k] = v.x;
          xi[u][k] = v.y;
        }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[tb]);
      tb = (tb + 1 == Cfg::NTB) ? 0 : tb + 1;
      if (P.exp & 1) continue;
      const int col = ct * NT + cc;
      const bool ok = cact && col < P.ncol;        // a sample of the volume
      const bool st_ok = cact && col < P.rpitch;   // a position of the (pitched) row
      const double qb = ok ? betaw_s[col / N] : 0.0;
      double s2 = 0.0, pr = 0.0, pi = 0.0, ir = 0.0, ii = 0.0, g0r = 0.0, g0i = 0.0;
      long long mx2 = 0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && !two) break;
        const int b = b0 + 4 * u;
        Radix<RL>::dft(xr[u], xi[u]);
        const int a0 = dif_last_freq0<N, RL>(b);
#pragma unroll
        for (int k = 0; k < RL; ++k) {
          const int a = a0 + k * (N / RL);
          const double vx = xr[u][k], vy = xi[u][k];
          const size_t pos = (size_t)a * P.rpitch + col;
          if (st_ok) {
            __stcs(o + pos, make_double2(vx, vy));
            if (mir) {
              const long long br = __double_as_longlong(vx) ^ mflip_r;
              const long long bim = __double_as_longlong(vy) ^ mflip_i;
              __stcs(om + pos, make_double2(__longlong_as_double(br), __longlong_as_double(bim)));
            }
          }
          if (ok) {
            const double a2 = fma(vx, vx, vy * vy);
            s2 += a2;
            mx2 = max(mx2, __double_as_longlong(a2));
            const double wgt = digest_weight((uint32_t)((size_t)a * P.ncol + col) * 0x9E3779B1u);
            pr = fma(wgt, vx, pr);
            pi = fma(wgt, vy, pi);
            ir += vx;
            ii += vy;
            if (a == 0 && col == 0) {
              g0r = vx;
              g0i = vy;
            }
          }
        }
      }
      ir *= qb;
      ii *= qb;
      // digest partial of (component ec, tile ct): fixed shuffle tree over the warp
      double v[8] = {s2, __longlong_as_double(mx2), pr, pi, g0r, g0i, ir, ii};
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int f = 0; f < 8; ++f) {
          const double x = __shfl_down_sync(0xffffffffu, v[f], off);
          v[f] = (f == 1) ? fmax(v[f], x) : v[f] + x;
        }
      if (lane == 0 && cact) {
        double* part = P.partials + ((size_t)(g * MT + ec) * nct + ct) * 8;
#pragma unroll
        for (int f = 0; f < 8; ++f) part[f] = v[f];
      }
    }
  }
}

}  // namespace slsht_cuda
