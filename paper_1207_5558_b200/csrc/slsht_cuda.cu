// Host side of the B200 directional-SLSHT engine: plan construction, chunk scheduling and the
// extern "C" ABI declared in include/slsht_cuda.h. All arithmetic runs in the kernels of
// kernels.cuh; the host only builds index tables (component lists, FFT plan, q offsets).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "kernels_chunk.cuh"
#include "kernels_couple.cuh"
#include "kernels_couple_ws.cuh"
#include "kernels_couple_lines.cuh"
#include "kernels_couple_reg.cuh"
#include "kernels_twopass.cuh"
#include "kernels_tpipe.cuh"
#include "kernels_fused.cuh"
#include "direct.cuh"
#include "window_solver.cuh"
#include "blas_fp64.cuh"
#include "kernels_setup.cuh"
#include "slsht_cuda.h"

using namespace slsht_cuda;

namespace {

thread_local std::string g_create_error;

struct CudaError {
  std::string msg;
};
struct Status {
  int code;
  std::string msg;
};

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      throw CudaError{std::string(#x) + ": " + cudaGetErrorString(e_)};               \
  } while (0)

#define CKL()                                                                         \
  do {                                                                                \
    cudaError_t e_ = cudaGetLastError();                                              \
    if (e_ != cudaSuccess) throw CudaError{std::string("launch: ") + cudaGetErrorString(e_)}; \
  } while (0)

inline int coeff_index(int l, int m) { return l * l + l + m; }
inline long long coeff_count(int L) { return (long long)(L + 1) * (L + 1); }

template <class T>
T* dalloc(size_t count) {
  T* p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

template <class T>
T* dupload(const std::vector<T>& v, cudaStream_t s) {
  T* p = dalloc<T>(v.size());
  if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

constexpr size_t kGuardBytes = 65536;

template <class T>
T* palloc(slsht_cuda_plan* p, size_t count);
void pfree(slsht_cuda_plan* p, void* ptr);
void check_guards(slsht_cuda_plan* p);

struct Chunk {
  long long comp0;
  int count;
  int seg0, nseg;
  int tile0, ntile;
  int buf;  // ring half (ring mode)
};

// ST_QFFT: the two-pass path's k_qfft (its k_tgemm is ST_COUPLE); 0 on the other paths
enum Stage { ST_SETUP = 0, ST_LEGENDRE, ST_MODGEMM, ST_COUPLE, ST_DIGEST, ST_QFFT, ST_COUNT };

// Warp-specialized persistent kernels (kernels_couple_ws.cuh) for the BASELINE lengths.
struct WsKernel {
  void (*fn)(WsParams);
  int threads;
  size_t smem;
  int MT, NT, RS;
};

}  // namespace

struct slsht_cuda_plan {
  slsht_cuda_desc desc{};
  int L_f = 0, L_h = 0, L_g = 0, lmax = 0, l_begin = 0, l_end = 0;
  int n = 0, nb = 0, ncol = 0, NPQ = 0, N = 0, n_nodes = 0, ldA = 0;
  int real_mode = 0, emit_neg = 0, mirror = 0, materialize = 0;
  int MG = 1, NG = 1, n_col_tiles = 0;
  long long vol = 0;            // complex elements per volume
  // device output layout: row a of a volume at a * rpitch, slots vstride apart. The two-pass
  // ring pads every row to whole 128-B lines (rpitch = ncol rounded up to 8) so the epilogue
  // writes aligned lines; elsewhere rpitch = ncol, vstride = vol (the So3Volume layout)
  int rpitch = 0;
  long long vstride = 0;
  long long slot_base = 0;      // coeff_index offset of the first materialized slot
  long long n_slots = 0;        // output slots allocated
  long long emitted = 0;
  int max_chunk = 0;
  FftPlan fft{};
  int generic_dft = 0;
  size_t couple_smem = 0;
  bool use_ws = false;  // warp-specialized persistent coupling kernel for this length
  bool use_reg = false; // thread-per-column register kernel (k_couple_reg, n = 17)
  WsKernel ws{};
  WsStages ws_stages{};
  int num_sms = 0;
  bool use_lines = false;  // line-aligned persistent coupling kernel (n <= 33, ncol % 8 == 1)
  void (*lines_fn)(LnParams) = nullptr;
  int lines_threads = 0;
  int lines_upad = 0;
  int lines_nseg = 1;      // line kernel: column segments per group (execution split, per chunk)
  int lines_nseg_dig = 1;  // digest segments per group (fixed per n: the digests do not depend
                           // on the execution split, the chunking or the sharding)
  int lines_urb[136] = {};
  bool use_tp = false;     // two-pass coupling: k_tgemm (T to HBM) + k_qfft (n = 49, 65, 129)
  int tp_KP = 0;           //   q-padded (p, q) rows
  int tp_ncolp = 0;        //   padded column stride of W and T
  int tp_ntiles = 0;       //   k_qfft column tiles (digest partials per component)
  int tp_nt = 32;          //   k_qfft columns per CTA
  int tp_threads = 0;
  size_t tp_gemm_smem = 0, tp_fft_smem = 0;
  int tp_bn = 64;          //   k_tgemm column tile (32 in the overlapped schedule)
  int tp_gv = 3;           //   k_tgemm variant (tgemm_variant)
  bool tp_overlap = false; //   k_qfft + digest of chunk i on fft_stream under k_tgemm of i+1
  bool use_fused = false;  // fused coupling (k_fused, n = 49): GEMM + FFT + epilogue in one
  int fu_KP = 0, fu_upad = 0;
  bool tp_col_fast = false; //  k_tgemm raster: column tiles fastest (W L2-resident)
  int tp_t_stream = 0;      //  k_tgemm: 1 T stores with the evict-first hint; 2 no T stores (timing)
  size_t tp_t_elems = 0;   //   one T buffer (two in the overlapped schedule)
  bool tp_pipe = false;    //   k_tpipe: GEMM and alpha-pass items in one persistent kernel over an
                           //   L2-resident ring of T slots (kernels_tpipe.cuh; n = 49, 65)
  int tp_ct = 0, tp_ncg = 0, tp_nqg = 0, tp_nslot = 3, tp_fb = 8, tp_lag = 1;
  size_t tp_slot_elems = 0, tp_pipe_smem = 0;
  int tp_sync_ints = 0;
  int tp_kc = 0;           //   T rows of at most tp_kc coupling terms are recomputed by k_qfft
  int tp_ks_lo = 0;        //   first k-step of k_tgemm's row range
  int tp_KPsub = 0;        //   rows of k_tgemm's range (whole stages)
  short tp_rc_urow[16] = {};
  signed char tp_rc_k[16] = {};
  bool tp_half = false;    //   k_qfft_half (n = 49, 65): last DIF stage fused into the epilogue, 4 partials per tile
  bool tp_lean = false;    //   k_qfft_lean (n = 49, 65): two smem passes, 4 digest partials per tile
  int tp_pipe_fv = 0;      //   lean alpha pass with per-warp digest partials (4 per tile)
  int* d_tp_sync = nullptr;
  int* d_qg = nullptr;     //   k-step bounds of the q groups
  void (*tp_pipe_fn)(TpParams) = nullptr;
  cudaStream_t fft_stream = nullptr;
  cudaEvent_t ev_tg[2] = {}, ev_fft[2] = {};
  bool fft_rec[2] = {false, false};  // ev_fft[b] recorded during the current call
  int fft_last = -1;
  void (*tp_fft)(QfParams) = nullptr;
  int* d_ubase = nullptr;  // stage-tiled U layout (ws path): per (p, q) row block offset
  int* d_ustr = nullptr;   //   and row stride
  int ct_fast = 0;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  cudaStream_t aux_stream = nullptr;  // window-table chain of the setup, overlapped
  cudaEvent_t ev_fork = nullptr, ev_wtab = nullptr;
  bool wtab_pending = false;
  cudaGraphExec_t graph = nullptr;  // forward_device replay (setup + every chunk), built once
  long long graph_launches = 0;
  bool own_stream = false;
  bool profile = false;
  bool built = false;  // build_plan completed (single-device plans)
  // SLSHT_CUDA_GUARD=1: every plan-owned device buffer is allocated with 64-KB guard bands on
  // both sides (pattern 0xA5), checked after every call (bounds checking of global memory; the
  // pool has no compute-sanitizer)
  struct GuardedBuf {
    void* user;
    char* base;
    size_t bytes;
  };
  bool guard = false;
  std::vector<GuardedBuf> guards;
  std::string last_error;
  long long launches = 0;
  double stage_ms[ST_COUNT] = {0, 0, 0, 0, 0, 0};

  std::vector<CompRec> comps;
  std::vector<Seg> segs;
  std::vector<MTile> tiles;
  std::vector<Chunk> chunks;

  // device
  double *d_f = nullptr, *d_h = nullptr;
  double *d_ncos = nullptr, *d_nsin = nullptr, *d_weights = nullptr, *d_betaw = nullptr;
  double2* d_itab = nullptr;
  double* d_lamh = nullptr;
  double* d_delta = nullptr;
  double* d_delta_ws = nullptr;  // k_delta workspace for large window band limits
  double* d_dtab = nullptr;
  double2* d_W = nullptr;
  double2* d_rou = nullptr;
  double2* d_phase = nullptr;
  int* d_perm = nullptr;
  int* d_qoff = nullptr;
  int* d_pq = nullptr;
  int* d_err = nullptr;
  CompRec* d_comps = nullptr;
  Seg* d_segs = nullptr;
  MTile* d_tiles = nullptr;
  double* d_A = nullptr;
  double2* d_U = nullptr;
  double2* d_T = nullptr;   // two-pass: T of one chunk
  short* d_qend = nullptr;  // two-pass: per k-step, the T row it completes (or -1)
  int* d_wrow = nullptr;    // two-pass: W row of every (p, q)
  double* d_r43 = nullptr;  // two-pass, n = 129: DMMA fragments of the radix-43 stage
  double2* d_out = nullptr;
  double* d_partials = nullptr;
  double* d_digest = nullptr;
  long long digest_rows = 0;
  // host staging for the host-sink mode
  double2* h_stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  cudaEvent_t ev_done[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_stage[ST_COUNT + 1] = {};
  // single-chunk plans: the coupling kernel's start and end, recorded on every call (also
  // inside the CUDA graph), read lazily by slsht_cuda_kernel_time
  cudaEvent_t ev_lazy[2] = {};
  bool lazy_valid = false;
  // multi-GPU plan (desc.n_devices > 1): one single-device plan per degree shard; this object
  // then only holds the group-level sizes and dispatches
  std::vector<slsht_cuda_plan*> parts;
  std::vector<int> part_bounds;  // shard k = degrees [part_bounds[k], part_bounds[k+1])
  bool group() const { return !parts.empty(); }
};

namespace {

template <class T>
T* palloc(slsht_cuda_plan* p, size_t count) {
  if (!p->guard) return dalloc<T>(count);
  if (count == 0) count = 1;
  const size_t bytes = count * sizeof(T);
  char* base = nullptr;
  CK(cudaMalloc(&base, bytes + 2 * kGuardBytes));
  CK(cudaMemset(base, 0xA5, kGuardBytes));
  CK(cudaMemset(base + kGuardBytes + bytes, 0xA5, kGuardBytes));
  p->guards.push_back({base + kGuardBytes, base, bytes});
  return reinterpret_cast<T*>(base + kGuardBytes);
}

void pfree(slsht_cuda_plan* p, void* ptr) {
  if (!ptr) return;
  for (auto& g : p->guards)
    if (g.user == ptr) {
      cudaFree(g.base);
      g.user = nullptr;
      return;
    }
  cudaFree(ptr);
}

// Every guard band still holds its pattern (after the device is idle).
void check_guards(slsht_cuda_plan* p) {
  if (!p->guard) return;
  CK(cudaDeviceSynchronize());
  std::vector<unsigned char> band(kGuardBytes);
  for (size_t i = 0; i < p->guards.size(); ++i) {
    const auto& g = p->guards[i];
    if (!g.user) continue;
    for (int side = 0; side < 2; ++side) {
      const char* src = side ? g.base + kGuardBytes + g.bytes : g.base;
      CK(cudaMemcpy(band.data(), src, kGuardBytes, cudaMemcpyDeviceToHost));
      for (size_t k = 0; k < kGuardBytes; ++k)
        if (band[k] != 0xA5) {
          char msg[160];
          std::snprintf(msg, sizeof msg,
                        "guard band %s device buffer #%zu (%zu bytes) overwritten at byte %zu",
                        side ? "after" : "before", i, g.bytes, k);
          throw Status{SLSHT_ERR_DEVICE, msg};
        }
    }
  }
}

void free_plan(slsht_cuda_plan* p) {
  if (!p) return;
  for (slsht_cuda_plan* q : p->parts) {
    cudaSetDevice(q->desc.device);
    free_plan(q);
  }
  p->parts.clear();
  pfree(p, p->d_f);
  pfree(p, p->d_T);
  pfree(p, p->d_qend);
  pfree(p, p->d_tp_sync);
  pfree(p, p->d_qg);
  pfree(p, p->d_wrow);
  pfree(p, p->d_r43);
  pfree(p, p->d_h);
  pfree(p, p->d_ncos);
  pfree(p, p->d_nsin);
  pfree(p, p->d_weights);
  pfree(p, p->d_betaw);
  pfree(p, p->d_itab);
  pfree(p, p->d_lamh);
  pfree(p, p->d_delta);
  pfree(p, p->d_delta_ws);
  pfree(p, p->d_dtab);
  pfree(p, p->d_W);
  pfree(p, p->d_rou);
  pfree(p, p->d_phase);
  pfree(p, p->d_perm);
  pfree(p, p->d_qoff);
  pfree(p, p->d_pq);
  pfree(p, p->d_ubase);
  pfree(p, p->d_ustr);
  pfree(p, p->d_err);
  pfree(p, p->d_comps);
  pfree(p, p->d_segs);
  pfree(p, p->d_tiles);
  pfree(p, p->d_A);
  pfree(p, p->d_U);
  pfree(p, p->d_out);
  pfree(p, p->d_partials);
  pfree(p, p->d_digest);
  for (int i = 0; i < 2; ++i) {
    if (p->h_stage[i]) cudaFreeHost(p->h_stage[i]);
    if (p->ev_done[i]) cudaEventDestroy(p->ev_done[i]);
    if (p->ev_copied[i]) cudaEventDestroy(p->ev_copied[i]);
  }
  for (auto& e : p->ev_stage)
    if (e) cudaEventDestroy(e);
  for (auto& e : p->ev_lazy)
    if (e) cudaEventDestroy(e);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->fft_stream) cudaStreamDestroy(p->fft_stream);
  for (int i = 0; i < 2; ++i) {
    if (p->ev_tg[i]) cudaEventDestroy(p->ev_tg[i]);
    if (p->ev_fft[i]) cudaEventDestroy(p->ev_fft[i]);
  }
  if (p->aux_stream) {
    cudaStreamSynchronize(p->aux_stream);
    cudaStreamDestroy(p->aux_stream);
  }
  if (p->graph) cudaGraphExecDestroy(p->graph);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  if (p->ev_wtab) cudaEventDestroy(p->ev_wtab);
  if (p->own_stream && p->stream) cudaStreamDestroy(p->stream);
  delete p;
}

std::vector<int> factor_odd(int n) {
  std::vector<int> f;
  int x = n;
  for (int p = 3; x > 1; p += 2)
    while (x % p == 0) {
      f.push_back(p);
      x /= p;
    }
  return f;
}

// Tile shape of k_couple per transform length: the CTA keeps 8*MG x 8*NG x n complex of T in
// shared memory (<= ~135 KB), DESIGN.md §3.3.
void couple_tile(int n, int& MG, int& NG) {
  // n = 49, 65: one 8x8 tile per CTA so that 3 CTAs share an SM and overlap their coupling,
  // FFT and store phases (a 16-component tile needs the whole shared memory)
  MG = (n <= 33) ? 2 : 1;
  NG = n <= 31 ? 2 : 1;
}

size_t couple_smem_bytes(int n, int MG, int NG) {
  return couple_t_bytes(n, MG, NG) + (size_t)n * 32 + (size_t)((n + 1) / 2) * 8 * 2 +
         (size_t)(2 * n + 1) * 4 + 64;
}

using CoupleFn = void (*)(CoupleParams);

// Compile-time instantiations: the BASELINE transform lengths get their own kernel (unrolled
// FFT plan, only the radices they need); every other odd length takes the runtime-plan kernel.
CoupleFn couple_kernel(int n, int MG, int NG) {
  switch (n) {
    case 17: return k_couple<17, 2, 2, 512, 1>;
    case 33: return k_couple<33, 2, 1, 256, 2>;
    case 49: return k_couple<49, 1, 1, 256, 3>;
    case 65: return k_couple<65, 1, 1, 256, 2>;
    case 129: return k_couple<129, 1, 1, 256, 1>;
    default: break;
  }
  if (MG == 2 && NG == 2) return k_couple<0, 2, 2, 256, 1>;
  if (MG == 2 && NG == 1) return k_couple<0, 2, 1, 256, 1>;
  return k_couple<0, 1, 1, 256, 1>;
}

// <N, MG, NG, stage rows, stages, warps per consumer group>

template <int N, int MG, int NG, int RS, int NSTAGE, int GW>
WsKernel ws_entry() {
  using Cfg = WsCfg<N, MG, NG, RS, NSTAGE, GW>;
  return WsKernel{k_couple_ws<N, MG, NG, RS, NSTAGE, GW>, Cfg::NTHREADS, Cfg::SMEM, Cfg::MT,
                  Cfg::NT, RS};
}

bool ws_kernel(int n, WsKernel& k) {
  switch (n) {
    case 17: k = ws_entry<17, 2, 2, 44, 3, 8>(); return true;
    case 33: k = ws_entry<33, 2, 1, 56, 3, 8>(); return true;
    // n = 49, 65, 129 (one 8x8 warp tile) stay on k_couple until the MMA warps of the
    // persistent kernel can split the k range of one q
    default: return false;
  }
}

using TgemmFn = void (*)(TgParams);
// k_tgemm variants (SLSHT_CUDA_TGEMM): <BN, WNF, stages, CTAs per SM>
struct TgemmVariant {
  TgemmFn fn;
  int bn, wnf, nst, per_sm, bm;
};
TgemmVariant tgemm_variant(int v) {
  switch (v) {
    case 0: return {k_tgemm<64, 2, 4, 1>, 64, 2, 4, 1, 64};
    case 2: return {k_tgemm<32, 2, 4, 1>, 32, 2, 4, 1, 64};
    case 3: return {k_tgemm<32, 2, 2, 3>, 32, 2, 2, 3, 64};
    default: return {k_tgemm<32, 2, 3, 2>, 32, 2, 3, 2, 64};
  }
}

// Two-pass coupling (kernels_twopass.cuh): the k_qfft instantiation per BASELINE length
// (n = 49, 65, 129; n = 17 and 33 keep their single-pass kernels).
bool tp_kernel(int n, void (*&fn)(QfParams), int& threads, int& nt) {
  // one component x 32 columns per CTA, 128 threads (k_qfft<129> shapes tried and not kept:
  // 96 threads, 16 x 64, 42 x 128, 64 x 256)
  threads = 128;
  nt = 32;
  // CTAs per SM: 6 (n = 49), 5 (n = 65) measured best (4 or 8 / 6 slower: DESIGN.md §7)
  switch (n) {
    case 49: fn = k_qfft<49, 32, 128, 6>; break;
    case 65: fn = k_qfft<65, 32, 128, 5>; break;
    case 129: fn = k_qfft<129, 32, 128, 3>; break;  // radix-43 stage on DMMA: 168 registers
    default:
      // longer transforms (n > 129) without a compile-time kernel: the runtime-plan alpha pass
      // (8 columns per CTA: the n x 8 tile of T fits in shared memory up to n ~ 1500)
      if (n <= 129) return false;
      fn = k_qfft_rt<8, 128>;
      nt = 8;
      break;
  }
  return true;
}

int couple_threads(int n) {
  switch (n) {
    case 17:
      return 512;
    default:
      return 256;
  }
}

// The dynamic shared-memory opt-in of this plan's kernels. The attribute belongs to the kernel
// function, not to the plan, and several plans can share a kernel with different sizes (the
// runtime-length kernels), so it is applied again at every entry point (cheap host calls,
// outside any stream capture) as well as at build time.
void set_func_attributes(const slsht_cuda_plan* p) {
  auto opt = [](auto fn, size_t bytes) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  };
  opt(k_modgemm, MG_SMEM);
  CK(configure_delta(p->L_h));
  opt(k_glnodes, 4 * sizeof(double) * (p->L_g + 2));
  if (p->use_fused) {
    opt(k_fused<49>, p->couple_smem);
  } else if (p->use_lines) {
    opt(p->lines_fn, p->couple_smem);
  } else if (p->use_tp) {
    opt(tgemm_variant(p->tp_gv).fn, p->tp_gemm_smem);
    opt(p->tp_fft, p->tp_fft_smem);
    if (p->tp_pipe) opt(p->tp_pipe_fn, p->tp_pipe_smem);
  } else if (p->use_reg) {
    opt(k_couple_reg<17>, p->couple_smem);
  } else if (p->use_ws) {
    opt(p->ws.fn, p->couple_smem);
  } else {
    opt(couple_kernel(p->n, p->MG, p->NG), p->couple_smem);
  }
}

void build_plan(slsht_cuda_plan* p) {
  const slsht_cuda_desc& d = p->desc;
  if (d.L_f < 0 || d.L_h < 0) throw Status{SLSHT_ERR_VALIDATION, "band limit must be non-negative"};
  {
    const char* g = std::getenv("SLSHT_CUDA_GUARD");
    p->guard = g && g[0] == '1';
  }
  p->L_f = d.L_f;
  p->L_h = d.L_h;
  p->L_g = d.L_f + d.L_h;
  p->lmax = d.lmax < 0 ? p->L_g : d.lmax;
  if (p->lmax > p->L_g)
    throw Status{SLSHT_ERR_VALIDATION, "fast engine computes components up to L_f + L_h only"};
  p->l_begin = std::max(0, d.l_begin);
  p->l_end = d.l_end < 0 ? p->lmax + 1 : std::min(d.l_end, p->lmax + 1);
  if (p->l_begin > p->l_end) throw Status{SLSHT_ERR_VALIDATION, "empty or inverted degree range"};
  p->real_mode = d.real_mode ? 1 : 0;
  p->emit_neg = d.emit_negative_m ? 1 : 0;
  p->mirror = p->real_mode && p->emit_neg;
  p->materialize = d.materialize ? 1 : 0;
  const int L = p->L_h;
  p->n = 2 * L + 1;
  p->nb = L + 1;
  p->ncol = p->n * p->nb;
  p->NPQ = (L + 1) * (L + 1);
  p->N = 2 * p->L_g;                // the reference rule S_{2L_g} (its residue check only)
  p->n_nodes = (p->L_g + 2) / 2;    // x >= 0 half of the (L_g + 1)-point Gauss-Legendre rule
  p->ldA = (p->n_nodes + MG_K - 1) / MG_K * MG_K;
  p->vol = (long long)p->n * p->n * p->nb;
  // two-pass coupling for the long transforms unless SLSHT_CUDA_TWO_PASS=0 (the single-pass
  // k_couple then runs); n = 33 keeps its line kernel, n = 17 its warp-specialized kernel
  {
    const char* e = std::getenv("SLSHT_CUDA_TWO_PASS");
    p->use_tp = !(e && e[0] == '0') && tp_kernel(p->n, p->tp_fft, p->tp_threads, p->tp_nt);
    if (const char* hf = std::getenv("SLSHT_CUDA_QFFT_HALF")) {
      const int mb = std::atoi(hf);  // CTAs per SM (0: off)
      if (p->use_tp && mb > 0 && (p->n == 49 || p->n == 65)) {
        p->tp_half = true;
        if (p->n == 49) p->tp_fft = mb >= 8 ? k_qfft_half<49, 32, 128, 8> : mb >= 6 ? k_qfft_half<49, 32, 128, 6> : k_qfft_half<49, 32, 128, 5>;
        else p->tp_fft = mb >= 6 ? k_qfft_half<65, 32, 128, 6> : mb >= 5 ? k_qfft_half<65, 32, 128, 5> : k_qfft_half<65, 32, 128, 4>;
      }
    }
    if (const char* ln = std::getenv("SLSHT_CUDA_QFFT_LEAN")) {
      const int mb = std::atoi(ln);  // CTAs per SM of the lean alpha pass (0: off)
      if (p->use_tp && mb > 0 && (p->n == 49 || p->n == 65)) {
        p->tp_lean = true;
        if (p->n == 49) p->tp_fft = mb >= 8 ? k_qfft_lean<49, 32, 128, 8> : mb >= 6 ? k_qfft_lean<49, 32, 128, 6> : k_qfft_lean<49, 32, 128, 4>;
        else p->tp_fft = mb >= 6 ? k_qfft_lean<65, 32, 128, 6> : mb >= 5 ? k_qfft_lean<65, 32, 128, 5> : k_qfft_lean<65, 32, 128, 4>;
      }
    }
    p->tp_ntiles = (p->ncol + p->tp_nt - 1) / p->tp_nt;
    // k_tgemm shape: <32, 2, 2, 3> (three 4-warp CTAs per SM, two stages) unless
    // SLSHT_CUDA_TGEMM selects <64, 2, 4, 1> (0), <32, 2, 3, 2> (1) or <32, 2, 4, 1> (2)
    const char* gv = std::getenv("SLSHT_CUDA_TGEMM");
    p->tp_gv = gv ? std::atoi(gv) : 3;
    if (p->tp_gv < 0 || p->tp_gv > 3) p->tp_gv = 3;
    p->tp_bn = tgemm_variant(p->tp_gv).bn;
    // T and W column stride: whole GEMM column tiles (a multiple of k_qfft's 32 columns)
    p->tp_ncolp = (p->ncol + p->tp_bn - 1) / p->tp_bn * p->tp_bn;
  }
  // fused coupling for n = 49 with SLSHT_CUDA_FUSED=1 (opt-in until it beats the two-pass
  // path)
  {
    const char* e = std::getenv("SLSHT_CUDA_FUSED");
    p->use_fused = p->n == 49 && e && e[0] == '1';
    if (p->use_fused) {
      p->use_tp = false;
      p->fu_KP = FuCfg<49>::KR;
      p->fu_upad = FuCfg<49>::UPAD;
    }
  }
  // ---- component list: orders m (all or m >= 0 in real mode), degrees in the shard
  for (int m = p->real_mode ? 0 : -p->lmax; m <= p->lmax; ++m) {
    const int lo = std::max(std::abs(m), p->l_begin), hi = std::min(p->lmax, p->l_end - 1);
    for (int l = lo; l <= hi; ++l) p->comps.push_back(CompRec{l, m, 0, -1});
  }
  const long long total = (long long)p->comps.size();
  p->emitted = 0;
  for (const auto& c : p->comps) p->emitted += (p->mirror && c.m > 0) ? 2 : 1;

  // ---- chunking and output slots
  p->rpitch = ((p->use_tp || p->use_fused) && !p->materialize) ? (p->ncol + 7) / 8 * 8 : p->ncol;
  p->vstride = (long long)p->n * p->rpitch;
  const size_t vol_bytes = (size_t)p->vstride * 16;
  if (p->materialize) {
    p->slot_base = (long long)p->l_begin * p->l_begin;
    p->n_slots = (long long)p->l_end * p->l_end - p->slot_base;
    p->max_chunk = (int)std::min<long long>(std::max<long long>(total, 1), 16384);
    if (p->use_tp) {  // the chunk's T buffer stays below 4 GiB
      const long long tcomp = (long long)p->n * p->tp_ncolp * 16;
      p->max_chunk = (int)std::max<long long>(
          TG_BM, std::min<long long>(p->max_chunk, (4LL << 30) / tcomp / TG_BM * TG_BM));
    }
  } else {
    long long ring = d.ring_bytes > 0 ? d.ring_bytes : (1LL << 31);
    const int per = p->mirror ? 2 : 1;
    long long ch = ring / (2LL * per * (long long)vol_bytes);
    ch = std::max<long long>(8, ch / 8 * 8);
    ch = std::min<long long>(ch, 16384);
    ch = std::min<long long>(ch, std::max<long long>(8, (total + 7) / 8 * 8));
    if (p->use_tp && ch >= 2 * TG_BM) {
      // whole 64-component GEMM blocks, as many as give full waves of k_tgemm CTAs
      int sms = 148;
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.device) != cudaSuccess)
        sms = 148;
      sms *= tgemm_variant(p->tp_gv).per_sm;  // resident k_tgemm CTAs
      const long long nct = p->tp_ncolp / p->tp_bn, bmax = ch / TG_BM;
      long long best_b = bmax;
      double best = 0.0;
      for (long long b = bmax; b >= (bmax + 1) / 2; --b) {
        const double eff = (double)(b * nct) / (double)(((b * nct + sms - 1) / sms) * sms);
        if (eff > best + 0.01) {
          best = eff;
          best_b = b;
        }
      }
      ch = best_b * TG_BM;
    }
    if (p->use_fused && ch >= 8) {
      // whole 8-component groups, a whole number of waves of the persistent CTAs when possible
      int sms = 148;
      if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.device) != cudaSuccess)
        sms = 148;
      const long long groups = ch / 8;
      ch = (groups >= sms ? groups / sms * sms : groups) * 8;
    }
    p->max_chunk = (int)ch;
    p->n_slots = 2LL * per * ch;
  }
  couple_tile(p->n, p->MG, p->NG);
  // line-aligned kernel for n = 33 (ncol == 1 mod 8); SLSHT_CUDA_LINES=0 selects the
  // column-strip kernel instead. Its digest partials use a fixed split of every component
  // group's column tiles into 4 segments (so the digests are bitwise independent of the
  // chunking and the sharding); its work units are (group, one of 1, 2 or 4 segments), chosen
  // per plan for balance over the SMs.
  bool lines = (p->ncol % 8) == 1 && p->n == 33;
  if (const char* e = std::getenv("SLSHT_CUDA_LINES")) lines = lines && e[0] != '0';
  if (lines) {
    p->use_lines = true;
    p->lines_nseg_dig = std::min(4, (p->ncol + 7) / 8);
    p->lines_nseg = p->lines_nseg_dig;
    p->MG = 1;
    p->NG = 1;
    p->lines_fn = k_couple_lines<33>;
    p->lines_threads = LnCfg<33>::NTHREADS;
    p->couple_smem = LnCfg<33>::SMEM;
    p->lines_upad = LnCfg<33>::UPAD;
  } else if (p->n == 17 && !(std::getenv("SLSHT_CUDA_REG") && std::getenv("SLSHT_CUDA_REG")[0] == '0') &&
             std::getenv("SLSHT_CUDA_NO_WS") == nullptr) {
    // n = 17 (L_h = 8, config 1): one thread per (component, column), all in registers
    p->use_reg = true;
    p->MG = 1;
    p->NG = RG_NT / 8;  // 32-column tiles
  } else if (std::getenv("SLSHT_CUDA_NO_WS") == nullptr && ws_kernel(p->n, p->ws)) {
    p->use_ws = true;
    p->MG = p->ws.MT / 8;
    p->NG = p->ws.NT / 8;
    // q-groups of consecutive rows jq with at most RS (p, q) rows per operand stage
    int cnt = 0, rows = 0;
    p->ws_stages.js[0] = 0;
    for (int jq = 0; jq < p->n; ++jq) {
      const int np = (L + 1 - std::abs(jq - L) + 3) / 4 * 4;  // padded to whole k-steps
      if (rows + np > p->ws.RS) {
        p->ws_stages.js[++cnt] = jq;
        rows = 0;
      }
      rows += np;
    }
    p->ws_stages.js[++cnt] = p->n;
    p->ws_stages.count = cnt;
  }
  p->n_col_tiles = p->use_fused ? (p->ncol + FuCfg<49>::NT - 1) / FuCfg<49>::NT
                   : p->use_tp  ? p->tp_ntiles
                                : (p->ncol + 8 * p->NG - 1) / (8 * p->NG);
  const char* prof = std::getenv("SLSHT_CUDA_PROFILE");
  p->profile = prof && prof[0] == '1';

  int dev_count = 0;
  if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
    throw Status{SLSHT_ERR_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
  if (d.device < 0 || d.device >= dev_count) throw Status{SLSHT_ERR_DEVICE, "invalid device ordinal"};
  CK(cudaSetDevice(d.device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, d.device));
  if (prop.major != 10) throw Status{SLSHT_ERR_DEVICE, "this build targets sm_100a (B200) only"};

  if (d.stream) {
    p->stream = (cudaStream_t)d.stream;
  } else {
    CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
    p->own_stream = true;
  }
  CK(cudaStreamCreateWithFlags(&p->copy_stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&p->aux_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&p->ev_wtab, cudaEventDisableTiming));
  cudaStream_t s = p->stream;

  // ---- q-major (p, q) ordering of the window band: c = qoff[q+L] + p - |q|
  std::vector<int> qoff(p->n + 1, 0), pq(2 * p->NPQ);
  for (int jq = 0; jq < p->n; ++jq) {
    const int q = jq - L, aq = std::abs(q);
    qoff[jq + 1] = qoff[jq] + (L + 1 - aq);
    for (int pp = aq; pp <= L; ++pp) {
      const int c = qoff[jq] + pp - aq;
      pq[2 * c] = q;
      pq[2 * c + 1] = pp;
    }
  }
  // ---- stage-tiled U layout of the warp-specialized coupling kernel: per component group,
  // stage s holds MT rows of USTR_s (>= the stage's (p, q) rows, == 4 mod 8) complex
  std::vector<int> ubase(p->NPQ, 0), ustr(p->NPQ, 0);
  if (p->use_ws) {
    const int MT = p->ws.MT;
    long long off = 0;
    for (int st = 0; st < p->ws_stages.count; ++st) {
      // each q's rows padded with zeros to whole k-steps of 4 (the MMA loop never masks)
      int rows_pad = 0;
      for (int jq = p->ws_stages.js[st]; jq < p->ws_stages.js[st + 1]; ++jq) {
        p->ws_stages.urb[jq] = rows_pad;
        rows_pad += (qoff[jq + 1] - qoff[jq] + 3) / 4 * 4;
      }
      const int us = rows_pad + (((4 - rows_pad) % 8) + 8) % 8;  // == 4 mod 8: no bank conflicts
      if (us + 8 > p->ws.RS + 8 + 8)
        throw Status{SLSHT_ERR_VALIDATION, "internal: operand stage exceeds its buffer"};
      p->ws_stages.uoff[st] = (int)off;
      p->ws_stages.ustr[st] = us;
      for (int jq = p->ws_stages.js[st]; jq < p->ws_stages.js[st + 1]; ++jq)
        for (int c = qoff[jq]; c < qoff[jq + 1]; ++c) {
          ubase[c] = (int)off + p->ws_stages.urb[jq] + (c - qoff[jq]);
          ustr[c] = us;
        }
      off += (long long)MT * us;
    }
    p->ws_stages.group_elems = off;
  }
  if (p->use_lines) {
    // one padded block per component: q rows padded with zeros to whole k-steps of 4
    int rows_pad = 0;
    for (int jq = 0; jq < p->n; ++jq) {
      p->lines_urb[jq] = rows_pad;
      rows_pad += (qoff[jq + 1] - qoff[jq] + 3) / 4 * 4;
    }
    if (rows_pad > p->lines_upad)
      throw Status{SLSHT_ERR_VALIDATION, "internal: padded U rows exceed the line kernel buffer"};
    for (int jq = 0; jq < p->n; ++jq)
      for (int c = qoff[jq]; c < qoff[jq + 1]; ++c) {
        ubase[c] = p->lines_urb[jq] + (c - qoff[jq]);
        ustr[c] = p->lines_upad;
      }
    p->ws_stages.group_elems = 8LL * p->lines_upad;
  }
  // ---- two-pass GEMM layout: every q's rows padded with zeros to whole k-steps of 4, the
  // same row positions in U (per component, stride KP) and W (stride ncolp); qend marks the
  // k-step that completes each q, with the T row (q mod n) it is stored to
  std::vector<int> wrow;
  std::vector<short> qend;
  if (p->use_tp) {
    int rows_pad = 0;
    wrow.assign(p->NPQ, 0);
    std::vector<int> urb(p->n + 1, 0);
    for (int jq = 0; jq < p->n; ++jq) {
      urb[jq] = rows_pad;
      rows_pad += (qoff[jq + 1] - qoff[jq] + 3) / 4 * 4;
    }
    urb[p->n] = rows_pad;
    rows_pad = (rows_pad + TG_KS - 1) / TG_KS * TG_KS;  // whole GEMM stages (zero rows)
    p->tp_KP = rows_pad;
    // k_tgemm raster: column tiles fastest when W (KP x ncolp complex) stays L2-resident, so a
    // chunk's U is read from HBM once (SLSHT_CUDA_TG_RASTER=0/1 forces either order)
    p->tp_col_fast = (size_t)p->tp_KP * p->tp_ncolp * 16 <= (48u << 20);
    if (const char* e = std::getenv("SLSHT_CUDA_TG_RASTER")) p->tp_col_fast = e[0] == '1';
    if (const char* e = std::getenv("SLSHT_CUDA_TG_STREAM")) p->tp_t_stream = std::atoi(e);
    qend.assign(rows_pad / 4, (short)-1);
    for (int jq = 0; jq < p->n; ++jq) {
      for (int c = qoff[jq]; c < qoff[jq + 1]; ++c) {
        ubase[c] = urb[jq] + (c - qoff[jq]);
        ustr[c] = 0;
        wrow[c] = ubase[c];
      }
      qend[urb[jq + 1] / 4 - 1] = (short)(jq >= L ? jq - L : jq + L + 1);
    }
    p->ws_stages.group_elems = rows_pad;
    // The q of few coupling terms (|q| > L - KC: K_q = L + 1 - |q| <= KC, the first and last KC
    // q of the q-major order) cost k_tgemm a whole k-step each and the T round trip 2 KC of n
    // rows; k_qfft recomputes them from U and W instead (n = 49, 65; not with the pipeline or
    // the lean alpha pass, which read every T row). SLSHT_CUDA_TP_KC=0..8 sets KC; with KC = 2
    // every k_qfft thread owns one recomputed (row, column) and requests its operands ahead of
    // the tile (config 4: k_tgemm 74.7 -> 70.8 ms, k_qfft +1 ms; KC = 4: slower, the W rows of
    // the recomputation are L2 traffic per (component, column tile)).
    p->tp_KPsub = p->tp_KP;
    {
      const char* pe = std::getenv("SLSHT_CUDA_TP_PIPE");
      const bool pipe_req = pe && pe[0] == '1';
      int kc = (p->n == 49 || p->n == 65) && !pipe_req && !p->tp_lean ? 2 : 0;  // measured best
      if (const char* e = std::getenv("SLSHT_CUDA_TP_KC")) kc = std::atoi(e);
      if (!(p->n == 49 || p->n == 65) || pipe_req || p->tp_lean) kc = 0;
      kc = std::max(0, std::min({kc, 8, L}));
      if (kc > 0) {
        const int ks_lo = urb[kc] / 4, ks_hi = urb[p->n - kc] / 4;
        std::vector<short> sub(qend.begin() + ks_lo, qend.begin() + ks_hi);
        while (sub.size() % (TG_KS / 4)) sub.push_back((short)-1);
        // the padding k-steps read the rows that follow (never stored): they must exist
        if ((int)sub.size() * 4 + ks_lo * 4 <= p->tp_KP) {
          p->tp_kc = kc;
          p->tp_ks_lo = ks_lo;
          p->tp_KPsub = (int)sub.size() * 4;
          qend = sub;
          for (int r = 0; r < 2 * kc; ++r) {
            const int trow = L + 1 - kc + r;          // T row = q mod n
            const int q = trow <= L ? trow : trow - p->n;
            p->tp_rc_urow[r] = (short)urb[q + L];
            p->tp_rc_k[r] = (signed char)(L + 1 - std::abs(q));
          }
        }
      }
    }
  }
  // ---- fused layout (k_fused, kernels_fused.cuh): T rows r = q mod n in G row groups
  // (rows j + G k); each group's sequence of k-steps (its rows in order, every row padded to
  // whole k-steps) is interleaved across the groups: K row ((s G + j) 4 + kl) holds position
  // 4 s + kl of group j's sequence. U (8-component groups, row stride UPAD) and W use it.
  if (p->use_fused) {
    using FC = FuCfg<49>;
    wrow.assign(p->NPQ, 0);
    for (int j = 0; j < FC::G; ++j) {
      int pos = 0;
      for (int k = 0; k < FC::R1; ++k) {
        const int r = j + FC::G * k;              // T row = q mod n
        const int q = r <= L ? r : r - p->n;
        const int jq = q + L;
        for (int c = qoff[jq]; c < qoff[jq + 1]; ++c, ++pos) {
          const int s0 = pos / 4, kl = pos % 4;
          wrow[c] = (s0 * FC::G + j) * 4 + kl;
          ubase[c] = wrow[c];
          ustr[c] = p->fu_upad;
        }
        pos = (pos + 3) / 4 * 4;
        if (pos / 4 != [&] { int t = 0; for (int e = 0; e <= k; ++e) t += FC::nks(j, e); return t; }())
          throw Status{SLSHT_ERR_VALIDATION, "internal: fused K layout mismatch"};
      }
      if (pos / 4 > FC::NST)
        throw Status{SLSHT_ERR_VALIDATION, "internal: fused K layout mismatch"};
    }
    p->ws_stages.group_elems = 8LL * p->fu_upad;
  }
  // ---- alpha-axis FFT plan: roots of unity, DIF stages, output permutation, phase shift
  const int n = p->n;
  std::vector<double2> rou(n), phase(n);
  for (int k = 0; k < n; ++k) {
    const double ang = -2.0 * kPi * k / n;
    rou[k] = make_double2(std::cos(ang), std::sin(ang));
  }
  for (int a = 0; a < n; ++a) {
    const int e = (int)(((long long)L * a) % n);  // e^{+2 pi i L a / n} = conj(rou[e])
    phase[a] = make_double2(rou[e].x, -rou[e].y);
  }
  const std::vector<int> fac = factor_odd(n);
  p->generic_dft = 0;
  for (int r : fac)
    if (r > kMaxGeneratedRadix) p->generic_dft = 1;
  if (fac.size() > 8) p->generic_dft = 1;
  std::vector<int> perm(n, 0);
  if (!p->generic_dft) {
    p->fft.nstages = (int)fac.size();
    int m = n;
    for (size_t i = 0; i < fac.size(); ++i) {
      p->fft.radix[i] = fac[i];
      p->fft.span[i] = m;
      m /= fac[i];
    }
    for (int pos = 0; pos < n; ++pos) {
      int rem = pos, freq = 0, mult = 1, mm = n;
      for (int r : fac) {
        const int mp = mm / r, k = rem / mp;
        rem %= mp;
        freq += k * mult;
        mult *= r;
        mm = mp;
      }
      perm[freq] = pos;
    }
  } else {
    p->fft.nstages = 0;
    for (int a = 0; a < n; ++a) perm[a] = a;
  }

  for (long long c0 = 0, ci = 0; c0 < total; c0 += p->max_chunk, ++ci) {
    Chunk ch{};
    ch.comp0 = c0;
    ch.count = (int)std::min<long long>(p->max_chunk, total - c0);
    ch.buf = (int)(ci & 1);
    ch.seg0 = (int)p->segs.size();
    ch.tile0 = (int)p->tiles.size();
    int i = 0;
    while (i < ch.count) {
      const int m = p->comps[c0 + i].m;
      int j = i;
      while (j + 1 < ch.count && p->comps[c0 + j + 1].m == m) ++j;
      const int l0 = p->comps[c0 + i].l, l1 = p->comps[c0 + j].l;
      p->segs.push_back(Seg{m, l0, l1, i});
      // GEMM tiles per parity class of l + m (A rows parity-sorted by k_agen)
      for (int par = 0; par < 2; ++par) {
        const int lf = ((l0 + m) & 1) == par ? l0 : l0 + 1;  // first degree of the class
        if (lf > l1) continue;
        const int cnt = (l1 - lf) / 2 + 1, arow = i + seg_arow(m, l0, l1, lf);
        for (int r = 0; r < cnt; r += MG_ROWS)
          p->tiles.push_back(MTile{m, arow + r, std::min(MG_ROWS, cnt - r), i + (lf - l0) + 2 * r, par});
      }
      i = j + 1;
    }
    ch.nseg = (int)p->segs.size() - ch.seg0;
    ch.ntile = (int)p->tiles.size() - ch.tile0;
    const int per = p->mirror ? 2 : 1;
    for (int k = 0; k < ch.count; ++k) {
      CompRec& r = p->comps[c0 + k];
      if (p->materialize) {
        r.slot = coeff_index(r.l, r.m) - p->slot_base;
        r.mslot = (p->mirror && r.m > 0) ? coeff_index(r.l, -r.m) - p->slot_base : -1;
      } else {
        const long long half = (long long)ch.buf * per * p->max_chunk;
        r.slot = half + k;
        r.mslot = (p->mirror && r.m > 0) ? half + p->max_chunk + k : -1;
      }
    }
    p->chunks.push_back(ch);
  }

  // ---- device memory
  const int Lf = p->L_f;
  p->d_f = palloc<double>(p, 2 * coeff_count(Lf));
  p->d_h = palloc<double>(p, 2 * coeff_count(L));
  CK(cudaMemsetAsync(p->d_h, 0, sizeof(double) * 2 * coeff_count(L), s));
  CK(cudaMemsetAsync(p->d_f, 0, sizeof(double) * 2 * coeff_count(Lf), s));
  p->d_ncos = palloc<double>(p, p->n_nodes);
  p->d_nsin = palloc<double>(p, p->n_nodes);
  p->d_weights = palloc<double>(p, p->n_nodes);
  p->d_betaw = palloc<double>(p, p->nb);
  // node stride ldA (a multiple of the modulated-SHT K chunk), padding zero for the 16-B copies
  p->d_itab = palloc<double2>(p, (size_t)2 * (2 * Lf + 1) * p->ldA);  // I_0, I_1 rows per order
  p->d_lamh = palloc<double>(p, (size_t)p->NPQ * p->ldA);
  CK(cudaMemsetAsync(p->d_itab, 0, sizeof(double2) * 2 * (2 * Lf + 1) * p->ldA, s));
  CK(cudaMemsetAsync(p->d_lamh, 0, sizeof(double) * p->NPQ * p->ldA, s));
  size_t dsz = 0;
  for (int pp = 0; pp <= L; ++pp) dsz += (size_t)(2 * pp + 1) * (2 * pp + 1);
  {
    // the window tables grow as L_h^4 (d(beta): sum (2p+1)^2 (L_h+1) doubles, W: ~(L_h+1)^2 x
    // n (L_h+1) complex); say so before allocating them
    const size_t wbytes = (size_t)(p->use_tp ? p->tp_KP : p->NPQ) *
                          (size_t)(p->use_tp ? p->tp_ncolp : p->ncol + 64) * 16;
    const size_t need = dsz * p->nb * 8 + wbytes;
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    if (need + (256u << 20) > free_b) {
      char msg[200];
      std::snprintf(msg, sizeof msg,
                    "window band limit %d: the window tables need %.1f GB of device memory, "
                    "%.1f GB are free",
                    L, need / 1e9, free_b / 1e9);
      throw Status{SLSHT_ERR_DEVICE, msg};
    }
  }
  p->d_delta = palloc<double>(p, dsz);
  if (delta_needs_gws(L)) p->d_delta_ws = palloc<double>(p, delta_ws_doubles(L));
  p->d_dtab = palloc<double>(p, dsz * p->nb);
  const int tile_nt_alloc = p->use_lines ? 8 : (p->use_ws ? p->ws.NT : 0);
  const size_t ncol_pad = tile_nt_alloc ? (size_t)p->n_col_tiles * tile_nt_alloc : (size_t)p->ncol;
  if (p->use_fused) {
    const size_t welems = (size_t)p->n_col_tiles * p->fu_KP * FuCfg<49>::NT;
    p->d_W = palloc<double2>(p, welems);
    CK(cudaMemsetAsync(p->d_W, 0, welems * 16, s));  // padding rows
    p->d_wrow = dupload(wrow, s);
  } else if (p->use_tp) {
    p->d_W = palloc<double2>(p, (size_t)p->tp_KP * p->tp_ncolp);
    CK(cudaMemsetAsync(p->d_W, 0, (size_t)p->tp_KP * p->tp_ncolp * 16, s));  // padding rows
    p->d_wrow = dupload(wrow, s);
    p->d_qend = dupload(qend, s);
    if (p->n == 129) {
      p->d_r43 = palloc<double>(p, 2 * 576);
      k_r43_table<<<3, 192, 0, s>>>(p->d_r43);
      CKL();
    }
  } else {
    p->d_W = palloc<double2>(p, (size_t)p->NPQ * ncol_pad);
  }
  p->ct_fast = (size_t)p->NPQ * ncol_pad * 16 < (48u << 20);
  p->d_ubase = dupload(ubase, s);
  p->d_ustr = dupload(ustr, s);
  p->d_rou = dupload(rou, s);
  p->d_phase = dupload(phase, s);
  p->d_perm = dupload(perm, s);
  p->d_qoff = dupload(qoff, s);
  p->d_pq = dupload(pq, s);
  p->d_err = palloc<int>(p, 1);
  CK(cudaMemsetAsync(p->d_err, 0, sizeof(int), s));
  p->d_comps = dupload(p->comps, s);
  p->d_segs = dupload(p->segs, s);
  p->d_tiles = dupload(p->tiles, s);
  p->d_A = palloc<double>(p, (size_t)p->max_chunk * p->ldA);
  if (p->use_fused) {
    const size_t uelems = (size_t)(p->max_chunk + 7) / 8 * 8 * p->fu_upad;
    p->d_U = palloc<double2>(p, uelems);
    CK(cudaMemsetAsync(p->d_U, 0, uelems * 16, s));  // padding rows stay zero
  } else if (p->use_tp) {
    p->d_U = palloc<double2>(p, (size_t)p->max_chunk * p->tp_KP);
    CK(cudaMemsetAsync(p->d_U, 0, (size_t)p->max_chunk * p->tp_KP * 16, s));  // padding rows
  } else if (p->use_ws || p->use_lines) {
    const int gmt = p->use_lines ? 8 : p->ws.MT;
    const size_t groups = (size_t)(p->max_chunk + gmt - 1) / gmt;
    p->d_U = palloc<double2>(p, groups * (size_t)p->ws_stages.group_elems);
    CK(cudaMemsetAsync(p->d_U, 0, groups * (size_t)p->ws_stages.group_elems * 16, s));
  } else {
    p->d_U = palloc<double2>(p, (size_t)p->max_chunk * p->NPQ);
  }
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const size_t out_bytes = (size_t)p->n_slots * vol_bytes;
  // overlapped schedule (multi-chunk plans, SLSHT_CUDA_TP_OVERLAP=1): two T buffers
  if (p->use_tp) {
    const char* e = std::getenv("SLSHT_CUDA_TP_OVERLAP");
    p->tp_overlap = p->chunks.size() > 1 && e && e[0] == '1';  // measured slower: opt-in
    if (p->tp_overlap && !std::getenv("SLSHT_CUDA_TGEMM")) {
      p->tp_gv = 2;
      p->tp_bn = 32;
    }
    p->tp_t_elems = (size_t)p->max_chunk * p->n * p->tp_ncolp;
    // k_tpipe (kernels_tpipe.cuh): one persistent kernel over an L2-resident ring of T slots.
    // SLSHT_CUDA_TP_PIPE=0/1 forces either path; _CT / _NQG / _NSLOT / _FB override the shape.
    {
      const char* e = std::getenv("SLSHT_CUDA_TP_PIPE");
      p->tp_pipe = (p->n == 49 || p->n == 65) && p->tp_bn == TP_BN && !p->tp_overlap && e && e[0] == '1';
    }
    if (p->tp_pipe) {
      auto env_int = [](const char* name, int dflt) {
        const char* e = std::getenv(name);
        return e ? std::atoi(e) : dflt;
      };
      p->tp_pipe_fv = (env_int("SLSHT_CUDA_TP_FV", 0) || p->tp_lean) ? 1 : 0;
      p->tp_pipe_fn = p->tp_pipe_fv ? (p->n == 49 ? k_tpipe<49, 1> : k_tpipe<65, 1>)
                                    : (p->n == 49 ? k_tpipe<49, 0> : k_tpipe<65, 0>);
      const int nct = p->tp_ncolp / TP_BN;
      const size_t tile_bytes = (size_t)TG_BM * p->n * TP_BN * 16;
      int ct = env_int("SLSHT_CUDA_TP_CT", (int)std::max<size_t>(1, (20u << 20) / tile_bytes));
      ct = std::max(1, std::min(ct, nct));
      p->tp_ncg = (nct + ct - 1) / ct;
      p->tp_ct = (nct + p->tp_ncg - 1) / p->tp_ncg;
      p->tp_lag = std::max(1, env_int("SLSHT_CUDA_TP_LAG", 1));
      p->tp_nslot = std::max(p->tp_lag + 1, env_int("SLSHT_CUDA_TP_NSLOT", p->tp_lag + 2));
      p->tp_fb = env_int("SLSHT_CUDA_TP_FB", 8);
      if (p->tp_fb < 1 || TG_BM % p->tp_fb) p->tp_fb = 8;
      // q groups: consecutive q (whole k-step ranges) with about equal k-step counts
      std::vector<int> qe;  // k-step after each q's last
      for (size_t k = 0; k < qend.size(); ++k)
        if (qend[k] >= 0) qe.push_back((int)k + 1);
      const int nks = qe.empty() ? 0 : qe.back();
      int nqg = env_int("SLSHT_CUDA_TP_NQG", std::max(1, (nks + 11) / 22));
      nqg = std::max(1, std::min<int>(nqg, (int)qe.size()));
      std::vector<int> qg(1, 0);
      for (size_t i = 0; i < qe.size(); ++i) {
        const int g = (int)qg.size();  // closing group g (1-based) at its target
        if (g < nqg && (long long)qe[i] * nqg >= (long long)nks * g &&
            (int)(qe.size() - 1 - i) >= nqg - g)
          qg.push_back(qe[i]);
      }
      qg.push_back(nks);
      // (degenerate targets can leave fewer groups than asked for)
      qg.erase(std::unique(qg.begin(), qg.end()), qg.end());
      p->tp_nqg = (int)qg.size() - 1;
      p->d_qg = dupload(qg, s);
      p->tp_slot_elems = (size_t)TG_BM * p->n * p->tp_ct * TP_BN;
      p->tp_t_elems = p->tp_slot_elems * p->tp_nslot;
      const int nsub_max = ((p->max_chunk + TG_BM - 1) / TG_BM) * p->tp_ncg;
      p->tp_sync_ints = 1 + nsub_max * (1 + p->tp_ct);
      p->d_tp_sync = palloc<int>(p, p->tp_sync_ints);
      p->tp_pipe_smem = tpipe_smem_bytes(p->n, p->tp_KP);
    }
  }
  const size_t t_bytes = p->use_tp ? p->tp_t_elems * 16 * (p->tp_overlap ? 2 : 1) : 0;
  if (out_bytes + t_bytes + (64u << 20) > free_b)
    throw Status{SLSHT_ERR_VALIDATION,
                 "device output buffer does not fit in HBM (use the streaming ring mode)"};
  p->d_out = palloc<double2>(p, (size_t)p->n_slots * p->vstride);
  if (p->use_tp) p->d_T = palloc<double2>(p, t_bytes / 16);
  const int parts_per_tile = p->use_fused ? FuCfg<49>::EPW : ((p->tp_pipe && p->tp_pipe_fv) || p->tp_lean || p->tp_half) ? TP_THREADS / 32 : 1;
  p->d_partials = palloc<double>(p, (size_t)p->max_chunk * p->n_col_tiles * parts_per_tile * 8);
  p->digest_rows = coeff_count(p->lmax);
  p->d_digest = palloc<double>(p, (size_t)p->digest_rows * 8);
  for (int i = 0; i < 2; ++i) {
    CK(cudaEventCreateWithFlags(&p->ev_done[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&p->ev_copied[i], cudaEventDisableTiming));
  }
  for (auto& e : p->ev_stage) CK(cudaEventCreate(&e));
  for (auto& e : p->ev_lazy) CK(cudaEventCreate(&e));

  p->num_sms = prop.multiProcessorCount;
  if (4 * sizeof(double) * (p->L_g + 2) > 227 * 1024)
    throw Status{SLSHT_ERR_VALIDATION, "band limit L_f + L_h too large for the node recursion table"};
  for (int c0 = 0; c0 < p->NPQ; c0 += MG_COLS) {  // distinct q per modulated-SHT column tile
    const int c1 = std::min(p->NPQ, c0 + MG_COLS) - 1;
    if (pq[2 * c1] - pq[2 * c0] + 1 > MG_NQ)
      throw Status{SLSHT_ERR_VALIDATION, "internal: column tile spans too many orders q"};
  }
  if (p->use_fused) {
    p->couple_smem = FuCfg<49>::SMEM;
  } else if (p->use_lines) {
  } else if (p->use_tp) {
    p->tp_gemm_smem = tgemm_smem_bytes(p->tp_KP, p->tp_bn, tgemm_variant(p->tp_gv).nst,
                                       tgemm_variant(p->tp_gv).bm);
    p->tp_fft_smem = qfft_smem_bytes(p->n, p->tp_nt);
    p->couple_smem = std::max(p->tp_gemm_smem, p->tp_fft_smem);
    if (p->tp_overlap) {
      CK(cudaStreamCreateWithFlags(&p->fft_stream, cudaStreamNonBlocking));
      for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&p->ev_tg[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&p->ev_fft[i], cudaEventDisableTiming));
      }
    }
  } else if (p->use_reg) {
    p->couple_smem = couple_reg_smem_bytes(p->n);
  } else if (p->use_ws) {
    p->couple_smem = p->ws.smem;
  } else {
    p->couple_smem = couple_smem_bytes(p->n, p->MG, p->NG);
  }
  if (p->use_lines) {
    // execution split: the divisor of the digest split with the best balance over the SMs for
    // a full chunk (each extra segment costs a warm-up tile per group)
    const int nct = p->n_col_tiles, G = (p->max_chunk + 7) / 8, sms = p->num_sms;
    double best = -1.0;
    for (int ns = 1; ns <= p->lines_nseg_dig; ++ns) {
      if (p->lines_nseg_dig % ns) continue;
      const long long units = (long long)G * ns, rounds = (units + sms - 1) / sms;
      const double eff = (double)units / (double)(rounds * sms) *
                         (double)nct / (double)(nct + ns - 1);
      if (eff > best + 1e-9) {
        best = eff;
        p->lines_nseg = ns;
      }
    }
    if (const char* e = std::getenv("SLSHT_CUDA_NSEG")) {  // experiments
      const int ns = std::atoi(e);
      if (ns >= 1 && p->lines_nseg_dig % ns == 0) p->lines_nseg = ns;
    }
  }
  if (p->couple_smem > (size_t)prop.sharedMemPerBlockOptin)
    throw Status{SLSHT_ERR_VALIDATION, "window band limit too large for the shared-memory tile"};
  set_func_attributes(p);
  p->built = true;
  CK(cudaStreamSynchronize(s));
}

void record(slsht_cuda_plan* p, int idx) {
  if (p->profile) CK(cudaEventRecord(p->ev_stage[idx], p->stream));
}

// Coupling-kernel boundary of a single-chunk plan (0: start, 1: end).
void record_lazy(slsht_cuda_plan* p, int lazy_idx) {
  if (p->chunks.size() != 1) return;
  // inside a stream capture an external record becomes an event-record node, so graph replays
  // record it too (a plain record would only order the capture)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(p->stream, &cs));
  if (cs == cudaStreamCaptureStatusActive)
    CK(cudaEventRecordWithFlags(p->ev_lazy[lazy_idx], p->stream, cudaEventRecordExternal));
  else
    CK(cudaEventRecord(p->ev_lazy[lazy_idx], p->stream));
}

void accumulate(slsht_cuda_plan* p, int st, int a, int b) {
  if (!p->profile) return;
  CK(cudaEventSynchronize(p->ev_stage[b]));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, p->ev_stage[a], p->ev_stage[b]));
  p->stage_ms[st] += ms;
}

// The main stream waits for the window-table chain (before the first coupling launch).
void join_aux(slsht_cuda_plan* p) {
  if (!p->wtab_pending) return;
  CK(cudaStreamWaitEvent(p->stream, p->ev_wtab, 0));
  p->wtab_pending = false;
}

// Setup stage: every table that depends on f, h or the band limits (recomputed per call).
// Two independent chains: nodes -> Legendre window rows -> I table (needed by the modulated
// SHT) on the main stream, and Delta -> d tables -> window table W (needed only by the
// coupling) on the auxiliary stream, where it overlaps the node chain and the modulated SHT.
// The main stream waits for the last k_qfft/digest of the overlapped schedule.
void join_fft(slsht_cuda_plan* p) {
  if (p->fft_last < 0) return;
  CK(cudaStreamWaitEvent(p->stream, p->ev_fft[p->fft_last], 0));
  p->fft_last = -1;
}

void run_setup(slsht_cuda_plan* p) {
  cudaStream_t s = p->stream;
  const int L = p->L_h;
  record(p, 0);
  CK(cudaEventRecord(p->ev_fork, s));  // after the inputs' upload on s
  CK(cudaStreamWaitEvent(p->aux_stream, p->ev_fork, 0));
  {
    SetupMainParams sp{};
    sp.N = p->N;
    sp.L_h = L;
    sp.L_f = p->L_f;
    sp.n_nodes = p->n_nodes;
    sp.ld = p->ldA;
    sp.nbx = (p->n_nodes + 127) / 128;
    sp.ni = sp.nbx * (2 * p->L_f + 1);
    sp.nw = sp.nbx * p->n;
    sp.f = p->d_f;
    sp.qoff = p->d_qoff;
    sp.ncos = p->d_ncos;
    sp.nsin = p->d_nsin;
    sp.betaw = p->d_betaw;
    sp.lamh = p->d_lamh;
    sp.itab = reinterpret_cast<double*>(p->d_itab);
    sp.err = p->d_err;
    const int nnodes_blocks = (p->N + 1 + L + 1 + 3) / 4;  // 4 warps (weights) per block
    const size_t sm = sizeof(double) * std::max<size_t>(3 * (L + 1), 5 * (p->L_f + 1) + 1);
    k_glnodes<<<(p->n_nodes + 63) / 64, 64, 4 * sizeof(double) * (p->L_g + 2), s>>>(
        p->L_g + 1, p->n_nodes, p->d_ncos, p->d_nsin, p->d_weights);
    CKL();
    k_setup_main<<<sp.ni + sp.nw + nnodes_blocks, 128, sm, s>>>(sp);
    CKL();
  }
  cudaStream_t a = p->aux_stream;
  CK(launch_delta(L, p->d_delta, a, p->d_delta_ws));
  const int wmax = (2 * L + 1) * (2 * L + 1) * p->nb;
  k_dtab<<<dim3((wmax + 255) / 256, L + 1), 256, 0, a>>>(L, p->d_delta, p->d_rou, p->d_dtab);
  CKL();
  const int tile_nt = p->use_lines ? 8 : (p->use_ws ? p->ws.NT : 0);
  const int ncol_pad = p->use_fused ? p->n_col_tiles * FuCfg<49>::NT
                       : p->use_tp  ? p->tp_ncolp
                                    : (tile_nt ? p->n_col_tiles * tile_nt : p->ncol);
  k_wtab<<<dim3((ncol_pad + 127) / 128, std::min(p->NPQ, 65535)), 128, 0, a>>>(
      L, p->d_h, p->d_dtab, p->d_rou, p->d_pq, tile_nt, ncol_pad,
      (p->use_tp || p->use_fused) ? p->d_wrow : nullptr, p->d_W, p->use_fused ? p->fu_KP : 0);
  CKL();
  CK(cudaEventRecord(p->ev_wtab, a));
  p->wtab_pending = true;
  p->launches += 5;  // k_glnodes, k_setup_main, k_delta, k_dtab, k_wtab
  record(p, 1);
  accumulate(p, ST_SETUP, 0, 1);
}

void run_chunk(slsht_cuda_plan* p, const Chunk& ch) {
  cudaStream_t s = p->stream;
  if (&ch == &p->chunks.front()) p->fft_rec[0] = p->fft_rec[1] = false;  // a new call
  const CompRec* comps = p->d_comps + ch.comp0;
  record(p, 0);
  k_agen<<<dim3(ch.nseg, (p->ldA + 127) / 128), 128, 3 * (p->L_g + 1) * sizeof(double), s>>>(
      p->d_segs + ch.seg0, p->L_g, p->n_nodes, p->ldA, p->d_ncos, p->d_nsin, p->d_weights, p->d_A);
  CKL();
  record(p, 1);
  k_modgemm<<<dim3(ch.ntile, (p->NPQ + MG_COLS - 1) / MG_COLS), 256, MG_SMEM, s>>>(
      p->d_tiles + ch.tile0, p->n_nodes, p->ldA, p->L_f, p->NPQ, p->d_A, p->d_itab, p->d_lamh,
      p->d_pq, (p->use_lines || p->use_fused) ? 8 : (p->use_ws ? p->ws.MT : (p->use_tp ? 1 : 0)),
      p->ws_stages.group_elems,
      p->d_ubase, p->d_ustr, p->d_U);
  CKL();
  join_aux(p);
  record(p, 2);
  record_lazy(p, 0);
  CoupleParams prm{};
  prm.U = p->d_U;
  prm.W = p->d_W;
  prm.out = p->d_out;
  prm.partials = p->d_partials;
  prm.comps = comps;
  prm.count = ch.count;
  prm.L = p->L_h;
  prm.n = p->n;
  prm.nb = p->nb;
  prm.ncol = p->ncol;
  prm.NPQ = p->NPQ;
  prm.n_col_tiles = p->n_col_tiles;
  prm.vol = p->vol;
  prm.mirror = p->mirror;
  prm.qoff = p->d_qoff;
  prm.rou = p->d_rou;
  prm.perm = p->d_perm;
  prm.phase = p->d_phase;
  prm.betaw = p->d_betaw;
  prm.fft = p->fft;
  prm.generic_dft = p->generic_dft;
  const int MT = 8 * p->MG;
  if (p->use_fused) {
    FuParams fp{};
    fp.U = p->d_U;
    fp.W = p->d_W;
    fp.out = p->d_out;
    fp.partials = p->d_partials;
    fp.comps = comps;
    fp.count = ch.count;
    fp.n_groups = (ch.count + 7) / 8;
    fp.n_col_tiles = p->n_col_tiles;
    fp.ncol = p->ncol;
    fp.vol = p->vstride;
    fp.rpitch = p->rpitch;
    if (const char* e = std::getenv("SLSHT_CUDA_FU_EXP")) fp.exp = std::atoi(e);
    fp.mirror = p->mirror;
    fp.rou = p->d_rou;
    fp.betaw = p->d_betaw;
    const int grid = std::min(fp.n_groups, p->num_sms);
    k_fused<49><<<grid, FuCfg<49>::NTHREADS, p->couple_smem, s>>>(fp);
  } else if (p->use_lines) {
    LnParams lp{};
    lp.c = prm;
    lp.group_elems = p->ws_stages.group_elems;
    for (int i = 0; i < p->n; ++i) lp.urb[i] = p->lines_urb[i];
    lp.n_groups = (ch.count + 7) / 8;
    lp.nseg = p->lines_nseg;
    lp.nseg_dig = p->lines_nseg_dig;
    lp.partials = p->d_partials;
    lp.trace = nullptr;
    const int grid = std::min(lp.n_groups * lp.nseg, p->num_sms);
#ifdef SLSHT_WS_TRACE
    static long long* d_ltrace = nullptr;
    if (!d_ltrace) CK(cudaMalloc(&d_ltrace, 1024 * sizeof(long long)));
    CK(cudaMemsetAsync(d_ltrace, 0, 1024 * sizeof(long long), s));
    lp.trace = d_ltrace;
#endif
    p->lines_fn<<<grid, p->lines_threads, p->couple_smem, s>>>(lp);
#ifdef SLSHT_WS_TRACE
    {
      long long h[1024];
      CK(cudaMemcpyAsync(h, d_ltrace, sizeof(h), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      fprintf(stderr, "lines grid %d groups %d\n", grid, lp.n_groups);
      for (int k = 0; k < 60; ++k) {
        const long long* r = h + 8 * k;
        fprintf(stderr, "tile %3d: start %8lld tfree %5lld wfull %5lld mma %5lld radix %5lld sync %5lld last %5lld | stores_done %8lld\n",
                k, r[0] - h[0], r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4], r[6] - r[5], r[7] - h[0]);
      }
    }
#endif
  } else if (p->use_reg) {
    RegParams rp{};
    rp.c = prm;
    rp.n_tiles = p->n_col_tiles;
    // components per CTA: one wave of two CTAs per SM when the chunk allows (each CTA stages its W
    // tile once), 8..256
    {
      const int groups = std::max(1, 2 * p->num_sms / std::max(1, p->n_col_tiles));
      rp.cpb = std::min(256, std::max(8, (ch.count + groups - 1) / groups));
      if (const char* e = std::getenv("SLSHT_CUDA_REG_CPB")) rp.cpb = std::max(1, std::atoi(e));
    }
    const dim3 grid(p->n_col_tiles, (ch.count + rp.cpb - 1) / rp.cpb);
    k_couple_reg<17><<<grid, RG_THREADS, p->couple_smem, s>>>(rp);
  } else if (p->use_ws) {
    WsParams wp{};
    wp.c = prm;
    wp.st = p->ws_stages;
    wp.n_groups = (ch.count + MT - 1) / MT;
    wp.n_tiles = wp.n_groups * p->n_col_tiles;
    wp.ct_fast = p->ct_fast;
    wp.trace = nullptr;
#ifdef SLSHT_WS_TRACE
    static long long* d_trace = nullptr;
    if (!d_trace) CK(cudaMalloc(&d_trace, 2048 * sizeof(long long)));
    CK(cudaMemsetAsync(d_trace, 0, 2048 * sizeof(long long), s));
    wp.trace = d_trace;
#endif
    int grid = std::min(wp.n_tiles, p->num_sms);
    if (const char* g = std::getenv("SLSHT_CUDA_WS_GRID")) grid = std::max(1, std::min(grid, std::atoi(g)));
    p->ws.fn<<<grid, p->ws.threads, p->couple_smem, s>>>(wp);
#ifdef SLSHT_WS_TRACE
    {
      long long h[2048];
      CK(cudaMemcpyAsync(h, d_trace, sizeof(h), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      const long long t0 = h[0];
      for (int k = 0; k < 12; ++k)
        fprintf(stderr, "tile %2d grp %d: start %8lld turn %6lld mma %6lld sync %6lld fft %6lld epi %6lld\n",
                k, k & 1, h[6 * k] - t0, h[6 * k + 1] - h[6 * k], h[6 * k + 2] - h[6 * k + 1],
                h[6 * k + 3] - h[6 * k + 2], h[6 * k + 4] - h[6 * k + 3], h[6 * k + 5] - h[6 * k + 4]);
      for (int k = 0; k < 6; ++k) {
        fprintf(stderr, "  tile %d stages (wait/compute):", k);
        for (int st = 0; st < 8; ++st)
          fprintf(stderr, " %lld/%lld", h[384 + k * 16 + 2 * st], h[384 + k * 16 + 2 * st + 1]);
        fprintf(stderr, "\n");
      }
    }
#endif
  } else if (p->use_tp && p->tp_pipe) {
    TpParams tp{};
    tp.U = p->d_U;
    tp.W = p->d_W;
    tp.T = p->d_T;
    tp.qend = p->d_qend;
    tp.count = ch.count;
    tp.KP = p->tp_KP;
    tp.wpitch = p->tp_ncolp;
    tp.n = p->n;
    tp.sync = p->d_tp_sync;
    tp.qg = p->d_qg;
    tp.nblk = (ch.count + TG_BM - 1) / TG_BM;
    tp.ncg = p->tp_ncg;
    tp.CT = p->tp_ct;
    tp.nct = p->tp_ncolp / TP_BN;
    tp.nqg = p->tp_nqg;
    tp.nslot = p->tp_nslot;
    tp.fb = p->tp_fb;
    tp.lag = p->tp_lag;
    if (const char* e = std::getenv("SLSHT_CUDA_TP_EXP")) tp.exp = std::atoi(e);
    tp.slot_elems = (long long)p->tp_slot_elems;
    tp.tpitch = p->tp_ct * TP_BN;
    tp.out = p->d_out;
    tp.partials = p->d_partials;
    tp.comps = comps;
    tp.ncol = p->ncol;
    tp.n_tiles = p->tp_ntiles;
    tp.vol = p->vstride;
    tp.rpitch = p->rpitch;
    tp.mirror = p->mirror;
    tp.rou = p->d_rou;
    tp.perm = p->d_perm;
    tp.betaw = p->d_betaw;
    CK(cudaMemsetAsync(p->d_tp_sync, 0, sizeof(int) * (1 + (size_t)tp.nblk * tp.ncg * (1 + tp.CT)), s));
    int grid = 3 * p->num_sms;
    if (const char* g = std::getenv("SLSHT_CUDA_TP_GRID")) grid = std::max(1, std::atoi(g));
    p->tp_pipe_fn<<<grid, TP_THREADS, p->tp_pipe_smem, s>>>(tp);
    CKL();
    record(p, 5);
    p->launches += 1;
  } else if (p->use_tp) {
    // overlapped schedule: T buffer b = chunk parity; k_tgemm waits until the k_qfft that read
    // T[b] two chunks ago is done, and k_qfft + digest run on fft_stream
    const bool overlap = p->tp_overlap && !p->profile;
    const int b = overlap ? ch.buf : 0;
    if (overlap && p->fft_rec[b]) CK(cudaStreamWaitEvent(s, p->ev_fft[b], 0));
    TgParams tg{};
    tg.U = p->d_U + 4 * p->tp_ks_lo;
    tg.W = p->d_W + (size_t)4 * p->tp_ks_lo * p->tp_ncolp;
    tg.ustride = p->tp_KP;
    tg.T = p->d_T + b * p->tp_t_elems;
    tg.qend = p->d_qend;
    tg.count = ch.count;
    tg.KP = p->tp_KPsub;
    tg.ncolp = p->tp_ncolp;
    tg.n = p->n;
    const int tbm = tgemm_variant(p->tp_gv).bm;
    tg.col_fast = p->tp_col_fast ? 1 : 0;
    tg.t_stream = p->tp_t_stream;
    const int nbm = (ch.count + tbm - 1) / tbm, nbn = p->tp_ncolp / p->tp_bn;
    const dim3 tgrid(tg.col_fast ? nbn : nbm, tg.col_fast ? nbm : nbn);
    if (p->tp_gv == 2) {
      // the GEMM of chunk i+1 is dispatched ahead of the FFT CTAs of chunk i (one GEMM CTA per
      // SM, one FFT CTA beside it)
      cudaLaunchConfig_t lc{};
      lc.gridDim = tgrid;
      lc.blockDim = dim3(tgemm_threads(32, 2));
      lc.dynamicSmemBytes = p->tp_gemm_smem;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributePriority;
      int lo = 0, hi = 0;
      CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      at[0].val.priority = hi;
      lc.attrs = at;
      lc.numAttrs = 1;
      CK(cudaLaunchKernelEx(&lc, k_tgemm<32, 2, 4, 1>, tg));
    } else {
      const TgemmVariant tv = tgemm_variant(p->tp_gv);
      tv.fn<<<tgrid, tgemm_threads(tv.bn, tv.wnf, tv.bm), p->tp_gemm_smem, s>>>(tg);
    }
    CKL();
    record(p, 5);
    cudaStream_t fs = s;
    if (overlap) {
      CK(cudaEventRecord(p->ev_tg[b], s));
      CK(cudaStreamWaitEvent(p->fft_stream, p->ev_tg[b], 0));
      fs = p->fft_stream;
    }
    QfParams qf{};
    qf.T = tg.T;
    qf.out = p->d_out;
    qf.partials = p->d_partials;
    qf.comps = comps;
    qf.count = ch.count;
    qf.n = p->n;
    qf.ncol = p->ncol;
    qf.ncolp = p->tp_ncolp;
    qf.n_tiles = p->tp_ntiles;
    qf.vol = p->vstride;
    qf.rpitch = p->rpitch;
    qf.mirror = p->mirror;
    qf.rou = p->d_rou;
    qf.perm = p->d_perm;
    qf.betaw = p->d_betaw;
    qf.r43 = p->d_r43;
    qf.fft = p->fft;
    qf.generic_dft = p->generic_dft;
    qf.U = p->d_U;
    qf.W = p->d_W;
    qf.ustride = p->tp_KP;
    qf.rc_lo = p->tp_kc ? p->L_h + 1 - p->tp_kc : 0;
    qf.rc_hi = p->tp_kc ? p->L_h + 1 + p->tp_kc : 0;
    for (int r = 0; r < 16; ++r) {
      qf.rc_urow[r] = p->tp_rc_urow[r];
      qf.rc_k[r] = p->tp_rc_k[r];
    }
    p->tp_fft<<<dim3(p->tp_ntiles, ch.count), p->tp_threads, p->tp_fft_smem, fs>>>(qf);
    CKL();
    if (overlap) {
      k_digest<<<(ch.count + 3) / 4, 128, 0, fs>>>(comps, ch.count, p->n_col_tiles * ((p->tp_lean || p->tp_half) ? TP_THREADS / 32 : 1), p->n,
                                                    p->d_partials, p->mirror, p->d_digest);
      CKL();
      CK(cudaEventRecord(p->ev_fft[b], fs));
      p->fft_rec[b] = true;
      p->fft_last = b;
      p->launches += 3;
      return;
    }
    p->launches += 1;
  } else {
    dim3 grid(p->n_col_tiles, (ch.count + MT - 1) / MT);
    couple_kernel(p->n, p->MG, p->NG)<<<grid, couple_threads(p->n), p->couple_smem, s>>>(prm);
  }
  CKL();
  record(p, 3);
  record_lazy(p, 1);
  k_digest<<<(ch.count + 3) / 4, 128, 0, s>>>(comps, ch.count,
                                                  p->use_lines   ? p->lines_nseg_dig
                                                  : p->use_fused ? p->n_col_tiles * FuCfg<49>::EPW
                                                  : ((p->tp_pipe && p->tp_pipe_fv) || p->tp_lean || p->tp_half) ? p->n_col_tiles * (TP_THREADS / 32)
                                                                 : p->n_col_tiles,
                                                  p->n, p->d_partials, p->mirror, p->d_digest);
  CKL();
  record(p, 4);
  p->launches += 4;
  if (p->profile) {
    accumulate(p, ST_LEGENDRE, 0, 1);
    accumulate(p, ST_MODGEMM, 1, 2);
    if (p->use_tp) {
      accumulate(p, ST_COUPLE, 2, 5);
      accumulate(p, ST_QFFT, 5, 3);
    } else {
      accumulate(p, ST_COUPLE, 2, 3);
    }
    accumulate(p, ST_DIGEST, 3, 4);
  }
}

void load_inputs(slsht_cuda_plan* p, const double* f, const double* h, bool on_device) {
  // device inputs may live on another GPU of a multi-GPU plan: UVA resolves the direction
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDefault : cudaMemcpyHostToDevice;
  CK(cudaMemcpyAsync(p->d_f, f, sizeof(double) * 2 * coeff_count(p->L_f), kind, p->stream));
  CK(cudaMemcpyAsync(p->d_h, h, sizeof(double) * 2 * coeff_count(p->L_h), kind, p->stream));
}

// Digest rows of the plan's degree range [l_begin, l_end) are the contiguous rows
// [l_begin^2, l_end^2) of the coeff_index table; only those are copied out.
void copy_digests(slsht_cuda_plan* p, double* digests, bool on_device) {
  const size_t r0 = (size_t)p->l_begin * p->l_begin, r1 = (size_t)p->l_end * p->l_end;
  if (r1 <= r0) return;
  if (digests == p->d_digest) return;  // already in place
  // the gather of a multi-GPU plan: a device destination may be a peer GPU (NVLink P2P)
  CK(cudaMemcpyAsync(digests + 8 * r0, p->d_digest + 8 * r0, (r1 - r0) * 8 * sizeof(double),
                     on_device ? cudaMemcpyDefault : cudaMemcpyDeviceToHost, p->stream));
}

void check_numeric(slsht_cuda_plan* p) {
  int flag = 0;
  CK(cudaMemcpyAsync(&flag, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, p->stream));
  CK(cudaStreamSynchronize(p->stream));
  if (flag == 1) throw Status{SLSHT_ERR_NUMERIC, "theta weight imaginary residue exceeds 1e-12"};
  if (flag == 2) throw Status{SLSHT_ERR_NUMERIC, "beta weight imaginary residue exceeds 1e-12"};
}

template <class F>
int guarded(slsht_cuda_plan* p, F&& fn) {
  try {
    if (p) CK(cudaSetDevice(p->desc.device));
    if (p && p->parts.empty() && p->built) set_func_attributes(p);
    fn();
    if (p && p->parts.empty() && p->built) check_guards(p);
    return SLSHT_OK;
  } catch (const Status& st) {
    if (p) p->last_error = st.msg;
    else g_create_error = st.msg;
    return st.code;
  } catch (const CudaError& e) {
    if (p) p->last_error = e.msg;
    else g_create_error = e.msg;
    return SLSHT_ERR_DEVICE;
  } catch (const std::exception& e) {
    if (p) p->last_error = e.what();
    else g_create_error = e.what();
    return SLSHT_ERR_DEVICE;
  }
}

// Degree shards of a multi-GPU plan, balanced by computed components: c(l) = 2l+1 (full-m) or
// l+1 (real mode); bound k is the first degree whose cumulative count reaches k/parts of the
// total (the same rule as paper_1207_5558_b200.configs.shard_degrees).
std::vector<int> shard_bounds(int l_begin, int l_end, bool real_mode, int parts) {
  std::vector<double> cum(1, 0.0);
  for (int l = l_begin; l < l_end; ++l) cum.push_back(cum.back() + (real_mode ? l + 1.0 : 2.0 * l + 1.0));
  const double total = cum.back();
  std::vector<int> b(parts + 1);
  b[0] = l_begin;
  for (int k = 1; k < parts; ++k) {
    const double x = total * k / parts;
    const int i = (int)(std::lower_bound(cum.begin(), cum.end(), x) - cum.begin());
    b[k] = std::min(std::max(l_begin + i, l_begin), l_end);
  }
  b[parts] = l_end;
  for (int k = 1; k <= parts; ++k) b[k] = std::max(b[k], b[k - 1]);
  return b;
}

// A multi-GPU plan: one single-device plan per shard.
void build_group(slsht_cuda_plan* p) {
  const slsht_cuda_desc& d = p->desc;
  if (!d.devices) throw Status{SLSHT_ERR_VALIDATION, "n_devices > 1 needs a device list"};
  if (d.L_f < 0 || d.L_h < 0) throw Status{SLSHT_ERR_VALIDATION, "band limit must be non-negative"};
  p->L_f = d.L_f;
  p->L_h = d.L_h;
  p->L_g = d.L_f + d.L_h;
  p->lmax = d.lmax < 0 ? p->L_g : d.lmax;
  if (p->lmax > p->L_g)
    throw Status{SLSHT_ERR_VALIDATION, "fast engine computes components up to L_f + L_h only"};
  p->l_begin = std::max(0, d.l_begin);
  p->l_end = d.l_end < 0 ? p->lmax + 1 : std::min(d.l_end, p->lmax + 1);
  if (p->l_begin > p->l_end) throw Status{SLSHT_ERR_VALIDATION, "empty or inverted degree range"};
  p->real_mode = d.real_mode ? 1 : 0;
  p->emit_neg = d.emit_negative_m ? 1 : 0;
  p->mirror = p->real_mode && p->emit_neg;
  p->materialize = d.materialize ? 1 : 0;
  p->n = 2 * d.L_h + 1;
  p->nb = d.L_h + 1;
  p->vol = (long long)p->n * p->n * p->nb;
  p->part_bounds = shard_bounds(p->l_begin, p->l_end, p->real_mode, d.n_devices);
  for (int k = 0; k < d.n_devices; ++k) {
    slsht_cuda_desc pd = d;
    pd.n_devices = 0;
    pd.devices = nullptr;
    pd.device = d.devices[k];
    pd.stream = nullptr;
    pd.l_begin = p->part_bounds[k];
    pd.l_end = p->part_bounds[k + 1];
    slsht_cuda_plan* q = new slsht_cuda_plan();
    q->desc = pd;
    p->parts.push_back(q);  // freed with the group on failure
    build_plan(q);
    p->emitted += q->emitted;
    p->launches = 0;
  }
  p->desc.device = d.devices[0];
  // direct NVLink P2P for the gather (the copies also work without it, staged by the driver)
  for (int a = 0; a < d.n_devices; ++a)
    for (int b = 0; b < d.n_devices; ++b) {
      int ok = 0;
      if (d.devices[a] == d.devices[b] ||
          cudaDeviceCanAccessPeer(&ok, d.devices[a], d.devices[b]) != cudaSuccess || !ok)
        continue;
      cudaSetDevice(d.devices[a]);
      if (cudaDeviceEnablePeerAccess(d.devices[b], 0) != cudaSuccess) cudaGetLastError();
    }
  CK(cudaSetDevice(p->desc.device));
}

long long group_computed(const slsht_cuda_plan* p) {
  long long c = 0;
  for (const slsht_cuda_plan* q : p->parts) c += (long long)q->comps.size();
  return c;
}

void run_forward_device(slsht_cuda_plan* p, const double* f, const double* h,
                        int inputs_on_device, double* digests, int digests_on_device,
                        int synchronize);

// Group forward_device: every shard is enqueued on its own device and stream, then each copies
// its digest rows into the caller's table (the final gather); the call returns after all
// shards finished.
void run_group_device(slsht_cuda_plan* p, const double* f, const double* h, int inputs_on_device,
                      double* digests, int digests_on_device) {
  p->launches = 0;
  for (slsht_cuda_plan* q : p->parts) {
    CK(cudaSetDevice(q->desc.device));
    run_forward_device(q, f, h, inputs_on_device, nullptr, 0, 0);
    if (digests) copy_digests(q, digests, digests_on_device != 0);
  }
  for (slsht_cuda_plan* q : p->parts) {
    CK(cudaSetDevice(q->desc.device));
    check_numeric(q);  // synchronizes the shard's stream
    p->launches += q->launches;
  }
  CK(cudaSetDevice(p->desc.device));
}

// tag passed as the sink of slsht_cuda_forward by slsht_cuda_forward_scatter (user = HostScatter)
void scatter_marker(int, int, const double*, void*) {}

struct LockedSink {
  slsht_host_sink sink;
  void* user;
  std::mutex* mu;
};
void locked_sink(int l, int m, const double* vol, void* u) {
  LockedSink* s = static_cast<LockedSink*>(u);
  std::lock_guard<std::mutex> lock(*s->mu);
  s->sink(l, m, vol, s->user);
}

// Materializing delivery: every emitted volume is copied to its own destination (disjoint
// rows), so the copies need no serialization and run on several host threads per chunk.
struct HostScatter {
  double* const* targets = nullptr;  // per coeff_index(l, m), or
  double* base = nullptr;            // one array of rows (slsht_copy_target)
  long long first_index = 0, count = 0;
  int threads = 0;
  std::atomic<long long> delivered{0}, dropped{0};
  double* dest(int l, int m, long long vol) const {
    const long long idx = (long long)coeff_index(l, m);
    if (targets) return idx < count ? targets[idx] : nullptr;
    const long long row = idx - first_index;
    return (row >= 0 && row < count && base) ? base + 2 * row * vol : nullptr;
  }
};
int host_threads(int asked) {
  if (asked <= 0) {
    if (const char* e = std::getenv("SLSHT_CUDA_HOST_THREADS")) asked = std::atoi(e);
  }
  if (asked <= 0) asked = (int)std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
  return std::min(asked, 64);
}

void run_forward_sink(slsht_cuda_plan* p, const double* f, const double* h, slsht_host_sink sink,
                      void* user, HostScatter* scatter = nullptr);
void run_capture(slsht_cuda_plan* p, const double* f, const double* h, double* digests, int count,
                 const int* l, const int* m, const int* slot, double* volumes);

}  // namespace

extern "C" {

int slsht_cuda_plan_create(const slsht_cuda_desc* desc, slsht_cuda_plan** out) {
  if (!desc || !out) {
    g_create_error = "null argument";
    return SLSHT_ERR_VALIDATION;
  }
  *out = nullptr;
  slsht_cuda_plan* p = new slsht_cuda_plan();
  p->desc = *desc;
  int rc = SLSHT_OK;
  try {
    if (desc->n_devices > 1) build_group(p);
    else build_plan(p);
  } catch (const Status& st) {
    g_create_error = st.msg;
    rc = st.code;
  } catch (const CudaError& e) {
    g_create_error = e.msg;
    rc = SLSHT_ERR_DEVICE;
  } catch (const std::exception& e) {
    g_create_error = e.what();
    rc = SLSHT_ERR_DEVICE;
  }
  if (rc != SLSHT_OK) {
    free_plan(p);
    return rc;
  }
  *out = p;
  return SLSHT_OK;
}

void slsht_cuda_plan_destroy(slsht_cuda_plan* p) {
  if (p) cudaSetDevice(p->desc.device);
  free_plan(p);
}

const char* slsht_cuda_last_error(const slsht_cuda_plan* p) {
  return p ? p->last_error.c_str() : g_create_error.c_str();
}

}  // extern "C"

namespace {

void run_forward_device(slsht_cuda_plan* p, const double* f, const double* h,
                        int inputs_on_device, double* digests, int digests_on_device,
                        int synchronize) {
  {
    if (!synchronize && digests && !digests_on_device)
      throw Status{SLSHT_ERR_VALIDATION, "asynchronous forward needs device digests"};
    p->launches = 0;
    for (double& v : p->stage_ms) v = 0.0;
    load_inputs(p, f, h, inputs_on_device != 0);
    // The device work only touches plan-owned buffers, so it is captured once into a CUDA graph
    // (both streams, with their fork/join events) and replayed: no per-kernel launch overhead.
    // A single-chunk graph carries its stage events as event-record nodes, so every call's
    // stage times are available (slsht_cuda_stage_times); profiling takes the stream path.
    const bool use_graph = !p->profile && std::getenv("SLSHT_CUDA_NO_GRAPH") == nullptr;
    if (use_graph && !p->graph) {
      CK(cudaStreamBeginCapture(p->stream, cudaStreamCaptureModeThreadLocal));
      cudaGraph_t graph = nullptr;
      try {
        run_setup(p);
        for (const Chunk& ch : p->chunks) run_chunk(p, ch);
        join_fft(p);
        join_aux(p);
      } catch (...) {
        cudaStreamEndCapture(p->stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      CK(cudaStreamEndCapture(p->stream, &graph));
      const cudaError_t e = cudaGraphInstantiate(&p->graph, graph, 0);
      cudaGraphDestroy(graph);
      CK(e);
      p->graph_launches = p->launches;
      p->launches = 0;
    }
    p->lazy_valid = p->chunks.size() == 1;
    if (use_graph) {
      CK(cudaGraphLaunch(p->graph, p->stream));
      p->launches += p->graph_launches;
    } else {
      run_setup(p);
      for (const Chunk& ch : p->chunks) run_chunk(p, ch);
      join_fft(p);
      join_aux(p);
    }
    if (digests) copy_digests(p, digests, digests_on_device != 0);
    if (synchronize) check_numeric(p);
  }
}

void run_capture(slsht_cuda_plan* p, const double* f, const double* h, double* digests, int count,
                 const int* l, const int* m, const int* slot, double* volumes) {
  {
    // locate every request: (chunk, slot) of the component or of its conjugate mirror
    struct Req {
      size_t chunk;
      long long slot;
      int i;
    };
    std::vector<Req> reqs;
    for (int i = 0; i < count; ++i) {
      bool found = false;
      for (size_t ci = 0; ci < p->chunks.size() && !found; ++ci) {
        const Chunk& ch = p->chunks[ci];
        for (int k = 0; k < ch.count; ++k) {
          const CompRec& r = p->comps[ch.comp0 + k];
          if (r.l != l[i]) continue;
          if (r.m == m[i]) {
            reqs.push_back({ci, r.slot, i});
            found = true;
            break;
          }
          if (r.mslot >= 0 && -r.m == m[i]) {
            reqs.push_back({ci, r.mslot, i});
            found = true;
            break;
          }
        }
      }
      if (!found) throw Status{SLSHT_ERR_VALIDATION, "requested component not produced by this plan"};
    }
    p->launches = 0;
    for (double& v : p->stage_ms) v = 0.0;
    load_inputs(p, f, h, false);
    run_setup(p);
    for (size_t ci = 0; ci < p->chunks.size(); ++ci) {
      run_chunk(p, p->chunks[ci]);
      join_fft(p);
      for (const Req& r : reqs)
        if (r.chunk == ci)
          CK(cudaMemcpy2DAsync(volumes + 2 * (size_t)(slot ? slot[r.i] : r.i) * p->vol,
                               (size_t)p->ncol * 16, p->d_out + (size_t)r.slot * p->vstride,
                               (size_t)p->rpitch * 16, (size_t)p->ncol * 16, (size_t)p->n,
                               cudaMemcpyDeviceToHost, p->stream));
    }
    if (digests) copy_digests(p, digests, false);
    check_numeric(p);
  }
}

void run_forward_sink(slsht_cuda_plan* p, const double* f, const double* h, slsht_host_sink sink,
                      void* user, HostScatter* scatter) {
  {
    if (p->materialize)
      throw Status{SLSHT_ERR_VALIDATION, "host-sink forward needs a streaming (ring) plan"};
    p->launches = 0;
    for (double& v : p->stage_ms) v = 0.0;
    const int per = p->mirror ? 2 : 1;
    const size_t chunk_bytes = (size_t)per * p->max_chunk * p->vol * 16;
    if (p->stage_bytes < chunk_bytes) {
      for (int i = 0; i < 2; ++i) {
        if (p->h_stage[i]) cudaFreeHost(p->h_stage[i]);
        p->h_stage[i] = nullptr;
        CK(cudaMallocHost(&p->h_stage[i], chunk_bytes));
      }
      p->stage_bytes = chunk_bytes;
    }
    load_inputs(p, f, h, false);
    run_setup(p);
    check_numeric(p);
    auto deliver = [&](size_t ci) {
      const Chunk& ch = p->chunks[ci];
      CK(cudaEventSynchronize(p->ev_copied[ch.buf]));
      const double2* base = p->h_stage[ch.buf];
      if (scatter) {
        // disjoint destinations: the chunk's volumes are copied by several host threads
        const size_t vbytes = (size_t)p->vol * 16;
        auto work = [&](int t, int nt) {
          long long del = 0, drop = 0;
          for (int k = t; k < ch.count; k += nt) {
            const CompRec& r = p->comps[ch.comp0 + k];
            for (int mir = 0; mir < (r.mslot >= 0 ? 2 : 1); ++mir) {
              double* dst = scatter->dest(r.l, mir ? -r.m : r.m, p->vol);
              if (!dst) {
                ++drop;
                continue;
              }
              std::memcpy(dst, base + (size_t)(mir ? p->max_chunk + k : k) * p->vol, vbytes);
              ++del;
            }
          }
          scatter->delivered += del;
          scatter->dropped += drop;
        };
        const int nt = (int)std::max<long long>(
            1, std::min<long long>(scatter->threads, (long long)ch.count * (long long)vbytes >> 20));
        std::vector<std::thread> pool;
        for (int t = 1; t < nt; ++t) pool.emplace_back(work, t, nt);
        work(0, nt);
        for (auto& th : pool) th.join();
        return;
      }
      for (int k = 0; k < ch.count; ++k) {
        const CompRec& r = p->comps[ch.comp0 + k];
        sink(r.l, r.m, reinterpret_cast<const double*>(base + (size_t)k * p->vol), user);
        if (r.mslot >= 0)
          sink(r.l, -r.m,
               reinterpret_cast<const double*>(base + (size_t)(p->max_chunk + k) * p->vol), user);
      }
    };
    for (size_t ci = 0; ci < p->chunks.size(); ++ci) {
      const Chunk& ch = p->chunks[ci];
      // the ring half and host stage of this chunk were last used by chunk ci-2
      if (ci >= 2) deliver(ci - 2);
      CK(cudaStreamWaitEvent(p->stream, p->ev_copied[ch.buf], 0));
      run_chunk(p, ch);
      CK(cudaEventRecord(p->ev_done[ch.buf], p->stream));
      CK(cudaStreamWaitEvent(p->copy_stream, p->ev_done[ch.buf], 0));
      if (p->fft_last >= 0) CK(cudaStreamWaitEvent(p->copy_stream, p->ev_fft[ch.buf], 0));
      // the ring's pitched rows to packed So3Volumes in the host stage
      const double2* src = p->d_out + (size_t)ch.buf * per * p->max_chunk * p->vstride;
      const size_t rw = (size_t)p->ncol * 16, sp = (size_t)p->rpitch * 16;
      const size_t rows = (size_t)ch.count * p->n;
      CK(cudaMemcpy2DAsync(p->h_stage[ch.buf], rw, src, sp, rw, rows, cudaMemcpyDeviceToHost,
                           p->copy_stream));
      if (per == 2)
        CK(cudaMemcpy2DAsync(p->h_stage[ch.buf] + (size_t)p->max_chunk * p->vol, rw,
                             src + (size_t)p->max_chunk * p->vstride, sp, rw, rows,
                             cudaMemcpyDeviceToHost, p->copy_stream));
      CK(cudaEventRecord(p->ev_copied[ch.buf], p->copy_stream));
    }
    const size_t nc = p->chunks.size();
    if (nc >= 2) deliver(nc - 2);
    if (nc >= 1) deliver(nc - 1);
    join_fft(p);
    CK(cudaStreamSynchronize(p->stream));
  }
}

}  // namespace

extern "C" {

int slsht_cuda_forward_device(slsht_cuda_plan* p, const double* f, const double* h,
                              int inputs_on_device, double* digests, int digests_on_device,
                              int synchronize) {
  if (!p) return SLSHT_ERR_VALIDATION;
  return guarded(p, [&] {
    if (p->group()) run_group_device(p, f, h, inputs_on_device, digests, digests_on_device);
    else run_forward_device(p, f, h, inputs_on_device, digests, digests_on_device, synchronize);
  });
}

int slsht_cuda_forward_capture(slsht_cuda_plan* p, const double* f, const double* h,
                               double* digests, int count, const int* l, const int* m,
                               double* volumes) {
  if (!p) return SLSHT_ERR_VALIDATION;
  return guarded(p, [&] {
    if (!p->group()) {
      run_capture(p, f, h, digests, count, l, m, nullptr, volumes);
      return;
    }
    // each request goes to the shard that owns its degree; volumes keep the caller's order
    std::vector<int> owner(count, -1);
    for (int i = 0; i < count; ++i)
      for (size_t k = 0; k < p->parts.size(); ++k)
        if (l[i] >= p->part_bounds[k] && l[i] < p->part_bounds[k + 1]) owner[i] = (int)k;
    for (int i = 0; i < count; ++i)
      if (owner[i] < 0) throw Status{SLSHT_ERR_VALIDATION, "requested component not produced by this plan"};
    for (size_t k = 0; k < p->parts.size(); ++k) {
      std::vector<int> ls, ms, slot;
      for (int i = 0; i < count; ++i)
        if (owner[i] == (int)k) {
          ls.push_back(l[i]);
          ms.push_back(m[i]);
          slot.push_back(i);
        }
      slsht_cuda_plan* q = p->parts[k];
      CK(cudaSetDevice(q->desc.device));
      run_capture(q, f, h, digests, (int)ls.size(), ls.data(), ms.data(), slot.data(), volumes);
    }
    CK(cudaSetDevice(p->desc.device));
  });
}

int slsht_cuda_forward(slsht_cuda_plan* p, const double* f, const double* h, slsht_host_sink sink,
                       void* user) {
  if (!p) return SLSHT_ERR_VALIDATION;
  return guarded(p, [&] {
    // the library's own copy sink writes disjoint rows: it is run as a parallel scatter
    HostScatter sc;
    HostScatter* scatter = nullptr;
    slsht_copy_target* ct = nullptr;
    if (sink == slsht_cuda_copy_sink && user) {
      ct = static_cast<slsht_copy_target*>(user);
      sc.base = ct->base;
      sc.first_index = ct->first_index;
      sc.count = ct->count;
      sc.threads = host_threads(0);
      scatter = &sc;
    } else if (sink == scatter_marker && user) {
      scatter = static_cast<HostScatter*>(user);
    }
    if (scatter && p->group())
      scatter->threads = std::max(1, scatter->threads / (int)p->parts.size());
    auto finish = [&] {
      if (ct) {
        ct->delivered += sc.delivered.load();
        ct->dropped += sc.dropped.load();
      }
    };
    if (!p->group()) {
      run_forward_sink(p, f, h, sink, user, scatter);
      finish();
      return;
    }
    // one host thread per shard; sink calls serialized under one mutex (transform.cpp:282-284)
    std::mutex mu;
    LockedSink ls{sink, user, &mu};
    std::vector<std::thread> pool;
    std::vector<Status> errors(p->parts.size(), Status{SLSHT_OK, ""});
    for (size_t k = 0; k < p->parts.size(); ++k)
      pool.emplace_back([&, k] {
        slsht_cuda_plan* q = p->parts[k];
        try {
          CK(cudaSetDevice(q->desc.device));
          run_forward_sink(q, f, h, locked_sink, &ls, scatter);
        } catch (const Status& st) {
          errors[k] = st;
        } catch (const CudaError& e) {
          errors[k] = Status{SLSHT_ERR_DEVICE, e.msg};
        } catch (const std::exception& e) {
          errors[k] = Status{SLSHT_ERR_DEVICE, e.what()};
        }
      });
    for (auto& t : pool) t.join();
    for (const Status& st : errors)
      if (st.code != SLSHT_OK) throw st;
    finish();
  });
}

int slsht_cuda_forward_scatter(slsht_cuda_plan* p, const double* f, const double* h,
                               double* const* targets, long long n_targets, int threads,
                               long long* delivered) {
  if (!p) return SLSHT_ERR_VALIDATION;
  if (!targets || n_targets < 0) {
    p->last_error = "null target table";
    return SLSHT_ERR_VALIDATION;
  }
  HostScatter sc;
  sc.targets = targets;
  sc.count = n_targets;
  sc.threads = host_threads(threads);
  const int rc = slsht_cuda_forward(p, f, h, scatter_marker, &sc);
  if (delivered) *delivered = sc.delivered.load();
  return rc;
}

void slsht_cuda_copy_sink(int l, int m, const double* volume, void* target) {
  slsht_copy_target* t = static_cast<slsht_copy_target*>(target);
  if (!t || !volume) return;
  const long long row = (long long)coeff_index(l, m) - t->first_index;
  if (row < 0 || row >= t->count || !t->base) {
    ++t->dropped;
    return;
  }
  std::memcpy(t->base + 2 * row * t->volume_elems, volume, sizeof(double) * 2 * t->volume_elems);
  ++t->delivered;
}

const double* slsht_cuda_device_output(const slsht_cuda_plan* p) {
  // a multi-GPU plan has no single device buffer
  return (p && p->materialize && !p->group()) ? reinterpret_cast<const double*>(p->d_out) : nullptr;
}
long long slsht_cuda_volume_elems(const slsht_cuda_plan* p) { return p ? p->vol : 0; }
long long slsht_cuda_computed_count(const slsht_cuda_plan* p) {
  if (!p) return 0;
  return p->group() ? group_computed(p) : (long long)p->comps.size();
}
long long slsht_cuda_emitted_count(const slsht_cuda_plan* p) { return p ? p->emitted : 0; }
void* slsht_cuda_stream(const slsht_cuda_plan* p) { return p ? (void*)p->stream : nullptr; }
long long slsht_cuda_launch_count(const slsht_cuda_plan* p) { return p ? p->launches : 0; }

int slsht_cuda_set_profiling(slsht_cuda_plan* p, int enable) {
  if (!p) return SLSHT_ERR_VALIDATION;
  p->profile = enable != 0;
  for (slsht_cuda_plan* q : p->parts) q->profile = enable != 0;
  return SLSHT_OK;
}

int slsht_cuda_stage_times(const slsht_cuda_plan* p, double* out_ms, int n) {
  if (!p || !out_ms) return 0;
  const int k = std::min(n, (int)ST_COUNT);
  for (int i = 0; i < k; ++i) {
    out_ms[i] = p->stage_ms[i];
    for (const slsht_cuda_plan* q : p->parts) out_ms[i] = std::max(out_ms[i], q->stage_ms[i]);
  }
  return k;
}

int slsht_cuda_device_count(void) {
  int n = 0, usable = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10) ++usable;
  }
  return usable;
}

int slsht_cuda_shard_bounds(int l_begin, int l_end, int real_mode, int parts, int* bounds) {
  if (parts < 1 || !bounds || l_begin < 0 || l_end < l_begin) return SLSHT_ERR_VALIDATION;
  const std::vector<int> b = shard_bounds(l_begin, l_end, real_mode != 0, parts);
  std::copy(b.begin(), b.end(), bounds);
  return SLSHT_OK;
}

int slsht_cuda_kernel_time(const slsht_cuda_plan* p, double* ms_out) {
  if (p && ms_out && p->group()) {  // the slowest shard
    double worst = -1.0;
    for (const slsht_cuda_plan* q : p->parts) {
      double ms = 0.0;
      if (slsht_cuda_kernel_time(q, &ms) != SLSHT_OK) return SLSHT_ERR_VALIDATION;
      worst = std::max(worst, ms);
    }
    *ms_out = worst;
    return SLSHT_OK;
  }
  if (!p || !ms_out || !p->lazy_valid) return SLSHT_ERR_VALIDATION;
  float ms = 0.f;
  if (cudaEventSynchronize(p->ev_lazy[1]) != cudaSuccess ||
      cudaEventElapsedTime(&ms, p->ev_lazy[0], p->ev_lazy[1]) != cudaSuccess) {
    cudaGetLastError();  // leave no error behind for the caller's runtime
    return SLSHT_ERR_DEVICE;
  }
  *ms_out = ms;
  return SLSHT_OK;
}

// ---------------------------------------------------------------------------------------------
// Slepian window (window.cpp:44-198) on the device; see window_solver.cuh.
namespace {

// theta_weights(N) (grids.cpp:76-92), the reference's serial k order: the same weights
std::vector<double> host_theta_weights(int N) {
  std::vector<double> w(N + 1);
  for (int t = 0; t <= N; ++t) {
    const double theta = kPi * (2 * t + 1) / (2 * N + 1);
    double sr = 0.0, si = 0.0;
    for (int k = -N; k <= N; ++k) {
      const int mk = -k;
      double wr = 0.0, wi = 0.0;
      if (mk == 0) wr = 2.0;
      else if (mk == 1) wi = kPi / 2.0;
      else if (mk == -1) wi = -kPi / 2.0;
      else if ((mk & 1) == 0) wr = 2.0 / (1.0 - (double)mk * mk);
      if (wr == 0.0 && wi == 0.0) continue;
      const double ck = std::cos(k * theta);
      sr += wr * ck;
      si += wi * ck;
    }
    if (std::fabs(si) >= 1e-12)
      throw Status{SLSHT_ERR_NUMERIC, "theta weight imaginary residue exceeds 1e-12"};
    w[t] = (t < N) ? 2.0 * sr / (2 * N + 1) : sr / (2 * N + 1);
  }
  return w;
}

double angular_distance(double t1, double p1, double t2, double p2) {
  const double c = std::sin(t1) * std::sin(t2) * std::cos(p1 - p2) + std::cos(t1) * std::cos(t2);
  return std::acos(std::min(1.0, std::max(-1.0, c)));
}

}  // namespace

int slsht_cuda_eigenfunction_window(int device, double theta_c, double a, int band_limit,
                                    int oversample, double* coeffs, double* lambda_out) {
  std::vector<void*> allocs;
  auto cleanup = [&]() {
    for (void* q : allocs) cudaFree(q);
  };
  try {
    if (!(theta_c >= 0.0) || !(theta_c <= a) || !(a <= kPi / 2.0))  // window.cpp:28-33
      throw Status{SLSHT_ERR_VALIDATION, "elliptical region requires 0 <= theta_c <= a <= pi/2"};
    if (band_limit < 0) throw Status{SLSHT_ERR_VALIDATION, "band limit must be non-negative"};
    if (oversample < 2) throw Status{SLSHT_ERR_VALIDATION, "oversample must be at least 2"};
    if (!coeffs || !lambda_out) throw Status{SLSHT_ERR_VALIDATION, "null output"};
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
      throw Status{SLSHT_ERR_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    CK(cudaSetDevice(device));
    const bool prof = std::getenv("SLSHT_CUDA_PROFILE") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t0 = now();
    auto lap = [&](const char* what) {
      if (!prof) return;
      CK(cudaDeviceSynchronize());
      fprintf(stderr, "window: %-24s %.3f s\n", what,
              std::chrono::duration<double>(now() - t0).count());
    };
    const int L = band_limit, dim = coeff_count(L), N = oversample * L;
    const int n_phi = 2 * N + 1;
    const std::vector<double> ring = host_theta_weights(N);
    const double dphi = 2.0 * kPi / n_phi;
    std::vector<double> st, sp, sw;  // mask samples (window.cpp:64-71)
    for (int t = 0; t <= N; ++t) {
      const double theta = kPi * (2 * t + 1) / (2 * N + 1);
      for (int q = 0; q < n_phi; ++q) {
        const double phi = 2.0 * kPi * q / n_phi;
        const double d = angular_distance(theta, phi, theta_c, 0.0) +
                         angular_distance(theta, phi, theta_c, kPi);
        if (d <= 2.0 * a) {
          st.push_back(theta);
          sp.push_back(phi);
          sw.push_back(ring[t] * dphi);
        }
      }
    }
    const int S = (int)st.size();
    lap("mask (host)");
    if (S < 10)
      throw Status{SLSHT_ERR_VALIDATION,
                   "region mask holds fewer than 10 grid samples; raise oversample or widen the "
                   "region"};
    auto dal = [&](size_t bytes) {
      void* q = nullptr;
      CK(cudaMalloc(&q, bytes));
      allocs.push_back(q);
      return q;
    };
    double* d_t = (double*)dal(sizeof(double) * S);
    double* d_p = (double*)dal(sizeof(double) * S);
    double* d_w = (double*)dal(sizeof(double) * S);
    CK(cudaMemcpy(d_t, st.data(), sizeof(double) * S, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_p, sp.data(), sizeof(double) * S, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_w, sw.data(), sizeof(double) * S, cudaMemcpyHostToDevice));
    double2* d_Y = (double2*)dal(sizeof(double2) * (size_t)S * dim);
    double2* d_B = (double2*)dal(sizeof(double2) * (size_t)S * dim);
    double2* d_K = (double2*)dal(sizeof(double2) * (size_t)dim * dim);
    double2* d_v = (double2*)dal(sizeof(double2) * dim);
    double2* d_x = (double2*)dal(sizeof(double2) * dim);
    double2* d_dn = (double2*)dal(sizeof(double2) * 2);  // v^H x, ||x||
    const int ny = S * (2 * L + 1);
    k_window_y<<<(ny + 127) / 128, 128>>>(L, S, d_t, d_p, d_Y);
    CKL();
    const size_t nb = (size_t)S * dim;
    k_window_scale<<<(unsigned)((nb + 255) / 256), 256>>>(dim, S, d_w, d_Y, d_B);
    CKL();
    // row-major Y[s][c] is the column-major dim x S matrix A; K (row-major) = A B^H
    // (column-major), B = A diag(w): K[r][c] = sum_s conj(Y[s][r]) w_s Y[s][c]
    // (blas_fp64.cuh: DMMA complex GEMM)
    CK(zgemm(kOpN, kOpC, dim, dim, S, d_Y, dim, d_B, dim, d_K, dim, 0));
    const size_t nk = (size_t)dim * dim;
    k_window_symmetrize<<<(unsigned)((nk + 255) / 256), 256>>>(dim, d_K);
    CKL();
    lap("Y, K (device)");
    // power iteration (window.cpp:129-157), v0 = e_(0,0)
    std::vector<double2> v(dim, make_double2(0.0, 0.0));
    v[0] = make_double2(1.0, 0.0);
    CK(cudaMemcpy(d_v, v.data(), sizeof(double2) * dim, cudaMemcpyHostToDevice));
    double lambda_prev = -1.0, lambda = 0.0;
    bool converged = false;
    for (int it = 0; it < 100000; ++it) {
      // w = K v: K row-major is the column-major K^T
      k_zgemv_t<<<(dim * 32 + 255) / 256, 256>>>(dim, d_K, dim, d_v, d_x);
      CKL();
      k_zdot_nrm<<<1, 1024>>>(dim, d_v, d_x, d_dn);
      CKL();
      double2 dn[2];
      CK(cudaMemcpy(dn, d_dn, sizeof dn, cudaMemcpyDeviceToHost));
      const double nw = dn[1].x;
      lambda = dn[0].x;
      if (nw == 0.0) throw Status{SLSHT_ERR_NUMERIC, "power iteration collapsed to zero"};
      k_zscale_inv<<<(dim + 255) / 256, 256>>>(dim, d_dn, d_x);
      CKL();
      std::swap(d_v, d_x);
      if (it > 0 && std::fabs(lambda - lambda_prev) <= 1e-12 * std::fabs(lambda)) {
        converged = true;
        break;
      }
      lambda_prev = lambda;
    }
    if (!converged)
      throw Status{SLSHT_ERR_NUMERIC, "power iteration did not converge within 1e5 steps"};
    lap("power iteration");
    CK(cudaMemcpy(v.data(), d_v, sizeof(double2) * dim, cudaMemcpyDeviceToHost));
    // north-pole phase, exact conjugate symmetry, unit norm (window.cpp:159-196)
    std::vector<std::complex<double>> z(dim);
    for (int i = 0; i < dim; ++i) z[i] = {v[i].x, v[i].y};
    std::complex<double> pole{0.0, 0.0};
    for (int l = 0; l <= L; ++l) pole += z[l * l + l] * std::sqrt((2.0 * l + 1.0) / (4.0 * kPi));
    if (std::abs(pole) > 0.0) {
      const std::complex<double> phase = std::conj(pole) / std::abs(pole);
      for (auto& x : z) x *= phase;
    }
    std::vector<std::complex<double>> c(dim);
    for (int l = 0; l <= L; ++l) {
      c[l * l + l] = {z[l * l + l].real(), 0.0};
      for (int m = 1; m <= l; ++m) {
        const double sign = (m & 1) ? -1.0 : 1.0;
        const std::complex<double> sym = 0.5 * (z[l * l + l + m] + sign * std::conj(z[l * l + l - m]));
        c[l * l + l + m] = sym;
        c[l * l + l - m] = sign * std::conj(sym);
      }
    }
    double norm = 0.0;
    for (const auto& x : c) norm += std::norm(x);
    norm = std::sqrt(norm);
    if (norm == 0.0) throw Status{SLSHT_ERR_NUMERIC, "eigenfunction window is zero"};
    for (auto& x : c) x /= norm;
    if (std::abs(c[0]) < 1e-10)
      throw Status{SLSHT_ERR_NUMERIC, "window DC component vanishes; inversion would be impossible"};
    for (int i = 0; i < dim; ++i) {
      coeffs[2 * i] = c[i].real();
      coeffs[2 * i + 1] = c[i].imag();
    }
    *lambda_out = lambda;
    cleanup();
    return SLSHT_OK;
  } catch (const Status& st) {
    cleanup();
    g_create_error = st.msg;
    return st.code;
  } catch (const CudaError& e) {  // CK / CKL: allocation or launch failure (memory ~ L^4)
    cleanup();
    g_create_error = e.msg;
    return SLSHT_ERR_DEVICE;
  } catch (const std::exception& e) {  // host vectors (mask samples, coefficients)
    cleanup();
    g_create_error = e.what();
    return SLSHT_ERR_DEVICE;
  }
}

// forward_direct (transform.cpp:313-388) on the device: direct.cuh. out[(l^2+l+m) * ncells + i]
// is g(l, m) at cell cells[i] (every cell of the So3Volume in order when cells == NULL).
int slsht_cuda_forward_direct(int device, int L_f, const double* f, int L_h, const double* h,
                              int lmax, const long long* cells, long long ncells, double* out) {
  std::vector<void*> allocs;
  cudaStream_t s = nullptr;
  auto cleanup = [&]() {
    if (s) cudaStreamDestroy(s);
    for (void* q : allocs) cudaFree(q);
  };
  try {
    if (L_f < 0 || L_h < 0) throw Status{SLSHT_ERR_VALIDATION, "band limit must be non-negative"};
    if (!f || !h || !out) throw Status{SLSHT_ERR_VALIDATION, "null argument"};
    const int L_g = L_f + L_h;
    if (lmax < 0) lmax = L_g;
    const int L = std::max(lmax, L_g);  // sphere-grid band (transform.cpp:319)
    const int n = 2 * L + 1, nt = L + 1, nh = 2 * L_h + 1, nb = L_h + 1, ncol = nh * nb;
    const int NPQ = (L_h + 1) * (L_h + 1), NN = 2 * L + 1;  // colatitudes of S_{2L}
    const long long vol = (long long)nh * ncol;
    if (!cells) ncells = vol;
    if (ncells <= 0) throw Status{SLSHT_ERR_VALIDATION, "no cells requested"};
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
      throw Status{SLSHT_ERR_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    auto dal = [&](size_t bytes) {
      void* q = nullptr;
      CK(cudaMalloc(&q, std::max<size_t>(bytes, 16)));
      allocs.push_back(q);
      return q;
    };
    auto up = [&](const void* src, size_t bytes) {
      void* d = dal(bytes);
      CK(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s));
      return d;
    };
    auto blocks = [](long long x, int b) { return (unsigned)((x + b - 1) / b); };
    // ---- inputs, colatitudes, quadrature weights
    const double2* d_f = (const double2*)up(f, 16 * (size_t)coeff_count(L_f));
    const double* d_h = (const double*)up(h, 16 * (size_t)coeff_count(L_h));
    std::vector<double> rings(nt), nodes(NN), wq = host_theta_weights(2 * L);
    for (int t = 0; t < nt; ++t) rings[t] = kPi * (2 * t + 1) / n;            // grids.cpp:34-35
    for (int j = 0; j < NN; ++j) nodes[j] = kPi * (2 * j + 1) / (4 * L + 1);  // harmonics.cpp:138
    for (double& w : wq) w *= 2.0 * kPi;                                        // harmonics.cpp:164
    const double* d_rings = (const double*)up(rings.data(), 8 * rings.size());
    const double* d_nodes = (const double*)up(nodes.data(), 8 * nodes.size());
    const double* d_wq = (const double*)up(wq.data(), 8 * wq.size());
    // ---- t1 = the window table W[(p,q)][b n + c] (q-major (p,q) rows), from Delta and d(beta)
    std::vector<int> pq(2 * NPQ), qoff(nh + 1, 0);
    for (int jq = 0; jq < nh; ++jq) {
      const int q = jq - L_h, aq = std::abs(q);
      qoff[jq + 1] = qoff[jq] + (L_h + 1 - aq);
      for (int pp = aq; pp <= L_h; ++pp) {
        pq[2 * (qoff[jq] + pp - aq)] = q;
        pq[2 * (qoff[jq] + pp - aq) + 1] = pp;
      }
    }
    const int* d_pq = (const int*)up(pq.data(), 4 * pq.size());
    std::vector<double2> rou(nh);
    for (int k = 0; k < nh; ++k)
      rou[k] = make_double2(std::cos(-2.0 * kPi * k / nh), std::sin(-2.0 * kPi * k / nh));
    const double2* d_rou = (const double2*)up(rou.data(), 16 * rou.size());
    size_t dsz = 0;
    for (int pp = 0; pp <= L_h; ++pp) dsz += (size_t)(2 * pp + 1) * (2 * pp + 1);
    double* d_delta = (double*)dal(8 * dsz);
    double* d_dtab = (double*)dal(8 * dsz * nb);
    double2* d_W = (double2*)dal(16 * (size_t)NPQ * ncol);
    CK(configure_delta(L_h));
    double* d_dws = delta_needs_gws(L_h) ? (double*)dal(8 * delta_ws_doubles(L_h)) : nullptr;
    CK(launch_delta(L_h, d_delta, s, d_dws));
    const int wmax = nh * nh * nb;
    k_dtab<<<dim3(blocks(wmax, 256), L_h + 1), 256, 0, s>>>(L_h, d_delta, d_rou, d_dtab);
    CKL();
    k_wtab<<<dim3(blocks(ncol, 128), std::min(NPQ, 65535)), 128, 0, s>>>(L_h, d_h, d_dtab, d_rou, d_pq, 0, ncol,
                                                       nullptr, d_W);
    CKL();
    // ---- synthesis tables: lambda_p^q(theta_t) in q-major (p,q) rows; F = sh_synthesis(f)
    double* d_ls = (double*)dal(8 * (size_t)NPQ * nt);
    for (int jq = 0; jq < nh; ++jq) {
      const int q = jq - L_h;
      k_dir_lrows<<<blocks(nt, 128), 128, 3 * (L_h + 2) * 8, s>>>(q, L_h, nt, d_rings, nullptr,
                                                                 d_ls + (size_t)qoff[jq] * nt, nt);
      CKL();
    }
    double2* d_fring = (double2*)dal(16 * (size_t)(2 * L_f + 1) * nt);
    double2* d_F = (double2*)dal(16 * (size_t)nt * n);
    k_dir_fring<<<dim3(blocks(nt, 128), 2 * L_f + 1), 128, 3 * (L_f + 2) * 8, s>>>(L_f, d_f, nt,
                                                                                 d_rings, d_fring);
    CKL();
    k_dir_fmap<<<blocks((long long)nt * n, 128), 128, 0, s>>>(L_f, nt, n, d_fring, d_F);
    CKL();
    // ring DFTs: Esyn[k][q + L_h] = e^{+2 pi i q k / n}, Eana[m + L][k] = e^{-2 pi i m k / n} / n
    double2* d_esyn = (double2*)dal(16 * (size_t)n * nh);
    double2* d_eana = (double2*)dal(16 * (size_t)n * n);
    k_dir_dft<<<blocks((long long)n * nh, 256), 256, 0, s>>>(n, nh, 0, -L_h, n, 1.0, 1.0, d_esyn);
    CKL();
    k_dir_dft<<<blocks((long long)n * n, 256), 256, 0, s>>>(n, n, -L, 0, n, -1.0, 1.0 / n, d_eana);
    CKL();
    // ---- analysis matrices Q_m = Lambda_m diag(2 pi v) B_{m mod 2}, rows l = |m|..lmax
    double* d_B = (double*)dal(8 * 2 * (size_t)NN * nt);
    k_dir_bpar<<<blocks((long long)NN * nt, 256), 256, 0, s>>>(L, NN, d_nodes, d_rings, d_B);
    CKL();
    std::vector<size_t> qm_off(2 * lmax + 2, 0);
    for (int m = -lmax; m <= lmax; ++m)
      qm_off[m + lmax + 1] = qm_off[m + lmax] + (size_t)(lmax - std::abs(m) + 1) * nt;
    double* d_Q = (double*)dal(8 * qm_off.back());
    double* d_la = (double*)dal(8 * (size_t)(lmax + 1) * NN);
    for (int m = -lmax; m <= lmax; ++m) {
      const int nl = lmax - std::abs(m) + 1;
      k_dir_lrows<<<blocks(NN, 128), 128, 3 * (lmax + 2) * 8, s>>>(m, lmax, NN, d_nodes, d_wq, d_la,
                                                                  NN);
      CKL();
      // row-major Q (nl x nt) = Lambda (nl x NN) B (NN x nt): column-major Q^T = B^T Lambda^T
      CK(dgemm(kOpN, kOpN, nt, nl, NN, d_B + (size_t)(m & 1) * NN * nt, nt, d_la, NN,
               d_Q + qm_off[m + lmax], nt, s));
    }
    // ---- cells in batches of R
    const size_t per_r = 16 * ((size_t)NPQ + (size_t)nt * nh + 2 * (size_t)nt * n +
                               (size_t)(2 * lmax + 1) * (lmax + 1) + (size_t)coeff_count(lmax)) +
                         8;
    const long long R = std::max<long long>(
        1, std::min<long long>(ncells, (long long)((6ull << 30) / per_r)));
    double2* d_HR = (double2*)dal(16 * (size_t)NPQ * R);
    double2* d_S = (double2*)dal(16 * (size_t)nt * nh * R);
    double2* d_H = (double2*)dal(16 * (size_t)nt * n * R);
    double2* d_FM = (double2*)dal(16 * (size_t)nt * n * R);
    double2* d_OUT = (double2*)dal(16 * (size_t)(2 * lmax + 1) * (lmax + 1) * R);
    double2* d_res = (double2*)dal(16 * (size_t)coeff_count(lmax) * R);
    long long* d_cells = (long long*)dal(8 * (size_t)R);
    std::vector<long long> hcells(R);
    for (long long c0 = 0; c0 < ncells; c0 += R) {
      const int r = (int)std::min<long long>(R, ncells - c0);
      for (int i = 0; i < r; ++i) {
        hcells[i] = cells ? cells[c0 + i] : c0 + i;
        if (hcells[i] < 0 || hcells[i] >= vol)
          throw Status{SLSHT_ERR_VALIDATION, "cell index outside the So3Volume"};
      }
      CK(cudaMemcpyAsync(d_cells, hcells.data(), 8 * (size_t)r, cudaMemcpyHostToDevice, s));
      k_dir_hr<<<dim3(blocks(r, 128), NPQ), 128, 0, s>>>(r, d_cells, NPQ, ncol, nh, d_pq, d_W, d_HR);
      CKL();
      // S[t][q][r] = sum_p lambda_p^q(theta_t) HR[(p,q)][r]  (real x complex: 2r real columns)
      for (int jq = 0; jq < nh; ++jq) {
        const int kq = qoff[jq + 1] - qoff[jq];
        CK(dgemm(kOpN, kOpT, 2 * r, nt, kq,
                 reinterpret_cast<const double*>(d_HR + (size_t)qoff[jq] * r), 2 * r,
                 d_ls + (size_t)qoff[jq] * nt, nt, reinterpret_cast<double*>(d_S + (size_t)jq * r),
                 2 * nh * r, s));
      }
      // H[t][k][r] = sum_q Esyn[k][q] S[t][q][r]
      CK(zgemm(kOpN, kOpN, r, n, nh, d_S, r, d_esyn, nh, d_H, r, s, nt, (long long)nh * r, 0,
               (long long)n * r));
      const long long tot = (long long)nt * n * r;
      k_dir_product<<<blocks(tot, 256), 256, 0, s>>>(tot, r, d_F, d_H);
      CKL();
      // FM[t][m][r] = sum_k Eana[m][k] P[t][k][r]
      CK(zgemm(kOpN, kOpN, r, n, n, d_H, r, d_eana, n, d_FM, r, s, nt, (long long)n * r, 0,
               (long long)n * r));
      // OUT[m][l - |m|][r] = sum_t Q_m[l][t] FM[t][m][r]
      for (int m = -lmax; m <= lmax; ++m) {
        const int nl = lmax - std::abs(m) + 1;
        CK(dgemm(kOpN, kOpN, 2 * r, nl, nt,
                 reinterpret_cast<const double*>(d_FM + (size_t)(m + L) * r), 2 * n * r,
                 d_Q + qm_off[m + lmax], nt,
                 reinterpret_cast<double*>(d_OUT + (size_t)(m + lmax) * (lmax + 1) * r), 2 * r,
                 s));
      }
      const long long nres = (long long)coeff_count(lmax) * r;
      k_dir_scatter<<<blocks(nres, 256), 256, 0, s>>>(lmax, r, nres, d_OUT, d_res);
      CKL();
      CK(cudaMemcpy2DAsync(out + 2 * c0, 16 * (size_t)ncells, d_res, 16 * (size_t)r, 16 * (size_t)r,
                           coeff_count(lmax), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    cleanup();
    return SLSHT_OK;
  } catch (const Status& st) {
    cleanup();
    g_create_error = st.msg;
    return st.code;
  } catch (const CudaError& e) {
    cleanup();
    g_create_error = e.msg;
    return SLSHT_ERR_DEVICE;
  } catch (const std::exception& e) {  // host allocation of the tables / cell lists
    cleanup();
    g_create_error = e.what();
    return SLSHT_ERR_DEVICE;
  }
}

}  // extern "C"

namespace {
// run fn on `device` with the ABI's error mapping (component-level entry points)
template <class F>
int on_device(int device, F&& fn) {
  std::vector<void*> allocs;
  auto dal = [&](size_t bytes) {
    void* q = nullptr;
    CK(cudaMalloc(&q, bytes ? bytes : 1));
    allocs.push_back(q);
    return q;
  };
  auto cleanup = [&]() {
    for (void* q : allocs) cudaFree(q);
  };
  try {
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
      throw Status{SLSHT_ERR_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    if (device < 0 || device >= dev_count) throw Status{SLSHT_ERR_DEVICE, "invalid device ordinal"};
    CK(cudaSetDevice(device));
    fn(dal);
    cleanup();
    return SLSHT_OK;
  } catch (const Status& st) {
    cleanup();
    g_create_error = st.msg;
    return st.code;
  } catch (const CudaError& e) {
    cleanup();
    g_create_error = e.msg;
    return SLSHT_ERR_DEVICE;
  } catch (const std::exception& e) {
    cleanup();
    g_create_error = e.what();
    return SLSHT_ERR_DEVICE;
  }
}
}  // namespace

extern "C" {

int slsht_cuda_theta_weights(int device, int N, double* out) {
  if (N < 0 || !out) {
    g_create_error = N < 0 ? "quadrature order must be non-negative" : "null output";
    return SLSHT_ERR_VALIDATION;
  }
  return on_device(device, [&](auto dal) {
    double* d = (double*)dal(sizeof(double) * (N + 1));
    int* err = (int*)dal(sizeof(int));
    CK(cudaMemset(err, 0, sizeof(int)));
    k_theta_weights<<<(N + 1 + 3) / 4, 128>>>(N, d, err);
    CKL();
    int herr = 0;
    CK(cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost));
    if (herr)  // grids.cpp:86-89
      throw Status{SLSHT_ERR_NUMERIC, "theta_weights: imaginary residue above tolerance"};
    CK(cudaMemcpy(out, d, sizeof(double) * (N + 1), cudaMemcpyDeviceToHost));
  });
}

int slsht_cuda_beta_weights(int device, int L, double* out) {
  if (L < 0 || !out) {
    g_create_error = L < 0 ? "band limit must be non-negative" : "null output";
    return SLSHT_ERR_VALIDATION;
  }
  return on_device(device, [&](auto dal) {
    double* d = (double*)dal(sizeof(double) * (L + 1));
    int* err = (int*)dal(sizeof(int));
    CK(cudaMemset(err, 0, sizeof(int)));
    k_beta_weights<<<(L + 1 + 3) / 4, 128>>>(L, d, err);
    CKL();
    int herr = 0;
    CK(cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost));
    if (herr)  // grids.cpp:66-69
      throw Status{SLSHT_ERR_NUMERIC, "beta_weights: imaginary residue above tolerance"};
    CK(cudaMemcpy(out, d, sizeof(double) * (L + 1), cudaMemcpyDeviceToHost));
  });
}

int slsht_cuda_legendre_rows(int device, int m, int lmax, const double* thetas, int n,
                             double* rows) {
  if (lmax < 0 || std::abs(m) > lmax || n < 0 || (n > 0 && (!thetas || !rows))) {
    g_create_error = "legendre_rows requires |m| <= lmax and n >= 0";
    return SLSHT_ERR_VALIDATION;
  }
  if (n == 0) return SLSHT_OK;
  return on_device(device, [&](auto dal) {
    const int nl = lmax - std::abs(m) + 1;
    double* dt = (double*)dal(sizeof(double) * n);
    double* dr = (double*)dal(sizeof(double) * (size_t)nl * n);
    CK(cudaMemcpy(dt, thetas, sizeof(double) * n, cudaMemcpyHostToDevice));
    const size_t sm = sizeof(double) * 3 * (lmax + 1);
    if (sm > 48 * 1024)
      CK(cudaFuncSetAttribute(k_legendre_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sm));
    k_legendre_rows<<<(n + 127) / 128, 128, sm>>>(m, lmax, dt, n, dr);
    CKL();
    CK(cudaMemcpy(rows, dr, sizeof(double) * (size_t)nl * n, cudaMemcpyDeviceToHost));
  });
}

int slsht_cuda_gauss_legendre_half(int device, int points, double* ncos, double* nsin,
                                   double* weights) {
  if (points < 1 || !ncos || !nsin || !weights) {
    g_create_error = points < 1 ? "the rule needs at least one point" : "null output";
    return SLSHT_ERR_VALIDATION;
  }
  if (4 * sizeof(double) * (points + 1) > 227 * 1024) {
    g_create_error = "rule too large for the node recursion table";
    return SLSHT_ERR_VALIDATION;
  }
  return on_device(device, [&](auto dal) {
    const int K = (points + 1) / 2;
    double* d = (double*)dal(sizeof(double) * 3 * K);
    const size_t sm = 4 * sizeof(double) * (points + 1);
    CK(cudaFuncSetAttribute(k_glnodes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    k_glnodes<<<(K + 63) / 64, 64, sm>>>(points, K, d, d + K, d + 2 * K);
    CKL();
    CK(cudaMemcpy(ncos, d, sizeof(double) * K, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(nsin, d + K, sizeof(double) * K, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(weights, d + 2 * K, sizeof(double) * K, cudaMemcpyDeviceToHost));
  });
}

int slsht_cuda_delta_tables(int device, int L, double* out) {
  double* d = nullptr;
  try {
    if (L < 0) throw Status{SLSHT_ERR_VALIDATION, "band limit must be non-negative"};
    if (!out) throw Status{SLSHT_ERR_VALIDATION, "null output"};
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || dev_count == 0)
      throw Status{SLSHT_ERR_DEVICE, "no CUDA device available (the engine has no CPU fallback)"};
    CK(cudaSetDevice(device));
    size_t dsz = 0;
    for (int pp = 0; pp <= L; ++pp) dsz += (size_t)(2 * pp + 1) * (2 * pp + 1);
    d = dalloc<double>(dsz + (delta_needs_gws(L) ? delta_ws_doubles(L) : 0));
    CK(configure_delta(L));
    CK(launch_delta(L, d, 0, delta_needs_gws(L) ? d + dsz : nullptr));
    CK(cudaMemcpy(out, d, dsz * sizeof(double), cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    return SLSHT_OK;
  } catch (const Status& st) {
    if (d) cudaFree(d);
    g_create_error = st.msg;
    return st.code;
  } catch (const CudaError& e) {
    if (d) cudaFree(d);
    g_create_error = e.msg;
    return SLSHT_ERR_DEVICE;
  } catch (const std::exception& e) {
    if (d) cudaFree(d);
    g_create_error = e.what();
    return SLSHT_ERR_DEVICE;
  }
}

int slsht_cuda_inverse(slsht_cuda_plan* p, const double* f, const double* h, double h00_re,
                       double h00_im, int signal_band_limit, double* f_rec) {
  if (!p) return SLSHT_ERR_VALIDATION;
  return guarded(p, [&] {
    if (std::hypot(h00_re, h00_im) <= 1e-10)  // transform.cpp:513-514
      throw Status{SLSHT_ERR_NUMERIC, "window DC component too small for inversion"};
    if (signal_band_limit < 0 || p->l_begin > 0 || p->l_end <= signal_band_limit)
      throw Status{SLSHT_ERR_VALIDATION, "distribution lacks components up to L_f"};
    if (!f_rec) throw Status{SLSHT_ERR_VALIDATION, "null output"};
    const int rows = coeff_count(signal_band_limit);
    // a multi-GPU plan gathers every shard's digest rows into its first shard's table (peer
    // copies) and inverts there
    slsht_cuda_plan* q = p->group() ? p->parts[0] : p;
    CK(cudaSetDevice(q->desc.device));
    double* d_rec = dalloc<double>((size_t)2 * rows);
    try {
      if (p->group()) run_group_device(p, f, h, 0, q->d_digest, 1);
      else run_forward_device(p, f, h, 0, nullptr, 0, 0);
      CK(cudaSetDevice(q->desc.device));
      k_inverse<<<(rows + 127) / 128, 128, 0, q->stream>>>(
          q->d_digest, signal_band_limit, p->real_mode && !p->emit_neg, h00_re, h00_im, d_rec);
      CKL();
      CK(cudaMemcpyAsync(f_rec, d_rec, sizeof(double) * 2 * rows, cudaMemcpyDeviceToHost,
                         q->stream));
      check_numeric(q);
    } catch (...) {
      cudaFree(d_rec);
      throw;
    }
    CK(cudaFree(d_rec));
  });
}

int slsht_cuda_modulated(slsht_cuda_plan* p, const double* f, int count, const int* l,
                         const int* m, double* out) {
  if (!p) return SLSHT_ERR_VALIDATION;
  if (p->group()) {  // every shard holds the whole modulated-SHT setup: the first one serves
    const int rc = slsht_cuda_modulated(p->parts[0], f, count, l, m, out);
    if (rc != SLSHT_OK) p->last_error = p->parts[0]->last_error;
    return rc;
  }
  return guarded(p, [&] {
    for (int i = 0; i < count; ++i)
      if (std::abs(m[i]) > l[i] || l[i] > p->L_g)
        throw Status{SLSHT_ERR_VALIDATION, "modulated transform requires |m| <= l <= L_f+L_h"};
    // one segment / tile per requested component (rows are independent)
    std::vector<Seg> segs;
    std::vector<MTile> tiles;
    for (int i = 0; i < count; ++i) {
      segs.push_back(Seg{m[i], l[i], l[i], i});
      tiles.push_back(MTile{m[i], i, 1, i, (l[i] + m[i]) & 1});
    }
    if (count <= 0) return;  // nothing requested: an empty result, no launch
    cudaStream_t s = p->stream;
    struct Scratch {  // freed on every exit, errors included
      Seg* ds = nullptr;
      MTile* dt = nullptr;
      double* A = nullptr;
      double2* U = nullptr;
      ~Scratch() {
        cudaFree(ds);
        cudaFree(dt);
        cudaFree(A);
        cudaFree(U);
      }
    } sc;
    CK(cudaMemcpyAsync(p->d_f, f, sizeof(double) * 2 * coeff_count(p->L_f), cudaMemcpyHostToDevice, s));
    run_setup(p);
    sc.ds = dupload(segs, s);
    sc.dt = dupload(tiles, s);
    sc.A = dalloc<double>((size_t)count * p->ldA);
    sc.U = dalloc<double2>((size_t)count * p->NPQ);
    k_agen<<<dim3(count, (p->ldA + 127) / 128), 128, 3 * (p->L_g + 1) * sizeof(double), s>>>(
        sc.ds, p->L_g, p->n_nodes, p->ldA, p->d_ncos, p->d_nsin, p->d_weights, sc.A);
    CKL();
    k_modgemm<<<dim3(count, (p->NPQ + MG_COLS - 1) / MG_COLS), 256, MG_SMEM, s>>>(
        sc.dt, p->n_nodes, p->ldA, p->L_f, p->NPQ, sc.A, p->d_itab, p->d_lamh, p->d_pq, 0, 0, nullptr,
        nullptr, sc.U);
    CKL();
    std::vector<double2> hU((size_t)count * p->NPQ);
    CK(cudaMemcpyAsync(hU.data(), sc.U, hU.size() * 16, cudaMemcpyDeviceToHost, s));
    join_aux(p);
    CK(cudaStreamSynchronize(s));
    // back to the reference's triangular coeff_index(p, q) order, un-conjugated
    const int L = p->L_h;
    for (int i = 0; i < count; ++i) {
      int c = 0;
      for (int q = -L; q <= L; ++q)
        for (int pp = std::abs(q); pp <= L; ++pp, ++c) {
          const double2 v = hU[(size_t)i * p->NPQ + c];
          double* o = out + 2 * ((size_t)i * p->NPQ + coeff_index(pp, q));
          o[0] = v.x;
          o[1] = -v.y;
        }
    }
  });
}

}  // extern "C"
