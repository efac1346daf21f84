/* slsht_cuda.h — C ABI of the B200-native directional-SLSHT forward engine.
 *
 * This is the drop-in boundary for the reference's hot path
 *   slsht::forward_fast(f, h, sink, opts)   /root/reference/proj/include/slsht/transform.hpp:162-163
 *   slsht::forward_fast(f, h, opts)         /root/reference/proj/include/slsht/transform.hpp:164-165
 * (implemented at /root/reference/proj/src/transform.cpp:244-311). The reference has no FFI;
 * its callers are C++ (proj/src/cli.cpp:223-224, proj/tests/acceptance_main.cpp:97). The C++
 * shim paper_1207_5558_b200/csrc/forward_fast_shim.cpp implements both forward_fast overloads
 * against the UNCHANGED reference headers on top of this ABI; Python tests and bench.py bind it
 * with ctypes (paper_1207_5558_b200/_lib.py). See INTEGRATION.md.
 *
 * Conventions (all from the reference):
 *  - complex arrays are interleaved (re, im) doubles == std::complex<double> storage;
 *  - coefficient arrays (f, h) are indexed coeff_index(l, m) = l*l + l + m
 *    (proj/include/slsht/harmonics.hpp:13), (L+1)^2 entries;
 *  - a component volume is an So3Volume: n*(L_h+1)*n complex, index (a*(L_h+1)+b)*n + c,
 *    n = 2*L_h+1 (proj/include/slsht/transform.hpp:15-29);
 *  - status codes: 0 ok, 2 validation (slsht::ValidationError, CLI exit 2), 3 numeric
 *    (slsht::NumericError, CLI exit 3), 4 device/runtime (CUDA), matching
 *    proj/include/slsht/errors.hpp and proj/src/cli.cpp:31-45.
 *
 * There is no CPU fallback: every entry point that computes runs CUDA kernels built for sm_100a
 * and returns SLSHT_ERR_DEVICE when no suitable device is present.
 */
#ifndef SLSHT_CUDA_H
#define SLSHT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLSHT_OK 0
#define SLSHT_ERR_VALIDATION 2
#define SLSHT_ERR_NUMERIC 3
#define SLSHT_ERR_DEVICE 4

/* Per-component digest computed on the device by the fused epilogue (8 doubles):
 *  [0] sum |g_i|^2          [1] max |g_i|
 *  [2,3] sum w_i g_i         with w_i = ((uint32(i) * 0x9E3779B1u) >> 8) * 2^-24 - 0.5
 *  [4,5] g at (a, b, c) = (0, 0, 0)
 *  [6,7] integrate_volume(g) = (2L_h+1)^-3 sum_{a,b,c} q(beta_b) g  (proj/src/transform.cpp:469-485)
 * Dividing [6,7] by sqrt(16 pi^3) h_0^0 gives the inverse coefficient f_l^m for l <= L_f
 * (InverseAccumulator, proj/src/transform.cpp:502-540). */
#define SLSHT_DIGEST_WIDTH 8

typedef struct slsht_cuda_plan slsht_cuda_plan;

typedef struct slsht_cuda_desc {
  int L_f;             /* f.band_limit */
  int L_h;             /* h.band_limit */
  int lmax;            /* ForwardOptions::lmax; -1 means L_f + L_h (transform.hpp:146-148) */
  int real_mode;       /* use_real_symmetry && f.real_signal && h.real_signal (transform.cpp:253-254) */
  int emit_negative_m; /* ForwardOptions::emit_negative_m (transform.hpp:154-156) */
  int device;          /* CUDA device ordinal */
  int l_begin;         /* first degree computed by this plan (multi-GPU shard); 0 for all */
  int l_end;           /* one past the last degree; -1 means lmax + 1 */
  int materialize;     /* 1: keep every emitted volume resident on the device at slot
                          coeff_index(l, m) (the materialized forward_fast, transform.cpp:297-311);
                          0: stream volumes through a device ring consumed by the epilogue */
  int n_devices;       /* 0 or 1: one device (`device`); > 1: a multi-GPU plan over devices[] */
  long long ring_bytes; /* ring capacity for materialize == 0 (0: automatic), per device */
  void* stream;        /* cudaStream_t to run on (NULL: the plan creates its own; ignored by
                          multi-GPU plans, which own one stream per device) */
  const int* devices;  /* n_devices > 1: CUDA ordinals, one degree shard each (an ordinal may
                          repeat: several shards on one device) */
} slsht_cuda_desc;

/* Multi-GPU plans (the reference's forward_fast owns its whole parallel
 * schedule, transform.cpp:260-294). The degree range [l_begin, l_end) is split into n_devices
 * contiguous shards balanced by computed components (c(l) = 2l+1, or l+1 in real mode), shard k
 * on devices[k]; the shards share nothing while computing. The only exchange is the final
 * gather: each shard's digest rows [l0^2, l1^2) are copied (cudaMemcpyDefault: peer-to-peer
 * over NVLink for a device destination) into the caller's table; rows are copied, never
 * reduced, so every result is bitwise the one-device result. Host-sink calls of the shards are
 * serialized under one mutex, as the reference's worker pool does (transform.cpp:282-284). */

/* Number of visible devices this build can run on (sm_100, B200); 0 when there is none. The
 * drop-in forward_fast uses all of them by default (one degree shard each). */
int slsht_cuda_device_count(void);

/* The shard rule of multi-GPU plans (host only, no device needed): bounds[0..parts] of the
 * degree range [l_begin, l_end) for `parts` shards. Returns 0, or SLSHT_ERR_VALIDATION. */
int slsht_cuda_shard_bounds(int l_begin, int l_end, int real_mode, int parts, int* bounds);

/* Host sink, called once per emitted component with a pointer valid only during the call
 * (the So3Volume& contract of ComponentSink, transform.hpp:142-143, transform.cpp:279-284).
 * Calls are serialized on the calling thread. */
typedef void (*slsht_host_sink)(int l, int m, const double* volume, void* user);

/* Host copy sink: the copy the materializing forward_fast performs for every component
 * (transform.cpp:297-311, `components[coeff_index(l, m)] = volume`). Pass it as the sink of
 * slsht_cuda_forward with user = a slsht_copy_target: the volume of (l, m) is copied to
 * base + (coeff_index(l, m) - first_index) * volume_elems complex when that row lies in
 * [first_index, first_index + count); other rows are counted in `dropped`. */
typedef struct slsht_copy_target {
  double* base;
  long long first_index;
  long long count;
  long long volume_elems;
  long long delivered; /* volumes copied */
  long long dropped;   /* volumes outside the target range */
} slsht_copy_target;
void slsht_cuda_copy_sink(int l, int m, const double* volume, void* target);

int slsht_cuda_plan_create(const slsht_cuda_desc* desc, slsht_cuda_plan** plan);
void slsht_cuda_plan_destroy(slsht_cuda_plan* plan);
/* Message of the last failure on this plan (or of the last failed plan_create when plan is NULL). */
const char* slsht_cuda_last_error(const slsht_cuda_plan* plan);

/* forward_fast(f, h, sink, opts): f, h host arrays; every emitted component of the plan's
 * degree range is delivered to the sink (pinned, double-buffered D2H). */
int slsht_cuda_forward(slsht_cuda_plan* plan, const double* f, const double* h,
                       slsht_host_sink sink, void* user);

/* The materializing forward_fast(f, h, opts) (transform.hpp:164-165, transform.cpp:297-311:
 * `components[coeff_index(l, m)] = volume`): the volume of every emitted (l, m) is copied to
 * targets[coeff_index(l, m)] (volume_elems complex each; NULL entries and indices >= n_targets
 * are skipped). The destinations are disjoint, so unlike the serialized sink of
 * slsht_cuda_forward the copies out of the pinned staging buffers run on `threads` host
 * threads (0: SLSHT_CUDA_HOST_THREADS, default min(16, cores)), divided over the devices of a
 * multi-GPU plan. slsht_cuda_forward with slsht_cuda_copy_sink takes the same parallel path.
 * delivered (may be NULL) receives the number of volumes copied. */
int slsht_cuda_forward_scatter(slsht_cuda_plan* plan, const double* f, const double* h,
                               double* const* targets, long long n_targets, int threads,
                               long long* delivered);

/* Device-consumer mode (the timed mode of bench.py). f, h are host pointers unless
 * inputs_on_device != 0. digests (may be NULL) receives coeff_count(lmax) x 8 doubles at
 * coeff_index(l, m) for every emitted component of the plan's shard (other rows untouched);
 * it is a host pointer unless digests_on_device != 0. With synchronize == 0 the call only
 * enqueues work on the plan's stream (digests must then be a device pointer). */
int slsht_cuda_forward_device(slsht_cuda_plan* plan, const double* f, const double* h,
                              int inputs_on_device, double* digests, int digests_on_device,
                              int synchronize);

/* Device-consumer forward that additionally copies the full volumes of the listed components
 * (l[i], m[i]) to volumes[i] (host, count x volume_elems complex) right after their chunk
 * is produced; components outside the plan's range are left untouched and reported by a
 * SLSHT_ERR_VALIDATION return. digests as in slsht_cuda_forward_device (host, may be NULL). */
int slsht_cuda_forward_capture(slsht_cuda_plan* plan, const double* f, const double* h,
                               double* digests, int count, const int* l, const int* m,
                               double* volumes);

/* Device pointer to the materialized distribution (materialize == 1): coeff_count(lmax)
 * volumes, volume k at offset k * volume_elems complex. NULL in ring mode. */
const double* slsht_cuda_device_output(const slsht_cuda_plan* plan);
long long slsht_cuda_volume_elems(const slsht_cuda_plan* plan);
long long slsht_cuda_computed_count(const slsht_cuda_plan* plan);
long long slsht_cuda_emitted_count(const slsht_cuda_plan* plan);
void* slsht_cuda_stream(const slsht_cuda_plan* plan);

/* Kernel launches issued by the last forward call, and per-stage device time (ms, CUDA
 * events on the plan stream) when profiling is on (slsht_cuda_set_profiling, or
 * SLSHT_CUDA_PROFILE=1 at plan creation):
 * out[0] setup tables, [1] Legendre rows, [2] modulated-SHT GEMM, [3] coupling + alpha FFT
 * + epilogue (two-pass path: the k_tgemm GEMM only), [4] digest reduction, [5] two-pass path:
 * k_qfft (alpha FFT + epilogue), 0 on the other paths. Returns the number of entries written. */
long long slsht_cuda_launch_count(const slsht_cuda_plan* plan);
int slsht_cuda_stage_times(const slsht_cuda_plan* plan, double* out_ms, int n);
/* Turn per-stage event timing on or off for subsequent forward calls (adds one host
 * synchronization per chunk while on). */
int slsht_cuda_set_profiling(slsht_cuda_plan* plan, int enable);

/* Device time (ms) of the coupling kernel in the last forward_device of a single-chunk
 * (materialized) plan, from CUDA events recorded around it on the plan's stream on every call
 * (also inside its CUDA graph). Blocks until that kernel has finished. SLSHT_ERR_VALIDATION if
 * the plan has several chunks or has not run forward_device. */
int slsht_cuda_kernel_time(const slsht_cuda_plan* plan, double* ms);

/* Component-level entry points (host arrays in/out), mirroring the reference's
 * DeltaTables (wigner.cpp:28-80), ModulatedSht::compute (transform.cpp:189-220) and the
 * window-side table of the coupling stage; used by the parity tests. */
int slsht_cuda_delta_tables(int device, int L, double* out);

/* Grid functions of the path on the device (component-level, as the engine computes them):
 *  - theta_weights(N): the N+1 colatitude weights of S_N (proj/src/grids.cpp:76-92),
 *    SLSHT_ERR_NUMERIC on an imaginary residue >= 1e-12 (grids.cpp:86-89);
 *  - beta_weights(L): the L+1 weights q(beta_b) of the inverse (grids.cpp:54-74);
 *  - legendre_rows(m, lmax, thetas, n): rows[(l-|m|) n + j] = lambda_l^m(theta_j) for
 *    |m| <= l <= lmax (proj/src/harmonics.cpp:60-89), (lmax-|m|+1) x n doubles;
 *  - gauss_legendre_half(points): the x = cos(theta) >= 0 half of the points-point
 *    Gauss-Legendre rule the engine's modulated SHT integrates with ((points+1)/2 nodes,
 *    decreasing x; the x = 0 node of an odd rule carries half its weight). */
int slsht_cuda_theta_weights(int device, int N, double* out);
int slsht_cuda_beta_weights(int device, int L, double* out);
int slsht_cuda_legendre_rows(int device, int m, int lmax, const double* thetas, int n,
                             double* rows);
int slsht_cuda_gauss_legendre_half(int device, int points, double* ncos, double* nsin,
                                   double* weights);
/* mod for (l[i], m[i]), i < count: out is count x coeff_count(L_h) complex, coeff_index(p, q). */
int slsht_cuda_modulated(slsht_cuda_plan* plan, const double* f, int count, const int* l,
                         const int* m, double* out);

/* Inversion from the SLSHT (transform.cpp:469-544: inverse_slsht / InverseAccumulator, the
 * reference's tau3 stage): runs the forward on the device and returns
 *   f_rec[coeff_index(l, m)] = integrate_volume(g(l, m)) / (sqrt(16 pi^3) h00),
 * l <= signal_band_limit, from the digest epilogue's quadrature integrals (no volume leaves
 * the device). Components not emitted (real mode without emit_negative_m) are filled by
 * conjugate symmetry, as InverseAccumulator(fill_negative_by_symmetry = true) does.
 * f_rec: coeff_count(signal_band_limit) complex (host memory).
 * Errors: SLSHT_ERR_NUMERIC if |h00| <= 1e-10; SLSHT_ERR_VALIDATION if the plan does not
 * cover every degree l <= signal_band_limit. */
int slsht_cuda_inverse(slsht_cuda_plan* plan, const double* f, const double* h,
                       double h00_re, double h00_im, int signal_band_limit, double* f_rec);

/* Slepian window (window.cpp:44-198: concentration_matrix + eigenfunction_window): the
 * dominant eigenfunction of the concentration kernel of the elliptical region (foci at
 * colatitude theta_c on phi = 0, pi; semi-major arc a) at band limit L, by mask quadrature on
 * S_{oversample L} and the reference's power iteration, on `device`.
 * coeffs: coeff_count(L) complex (host), unit norm, real-signal symmetric; lambda: the
 * concentration ratio. Errors as the reference (ValidationError / NumericError codes); the
 * message is slsht_cuda_last_error(NULL). */
int slsht_cuda_eigenfunction_window(int device, double theta_c, double a, int band_limit,
                                    int oversample, double* coeffs, double* lambda);

/* forward_direct (transform.hpp:167-168, transform.cpp:313-388), the reference's independent
 * direct engine, on the device: g(l, m; rho) = sh_analysis(sh_synthesis(f) sh_synthesis(R_rho h))
 * on the sphere grid of band max(lmax, L_f + L_h), every component l <= lmax (lmax < 0: L_f +
 * L_h) at the So3Volume cells `cells` (indices (a (L_h+1) + b)(2L_h+1) + c; NULL = every cell
 * in order, ncells ignored). Host arrays; out: coeff_count(lmax) x ncells complex, row
 * coeff_index(l, m), column = requested cell. Status codes as above. */
int slsht_cuda_forward_direct(int device, int L_f, const double* f, int L_h, const double* h,
                              int lmax, const long long* cells, long long ncells, double* out);

#ifdef __cplusplus
}
#endif
#endif /* SLSHT_CUDA_H */
