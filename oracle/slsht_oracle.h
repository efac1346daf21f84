/* CPU oracle for the directional-SLSHT fast forward path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of slsht::forward_fast and the pieces it calls
 * (/root/reference/proj/src/{transform,grids,harmonics,wigner}.cpp). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and only as the
 * checker. The product (libslsht_cuda.so) never links or calls it.
 *
 * Complex arrays are interleaved (re, im) doubles, i.e. std::complex<double> layout.
 * Coefficient arrays use coeff_index(l, m) = l*l + l + m (proj/include/slsht/harmonics.hpp:13).
 * Status codes: 0 ok, 2 validation error, 3 numeric error (proj/include/slsht/errors.hpp).
 */
#ifndef SLSHT_ORACLE_H
#define SLSHT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void (*oracle_sink_fn)(int l, int m, const double* volume, void* user);

const char* oracle_last_error(void);

/* grids.cpp:20-26 (real and imaginary part of w(m)) */
void oracle_fourier_sin_integral(int m, double* re, double* im);
/* grids.cpp:76-92; out has band_limit+1 entries */
int oracle_theta_weights(int band_limit, double* out);
/* grids.cpp:54-74; out has band_limit+1 entries */
int oracle_beta_weights(int band_limit, double* out);
/* harmonics.cpp:60-89; rows is (lmax-|m|+1) x n */
int oracle_legendre_rows(int m, int lmax, const double* thetas, int n, double* rows);
/* wigner.cpp:28-80; out holds sum_p (2p+1)^2 doubles, level p row-major [q+p][q'+p] */
int oracle_delta_tables(int band_limit, double* out);
size_t oracle_delta_size(int band_limit);

/* ModulatedSht (transform.cpp:147-220). itab rows are built lazily per order mu, so a
 * handful of components at L_f = 1024 cost seconds instead of the constructor's minute. */
typedef struct oracle_ctx oracle_ctx;
oracle_ctx* oracle_ctx_create(int L_f, const double* f, int L_h);
void oracle_ctx_destroy(oracle_ctx* ctx);
/* out: coeff_count(L_h) complex, triangular coeff_index(p, q) */
int oracle_modulated_sht(oracle_ctx* ctx, int l, int m, double* out);
/* transform.cpp:23-58; out: n^3 complex, layout [q''][q][q'] */
int oracle_c_tensor(int L_h, const double* mod, const double* h, const double* delta,
                    double* out);
/* transform.cpp:78-135; out: n*(L_h+1)*n complex, So3Volume layout (a*(L+1)+b)*n+c */
int oracle_evaluate(int L_h, const double* ctensor, double* out);
/* transform.cpp:469-485 */
int oracle_integrate_volume(int L_h, const double* volume, double* out2);

/* One component (l, m): mod -> C -> evaluate. */
int oracle_component(oracle_ctx* ctx, const double* h, const double* delta, int l, int m,
                     double* out_volume);

/* transform.cpp:244-295, single-threaded; emission order m ascending, then l. */
int oracle_forward_fast(int L_f, const double* f, int f_real, int L_h, const double* h,
                        int h_real, int lmax, int use_real_symmetry, int emit_negative_m,
                        oracle_sink_fn sink, void* user);

/* Digest of a volume (8 doubles): sum |g|^2, max |g|, sum w_i g_i (re, im),
 * g[0] (re, im), integrate_volume (re, im); w_i = ((uint32(i)*0x9E3779B1) >> 8) 2^-24 - 0.5.
 * The same definition is used by the device consumer (include/slsht_cuda.h). */
void oracle_digest(int L_h, const double* volume, double* out8);

#ifdef __cplusplus
}
#endif
#endif
