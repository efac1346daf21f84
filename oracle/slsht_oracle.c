/* CPU oracle for the directional-SLSHT fast forward path — TEST INFRASTRUCTURE ONLY.
 *
 * Restates, in plain C, the algorithm of slsht::forward_fast from the reference
 * (/root/reference/proj). Each function cites the file:line it follows. This code is the
 * checker the CUDA path is compared against; it is never linked into the product and the
 * product never falls back to it. The restatement itself is pinned against the compiled
 * reference (oracle/_ref, tests/test_oracle_vs_reference.py) and against the committed
 * golden fixtures generated from the reference (tests/golden/).
 */
#include "slsht_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define K_PI 3.14159265358979323846

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* oracle_last_error(void) { return g_err; }

static inline int coeff_index(int l, int m) { return l * l + l + m; }
static inline int coeff_count(int L) { return (L + 1) * (L + 1); }

/* i^k as (re, im); transform.cpp:20-21 */
static void ipow(int k, double* re, double* im) {
  static const double tr[4] = {1.0, 0.0, -1.0, 0.0};
  static const double ti[4] = {0.0, 1.0, 0.0, -1.0};
  const int r = ((k % 4) + 4) % 4;
  *re = tr[r];
  *im = ti[r];
}

/* grids.cpp:20-26 */
void oracle_fourier_sin_integral(int m, double* re, double* im) {
  *re = 0.0;
  *im = 0.0;
  if (m == 0) { *re = 2.0; return; }
  if (m == 1) { *im = K_PI / 2.0; return; }
  if (m == -1) { *im = -K_PI / 2.0; return; }
  if (m % 2 != 0) return;
  *re = 2.0 / (1.0 - (double)m * m);
}

/* grids.cpp:76-92 */
int oracle_theta_weights(int band_limit, double* out) {
  if (band_limit < 0) return fail(2, "band limit must be non-negative");
  const int L = band_limit, n = 2 * L + 1;
  for (int t = 0; t <= L; ++t) {
    const double theta = K_PI * (2 * t + 1) / n;
    double sr = 0.0, si = 0.0;
    for (int k = -L; k <= L; ++k) {
      double wr, wi;
      oracle_fourier_sin_integral(-k, &wr, &wi);
      const double c = cos(k * theta);
      sr += wr * c;
      si += wi * c;
    }
    if (fabs(si) >= 1e-12) return fail(3, "theta weight imaginary residue exceeds 1e-12");
    out[t] = (t < L) ? 2.0 * sr / n : sr / n;
  }
  return 0;
}

/* grids.cpp:54-74 */
int oracle_beta_weights(int band_limit, double* out) {
  if (band_limit < 0) return fail(2, "band limit must be non-negative");
  const int L = band_limit, n = 2 * L + 1;
  out[0] = 4.0 * K_PI * K_PI / (L / 2 + 0.5);
  for (int b = 1; b <= L; ++b) {
    const double beta = 2.0 * K_PI * b / n;
    double sr = 0.0, si = 0.0;
    for (int m = -L; m <= L; ++m) {
      double wr, wi;
      oracle_fourier_sin_integral(-m, &wr, &wi);
      const double c = cos(m * beta);
      sr += wr * c;
      si += wi * c;
    }
    if (fabs(si) >= 1e-12) return fail(3, "beta weight imaginary residue exceeds 1e-12");
    out[b] = 8.0 * K_PI * K_PI * sr;
  }
  return 0;
}

/* harmonics.cpp:60-89: normalized lambda_l^m(theta) with the Condon-Shortley phase,
 * sectoral seed then the three-term recursion in l. */
int oracle_legendre_rows(int m, int lmax, const double* thetas, int n, double* rows) {
  const int am = abs(m);
  if (am > lmax) return fail(2, "legendre order exceeds degree");
  double* r0 = rows;
  for (int j = 0; j < n; ++j) {
    double sect = 1.0 / sqrt(4.0 * K_PI);
    const double s = sin(thetas[j]);
    for (int k = 1; k <= am; ++k) sect *= -s * sqrt((2.0 * k + 1.0) / (2.0 * k));
    if (m < 0 && (am & 1)) sect = -sect;
    r0[j] = sect;
  }
  if (lmax == am) return 0;
  double* r1 = rows + n;
  const double c1 = sqrt(2.0 * am + 3.0);
  for (int j = 0; j < n; ++j) r1[j] = cos(thetas[j]) * c1 * r0[j];
  for (int l = am + 2; l <= lmax; ++l) {
    const double ll = (double)l * l;
    const double l1 = (double)(l - 1) * (l - 1);
    const double a = sqrt((4.0 * ll - 1.0) / (ll - am * am));
    const double b = sqrt((l1 - am * am) / (4.0 * l1 - 1.0));
    const double* p1 = rows + (size_t)(l - am - 1) * n;
    const double* p2 = rows + (size_t)(l - am - 2) * n;
    double* cur = rows + (size_t)(l - am) * n;
    for (int j = 0; j < n; ++j) cur[j] = a * (cos(thetas[j]) * p1[j] - b * p2[j]);
  }
  return 0;
}

size_t oracle_delta_size(int band_limit) {
  size_t total = 0;
  for (int p = 0; p <= band_limit; ++p) total += (size_t)(2 * p + 1) * (2 * p + 1);
  return total;
}

static size_t delta_offset(int p) {
  /* sum_{p'<p} (2p'+1)^2 = p(2p-1)(2p+1)/3 */
  return (size_t)p * (2 * p - 1) * (2 * p + 1) / 3;
}

static inline double* dslot(double* d, int p, int q, int qp) {
  return d + delta_offset(p) + (size_t)(q + p) * (2 * p + 1) + (qp + p);
}

static inline double parity(int k) { return (k & 1) ? -1.0 : 1.0; }

/* wigner.cpp:28-80: Trapani seeds from the previous level's top row, downward three-term
 * recursion over the sector m >= m' >= 0, transpose, then the d-matrix symmetries. */
int oracle_delta_tables(int band_limit, double* d) {
  if (band_limit < 0) return fail(2, "band limit must be non-negative");
  memset(d, 0, sizeof(double) * oracle_delta_size(band_limit));
  *dslot(d, 0, 0, 0) = 1.0;
  for (int l = 1; l <= band_limit; ++l) {
    *dslot(d, l, l, 0) = -sqrt((2.0 * l - 1.0) / (2.0 * l)) * *dslot(d, l - 1, l - 1, 0);
    for (int mp = 1; mp <= l; ++mp)
      *dslot(d, l, l, mp) =
          sqrt(l * (2.0 * l - 1.0) / (2.0 * (l + mp) * ((double)l + mp - 1.0))) *
          *dslot(d, l - 1, l - 1, mp - 1);
    for (int mp = 0; mp <= l - 1; ++mp) {
      for (int m = l - 1; m >= mp; --m) {
        const double denom = sqrt((double)(l - m) * (l + m + 1.0));
        double value = 2.0 * mp / denom * *dslot(d, l, m + 1, mp);
        if (m + 2 <= l)
          value -= sqrt((l - m - 1.0) * (l + m + 2.0)) / denom * *dslot(d, l, m + 2, mp);
        *dslot(d, l, m, mp) = value;
      }
    }
    for (int m = 0; m <= l; ++m)
      for (int mp = m + 1; mp <= l; ++mp)
        *dslot(d, l, m, mp) = parity(mp - m) * *dslot(d, l, mp, m);
    for (int m = 0; m <= l; ++m)
      for (int mp = 0; mp <= l; ++mp) {
        const double value = *dslot(d, l, m, mp);
        if (m > 0) *dslot(d, l, -m, mp) = parity(l + mp) * value;
        if (mp > 0) *dslot(d, l, m, -mp) = parity(l + m) * value;
        if (m > 0 && mp > 0) *dslot(d, l, -m, -mp) = parity(m + mp) * value;
      }
  }
  return 0;
}

/* ---------------------------------------------------------------- ModulatedSht */

struct oracle_ctx {
  int L_f, L_h, L_g, n_nodes;
  const double* f;  /* borrowed, coeff_count(L_f) complex */
  double* nodes;    /* transform.cpp:151-155 */
  double* weights;  /* transform.cpp:156 */
  double* itab;     /* (2L_f+1) x n_nodes complex, built lazily per mu */
  char* itab_ready;
  double* lamh;     /* coeff_count(L_h) x n_nodes, transform.cpp:175-186 */
  double* rows;     /* scratch */
  int lamf_m;       /* cached order of lamf (transform.cpp:194-199) */
  double* lamf;
};

oracle_ctx* oracle_ctx_create(int L_f, const double* f, int L_h) {
  if (L_h < 0 || L_f < 0) {
    fail(2, "window band limit must be non-negative");
    return NULL;
  }
  oracle_ctx* c = (oracle_ctx*)calloc(1, sizeof *c);
  c->L_f = L_f;
  c->L_h = L_h;
  c->L_g = L_f + L_h;
  const int N = 2 * c->L_g;
  c->n_nodes = N + 1;
  c->f = f;
  c->nodes = (double*)malloc(sizeof(double) * c->n_nodes);
  for (int j = 0; j < c->n_nodes; ++j) c->nodes[j] = K_PI * (2 * j + 1) / (2 * N + 1);
  c->weights = (double*)malloc(sizeof(double) * c->n_nodes);
  if (oracle_theta_weights(N, c->weights) != 0) {
    oracle_ctx_destroy(c);
    return NULL;
  }
  c->itab = (double*)malloc(sizeof(double) * 2 * (size_t)(2 * L_f + 1) * c->n_nodes);
  c->itab_ready = (char*)calloc(2 * L_f + 1, 1);
  c->rows = (double*)malloc(sizeof(double) * (size_t)(c->L_g + 1) * c->n_nodes);
  c->lamf = (double*)malloc(sizeof(double) * (size_t)(c->L_g + 1) * c->n_nodes);
  c->lamf_m = 1 << 30;
  c->lamh = (double*)malloc(sizeof(double) * (size_t)coeff_count(L_h) * c->n_nodes);
  for (int q = -L_h; q <= L_h; ++q) {
    const int aq = abs(q);
    oracle_legendre_rows(q, L_h, c->nodes, c->n_nodes, c->rows);
    for (int p = aq; p <= L_h; ++p)
      memcpy(c->lamh + (size_t)coeff_index(p, q) * c->n_nodes,
             c->rows + (size_t)(p - aq) * c->n_nodes, sizeof(double) * c->n_nodes);
  }
  return c;
}

void oracle_ctx_destroy(oracle_ctx* c) {
  if (!c) return;
  free(c->nodes);
  free(c->weights);
  free(c->itab);
  free(c->itab_ready);
  free(c->rows);
  free(c->lamf);
  free(c->lamh);
  free(c);
}

/* transform.cpp:158-173: I(theta_j, mu) = 2 pi conj(sum_l f_l^mu lambda_l^mu(theta_j)) */
static const double* itab_row(oracle_ctx* c, int mu) {
  double* dst = c->itab + 2 * (size_t)(mu + c->L_f) * c->n_nodes;
  if (c->itab_ready[mu + c->L_f]) return dst;
  const int amu = abs(mu);
  const int nn = c->n_nodes;
  oracle_legendre_rows(mu, c->L_f, c->nodes, nn, c->rows);
  for (int j = 0; j < nn; ++j) {
    double ar = 0.0, ai = 0.0;
    for (int l = amu; l <= c->L_f; ++l) {
      const double lam = c->rows[(size_t)(l - amu) * nn + j];
      const double* fv = c->f + 2 * coeff_index(l, mu);
      ar += fv[0] * lam;
      ai += fv[1] * lam;
    }
    dst[2 * j] = 2.0 * K_PI * ar;
    dst[2 * j + 1] = -(2.0 * K_PI * ai);
  }
  c->itab_ready[mu + c->L_f] = 1;
  return dst;
}

/* transform.cpp:189-220 */
int oracle_modulated_sht(oracle_ctx* c, int l, int m, double* out) {
  if (abs(m) > l || l > c->L_g)
    return fail(2, "modulated transform requires |m| <= l <= L_f+L_h");
  const int am = abs(m), nn = c->n_nodes, L_h = c->L_h;
  if (c->lamf_m != m) {
    oracle_legendre_rows(m, c->L_g, c->nodes, nn, c->lamf);
    c->lamf_m = m;
  }
  const double* lamf = c->lamf + (size_t)(l - am) * nn;
  memset(out, 0, sizeof(double) * 2 * coeff_count(L_h));
  double* row = (double*)malloc(sizeof(double) * 2 * nn);
  for (int q = -L_h; q <= L_h; ++q) {
    const int mu = m - q;
    if (abs(mu) > c->L_f) continue;
    const double* it = itab_row(c, mu);
    for (int j = 0; j < nn; ++j) {
      const double s = c->weights[j] * lamf[j];
      row[2 * j] = s * it[2 * j];
      row[2 * j + 1] = s * it[2 * j + 1];
    }
    for (int p = abs(q); p <= L_h; ++p) {
      const double* lam = c->lamh + (size_t)coeff_index(p, q) * nn;
      double ar = 0.0, ai = 0.0;
      for (int j = 0; j < nn; ++j) {
        ar += row[2 * j] * lam[j];
        ai += row[2 * j + 1] * lam[j];
      }
      out[2 * coeff_index(p, q)] = ar;
      out[2 * coeff_index(p, q) + 1] = ai;
    }
  }
  free(row);
  return 0;
}

/* transform.cpp:23-58: C[q''][q][q'] = sum_p (Delta^p_{q''q} u_q)(Delta^p_{q''q'} v_q'),
 * u_q = i^q conj(mod_p^q), v_q' = i^{-q'} h_p^{q'}. */
int oracle_c_tensor(int L, const double* mod, const double* h, const double* delta,
                    double* out) {
  const int n = 2 * L + 1;
  memset(out, 0, sizeof(double) * 2 * (size_t)n * n * n);
  double* u = (double*)malloc(sizeof(double) * 2 * n);
  double* v = (double*)malloc(sizeof(double) * 2 * n);
  double* au = (double*)malloc(sizeof(double) * 2 * n);
  double* av = (double*)malloc(sizeof(double) * 2 * n);
  for (int p = 0; p <= L; ++p) {
    const int w = 2 * p + 1;
    for (int q = -p; q <= p; ++q) {
      double ir, ii;
      ipow(q, &ir, &ii);
      const double mr = mod[2 * coeff_index(p, q)], mi = -mod[2 * coeff_index(p, q) + 1];
      u[2 * (q + p)] = ir * mr - ii * mi;
      u[2 * (q + p) + 1] = ir * mi + ii * mr;
    }
    for (int qp = -p; qp <= p; ++qp) {
      double ir, ii;
      ipow(-qp, &ir, &ii);
      const double hr = h[2 * coeff_index(p, qp)], hi = h[2 * coeff_index(p, qp) + 1];
      v[2 * (qp + p)] = ir * hr - ii * hi;
      v[2 * (qp + p) + 1] = ir * hi + ii * hr;
    }
    for (int qpp = -p; qpp <= p; ++qpp) {
      const double* drow = delta + delta_offset(p) + (size_t)(qpp + p) * w;
      for (int i = 0; i < w; ++i) {
        au[2 * i] = drow[i] * u[2 * i];
        au[2 * i + 1] = drow[i] * u[2 * i + 1];
        av[2 * i] = drow[i] * v[2 * i];
        av[2 * i + 1] = drow[i] * v[2 * i + 1];
      }
      /* base = index(-p, -p, qpp) */
      double* base = out + 2 * (((size_t)(qpp + L) * n + (L - p)) * n + (L - p));
      for (int iq = 0; iq < w; ++iq) {
        const double lr = au[2 * iq], li = au[2 * iq + 1];
        double* row = base + 2 * (size_t)iq * n;
        for (int iqp = 0; iqp < w; ++iqp) {
          row[2 * iqp] += lr * av[2 * iqp] - li * av[2 * iqp + 1];
          row[2 * iqp + 1] += lr * av[2 * iqp + 1] + li * av[2 * iqp];
        }
      }
    }
  }
  free(u);
  free(v);
  free(au);
  free(av);
  return 0;
}

/* transform.cpp:78-135: kernel K[x][j] = e^{-2 pi i x (j-L)/n}; pass beta (b <= L only),
 * then alpha over q, then gamma over q'. */
int oracle_evaluate(int L, const double* c, double* out) {
  const int n = 2 * L + 1, nb = L + 1;
  const size_t nn = (size_t)n * n;
  double* K = (double*)malloc(sizeof(double) * 2 * nn);
  for (int x = 0; x < n; ++x)
    for (int j = 0; j < n; ++j) {
      const double ang = -2.0 * K_PI * x * (j - L) / (double)n;
      K[2 * ((size_t)x * n + j)] = cos(ang);
      K[2 * ((size_t)x * n + j) + 1] = sin(ang);
    }
  double* v1 = (double*)calloc(2 * (size_t)nb * nn, sizeof(double));
  for (int b = 0; b < nb; ++b) {
    double* acc = v1 + 2 * (size_t)b * nn;
    for (int jpp = 0; jpp < n; ++jpp) {
      const double wr = K[2 * ((size_t)b * n + jpp)], wi = K[2 * ((size_t)b * n + jpp) + 1];
      const double* src = c + 2 * (size_t)jpp * nn;
      for (size_t i = 0; i < nn; ++i) {
        acc[2 * i] += wr * src[2 * i] - wi * src[2 * i + 1];
        acc[2 * i + 1] += wr * src[2 * i + 1] + wi * src[2 * i];
      }
    }
  }
  double* plane = (double*)malloc(sizeof(double) * 2 * nn);
  for (int b = 0; b < nb; ++b) {
    memset(plane, 0, sizeof(double) * 2 * nn);
    const double* vb = v1 + 2 * (size_t)b * nn;
    for (int a = 0; a < n; ++a) {
      double* dst = plane + 2 * (size_t)a * n;
      for (int jq = 0; jq < n; ++jq) {
        const double wr = K[2 * ((size_t)a * n + jq)], wi = K[2 * ((size_t)a * n + jq) + 1];
        const double* src = vb + 2 * (size_t)jq * n;
        for (int i = 0; i < n; ++i) {
          dst[2 * i] += wr * src[2 * i] - wi * src[2 * i + 1];
          dst[2 * i + 1] += wr * src[2 * i + 1] + wi * src[2 * i];
        }
      }
    }
    for (int a = 0; a < n; ++a) {
      const double* arow = plane + 2 * (size_t)a * n;
      double* orow = out + 2 * (((size_t)a * nb + b) * n);
      for (int cc = 0; cc < n; ++cc) {
        const double* kr = K + 2 * (size_t)cc * n;
        double ar = 0.0, ai = 0.0;
        for (int j = 0; j < n; ++j) {
          ar += arow[2 * j] * kr[2 * j] - arow[2 * j + 1] * kr[2 * j + 1];
          ai += arow[2 * j] * kr[2 * j + 1] + arow[2 * j + 1] * kr[2 * j];
        }
        orow[2 * cc] = ar;
        orow[2 * cc + 1] = ai;
      }
    }
  }
  free(plane);
  free(v1);
  free(K);
  return 0;
}

/* transform.cpp:469-485 */
int oracle_integrate_volume(int L, const double* vol, double* out2) {
  const int n = 2 * L + 1, nb = L + 1;
  double* qb = (double*)malloc(sizeof(double) * nb);
  const int rc = oracle_beta_weights(L, qb);
  if (rc) {
    free(qb);
    return rc;
  }
  double ar = 0.0, ai = 0.0;
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < nb; ++b) {
      const double* row = vol + 2 * (((size_t)a * nb + b) * n);
      double rr = 0.0, ri = 0.0;
      for (int cc = 0; cc < n; ++cc) {
        rr += row[2 * cc];
        ri += row[2 * cc + 1];
      }
      ar += qb[b] * rr;
      ai += qb[b] * ri;
    }
  const double s = (double)n * n * n;
  out2[0] = ar / s;
  out2[1] = ai / s;
  free(qb);
  return 0;
}

void oracle_digest(int L, const double* vol, double* d) {
  const int n = 2 * L + 1, nb = L + 1;
  const size_t V = (size_t)n * n * nb;
  double s2 = 0.0, mx = 0.0, pr = 0.0, pi = 0.0;
  for (size_t i = 0; i < V; ++i) {
    const double gr = vol[2 * i], gi = vol[2 * i + 1];
    const double a2 = gr * gr + gi * gi;
    s2 += a2;
    const double a = sqrt(a2);
    if (a > mx) mx = a;
    const uint32_t hsh = (uint32_t)i * 0x9E3779B1u;
    const double w = (double)(hsh >> 8) * (1.0 / 16777216.0) - 0.5;
    pr += w * gr;
    pi += w * gi;
  }
  d[0] = s2;
  d[1] = mx;
  d[2] = pr;
  d[3] = pi;
  d[4] = vol[0];
  d[5] = vol[1];
  oracle_integrate_volume(L, vol, d + 6);
}

int oracle_component(oracle_ctx* ctx, const double* h, const double* delta, int l, int m,
                     double* out_volume) {
  const int L = ctx->L_h, n = 2 * L + 1;
  double* mod = (double*)malloc(sizeof(double) * 2 * coeff_count(L));
  double* ct = (double*)malloc(sizeof(double) * 2 * (size_t)n * n * n);
  int rc = oracle_modulated_sht(ctx, l, m, mod);
  if (!rc) rc = oracle_c_tensor(L, mod, h, delta, ct);
  if (!rc) rc = oracle_evaluate(L, ct, out_volume);
  free(mod);
  free(ct);
  return rc;
}

/* transform.cpp:244-295 (single worker; the reference emits (l, -m) right after (l, m)
 * in real mode, transform.cpp:280-284). */
int oracle_forward_fast(int L_f, const double* f, int f_real, int L_h, const double* h,
                        int h_real, int lmax, int use_real_symmetry, int emit_negative_m,
                        oracle_sink_fn sink, void* user) {
  const int L_g = L_f + L_h;
  if (lmax < 0) lmax = L_g;
  if (lmax > L_g) return fail(2, "fast engine computes components up to L_f + L_h only");
  const int real_mode = use_real_symmetry && f_real && h_real;
  oracle_ctx* ctx = oracle_ctx_create(L_f, f, L_h);
  if (!ctx) return 2;
  double* delta = (double*)malloc(sizeof(double) * oracle_delta_size(L_h));
  oracle_delta_tables(L_h, delta);
  const int n = 2 * L_h + 1;
  const size_t V = (size_t)n * n * (L_h + 1);
  double* vol = (double*)malloc(sizeof(double) * 2 * V);
  double* neg = (double*)malloc(sizeof(double) * 2 * V);
  int rc = 0;
  for (int m = real_mode ? 0 : -lmax; m <= lmax && !rc; ++m) {
    for (int l = abs(m); l <= lmax && !rc; ++l) {
      rc = oracle_component(ctx, h, delta, l, m, vol);
      if (rc) break;
      const int mirror = real_mode && emit_negative_m && m > 0;
      sink(l, m, vol, user);
      if (mirror) {
        /* transform.cpp:60-66 */
        const double sign = (m & 1) ? -1.0 : 1.0;
        for (size_t i = 0; i < V; ++i) {
          neg[2 * i] = sign * vol[2 * i];
          neg[2 * i + 1] = sign * -vol[2 * i + 1];
        }
        sink(l, -m, neg, user);
      }
    }
  }
  free(vol);
  free(neg);
  free(delta);
  oracle_ctx_destroy(ctx);
  return rc;
}
