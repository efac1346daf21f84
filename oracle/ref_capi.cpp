// extern "C" harness around the UNMODIFIED reference library (TEST INFRASTRUCTURE ONLY).
//
// Compiled by oracle/Makefile together with the reference's own sources under
// /root/reference/proj/src into oracle/_ref/libslsht_ref.so. It is used (a) to pin our
// C restatement (oracle/slsht_oracle.c) against the real reference, (b) to generate the
// committed golden fixtures (tests/golden/make_golden.py) and (c) as the CPU baseline arm
// of bench.py (`--impl reference`). It is never linked into the product library.
//
// Every entry point returns 0 on success, 2 for slsht::ValidationError, 3 for
// slsht::NumericError and 1 for anything else, mirroring the reference CLI's exit codes
// (proj/src/cli.cpp:31-45).
#include <algorithm>
#include <atomic>
#include <mutex>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "slsht/errors.hpp"
#include "slsht/grids.hpp"
#include "slsht/harmonics.hpp"
#include "slsht/signals.hpp"
#include "slsht/transform.hpp"
#include "slsht/wigner.hpp"
#include "slsht/window.hpp"

using cplx = std::complex<double>;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return 0;
  } catch (const slsht::ValidationError& e) {
    g_err = e.what();
    return 2;
  } catch (const slsht::NumericError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

slsht::SphCoeffs make_coeffs(int L, const double* data, int real_signal) {
  slsht::SphCoeffs c = slsht::SphCoeffs::zeros(L, real_signal != 0);
  std::memcpy(c.data.data(), data, sizeof(double) * 2 * c.data.size());
  return c;
}

// Digest of one So3Volume; the definition is shared with oracle/slsht_oracle.c and the
// device consumer (include/slsht_cuda.h, SLSHT_DIGEST_*).
void digest_volume(const slsht::So3Volume& v, const slsht::QuadratureWeights& qw,
                   double* d) {
  const int L = v.band_limit;
  const int n = 2 * L + 1, nb = L + 1;
  double s2 = 0.0, mx = 0.0;
  cplx proj{0.0, 0.0};
  for (std::size_t i = 0; i < v.values.size(); ++i) {
    const cplx g = v.values[i];
    const double a2 = g.real() * g.real() + g.imag() * g.imag();
    s2 += a2;
    mx = std::max(mx, std::sqrt(a2));
    const uint32_t hsh = static_cast<uint32_t>(i) * 0x9E3779B1u;
    const double w = static_cast<double>(hsh >> 8) * 0x1.0p-24 - 0.5;
    proj += w * g;
  }
  const cplx integ = slsht::integrate_volume(v, qw);
  (void)n;
  (void)nb;
  d[0] = s2;
  d[1] = mx;
  d[2] = proj.real();
  d[3] = proj.imag();
  d[4] = v.values[0].real();
  d[5] = v.values[0].imag();
  d[6] = integ.real();
  d[7] = integ.imag();
}
}  // namespace

extern "C" {

typedef void (*ref_sink_fn)(int l, int m, const double* volume, void* user);

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_forward_fast(int L_f, const double* f, int f_real, int L_h, const double* h,
                     int h_real, int lmax, int threads, int use_real_symmetry,
                     int emit_negative_m, ref_sink_fn cb, void* user) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, f_real);
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, h_real);
    slsht::ForwardOptions opts;
    opts.lmax = lmax;
    opts.threads = threads;
    opts.use_real_symmetry = use_real_symmetry != 0;
    opts.emit_negative_m = emit_negative_m != 0;
    slsht::forward_fast(
        fc, hc,
        [&](int l, int m, const slsht::So3Volume& v) {
          cb(l, m, reinterpret_cast<const double*>(v.values.data()), user);
        },
        opts);
  });
}

// forward_fast with a digest sink (8 doubles per component, slot coeff_index(l, m)),
// timed with steady_clock around the call (the CPU-baseline recipe of BASELINE.md §3).
int ref_forward_fast_digest(int L_f, const double* f, int f_real, int L_h,
                            const double* h, int h_real, int lmax, int threads,
                            int use_real_symmetry, int emit_negative_m, double* digests,
                            double* seconds) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, f_real);
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, h_real);
    slsht::ForwardOptions opts;
    opts.lmax = lmax;
    opts.threads = threads;
    opts.use_real_symmetry = use_real_symmetry != 0;
    opts.emit_negative_m = emit_negative_m != 0;
    const slsht::QuadratureWeights qw = slsht::beta_weights(L_h);
    const auto t0 = std::chrono::steady_clock::now();
    slsht::forward_fast(
        fc, hc,
        [&](int l, int m, const slsht::So3Volume& v) {
          digest_volume(v, qw, digests + 8 * static_cast<std::size_t>(slsht::coeff_index(l, m)));
        },
        opts);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

int ref_delta_tables(int L, double* out) {
  return guarded([&] {
    const slsht::DeltaTables d(L);
    std::size_t k = 0;
    for (int p = 0; p <= L; ++p)
      for (int q = -p; q <= p; ++q)
        for (int qp = -p; qp <= p; ++qp) out[k++] = d.at(p, q, qp);
  });
}

int ref_theta_weights(int N, double* out) {
  return guarded([&] {
    const std::vector<double> w = slsht::theta_weights(N);
    std::copy(w.begin(), w.end(), out);
  });
}

int ref_beta_weights(int L, double* out) {
  return guarded([&] {
    const slsht::QuadratureWeights qw = slsht::beta_weights(L);
    std::copy(qw.beta_weights.begin(), qw.beta_weights.end(), out);
  });
}

int ref_legendre_rows(int m, int lmax, const double* thetas, int n, double* rows) {
  return guarded([&] { slsht::legendre_rows(m, lmax, thetas, n, rows); });
}

int ref_modulated_sht(int L_f, const double* f, int l, int m, int L_h, double* out) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, 0);
    const slsht::ModulatedCoeffs mod = slsht::modulated_sht(fc, l, m, L_h);
    std::memcpy(out, mod.data.data(), sizeof(double) * 2 * mod.data.size());
  });
}

int ref_build_c_tensor(int L_h, const double* mod, const double* h, double* out) {
  return guarded([&] {
    slsht::ModulatedCoeffs mc;
    mc.band_limit = L_h;
    mc.data.resize(slsht::coeff_count(L_h));
    std::memcpy(mc.data.data(), mod, sizeof(double) * 2 * mc.data.size());
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, 0);
    const slsht::DeltaTables delta(L_h);
    const slsht::CTensor c = slsht::build_c_tensor(mc, hc, delta);
    std::memcpy(out, c.data.data(), sizeof(double) * 2 * c.data.size());
  });
}

int ref_evaluate(int L_h, const double* ctensor, double* out) {
  return guarded([&] {
    const int n = 2 * L_h + 1;
    slsht::CTensor c;
    c.band_limit = L_h;
    c.data.resize(static_cast<std::size_t>(n) * n * n);
    std::memcpy(c.data.data(), ctensor, sizeof(double) * 2 * c.data.size());
    const slsht::So3Evaluator ev(L_h);
    slsht::So3Evaluator::Scratch s;
    slsht::So3Volume vol;
    ev.evaluate(c, s, vol);
    std::memcpy(out, vol.values.data(), sizeof(double) * 2 * vol.values.size());
  });
}

int ref_integrate_volume(int L_h, const double* vol, double* out2) {
  return guarded([&] {
    slsht::So3Volume v = slsht::So3Volume::zeros(L_h);
    std::memcpy(v.values.data(), vol, sizeof(double) * 2 * v.values.size());
    const cplx r = slsht::integrate_volume(v, slsht::beta_weights(L_h));
    out2[0] = r.real();
    out2[1] = r.imag();
  });
}

// Streaming round trip exactly as acceptance criterion 1 runs it
// (proj/tests/acceptance_main.cpp:87-107): forward_fast into an InverseAccumulator.
int ref_roundtrip(int L_f, const double* f, int f_real, int L_h, const double* h,
                  int h_real, double* f_rec) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, f_real);
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, h_real);
    slsht::InverseAccumulator acc(L_f, L_h, hc.at(0, 0), true);
    slsht::ForwardOptions opts;
    opts.lmax = L_f;
    opts.emit_negative_m = false;
    slsht::forward_fast(fc, hc, acc.sink(), opts);
    const slsht::SphCoeffs back = acc.finish();
    std::memcpy(f_rec, back.data.data(), sizeof(double) * 2 * back.data.size());
  });
}

// Selected components (l[i], m[i]) through the reference's component-level public API, exactly
// as its bench_pass does (proj/src/cli.cpp:94-143): one ModulatedSht, DeltaTables and
// So3Evaluator, then compute -> build_c_tensor -> evaluate per component.
int ref_components(int L_f, const double* f, int L_h, const double* h, int count, const int* l,
                   const int* m, double* out) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, 0);
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, 0);
    const slsht::ModulatedSht ctx(fc, L_h);
    const slsht::DeltaTables delta(L_h);
    const slsht::So3Evaluator ev(L_h);
    slsht::ModulatedSht::Scratch scratch;
    slsht::So3Evaluator::Scratch es;
    slsht::ModulatedCoeffs mod;
    slsht::CTensor c;
    slsht::So3Volume vol;
    const std::size_t V = static_cast<std::size_t>(2 * L_h + 1) * (2 * L_h + 1) * (L_h + 1);
    for (int i = 0; i < count; ++i) {
      ctx.compute(l[i], m[i], scratch, mod);
      slsht::build_c_tensor(mod, hc, delta, c);
      ev.evaluate(c, es, vol);
      std::memcpy(out + 2 * V * static_cast<std::size_t>(i), vol.values.data(), sizeof(double) * 2 * V);
    }
  });
}

// The same chain on `threads` worker threads (each with its own scratch, as forward_fast's pool
// does, transform.cpp:263-294); the shared ModulatedSht / DeltaTables / So3Evaluator are const.
// Components are independent, so every volume is bitwise the single-threaded one.
int ref_components_mt(int L_f, const double* f, int L_h, const double* h, int count, const int* l,
                      const int* m, int threads, double* out) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, 0);
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, 0);
    const slsht::ModulatedSht ctx(fc, L_h);
    const slsht::DeltaTables delta(L_h);
    const slsht::So3Evaluator ev(L_h);
    const std::size_t V = static_cast<std::size_t>(2 * L_h + 1) * (2 * L_h + 1) * (L_h + 1);
    std::atomic<int> next{0};
    std::string first_error;
    std::mutex err_mutex;
    auto worker = [&] {
      try {
        slsht::ModulatedSht::Scratch scratch;
        slsht::So3Evaluator::Scratch es;
        slsht::ModulatedCoeffs mod;
        slsht::CTensor c;
        slsht::So3Volume vol;
        for (;;) {
          const int i = next.fetch_add(1);
          if (i >= count) break;
          ctx.compute(l[i], m[i], scratch, mod);
          slsht::build_c_tensor(mod, hc, delta, c);
          ev.evaluate(c, es, vol);
          std::memcpy(out + 2 * V * static_cast<std::size_t>(i), vol.values.data(),
                      sizeof(double) * 2 * V);
        }
      } catch (const std::exception& e) {
        std::lock_guard<std::mutex> lock(err_mutex);
        if (first_error.empty()) first_error = e.what();
        next.store(count);
      }
    };
    const int nt = std::max(1, std::min(threads, count));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (!first_error.empty()) throw slsht::ValidationError(first_error);
  });
}

// The per-call setup of forward_fast (transform.cpp:256-258): ModulatedSht (serial: the I table
// and the window Legendre table), DeltaTables and So3Evaluator, timed with steady_clock. The
// CPU-baseline extrapolation of SURVEY.md §8(d) subtracts it from a sampled run.
int ref_setup_seconds(int L_f, const double* f, int f_real, int L_h, const double* h, int h_real,
                      double* seconds) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, f_real);
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, h_real);
    const auto t0 = std::chrono::steady_clock::now();
    const slsht::ModulatedSht ctx(fc, L_h);
    const slsht::DeltaTables delta(L_h);
    const slsht::So3Evaluator ev(L_h);
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

// The reference's independent direct engine (transform.cpp:313-388): every component's
// So3Volume, out[(coeff_index(l, m) * V + cell) * 2].
int ref_forward_direct(int L_f, const double* f, int L_h, const double* h, int lmax, int threads,
                       double* out) {
  return guarded([&] {
    const slsht::SphCoeffs fc = make_coeffs(L_f, f, 0);
    const slsht::SphCoeffs hc = make_coeffs(L_h, h, 0);
    slsht::ForwardOptions opts;
    opts.lmax = lmax;
    opts.threads = threads;
    const slsht::SlshtDistribution d = slsht::forward_direct(fc, hc, opts);
    const std::size_t V = static_cast<std::size_t>(2 * L_h + 1) * (2 * L_h + 1) * (L_h + 1);
    for (std::size_t i = 0; i < d.components.size(); ++i)
      std::memcpy(out + 2 * V * i, d.components[i].values.data(), sizeof(double) * 2 * V);
  });
}

int ref_eigenfunction_window(double theta_c, double a, int L, int oversample,
                             double* out, double* lambda) {
  return guarded([&] {
    const slsht::Window w = slsht::eigenfunction_window({theta_c, a}, L, oversample);
    std::memcpy(out, w.coeffs.data.data(), sizeof(double) * 2 * w.coeffs.data.size());
    *lambda = w.lambda;
  });
}

int ref_random_coeffs(int L, uint64_t seed, int real_signal, double* out) {
  return guarded([&] {
    const slsht::SphCoeffs c = slsht::random_coeffs(L, seed, real_signal != 0);
    std::memcpy(out, c.data.data(), sizeof(double) * 2 * c.data.size());
  });
}

int ref_rotate_coeffs(int L, const double* in, double alpha, double beta, double gamma,
                      double* out) {
  return guarded([&] {
    const slsht::SphCoeffs c = make_coeffs(L, in, 0);
    const slsht::SphCoeffs r = slsht::rotate_coeffs(c, {alpha, beta, gamma});
    std::memcpy(out, r.data.data(), sizeof(double) * 2 * r.data.size());
  });
}

}  // extern "C"
