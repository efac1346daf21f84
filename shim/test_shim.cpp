// Drop-in check of the shim: the reference's own library (sources under /root/reference,
// with transform.cpp compiled as -Dforward_fast=reference_forward_fast so both engines can
// live in one binary) drives the B200 forward_fast through its UNCHANGED headers:
//  * engine equivalence against the reference CPU forward_fast (test_transform.cpp:229-262
//    shapes, real and complex, windows from the reference's eigenfunction_window);
//  * the streaming contract: every component once, sink == materialized (test_transform.cpp:331-348);
//  * the reference's InverseAccumulator consuming the shim's stream: acceptance criterion 1
//    (acceptance_main.cpp:87-107, error < 1e-9);
//  * ValidationError for lmax > L_f + L_h (transform.cpp:250-252);
//  * eigenfunction_window through the shim (window.cpp:126-198 on the device) against the
//    reference's CPU solver;
//  * the CLI's `forward --engine fast` path (cli.cpp:220-224): the reference's
//    io::DistributionWriter as the sink, read back with io::read_component (SURVEY 8(f)
//    next-2: host sink delivery and on-disk format through the drop-in).
// Prints one PASS/FAIL line per check; exit status 0 iff all pass.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <complex>
#include <cstdio>
#include <map>
#include <numbers>
#include <random>
#include <vector>

#include <filesystem>

#include "slsht/errors.hpp"
#include "slsht/io.hpp"
#include "slsht/signals.hpp"
#include "slsht/transform.hpp"
#include "slsht/window.hpp"

namespace slsht {
// the reference's CPU engine, renamed at compile time (see Makefile)
void reference_forward_fast(const SphCoeffs& f, const SphCoeffs& h, const ComponentSink& sink,
                            const ForwardOptions& opts);
SlshtDistribution reference_forward_fast(const SphCoeffs& f, const SphCoeffs& h,
                                         const ForwardOptions& opts);
SlshtDistribution reference_forward_direct(const SphCoeffs& f, const SphCoeffs& h,
                                           const ForwardOptions& opts);
// the reference's CPU window solver, renamed at compile time (see Makefile)
Window reference_eigenfunction_window(const EllipticalRegion& region, int band_limit,
                                      int oversample);
}  // namespace slsht

using namespace slsht;
using cplx = std::complex<double>;

static int failures = 0;
static void report(bool ok, const char* name, double value, double limit) {
  std::printf("%s %-58s %.3e (limit %.0e)\n", ok ? "PASS" : "FAIL", name, value, limit);
  if (!ok) ++failures;
}

static SphCoeffs random_complex(int L, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  SphCoeffs c = SphCoeffs::zeros(L);
  for (auto& v : c.data)
    v = cplx(static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5,
             static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5);
  return c;
}

static double max_diff(const SlshtDistribution& a, const SlshtDistribution& b) {
  double worst = 0.0;
  for (int l = 0; l <= a.lmax; ++l)
    for (int m = -l; m <= l; ++m) {
      const auto& va = a.component(l, m).values;
      const auto& vb = b.component(l, m).values;
      if (va.size() != vb.size()) return INFINITY;
      for (std::size_t i = 0; i < va.size(); ++i) worst = std::max(worst, std::abs(va[i] - vb[i]));
    }
  return worst;
}

int main() {
  {
    // forward_direct drop-in (the device direct engine) against the reference's CPU direct
    // engine, and against the fast engine
    const SphCoeffs f = random_complex(6, 45), h = random_complex(3, 46);
    const SlshtDistribution a = forward_direct(f, h);
    const SlshtDistribution b = reference_forward_direct(f, h, {});
    report(max_diff(a, b) < 1e-12, "forward_direct (6, 3) vs reference forward_direct",
           max_diff(a, b), 1e-12);
    ForwardOptions lo;
    lo.lmax = 4;
    const double d2 = max_diff(forward_direct(f, h, lo), reference_forward_direct(f, h, lo));
    report(d2 < 1e-12, "forward_direct lmax = 4 < L_g vs reference", d2, 1e-12);
    const double d3 = max_diff(a, forward_fast(f, h));
    report(d3 < 1e-12, "forward_direct vs forward_fast (6, 3)", d3, 1e-12);
  }
  {
    const SphCoeffs f = random_complex(3, 41), h = random_complex(2, 42);
    report(max_diff(forward_fast(f, h), reference_forward_fast(f, h, {})) < 1e-12,
           "complex (L_f, L_h) = (3, 2) vs reference forward_fast",
           max_diff(forward_fast(f, h), reference_forward_fast(f, h, {})), 1e-12);
  }
  {
    const SphCoeffs f = random_coeffs(6, 43, true);
    const Window w = eigenfunction_window({0.3, 0.7}, 3, 4);
    const double d = max_diff(forward_fast(f, w.coeffs), reference_forward_fast(f, w.coeffs, {}));
    report(d < 1e-12, "real mode (6, 3), eigenfunction window, mirrored m < 0", d, 1e-12);
    ForwardOptions full;
    full.use_real_symmetry = false;
    const double d2 = max_diff(forward_fast(f, w.coeffs, full), reference_forward_fast(f, w.coeffs, {}));
    report(d2 < 1e-12, "full-m mode vs reference real mode (conjugate symmetry)", d2, 1e-12);
  }
  {
    const SphCoeffs f = random_complex(32, 1), h = random_complex(8, 2);
    const SlshtDistribution a = forward_fast(f, h);
    const SlshtDistribution b = reference_forward_fast(f, h, {});
    double scale = 0.0;
    for (const auto& c : b.components)
      for (const auto& v : c.values) scale = std::max(scale, std::abs(v));
    const double d = max_diff(a, b) / scale;
    report(d < 1e-10, "config-1 shape (32, 8): eps_inf relative to max |g|", d, 1e-10);
  }
  {
    const SphCoeffs f = random_complex(3, 71), h = random_complex(2, 72);
    const SlshtDistribution dist = forward_fast(f, h);
    std::map<std::pair<int, int>, So3Volume> seen;
    bool once = true;
    forward_fast(f, h, [&](int l, int m, const So3Volume& v) {
      once = once && seen.emplace(std::make_pair(l, m), v).second;
    });
    double d = 0.0;
    for (const auto& [key, vol] : seen) {
      const auto& ref = dist.component(key.first, key.second).values;
      for (std::size_t i = 0; i < ref.size(); ++i) d = std::max(d, std::abs(vol.values[i] - ref[i]));
    }
    const bool ok = once && seen.size() == static_cast<std::size_t>(coeff_count(5)) && d == 0.0;
    report(ok, "streaming sink sees every component once, == materialized", d, 0.0);
  }
  {
    const Window win18 = eigenfunction_window(
        {std::numbers::pi / 6.0, std::numbers::pi / 6.0 + std::numbers::pi / 240.0}, 18, 4);
    double worst = 0.0;
    for (const int lf : {18, 32}) {
      const SphCoeffs f = random_coeffs(lf, 100 + lf, true);
      InverseAccumulator acc(lf, 18, win18.coeffs.at(0, 0), true);
      ForwardOptions opts;
      opts.lmax = lf;
      opts.emit_negative_m = false;
      forward_fast(f, win18.coeffs, acc.sink(), opts);
      const SphCoeffs back = acc.finish();
      for (int i = 0; i < coeff_count(lf); ++i)
        worst = std::max(worst, std::abs(back.data[i] - f.data[i]));
    }
    report(worst < 1e-9, "round trip via the reference InverseAccumulator (L_h = 18)", worst, 1e-9);
  }
  {
    bool threw = false;
    try {
      ForwardOptions opts;
      opts.lmax = 9;
      forward_fast(random_complex(4, 5), random_complex(3, 6), opts);
    } catch (const ValidationError&) {
      threw = true;
    }
    report(threw, "lmax > L_f + L_h throws ValidationError", threw ? 0.0 : 1.0, 0.0);
  }
  {
    // cli.cpp:220-224 with the drop-in: DistributionWriter sink, files read back
    const SphCoeffs f = random_coeffs(12, 41, true);
    const Window win = eigenfunction_window(
        {std::numbers::pi / 5.0, std::numbers::pi / 5.0 + std::numbers::pi / 200.0}, 6, 3);
    const int top = 12 + 6;
    const std::filesystem::path dir =
        std::filesystem::temp_directory_path() / "slsht_shim_writer_test";
    std::filesystem::remove_all(dir);
    {
      io::DistributionWriter writer(dir, 12, 6, top, true);
      ForwardOptions opts;
      opts.lmax = top;
      forward_fast(f, win.coeffs, writer.sink(), opts);
      writer.finalize();
    }
    const io::DistributionManifest man = io::read_manifest(dir);
    ForwardOptions opts;
    opts.lmax = top;
    const SlshtDistribution ref = reference_forward_fast(f, win.coeffs, opts);
    double num = 0.0, den = 0.0;
    bool complete = man.components.size() == static_cast<std::size_t>(coeff_count(top));
    for (const auto& [l, m] : man.components) {
      const So3Volume v = io::read_component(dir, man, l, m);
      const So3Volume& r = ref.component(l, m);
      for (std::size_t i = 0; i < r.values.size(); ++i) {
        num = std::max(num, std::abs(v.values[i] - r.values[i]));
        den = std::max(den, std::abs(r.values[i]));
      }
    }
    std::filesystem::remove_all(dir);
    const double rel = complete ? num / den : 1.0;
    report(complete && rel < 1e-12, "CLI path: DistributionWriter sink, files vs reference", rel,
           1e-12);
  }
  {
    // eigenfunction_window: device solver (shim) vs the reference's CPU solver
    double worst = 0.0, dl = 0.0;
    const EllipticalRegion regions[] = {{std::numbers::pi / 9.0, std::numbers::pi / 6.0},
                                        {0.3, 0.7}};
    const int bls[] = {16, 6};
    for (int i = 0; i < 2; ++i) {
      const Window a = eigenfunction_window(regions[i], bls[i], 4);
      const Window b = reference_eigenfunction_window(regions[i], bls[i], 4);
      for (std::size_t k = 0; k < a.coeffs.data.size(); ++k)
        worst = std::max(worst, std::abs(a.coeffs.data[k] - b.coeffs.data[k]));
      dl = std::max(dl, std::abs(a.lambda - b.lambda));
    }
    report(worst < 1e-9 && dl < 1e-12, "eigenfunction_window (device) vs reference solver", worst,
           1e-9);
    bool threw = false;
    try {
      eigenfunction_window({0.8, 0.5}, 4, 4);
    } catch (const ValidationError&) {
      threw = true;
    }
    report(threw, "eigenfunction_window: theta_c > a throws ValidationError", threw ? 0.0 : 1.0,
           0.0);
  }
  {
    // the shim's plan cache: repeated calls (same and interleaved shapes, with a validation
    // error in between) give bitwise the results of fresh plans
    const SphCoeffs f = random_complex(10, 61), h = random_complex(4, 62);
    const SphCoeffs f2 = random_complex(7, 63), h2 = random_complex(3, 64);
    const SlshtDistribution a1 = forward_fast(f, h);
    const SlshtDistribution b1 = forward_fast(f2, h2);
    ForwardOptions bad;
    bad.lmax = 99;
    try {
      forward_fast(f, h, bad);
    } catch (const ValidationError&) {
    }
    const SlshtDistribution a2 = forward_fast(f, h);
    const SlshtDistribution b2 = forward_fast(f2, h2);
    setenv("SLSHT_CUDA_PLAN_CACHE", "0", 1);
    const SlshtDistribution a3 = forward_fast(f, h);
    unsetenv("SLSHT_CUDA_PLAN_CACHE");
    const double d = std::max({max_diff(a1, a2), max_diff(b1, b2), max_diff(a1, a3)});
    report(d == 0.0, "plan cache: repeated calls bitwise equal to fresh plans", d, 0.0);
    // device selection: two degree shards (here both on device 0, the test box's one GPU)
    // give bitwise the one-device result, through the multi-GPU plan of the C ABI
    setenv("SLSHT_CUDA_DEVICES", "0,0", 1);
    const SlshtDistribution a4 = forward_fast(f, h);
    unsetenv("SLSHT_CUDA_DEVICES");
    const double d4 = max_diff(a1, a4);
    report(d4 == 0.0, "two-shard plan (SLSHT_CUDA_DEVICES) bitwise equal to one device", d4, 0.0);
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "ALL PASSED", failures);
  return failures ? 1 : 0;
}
