// Drop-in replacement of slsht::forward_fast (both overloads) for the reference library,
// compiled against its UNCHANGED public headers (/root/reference/proj/include/slsht) and
// implemented on top of the C ABI of the B200 engine (include/slsht_cuda.h).
//
//   void forward_fast(const SphCoeffs&, const SphCoeffs&, const ComponentSink&, const ForwardOptions&)
//        proj/include/slsht/transform.hpp:162-163, proj/src/transform.cpp:244-295
//   SlshtDistribution forward_fast(const SphCoeffs&, const SphCoeffs&, const ForwardOptions&)
//        proj/include/slsht/transform.hpp:164-165, proj/src/transform.cpp:297-311
//
// Semantics kept from the reference: lmax validation and real-mode selection
// (transform.cpp:249-254), every component emitted once with (l, -m) right after (l, m) in
// real mode (transform.cpp:280-284), serialized sink calls with a volume reference valid only
// during the call, ValidationError / NumericError for the C status codes 2 / 3
// (errors.hpp:7-16). ForwardOptions::threads has no meaning on the device and is ignored.
// Environment: SLSHT_CUDA_DEVICE (default 0), SLSHT_CUDA_RING_MB (default 256).
#include <cstdlib>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

#include "slsht/errors.hpp"
#include "slsht/grids.hpp"
#include "slsht/transform.hpp"
#include "slsht_cuda.h"

namespace slsht {
namespace {

int env_int(const char* name, int fallback) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : fallback;
}

[[noreturn]] void raise_status(int rc, const slsht_cuda_plan* plan) {
  const std::string msg = slsht_cuda_last_error(plan);
  if (rc == SLSHT_ERR_VALIDATION) throw ValidationError(msg);
  if (rc == SLSHT_ERR_NUMERIC) throw NumericError(msg);
  throw std::runtime_error("slsht_cuda: " + msg);
}

struct SinkContext {
  const ComponentSink* sink;
  So3Volume volume;
  std::exception_ptr error;
};

extern "C" void deliver(int l, int m, const double* data, void* user) {
  auto* ctx = static_cast<SinkContext*>(user);
  if (ctx->error) return;  // a sink threw: drain the remaining callbacks, rethrow afterwards
  try {
    std::memcpy(ctx->volume.values.data(), data, sizeof(double) * 2 * ctx->volume.values.size());
    (*ctx->sink)(l, m, ctx->volume);
  } catch (...) {
    ctx->error = std::current_exception();
  }
}

}  // namespace

void forward_fast(const SphCoeffs& f, const SphCoeffs& h, const ComponentSink& sink,
                  const ForwardOptions& opts) {
  const int L_f = f.band_limit;
  const int L_h = h.band_limit;
  const int L_g = L_f + L_h;
  const int lmax = opts.lmax < 0 ? L_g : opts.lmax;
  if (lmax > L_g) throw ValidationError("fast engine computes components up to L_f + L_h only");
  slsht_cuda_desc desc{};
  desc.L_f = L_f;
  desc.L_h = L_h;
  desc.lmax = lmax;
  desc.real_mode = opts.use_real_symmetry && f.real_signal && h.real_signal;
  desc.emit_negative_m = opts.emit_negative_m;
  desc.device = env_int("SLSHT_CUDA_DEVICE", 0);
  desc.l_begin = 0;
  desc.l_end = -1;
  desc.materialize = 0;
  desc.ring_bytes = static_cast<long long>(env_int("SLSHT_CUDA_RING_MB", 256)) << 20;
  slsht_cuda_plan* plan = nullptr;
  int rc = slsht_cuda_plan_create(&desc, &plan);
  if (rc != SLSHT_OK) raise_status(rc, nullptr);
  SinkContext ctx{&sink, So3Volume::zeros(L_h), nullptr};
  rc = slsht_cuda_forward(plan, reinterpret_cast<const double*>(f.data.data()),
                          reinterpret_cast<const double*>(h.data.data()), deliver, &ctx);
  if (rc != SLSHT_OK) {
    const std::string msg = slsht_cuda_last_error(plan);
    slsht_cuda_plan_destroy(plan);
    if (rc == SLSHT_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == SLSHT_ERR_NUMERIC) throw NumericError(msg);
    throw std::runtime_error("slsht_cuda: " + msg);
  }
  slsht_cuda_plan_destroy(plan);
  if (ctx.error) std::rethrow_exception(ctx.error);
}

SlshtDistribution forward_fast(const SphCoeffs& f, const SphCoeffs& h, const ForwardOptions& opts) {
  SlshtDistribution dist;
  dist.L_f = f.band_limit;
  dist.L_h = h.band_limit;
  dist.L_g = dist.L_f + dist.L_h;
  dist.lmax = opts.lmax < 0 ? dist.L_g : opts.lmax;
  if (dist.lmax > dist.L_g)
    throw ValidationError("fast engine computes components up to L_f + L_h only");
  dist.grid = so3_grid(dist.L_h);
  dist.components.assign(coeff_count(dist.lmax), So3Volume{});
  forward_fast(
      f, h, [&dist](int l, int m, const So3Volume& v) { dist.component(l, m) = v; }, opts);
  return dist;
}

}  // namespace slsht
