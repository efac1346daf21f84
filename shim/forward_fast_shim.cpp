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
//
// Devices: like the reference's worker pool (transform.cpp:260-294) the call uses the whole
// machine: every visible B200, one degree shard each (a multi-GPU plan);
// SLSHT_CUDA_DEVICES="0,2,..." picks the devices, SLSHT_CUDA_DEVICE=k a single one. Results are
// bitwise the same for any device count.
// Plans: the reference's callers make many small calls (tests, the CLI), so plans (tables,
// ring, pinned staging, streams) are cached per (L_f, L_h, lmax, mode, devices, ring), up to
// SLSHT_CUDA_PLAN_CACHE entries (default 4, least recently used evicted; 0 disables), and reused
// under one mutex: calls from several threads are serialized, as the device is shared anyway.
// Environment: SLSHT_CUDA_RING_MB (default 256, per device).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <list>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

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

std::vector<int> device_list() {
  if (const char* v = std::getenv("SLSHT_CUDA_DEVICES")) {
    std::vector<int> out;
    for (const char* p = v; *p;) {
      char* end = nullptr;
      const long d = std::strtol(p, &end, 10);
      if (end == p) break;
      out.push_back(static_cast<int>(d));
      p = (*end == ',') ? end + 1 : end;
    }
    if (!out.empty()) return out;
  }
  if (std::getenv("SLSHT_CUDA_DEVICE")) return {env_int("SLSHT_CUDA_DEVICE", 0)};
  const int n = slsht_cuda_device_count();
  std::vector<int> out;
  for (int d = 0; d < std::max(n, 1); ++d) out.push_back(d);
  return out;
}

struct PlanKey {
  int L_f, L_h, lmax, real_mode, emit_neg;
  long long ring;
  std::vector<int> devices;
  bool operator==(const PlanKey& o) const {
    return L_f == o.L_f && L_h == o.L_h && lmax == o.lmax && real_mode == o.real_mode &&
           emit_neg == o.emit_neg && ring == o.ring && devices == o.devices;
  }
};

// Plans in use order (front: most recent). Cached plans are never destroyed at exit (the CUDA
// runtime may already be shut down by then); the process exit releases them.
std::mutex g_mutex;
std::list<std::pair<PlanKey, slsht_cuda_plan*>> g_plans;

// Returns a plan for the key (cached or new); the caller holds g_mutex.
slsht_cuda_plan* acquire_plan(const PlanKey& key, bool& owned) {
  const int cap = env_int("SLSHT_CUDA_PLAN_CACHE", 4);
  owned = cap <= 0;
  if (!owned)
    for (auto it = g_plans.begin(); it != g_plans.end(); ++it)
      if (it->first == key) {
        g_plans.splice(g_plans.begin(), g_plans, it);
        return it->second;
      }
  slsht_cuda_desc desc{};
  desc.L_f = key.L_f;
  desc.L_h = key.L_h;
  desc.lmax = key.lmax;
  desc.real_mode = key.real_mode;
  desc.emit_negative_m = key.emit_neg;
  desc.device = key.devices.front();
  desc.n_devices = static_cast<int>(key.devices.size());
  desc.devices = key.devices.size() > 1 ? key.devices.data() : nullptr;
  desc.l_begin = 0;
  desc.l_end = -1;
  desc.materialize = 0;
  desc.ring_bytes = key.ring;
  slsht_cuda_plan* plan = nullptr;
  const int rc = slsht_cuda_plan_create(&desc, &plan);
  if (rc != SLSHT_OK) raise_status(rc, nullptr);
  if (owned) return plan;
  g_plans.emplace_front(key, plan);
  while (static_cast<int>(g_plans.size()) > cap) {
    slsht_cuda_plan_destroy(g_plans.back().second);
    g_plans.pop_back();
  }
  return plan;
}

}  // namespace

void forward_fast(const SphCoeffs& f, const SphCoeffs& h, const ComponentSink& sink,
                  const ForwardOptions& opts) {
  const int L_f = f.band_limit;
  const int L_h = h.band_limit;
  const int L_g = L_f + L_h;
  const int lmax = opts.lmax < 0 ? L_g : opts.lmax;
  if (lmax > L_g) throw ValidationError("fast engine computes components up to L_f + L_h only");
  const PlanKey key{L_f, L_h, lmax, opts.use_real_symmetry && f.real_signal && h.real_signal,
                    opts.emit_negative_m ? 1 : 0,
                    static_cast<long long>(env_int("SLSHT_CUDA_RING_MB", 256)) << 20,
                    device_list()};
  std::lock_guard<std::mutex> lock(g_mutex);
  bool owned = false;
  slsht_cuda_plan* plan = acquire_plan(key, owned);
  SinkContext ctx{&sink, So3Volume::zeros(L_h), nullptr};
  const int rc = slsht_cuda_forward(plan, reinterpret_cast<const double*>(f.data.data()),
                                    reinterpret_cast<const double*>(h.data.data()), deliver, &ctx);
  if (rc != SLSHT_OK) {
    const std::string msg = slsht_cuda_last_error(plan);
    // a failed call leaves the plan reusable (validation errors) or suspect (device errors):
    // drop device-error plans from the cache
    if (rc == SLSHT_ERR_DEVICE && !owned)
      g_plans.remove_if([plan](const auto& e) { return e.second == plan; });
    if (owned || rc == SLSHT_ERR_DEVICE) slsht_cuda_plan_destroy(plan);
    if (rc == SLSHT_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == SLSHT_ERR_NUMERIC) throw NumericError(msg);
    throw std::runtime_error("slsht_cuda: " + msg);
  }
  if (owned) slsht_cuda_plan_destroy(plan);
  if (ctx.error) std::rethrow_exception(ctx.error);
}

SlshtDistribution forward_fast(const SphCoeffs& f, const SphCoeffs& h, const ForwardOptions& opts) {
  // transform.cpp:297-311. Every emitted volume is copied straight from the engine's pinned
  // staging buffers into its So3Volume (slsht_cuda_forward_scatter: disjoint destinations,
  // several host threads), instead of through the serialized sink and two more copies.
  SlshtDistribution dist;
  dist.L_f = f.band_limit;
  dist.L_h = h.band_limit;
  dist.L_g = dist.L_f + dist.L_h;
  dist.lmax = opts.lmax < 0 ? dist.L_g : opts.lmax;
  if (dist.lmax > dist.L_g)
    throw ValidationError("fast engine computes components up to L_f + L_h only");
  dist.grid = so3_grid(dist.L_h);
  dist.components.assign(coeff_count(dist.lmax), So3Volume{});
  const bool real_mode = opts.use_real_symmetry && f.real_signal && h.real_signal;
  const PlanKey key{dist.L_f, dist.L_h, dist.lmax, real_mode, opts.emit_negative_m ? 1 : 0,
                    static_cast<long long>(env_int("SLSHT_CUDA_RING_MB", 256)) << 20,
                    device_list()};
  // the components the call emits (transform.cpp:262-284): all (l, m) of l <= lmax, or in real
  // mode m >= 0 and, with emit_negative_m, their mirrors; the others stay empty
  std::vector<double*> targets(dist.components.size(), nullptr);
  {
    // allocation (first touch of every page) on several host threads, degree-interleaved
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nt = std::max(1, std::min<int>({env_int("SLSHT_CUDA_HOST_THREADS", 16), (int)hw,
                                              dist.lmax + 1}));
    auto work = [&](int t) {
      for (int l = t; l <= dist.lmax; l += nt)
        for (int m = -l; m <= l; ++m) {
          if (real_mode && m < 0 && !opts.emit_negative_m) continue;
          So3Volume& v = dist.component(l, m);
          v = So3Volume::zeros(dist.L_h);
          targets[coeff_index(l, m)] = reinterpret_cast<double*>(v.values.data());
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
  }
  std::lock_guard<std::mutex> lock(g_mutex);
  bool owned = false;
  slsht_cuda_plan* plan = acquire_plan(key, owned);
  long long delivered = 0;
  const int rc = slsht_cuda_forward_scatter(
      plan, reinterpret_cast<const double*>(f.data.data()),
      reinterpret_cast<const double*>(h.data.data()), targets.data(),
      static_cast<long long>(targets.size()), 0, &delivered);
  if (rc != SLSHT_OK) {
    const std::string msg = slsht_cuda_last_error(plan);
    if (rc == SLSHT_ERR_DEVICE && !owned)
      g_plans.remove_if([plan](const auto& e) { return e.second == plan; });
    if (owned || rc == SLSHT_ERR_DEVICE) slsht_cuda_plan_destroy(plan);
    if (rc == SLSHT_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == SLSHT_ERR_NUMERIC) throw NumericError(msg);
    throw std::runtime_error("slsht_cuda: " + msg);
  }
  if (owned) slsht_cuda_plan_destroy(plan);
  return dist;
}

}  // namespace slsht
