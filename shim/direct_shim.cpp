// Drop-in replacement of slsht::forward_direct (proj/include/slsht/transform.hpp:167-168 and the
// Window overload at :185-188, proj/src/transform.cpp:313-388) on the C ABI of the B200 engine:
// the reference's independent direct engine, computed on the device
// (slsht_cuda_forward_direct). Same result layout (SlshtDistribution over so3_grid(L_h), every
// component l <= lmax), same sphere band max(lmax, L_f + L_h). ForwardOptions::threads has no
// meaning on the device and is ignored. Environment: SLSHT_CUDA_DEVICE (default 0).
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "slsht/errors.hpp"
#include "slsht/grids.hpp"
#include "slsht/transform.hpp"
#include "slsht_cuda.h"

namespace slsht {

SlshtDistribution forward_direct(const SphCoeffs& f, const SphCoeffs& h, const ForwardOptions& opts) {
  SlshtDistribution dist;
  dist.L_f = f.band_limit;
  dist.L_h = h.band_limit;
  dist.L_g = dist.L_f + dist.L_h;
  dist.lmax = opts.lmax < 0 ? dist.L_g : opts.lmax;
  dist.grid = so3_grid(dist.L_h);
  const std::size_t V = static_cast<std::size_t>(2 * dist.L_h + 1) * (2 * dist.L_h + 1) *
                        (dist.L_h + 1);
  const int rows = coeff_count(dist.lmax);
  std::vector<double> out(2 * V * static_cast<std::size_t>(rows));
  const char* dev = std::getenv("SLSHT_CUDA_DEVICE");
  const int rc = slsht_cuda_forward_direct(
      dev ? std::atoi(dev) : 0, dist.L_f, reinterpret_cast<const double*>(f.data.data()), dist.L_h,
      reinterpret_cast<const double*>(h.data.data()), dist.lmax, nullptr, 0, out.data());
  if (rc != SLSHT_OK) {
    const std::string msg = slsht_cuda_last_error(nullptr);
    if (rc == SLSHT_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == SLSHT_ERR_NUMERIC) throw NumericError(msg);
    throw std::runtime_error("slsht_cuda: " + msg);
  }
  dist.components.assign(rows, So3Volume{});
  for (int i = 0; i < rows; ++i) {
    So3Volume& v = dist.components[i];
    v = So3Volume::zeros(dist.L_h);
    const double* src = out.data() + 2 * V * static_cast<std::size_t>(i);
    for (std::size_t k = 0; k < V; ++k) v.values[k] = {src[2 * k], src[2 * k + 1]};
  }
  return dist;
}

}  // namespace slsht
