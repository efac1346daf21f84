// Drop-in replacement of slsht::eigenfunction_window for the reference library
// (proj/include/slsht/window.hpp:61-63, proj/src/window.cpp:126-198), compiled against its
// UNCHANGED headers and implemented on the C ABI (slsht_cuda_eigenfunction_window): the
// concentration kernel by one ZGEMM and the reference's power iteration on the device.
// Same validation (ValidationError) and numeric failures (NumericError) as the reference.
// Environment: SLSHT_CUDA_DEVICE (default 0).
#include <complex>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "slsht/errors.hpp"
#include "slsht/window.hpp"
#include "slsht_cuda.h"

namespace slsht {

Window eigenfunction_window(const EllipticalRegion& region, int band_limit, int oversample) {
  const char* dv = std::getenv("SLSHT_CUDA_DEVICE");
  const int device = dv ? std::atoi(dv) : 0;
  Window win;
  win.region = region;
  win.coeffs = SphCoeffs::zeros(band_limit < 0 ? 0 : band_limit, true);
  double lambda = 0.0;
  const int rc = slsht_cuda_eigenfunction_window(
      device, region.theta_c, region.a, band_limit, oversample,
      reinterpret_cast<double*>(win.coeffs.data.data()), &lambda);
  if (rc != SLSHT_OK) {
    const std::string msg = slsht_cuda_last_error(nullptr);
    if (rc == SLSHT_ERR_VALIDATION) throw ValidationError(msg);
    if (rc == SLSHT_ERR_NUMERIC) throw NumericError(msg);
    throw std::runtime_error("slsht_cuda: " + msg);
  }
  win.lambda = lambda;
  return win;
}

}  // namespace slsht
