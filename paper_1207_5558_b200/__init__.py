"""B200-native directional SLSHT forward engine (arXiv 1207.5558), sm_100a CUDA behind a C ABI.

Drop-in for the reference's hot path slsht::forward_fast
(/root/reference/proj/include/slsht/transform.hpp:159-165). See DESIGN.md and INTEGRATION.md.
"""
from ._lib import DIGEST_WIDTH, LIB_PATH, load
from .transform import (DeviceError, ForwardOptions, NumericError, Plan, SlshtDistribution,
                        SphCoeffs, ValidationError, beta_weights, coeff_count, coeff_index,
                        delta_tables, eigenfunction_window, forward_direct, forward_fast,
                        gauss_legendre_half, legendre_rows, modulated_sht, shard_bounds,
                        theta_weights, volume_shape)

__all__ = [
    "DIGEST_WIDTH", "LIB_PATH", "load", "DeviceError", "ForwardOptions", "NumericError", "Plan",
    "SlshtDistribution", "SphCoeffs", "ValidationError", "coeff_count", "coeff_index",
    "delta_tables", "eigenfunction_window", "forward_direct", "forward_fast", "modulated_sht",
    "shard_bounds", "volume_shape", "theta_weights", "beta_weights", "legendre_rows",
    "gauss_legendre_half",
]
