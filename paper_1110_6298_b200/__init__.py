"""B200-native McEwen-Wiaux spin spherical-harmonic transforms.

Drop-in for the reference package's transform path (torusht: forward,
inverse, forward_real, inverse_real, HarmonicCoeffs, MwSignal, the error
types), computed by hand-written sm_100a FP64 kernels (FFT stages included) behind the C ABI
in include/mwsht.h.  See DESIGN.md.
"""

from .errors import (ContractViolationError, ConvergenceError, DeviceError,
                     InvalidBandLimitError, InvalidSpinError, SymmetryError, TorushtError,
                     UnsupportedDegreeError)
from .mw import (HarmonicCoeffs, MwSignal, Plan, check_band_limit, clear_plans, forward,
                 forward_batch, forward_multi_spin, forward_real, get_plan, inverse, inverse_batch,
                 inverse_multi_spin, inverse_real,
                 mw_grid_phis, mw_grid_thetas, reality_residual)
from .gl import GlGrid, STABLE_BAND_LIMIT, gl_forward, gl_inverse, gl_nodes
from .io import load_coeffs, load_signal, read_coeffs_to, read_signal_to, save_coeffs, save_signal
from .pipeline import HostPipeline
from .quadrature import (QuadWeights, integrate, quad_weights, quad_weights_q, ring_weights_v,
                         synthesize_reduced, weight_w)

__all__ = [
    "HarmonicCoeffs", "MwSignal", "forward", "inverse", "forward_real", "inverse_real",
    "forward_batch", "inverse_batch", "forward_multi_spin", "inverse_multi_spin", "reality_residual", "HostPipeline", "check_band_limit",
    "mw_grid_thetas", "mw_grid_phis", "Plan", "get_plan", "clear_plans",
    "synthesize_reduced", "quad_weights", "quad_weights_q", "ring_weights_v", "weight_w",
    "integrate", "QuadWeights", "GlGrid", "gl_nodes", "gl_forward", "gl_inverse",
    "STABLE_BAND_LIMIT",
    "save_coeffs", "load_coeffs", "save_signal", "load_signal", "read_coeffs_to", "read_signal_to",
    "TorushtError", "InvalidBandLimitError", "InvalidSpinError", "ContractViolationError",
    "UnsupportedDegreeError", "SymmetryError", "ConvergenceError", "DeviceError",
]
