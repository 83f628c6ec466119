"""Reduced-grid synthesis and the MW quadrature.

Mirrors the reference's quadrature and reduced-grid functions
(pkg/src/torusht/quadrature.py:34-139, mw.py:449-466): the same names,
arguments and error types.  The O(L^3) part of ``synthesize_reduced`` is the
inverse core plus the theta synthesis of the CUDA inverse pipeline
(``mwsht_shard_inverse_front`` over all orders).  The residue fold and the
L-point azimuthal DFT run on the device through torch (cuFFT).  The weights
are O(L) device FFTs.  Nothing here runs on the host CPU.

* ``quad_weights(L, spin)`` -> QuadWeights(band_limit, spin, w, v, q):
  w(m') for |m'| <= 2(L-1), ring weights v(theta_t) over the 2L-1 extended
  rings (quadrature.py:77-93), quadrature weights q(theta_t) over the L
  physical rings (quadrature.py:96-111).
* ``synthesize_reduced(coeffs)`` -> samples on the reduced grid
  (theta_t, 2 pi p / L), (L, L) complex (mw.py:449-466).
* ``integrate(samples, weights)`` -> the exact integral over the sphere of
  a band-limited f sampled on that grid (quadrature.py:123-139).
"""

import math
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ContractViolationError, SymmetryError
from .mw import (_back, _check_recursion, _check_spin, _stream, _target_device, _to_device,
                 check_band_limit, get_plan)

IMAG_GUARD = 1e-12  # quadrature.py:31


@dataclass(frozen=True)
class QuadWeights:
    """Weights for one (band_limit, spin): ``w`` over m' in [-2(L-1), 2(L-1)],
    ``v`` over the 2L-1 extended rings, ``q`` over the L physical rings."""

    band_limit: int
    spin: int
    w: torch.Tensor
    v: torch.Tensor
    q: torch.Tensor


def _device():
    if not torch.cuda.is_available():
        from .errors import DeviceError
        raise DeviceError("the quadrature runs on a CUDA device; none is available")
    return torch.cuda.current_device()


def weight_w(k, device=None):
    """w(k) = int_0^pi sin(theta) e^{i k theta} d theta (quadrature.py:54-74):
    w(0) = 2, w(+-1) = +-i pi/2, 0 for other odd k, 2/(1-k^2) for even k."""
    dev = _device() if device is None else device
    k = torch.as_tensor(k, dtype=torch.int64, device=f"cuda:{dev}")
    kd = k.to(torch.float64)
    even = (k % 2) == 0
    re = torch.where(even, 2.0 / (1.0 - kd * kd), torch.zeros_like(kd))
    im = torch.where(k == 1, torch.full_like(kd, math.pi / 2),
                     torch.where(k == -1, torch.full_like(kd, -math.pi / 2), torch.zeros_like(kd)))
    return torch.complex(re, im)


def _check_imag(x, label):
    peak = float(x.imag.abs().max()) if x.numel() else 0.0
    if peak > IMAG_GUARD:
        raise SymmetryError(f"{label} should be real to rounding, found imaginary part {peak:.3e}")


def ring_weights_v(band_limit, device=None):
    """v(theta_t) = (1/(2L-1)) sum_{|m'|<=L-1} w(-m') e^{i m' theta_t}, t < 2L-1."""
    check_band_limit(band_limit)
    L = int(band_limit)
    dev = _device() if device is None else device
    mp = torch.arange(-(L - 1), L, device=f"cuda:{dev}")
    theta0 = math.pi / (2 * L - 1)
    spectrum = weight_w(-mp, dev) * torch.polar(torch.ones(mp.shape, dtype=torch.float64,
                                                            device=mp.device),
                                                mp.to(torch.float64) * theta0)
    v = torch.fft.ifft(torch.fft.ifftshift(spectrum))
    _check_imag(v, "ring weights v")
    return v


def quad_weights_q(band_limit, spin, device=None):
    """q(theta_t) = (2 pi/L) [v(theta_t) + (-1)^s v(theta_{2L-2-t})], t < L;
    the reflected term is dropped at t = L-1."""
    check_band_limit(band_limit)
    L = int(band_limit)
    v = ring_weights_v(L, device)
    q = v[:L].clone()
    if L > 1:
        q[: L - 1] += (-1.0 if spin % 2 else 1.0) * torch.flip(v[L:2 * L - 1], dims=[0])
    q = q * (2.0 * math.pi / L)
    _check_imag(q, "quadrature weights q")
    return q


def quad_weights(band_limit, spin=0):
    check_band_limit(band_limit)
    L = int(band_limit)
    dev = _device()
    mp = torch.arange(-2 * (L - 1), 2 * (L - 1) + 1, device=f"cuda:{dev}")
    return QuadWeights(L, spin, weight_w(mp, dev), ring_weights_v(L, dev),
                       quad_weights_q(L, spin, dev))


def synthesize_reduced(coeffs, recursion="trapani"):
    """Samples on the reduced grid (theta_t, 2 pi p / L), p < L  (mw.py:449-466).

    The CUDA inverse pipeline produces the theta-synthesised rows F_m(theta_t)
    (core + theta stage over all orders).  Orders m and m - L land on the same
    bin of an L-point ring, so they are folded by residue, then one L-point
    inverse DFT per ring gives the samples.
    """
    L, spin = coeffs.band_limit, coeffs.spin
    _check_spin(L, spin)
    _check_recursion(recursion)
    dev = _target_device(coeffs.values)
    f = _to_device(coeffs.values, torch.complex128, dev)
    N = 2 * L - 1
    rows = torch.empty((L, N), dtype=torch.complex128, device=f"cuda:{dev}")  # [t][bin(m)]
    plan = get_plan(L, dev)
    _lib.check(_lib.load().mwsht_shard_inverse_front(plan.handle, f.data_ptr(), 0, L, int(spin), None,
                                                      rows.data_ptr(), _stream(dev)),
               "synthesize_reduced")
    k = torch.arange(N, device=rows.device)
    residue = torch.where(k < L, k, k - N) % L          # order m of bin k, folded mod L
    bins = torch.zeros((L, L), dtype=torch.complex128, device=rows.device)
    bins.index_add_(1, residue, rows)
    samples = torch.fft.ifft(bins, dim=1) * L
    return _back(samples, coeffs.values)


def integrate(samples, weights):
    """sum_t q_t sum_p f[t, p] on the reduced L x L grid: the exact integral
    over the sphere for f band-limited at the weights' band limit."""
    L = weights.band_limit
    dev = weights.q.device.index
    f = _to_device(samples, torch.complex128, dev)
    if tuple(f.shape) != (L, L):
        raise ContractViolationError(
            f"samples must have shape ({L}, {L}) for band limit {L}, got {tuple(f.shape)}")
    return complex((f.sum(dim=1) * weights.q).sum().item())
