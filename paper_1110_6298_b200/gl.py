"""Gauss-Legendre sampling comparator on the GPU.

Mirrors the reference's pkg/src/torusht/gl.py: ``gl_nodes`` (Legendre roots
and weights by Newton refinement, :60-95), ``gl_forward`` (:114-148) and
``gl_inverse`` (:151-178), with the same arguments, stability gate
(``STABLE_BAND_LIMIT`` = 1024 unless ``allow_unstable``, :30, :98-104) and
exception types.  The O(L^3) colatitude stages (the reference's numba
gl_flm_core / gl_fm_core, kernels/_numba.py:211-268) run in libmwsht.so
(csrc/gl.cu); the azimuthal FFT of each ring (numpy in the reference) runs
through torch on the same device.  Node computation stays on the host, like
the reference's.
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ContractViolationError, ConvergenceError, UnsupportedDegreeError
from .mw import (HarmonicCoeffs, _back, _check_spin, _stream, _target_device, _to_device,
                 _trusted, check_band_limit)

STABLE_BAND_LIMIT = 1024

_NEWTON_CAP = 100
_NEWTON_TOL = 1e-15
_STALL_STEP = 2.5e-16


@dataclass(frozen=True)
class GlGrid:
    """Nodes x_i = cos(theta_i) (strictly decreasing), weights, azimuths (gl.py:33-46)."""

    band_limit: int
    nodes: np.ndarray
    weights: np.ndarray
    phis: np.ndarray

    def __post_init__(self):
        self.nodes.flags.writeable = False
        self.weights.flags.writeable = False
        self.phis.flags.writeable = False


def _legendre_and_deriv(L, x):
    """P_L and P'_L at x by the degree recurrence (gl.py:49-57)."""
    p0 = np.ones_like(x)
    p1 = x.copy()
    for k in range(2, L + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
    if L == 0:
        return p0, np.zeros_like(x)
    if L == 1:
        return x.copy(), np.ones_like(x)
    return p1, L * (x * p1 - p0) / (x * x - 1.0)


def gl_nodes(band_limit):
    """Legendre roots and Gauss-Legendre weights (gl.py:60-95): Newton from the
    Chebyshev-angle guess until |P_L| <= 1e-15 or the step is below one ulp of
    the node scale; more than 100 iterations raise ConvergenceError."""
    check_band_limit(band_limit)
    L = int(band_limit)
    i = np.arange(L)
    x = np.cos(math.pi * (i + 0.75) / (L + 0.5))
    for _ in range(_NEWTON_CAP):
        p, dp = _legendre_and_deriv(L, x)
        if np.max(np.abs(p)) <= _NEWTON_TOL:
            break
        step = p / dp
        x = x - step
        if np.max(np.abs(step)) <= _STALL_STEP:
            break
    else:
        raise ConvergenceError(f"Legendre root refinement did not converge within "
                               f"{_NEWTON_CAP} iterations at L={L}")
    p, dp = _legendre_and_deriv(L, x)
    weights = 2.0 / ((1.0 - x * x) * dp * dp)
    phis = 2.0 * math.pi * np.arange(2 * L - 1) / (2 * L - 1)
    return GlGrid(L, x, weights, phis)


def _check_stability(L, allow_unstable):
    if L > STABLE_BAND_LIMIT and not allow_unstable:
        raise UnsupportedDegreeError(
            f"the pointwise degree recursion is unstable beyond L={STABLE_BAND_LIMIT}; pass "
            f"allow_unstable=True to proceed at L={L} anyway")


def _libm():
    """The C math library's lgamma/exp: the reference's numba _seed_d
    (_numba.py:191-208) calls these, not CPython's own math.lgamma."""
    import ctypes
    import ctypes.util
    lib = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
    for name in ("lgamma", "exp"):
        getattr(lib, name).restype = ctypes.c_double
        getattr(lib, name).argtypes = [ctypes.c_double]
    return lib


_LIBM = _libm()


def seed_tables(L, spin):
    """Per order row mi the seed of d^l_{m,n} at l0 = max(|m|, |n|), n = -spin:
    (const, ec, es, l0) exactly as the reference's _seed_d (_numba.py:191-208),
    with the C library's lgamma/exp as the reference's numba code calls them
    (so the GPU starts every chain from the reference's own constant)."""
    n = -spin
    N = 2 * L - 1
    cst = np.zeros(N)
    ints = np.zeros((N, 4), dtype=np.int32)
    for mi in range(N):
        m = mi - (L - 1)
        if n >= abs(m):
            mm, nn, sign = m, n, 1.0
        elif n <= -abs(m):
            mm, nn, sign = -m, -n, (-1.0 if (m - n) % 2 else 1.0)
        elif m >= abs(n):
            mm, nn, sign = n, m, (-1.0 if (m - n) % 2 else 1.0)
        else:
            mm, nn, sign = -n, -m, 1.0
        cst[mi] = sign * _LIBM.exp(0.5 * (_LIBM.lgamma(2 * nn + 1.0) - _LIBM.lgamma(nn + mm + 1.0)
                                          - _LIBM.lgamma(nn - mm + 1.0)))
        ints[mi] = (nn + mm, nn - mm, nn, 0)
    return cst, ints


class _GlDevice:
    """Node arrays and seeds of one (grid, spin) on one device."""

    def __init__(self, grid, spin, dev):
        L = grid.band_limit
        d = f"cuda:{dev}"
        nodes = np.array(grid.nodes)  # writable copy for torch
        self.x = torch.from_numpy(np.ascontiguousarray(nodes)).to(d)
        self.ch = torch.from_numpy(np.sqrt((1.0 + nodes) / 2.0)).to(d)   # gl.py:107-111
        self.sh = torch.from_numpy(np.sqrt((1.0 - nodes) / 2.0)).to(d)
        self.w = torch.from_numpy(np.array(grid.weights)).to(d)
        cst, ints = seed_tables(L, spin)
        self.cst = torch.from_numpy(cst).to(d)
        self.ints = torch.from_numpy(ints).to(d)


def _core(name, inp, dg, L, spin, out, dev):
    _lib.call(name, inp.data_ptr(), dg.x.data_ptr(), dg.ch.data_ptr(), dg.sh.data_ptr(),
              dg.cst.data_ptr(), dg.ints.data_ptr(), int(L), int(spin), out.data_ptr(),
              _stream(dev))


def _cl(L, dev):
    return torch.sqrt((2.0 * torch.arange(L, dtype=torch.float64, device=dev) + 1.0)
                      / (4.0 * math.pi))


def _layout(L, dev):
    """(row l, column L-1+m) of every flat index l(l+1)+m (mw.py:341-362)."""
    idx = torch.arange(L * L, device=dev)
    ell = torch.floor(torch.sqrt(idx.to(torch.float64))).to(torch.int64)
    ell = torch.where(ell * ell > idx, ell - 1, ell)
    ell = torch.where((ell + 1) * (ell + 1) <= idx, ell + 1, ell)
    m = idx - ell * (ell + 1)
    return ell, L - 1 + m


def gl_forward(samples, spin, grid=None, allow_unstable=False):
    """Harmonic coefficients from samples on the Gauss-Legendre grid (gl.py:114-148):
    per ring the phi FFT G_m(theta_i) (2 pi/N scaled, fftshift), then
    f_lm = (-1)^s c_l sum_i lambda_i d^l_{m,-s}(theta_i) G_m(theta_i) on the GPU."""
    shape = tuple(samples.shape)
    if len(shape) != 2 or shape[1] != 2 * shape[0] - 1:
        raise ContractViolationError(f"samples must have shape (L, 2L-1), got {shape}")
    L = shape[0]
    _check_spin(L, spin)
    _check_stability(L, allow_unstable)
    if grid is None:
        grid = gl_nodes(L)
    elif grid.band_limit != L:
        raise ContractViolationError(
            f"grid band limit {grid.band_limit} does not match samples at L={L}")
    dev = _target_device(samples)
    dg = _GlDevice(grid, spin, dev)
    f = _to_device(samples, torch.complex128, dev)
    gm = torch.fft.fftshift(torch.fft.fft(f, dim=1), dim=1) * (2.0 * math.pi / (2 * L - 1))
    a = (gm.T * dg.w[None, :]).contiguous()                       # (N, L): [mi, node]
    R = torch.empty((L, 2 * L - 1), dtype=torch.complex128, device=f"cuda:{dev}")
    _core("mwsht_gl_flm_core", a, dg, L, spin, R, dev)
    out2d = R * _cl(L, R.device)[:, None]
    if spin % 2:
        out2d = -out2d
    rows, cols = _layout(L, R.device)
    return _trusted(HarmonicCoeffs, L, spin, _back(out2d[rows, cols].contiguous(), samples))


def gl_inverse(coeffs, spin=None, grid=None, allow_unstable=False):
    """Samples on the Gauss-Legendre grid (gl.py:151-178): per order the degree
    sum F_m(theta_i) on the GPU, then an inverse FFT per ring.  Returns a plain
    array (numpy for numpy input), like the reference."""
    if spin is None:
        spin = coeffs.spin
    elif spin != coeffs.spin:
        raise ContractViolationError(f"requested spin {spin} does not match the coefficients' "
                                     f"spin {coeffs.spin}")
    L = coeffs.band_limit
    _check_spin(L, spin)
    _check_stability(L, allow_unstable)
    if grid is None:
        grid = gl_nodes(L)
    elif grid.band_limit != L:
        raise ContractViolationError(
            f"grid band limit {grid.band_limit} does not match coefficients at L={L}")
    dev = _target_device(coeffs.values)
    dg = _GlDevice(grid, spin, dev)
    v = _to_device(coeffs.values, torch.complex128, dev)
    flm2d = torch.zeros((L, 2 * L - 1), dtype=torch.complex128, device=v.device)
    rows, cols = _layout(L, v.device)
    flm2d[rows, cols] = v
    flm2d *= _cl(L, v.device)[:, None]
    if spin % 2:
        flm2d = -flm2d
    F = torch.empty((2 * L - 1, L), dtype=torch.complex128, device=v.device)
    _core("mwsht_gl_fm_core", flm2d.contiguous(), dg, L, spin, F, dev)
    out = torch.fft.ifft(torch.fft.ifftshift(F.T, dim=1), dim=1) * (2 * L - 1)
    return _back(out.contiguous(), coeffs.values)
