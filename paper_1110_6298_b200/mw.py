"""MW spin spherical-harmonic transforms on B200 — the drop-in entry points.

Mirrors the reference's public path (pkg/src/torusht/mw.py): the containers
``HarmonicCoeffs`` (:46-80) and ``MwSignal`` (:83-99) and the transforms
``forward`` (:365), ``inverse`` (:419), ``forward_real`` (:469) and
``inverse_real`` (:524), with the same arguments, flat coefficient layout
l(l+1)+m, MW grid (L rings x 2L-1 azimuths), validation order and exception
types.  All arithmetic runs in libmwsht.so (hand-written sm_100a kernels,
including the FFT stages; no cuFFT/cuBLAS) through the C ABI in
include/mwsht.h; there is no CPU fallback.

Band limits: every L >= 1 up to L = 8192 (the FFT engine's documented cap:
half-split convolutions up to L = 4096, quarter-split above); larger L raises
UnsupportedDegreeError (errors.py:24-25) when the plan is built.  Calls are reentrant: plans are shared per (L, device), and the
library orders calls from different threads/streams on the device so they
never share scratch in flight (include/mwsht.h).

Arrays may be numpy arrays (drop-in: results come back as numpy, host<->device
copies included) or torch tensors (results stay on the tensor's CUDA device;
calls are asynchronous on the current torch stream except where a check
needs a value on the host, as noted per function).

``recursion`` accepts "trapani" and "risbo" like the reference
(mw.py:43,562-566) and raises ValueError otherwise.  Both names run the same
stable GPU recursions: outputs agree with the reference's
Trapani path to round-off for L <= 1024 and with its Risbo path beyond, and
neither reproduces the reference Trapani's silent blow-up above l ~ 1040.
"""

import math
import threading
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import (ContractViolationError, InvalidBandLimitError, InvalidSpinError,
                     SymmetryError)

_RECURSIONS = ("trapani", "risbo")
_REC_ID = {"trapani": _lib.TRAPANI, "risbo": _lib.RISBO}


def check_band_limit(band_limit):
    """Reject band-limits below 1 (grid.py:37-42)."""
    if not isinstance(band_limit, (int, np.integer)) or isinstance(band_limit, bool) \
            or band_limit < 1:
        raise InvalidBandLimitError(f"band limit must be an integer >= 1, got {band_limit!r}")


def _shape(x):
    return tuple(x.shape)


def _lead_nonzero(values, lead):
    if lead <= 0:
        return False
    head = values[:lead]
    if isinstance(head, torch.Tensor):
        return bool((head != 0).any().item())
    return bool(np.any(head != 0))


def _freeze(x):
    if isinstance(x, np.ndarray):
        x.flags.writeable = False


@dataclass(frozen=True)
class HarmonicCoeffs:
    """Coefficients f_lm as a flat complex array of length L^2 (mw.py:46-80).

    Flat index l(l+1)+m for 0 <= l < L, |m| <= l; entries with l < |spin| must
    be exactly zero.  ``values`` is a numpy array or a torch tensor.
    """

    band_limit: int
    spin: int
    values: object

    def __post_init__(self):
        check_band_limit(self.band_limit)
        L = self.band_limit
        if _shape(self.values) != (L * L,):
            raise ContractViolationError(
                f"coefficients for L={L} must have shape ({L * L},), got {_shape(self.values)}")
        lead = min(self.spin * self.spin, L * L)
        if _lead_nonzero(self.values, lead):
            raise ContractViolationError(
                f"coefficients with degree below |spin|={abs(self.spin)} must be exactly zero")
        _freeze(self.values)

    def value(self, ell, m):
        """Coefficient at (ell, m)."""
        if not (0 <= ell < self.band_limit and abs(m) <= ell):
            raise ContractViolationError(
                f"(ell, m) = ({ell}, {m}) out of range for L={self.band_limit}")
        return self.values[ell * (ell + 1) + m]


@dataclass(frozen=True)
class MwSignal:
    """Samples on the L x (2L-1) MW grid, theta rows by phi columns (mw.py:83-99)."""

    band_limit: int
    spin: int
    samples: object

    def __post_init__(self):
        check_band_limit(self.band_limit)
        L = self.band_limit
        if _shape(self.samples) != (L, 2 * L - 1):
            raise ContractViolationError(
                f"signal for L={L} must have shape ({L}, {2 * L - 1}), got {_shape(self.samples)}")
        _freeze(self.samples)


def _trusted(cls, band_limit, spin, data, lead_checked=False):
    """Build a container from our own (already valid) output without re-validating
    (avoids a device sync on torch outputs).  lead_checked: the l < |spin| zeros
    were verified by the caller (e.g. on the host copy), inverse() skips them."""
    obj = object.__new__(cls)
    if lead_checked:
        object.__setattr__(obj, "_lead_checked", True)
    object.__setattr__(obj, "band_limit", band_limit)
    object.__setattr__(obj, "spin", spin)
    object.__setattr__(obj, "values" if cls is HarmonicCoeffs else "samples", data)
    _freeze(data)
    return obj


def mw_grid_thetas(L):
    """theta_t = pi (2t+1)/(2L-1), t = 0..L-1 (grid.py:45-53)."""
    return math.pi * (2 * np.arange(L) + 1) / (2 * L - 1)


def mw_grid_phis(L):
    """phi_p = 2 pi p/(2L-1) (grid.py:45-53)."""
    return 2.0 * math.pi * np.arange(2 * L - 1) / (2 * L - 1)


# ------------------------------------------------------------------ plans

class Plan:
    """Owns one native plan (FFT tables, recursion tables, scratch) for (L, device, batch)."""

    def __init__(self, L, device, max_batch=1):
        lib = _lib.load()
        handle = _lib._P()
        with torch.cuda.device(device):
            _lib.check(lib.mwsht_plan_create(int(L), int(device), int(max_batch),
                                             _lib.ctypes.byref(handle)), "plan_create")
        self.handle = handle
        self.L = L
        self.device = device
        self.max_batch = max_batch

    def device_bytes(self):
        return int(_lib.load().mwsht_plan_device_bytes(self.handle))

    def last_launches(self):
        """Kernel launches of the most recent call on this plan (all our own)."""
        own = _lib.ctypes.c_int()
        _lib.load().mwsht_plan_last_launches(self.handle, _lib.ctypes.byref(own))
        return own.value

    def set_paired(self, mode):
        """Inverse-core tiling for spin 0: -1 (default) paired tiles for single
        maps (one recursion feeds T[m',m] and its transpose; batches share the
        recursion between maps instead), 1 paired always, 0 plain tiles."""
        _lib.call("mwsht_plan_set_paired", self.handle, int(mode))

    def prepare_spin(self, spin):
        _lib.call("mwsht_plan_prepare_spin", self.handle, int(spin))

    def close(self):
        if self.handle:
            _lib.load().mwsht_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


_PLANS = {}
_PLANS_LOCK = threading.Lock()


def get_plan(L, device=None, max_batch=1):
    """Cached plan for band-limit L on a CUDA device (cf. _CONV_CACHE, mw.py:225).

    One plan per (L, device): batch capacity is rounded up to a power of two,
    and a request beyond the cached capacity replaces the cached plan (the old
    one is freed once no caller holds it), so growing batches never keep
    several plans' scratch alive."""
    if device is None:
        device = torch.cuda.current_device()
    device = int(device)
    cap = 1
    while cap < max_batch:
        cap *= 2
    with _PLANS_LOCK:
        p = _PLANS.get((L, device))
        if p is None or p.max_batch < cap:
            if p is not None:
                del _PLANS[(L, device)]
                p = None  # freed when the last in-flight caller drops it
            p = Plan(L, device, cap)
            _PLANS[(L, device)] = p
        return p


def clear_plans():
    with _PLANS_LOCK:
        for p in _PLANS.values():
            p.close()
        _PLANS.clear()


# ------------------------------------------------------------ array moves

def _target_device(x):
    if isinstance(x, torch.Tensor) and x.is_cuda:
        return x.device.index
    if not torch.cuda.is_available():
        from .errors import DeviceError
        raise DeviceError("no CUDA device available: the MW transforms run on the GPU only")
    return torch.cuda.current_device()


def _to_device(x, dtype, device):
    """Contiguous CUDA tensor of `dtype` holding x (numpy or torch)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=f"cuda:{device}", dtype=dtype).contiguous()
    arr = np.ascontiguousarray(x)
    with warnings.catch_warnings():  # read-only input: the tensor is only copied to the device
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.to(f"cuda:{device}", non_blocking=False)


def _back(out, like):
    """Return `out` in the caller's array type: numpy in -> numpy out."""
    if isinstance(like, torch.Tensor):
        return out
    return out.cpu().numpy()


def _stream(device):
    return _lib._P(torch.cuda.current_stream(device).cuda_stream)


def _check_spin(band_limit, spin):
    if abs(spin) >= band_limit:
        raise InvalidSpinError(
            f"|spin| must be below the band limit, got spin={spin} at L={band_limit}")


def _check_recursion(recursion):
    if recursion not in _RECURSIONS:
        raise ValueError(f"recursion must be one of {_RECURSIONS}, got {recursion!r}")


# ------------------------------------------------------------- transforms

def forward(signal, recursion="trapani"):
    """Harmonic coefficients of a sampled signal (mw.py:365-375).

    phi FFT -> periodic extension -> theta FFT -> quadrature-weight
    correlation -> m' fold -> fused Delta recursion + contraction, all on the
    GPU.  Like the reference, any dtype is accepted and treated as complex.
    """
    L, s = signal.band_limit, signal.spin
    _check_spin(L, s)
    _check_recursion(recursion)
    dev = _target_device(signal.samples)
    x = _to_device(signal.samples, torch.complex128, dev)
    out = torch.empty(L * L, dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_forward_z", plan.handle, x.data_ptr(), out.data_ptr(), s,
              _REC_ID[recursion], _stream(dev))
    return _trusted(HarmonicCoeffs, L, s, _back(out, signal.samples))


def inverse(coeffs, recursion="trapani"):
    """Sampled signal of the given harmonic coefficients (mw.py:419-438).

    For spin != 0 the l < |s| zero check reads s^2 values on the host (a
    device sync for torch inputs), as the reference's check does.
    """
    L, s = coeffs.band_limit, coeffs.spin
    _check_spin(L, s)
    if not getattr(coeffs, "_lead_checked", False) and _lead_nonzero(coeffs.values, s * s):
        raise ContractViolationError(
            f"coefficients with degree below |spin|={abs(s)} must be zero on input to the "
            "inverse transform")
    _check_recursion(recursion)
    dev = _target_device(coeffs.values)
    f = _to_device(coeffs.values, torch.complex128, dev)
    out = torch.empty((L, 2 * L - 1), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_inverse_z", plan.handle, f.data_ptr(), out.data_ptr(), s,
              _REC_ID[recursion], _stream(dev))
    return _trusted(MwSignal, L, s, _back(out, coeffs.values))


def forward_real(signal, recursion="trapani"):
    """Spin-0 forward transform of a real signal (mw.py:469-501).

    Complex input must have an identically zero imaginary part (checked on
    the host: a device sync for complex torch inputs).
    """
    if signal.spin != 0:
        raise InvalidSpinError(f"the real-signal path supports spin 0 only, got {signal.spin}")
    samples = signal.samples
    is_complex = samples.is_complex() if isinstance(samples, torch.Tensor) \
        else np.iscomplexobj(samples)
    if is_complex:
        imag = samples.imag
        bad = bool((imag != 0).any().item()) if isinstance(imag, torch.Tensor) \
            else bool(np.any(imag != 0))
        if bad:
            raise ContractViolationError("real-path input must have identically zero imaginary part")
        samples = samples.real
    L = signal.band_limit
    _check_recursion(recursion)
    dev = _target_device(samples)
    x = _to_device(samples, torch.float64, dev)
    out = torch.empty(L * L, dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_forward_real_d", plan.handle, x.data_ptr(), out.data_ptr(),
              _REC_ID[recursion], _stream(dev))
    return _trusted(HarmonicCoeffs, L, 0, _back(out, signal.samples))


def reality_residual(coeffs):
    """(worst, tol) of the reality condition checked by inverse_real (mw.py:537-547)."""
    L = coeffs.band_limit
    dev = _target_device(coeffs.values)
    f = _to_device(coeffs.values, torch.complex128, dev)
    plan = get_plan(L, dev)
    worst, tol = _lib.ctypes.c_double(), _lib.ctypes.c_double()
    _lib.call("mwsht_reality_residual", plan.handle, f.data_ptr(), _lib.ctypes.byref(worst),
              _lib.ctypes.byref(tol), _stream(dev))
    return worst.value, tol.value, f


def inverse_real(coeffs, recursion="trapani"):
    """Spin-0 inverse transform onto real samples (mw.py:524-559).

    Raises SymmetryError unless conj(f_lm) = (-1)^m f_l,-m holds to
    1e-12 max(1, max|f|); the check reduces on the GPU and reads two numbers
    back (one device sync).
    """
    if coeffs.spin != 0:
        raise InvalidSpinError(f"the real-signal path supports spin 0 only, got {coeffs.spin}")
    L = coeffs.band_limit
    _check_recursion(recursion)
    worst, tol, f = reality_residual(coeffs)
    if worst > tol:
        raise SymmetryError(
            f"coefficients violate the reality condition by {worst:.3e} (tolerance {tol:.3e})")
    out = _inverse_real_unchecked(f, L, recursion)
    return _trusted(MwSignal, L, 0, _back(out, coeffs.values))


def _inverse_real_unchecked(f, L, recursion):
    """inverse_real's transform on a device tensor whose reality condition the
    caller checks (HostPipeline defers it to synchronize())."""
    dev = f.device.index
    out = torch.empty((L, 2 * L - 1), dtype=torch.float64, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_inverse_real_d", plan.handle, f.data_ptr(), out.data_ptr(),
              _REC_ID[recursion], _stream(dev))
    return out


# ------------------------------------------------------------- batches

def forward_batch(samples, band_limit, spin, recursion="trapani"):
    """forward() of B independent maps, samples (B, L, 2L-1) -> (B, L^2).

    One plan, one launch per stage for the whole batch (cli.py:159-224 loops
    over maps one by one).
    """
    L = band_limit
    check_band_limit(L)
    _check_spin(L, spin)
    _check_recursion(recursion)
    if _shape(samples)[1:] != (L, 2 * L - 1):
        raise ContractViolationError(f"batch samples must be (B, {L}, {2 * L - 1})")
    B = _shape(samples)[0]
    dev = _target_device(samples)
    x = _to_device(samples, torch.complex128, dev)
    out = torch.empty((B, L * L), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev, max_batch=max(1, B))
    _lib.call("mwsht_forward_z_batch", plan.handle, B, x.data_ptr(), out.data_ptr(), spin,
              _REC_ID[recursion], _stream(dev))
    return _back(out, samples)


def inverse_batch(values, band_limit, spin, recursion="trapani"):
    """inverse() of B independent coefficient sets, (B, L^2) -> (B, L, 2L-1)."""
    L = band_limit
    check_band_limit(L)
    _check_spin(L, spin)
    if _shape(values)[1:] != (L * L,):
        raise ContractViolationError(f"batch coefficients must be (B, {L * L})")
    B = _shape(values)[0]
    for b in range(B) if spin else ():
        if _lead_nonzero(values[b], spin * spin):
            raise ContractViolationError(
                f"coefficients with degree below |spin|={abs(spin)} must be zero")
    _check_recursion(recursion)
    dev = _target_device(values)
    f = _to_device(values, torch.complex128, dev)
    out = torch.empty((B, L, 2 * L - 1), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev, max_batch=max(1, B))
    _lib.call("mwsht_inverse_z_batch", plan.handle, B, f.data_ptr(), out.data_ptr(), spin,
              _REC_ID[recursion], _stream(dev))
    return _back(out, values)


# ------------------------------------------------------- multi-spin batches

MAX_MULTI_SPIN = 16  # maps per native call (include/mwsht.h)


def _spins_arg(spins, B, L):
    spins = [int(s) for s in spins]
    if len(spins) != B:
        raise ContractViolationError(f"need one spin per map: {B} maps, {len(spins)} spins")
    for s in spins:
        _check_spin(L, s)
    return spins


def inverse_multi_spin(values, band_limit, spins, recursion="trapani"):
    """inverse() of B coefficient sets of different spins, (B, L^2) -> (B, L, 2L-1).

    The maps share every Wigner chain's recursion, which does not depend on the
    spin; each map contracts with its own
    spin's row weights.  Results equal inverse() of each map with its spin.
    """
    L = band_limit
    check_band_limit(L)
    if _shape(values)[1:] != (L * L,):
        raise ContractViolationError(f"batch coefficients must be (B, {L * L})")
    B = _shape(values)[0]
    spins = _spins_arg(spins, B, L)
    for b, s in enumerate(spins):
        if _lead_nonzero(values[b], s * s):
            raise ContractViolationError(
                f"map {b}: coefficients with degree below |spin|={abs(s)} must be zero")
    _check_recursion(recursion)
    dev = _target_device(values)
    f = _to_device(values, torch.complex128, dev)
    out = torch.empty((B, L, 2 * L - 1), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev, max_batch=min(B, MAX_MULTI_SPIN))
    for b0 in range(0, B, MAX_MULTI_SPIN):
        nb = min(MAX_MULTI_SPIN, B - b0)
        arr = (_lib.ctypes.c_int * nb)(*spins[b0:b0 + nb])
        _lib.call("mwsht_inverse_z_multi", plan.handle, nb, f[b0].data_ptr(), out[b0].data_ptr(),
                  arr, _REC_ID[recursion], _stream(dev))
    return _back(out, values)


def forward_multi_spin(samples, band_limit, spins, recursion="trapani"):
    """forward() of B maps of different spins, (B, L, 2L-1) -> (B, L^2), sharing
    the recursion like inverse_multi_spin."""
    L = band_limit
    check_band_limit(L)
    if _shape(samples)[1:] != (L, 2 * L - 1):
        raise ContractViolationError(f"batch samples must be (B, {L}, {2 * L - 1})")
    B = _shape(samples)[0]
    spins = _spins_arg(spins, B, L)
    _check_recursion(recursion)
    dev = _target_device(samples)
    x = _to_device(samples, torch.complex128, dev)
    out = torch.empty((B, L * L), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev, max_batch=min(B, MAX_MULTI_SPIN))
    for b0 in range(0, B, MAX_MULTI_SPIN):
        nb = min(MAX_MULTI_SPIN, B - b0)
        arr = (_lib.ctypes.c_int * nb)(*spins[b0:b0 + nb])
        _lib.call("mwsht_forward_z_multi", plan.handle, nb, x[b0].data_ptr(), out[b0].data_ptr(),
                  arr, _REC_ID[recursion], _stream(dev))
    return _back(out, samples)
