"""Kernel-level mirrors of torusht.kernels (kernels/__init__.py:67-80).

Same names, arguments and array layouts as the reference dispatchers, for
stage-by-stage parity (the reference's test_kernels.py:52-92 shape):

    fmm_core(flm2d (L,2L-1), cl (L,), L, spin, use_trapani) -> T (L, 2L-1)
    flm_core(gfold (2L-1,L), L, spin, use_trapani)          -> R (L, 2L-1)
    fmm_core_real(flm_half (L,L), cl, L, use_trapani)       -> T (L, L)
    flm_core_real(gfold (L,L), L, use_trapani)              -> R (L, L)

Each call runs the sm_100a core kernel (core_inverse.cu / core_forward.cu)
via the C ABI; numpy in -> numpy out, torch CUDA tensors stay on device.
``use_trapani`` is accepted and ignored: both recursions map onto the same
stable GPU recursion (see mw.py).  There is no backend switch and no CPU path.
"""

import torch

from . import _lib
from .mw import _back, _stream, _target_device, _to_device, get_plan

BACKEND = "cuda-sm100a"


def fmm_core(flm2d, cl, L, spin, use_trapani):
    dev = _target_device(flm2d)
    f = _to_device(flm2d, torch.complex128, dev)
    c = _to_device(cl, torch.float64, dev)
    out = torch.empty((L, 2 * L - 1), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_fmm_core", plan.handle, f.data_ptr(), c.data_ptr(), int(spin),
              int(bool(use_trapani)), out.data_ptr(), _stream(dev))
    return _back(out, flm2d)


def flm_core(gfold, L, spin, use_trapani):
    dev = _target_device(gfold)
    g = _to_device(gfold, torch.complex128, dev)
    out = torch.empty((L, 2 * L - 1), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_flm_core", plan.handle, g.data_ptr(), int(spin), int(bool(use_trapani)),
              out.data_ptr(), _stream(dev))
    return _back(out, gfold)


def fmm_core_real(flm_half, cl, L, use_trapani):
    dev = _target_device(flm_half)
    f = _to_device(flm_half, torch.complex128, dev)
    c = _to_device(cl, torch.float64, dev)
    out = torch.empty((L, L), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_fmm_core_real", plan.handle, f.data_ptr(), c.data_ptr(),
              int(bool(use_trapani)), out.data_ptr(), _stream(dev))
    return _back(out, flm_half)


def flm_core_real(gfold, L, use_trapani):
    dev = _target_device(gfold)
    g = _to_device(gfold, torch.complex128, dev)
    out = torch.empty((L, L), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_flm_core_real", plan.handle, g.data_ptr(), int(bool(use_trapani)),
              out.data_ptr(), _stream(dev))
    return _back(out, gfold)


def forward_stages(samples, L, spin):
    """phi FFT .. m' fold (mw.py:149-285): samples (L, 2L-1) -> gfold (2L-1, L)."""
    dev = _target_device(samples)
    x = _to_device(samples, torch.complex128, dev)
    out = torch.empty((2 * L - 1, L), dtype=torch.complex128, device=f"cuda:{dev}")
    plan = get_plan(L, dev)
    _lib.call("mwsht_forward_stages_z", plan.handle, x.data_ptr(), out.data_ptr(), int(spin),
              _stream(dev))
    return _back(out, samples)
