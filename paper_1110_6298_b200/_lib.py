"""ctypes binding of libmwsht.so (include/mwsht.h).

The native library is the only compute path: if it cannot be loaded, every
transform raises DeviceError (there is no CPU fallback).
"""

import ctypes
import os

from .errors import (ContractViolationError, DeviceError, InvalidBandLimitError,
                     InvalidSpinError, SymmetryError, UnsupportedDegreeError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmwsht.so")

TRAPANI, RISBO = 0, 1
_lib = None

# status -> exception type (mwsht_status)
_EXC = {
    1: InvalidBandLimitError,
    2: InvalidSpinError,
    3: ContractViolationError,
    4: SymmetryError,
    5: ValueError,
    6: DeviceError,
    7: UnsupportedDegreeError,
    8: MemoryError,
    9: DeviceError,
}

_P = ctypes.c_void_p
_I = ctypes.c_int
_SIGS = {
    "mwsht_version": ([], ctypes.c_char_p),
    "mwsht_status_string": ([_I], ctypes.c_char_p),
    "mwsht_last_error": ([], ctypes.c_char_p),
    "mwsht_plan_create": ([_I, _I, _I, ctypes.POINTER(_P)], _I),
    "mwsht_plan_destroy": ([_P], _I),
    "mwsht_plan_device_bytes": ([_P], ctypes.c_size_t),
    "mwsht_plan_prepare_spin": ([_P, _I], _I),
    "mwsht_forward_z": ([_P, _P, _P, _I, _I, _P], _I),
    "mwsht_inverse_z": ([_P, _P, _P, _I, _I, _P], _I),
    "mwsht_forward_real_d": ([_P, _P, _P, _I, _P], _I),
    "mwsht_inverse_real_d": ([_P, _P, _P, _I, _P], _I),
    "mwsht_reality_residual": ([_P, _P, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double), _P], _I),
    "mwsht_reality_residual_async": ([_P, _P, _P, _P], _I),
    "mwsht_forward_z_batch": ([_P, _I, _P, _P, _I, _I, _P], _I),
    "mwsht_inverse_z_batch": ([_P, _I, _P, _P, _I, _I, _P], _I),
    "mwsht_forward_z_multi": ([_P, _I, _P, _P, ctypes.POINTER(_I), _I, _P], _I),
    "mwsht_inverse_z_multi": ([_P, _I, _P, _P, ctypes.POINTER(_I), _I, _P], _I),
    "mwsht_gl_fm_core": ([_P, _P, _P, _P, _P, _P, _I, _I, _P, _P], _I),
    "mwsht_gl_flm_core": ([_P, _P, _P, _P, _P, _P, _I, _I, _P, _P], _I),
    "mwsht_fmm_core": ([_P, _P, _P, _I, _I, _P, _P], _I),
    "mwsht_flm_core": ([_P, _P, _I, _I, _P, _P], _I),
    "mwsht_fmm_core_real": ([_P, _P, _P, _I, _P, _P], _I),
    "mwsht_flm_core_real": ([_P, _P, _I, _P, _P], _I),
    "mwsht_forward_stages_z": ([_P, _P, _P, _I, _P], _I),
    "mwsht_plan_last_launches": ([_P, ctypes.POINTER(_I)], _I),
    "mwsht_plan_set_timing": ([_P, _I], _I),
    "mwsht_plan_set_paired": ([_P, _I], _I),
    "mwsht_shard_forward_phi": ([_P, _P, _I, _I, _P, _P, _P], _I),
    "mwsht_shard_forward_rest": ([_P, _P, _I, _I, _P, _P, _I, _P, _I, _P], _I),
    "mwsht_shard_inverse_front": ([_P, _P, _I, _I, _I, _P, _P, _P], _I),
    "mwsht_shard_inverse_phi": ([_P, _P, _I, _I, _P, _P, _P, _P], _I),
    "mwsht_shard_unpack_flm": ([_P, _P, ctypes.c_longlong, _P, _I, _P, _P], _I),
    "mwsht_plan_last_timing": ([_P, _I, ctypes.POINTER(ctypes.c_float),
                                ctypes.POINTER(ctypes.c_float)], _I),
    "mwsht_fp64_probe": ([_I, ctypes.POINTER(ctypes.c_double),
                          ctypes.POINTER(ctypes.c_double)], _I),
}

EXPORTED = tuple(_SIGS)


def load(path=None):
    """Load (once) and return the native library; raises DeviceError if absent.

    MWSHT_LIB overrides the in-tree path (used to A/B kernel variants)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("MWSHT_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise DeviceError(
            f"native library {path} is missing: build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    try:
        lib = ctypes.CDLL(path)
    except OSError as exc:  # pragma: no cover - depends on the host
        raise DeviceError(f"cannot load {path}: {exc}") from exc
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc, what=""):
    """Raise the reference's exception type for a nonzero status."""
    if rc == 0:
        return
    lib = load()
    detail = lib.mwsht_last_error().decode(errors="replace")
    exc = _EXC.get(rc, DeviceError)
    raise exc(f"{what}: {lib.mwsht_status_string(rc).decode()} ({detail})")


def call(name, *args):
    check(getattr(load(), name)(*args), name)
