"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/mwsht.h declares; the host binding maps status codes to the
reference's exception types.  No GPU compute here."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "mwsht.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(mwsht_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_drop_in_entry_points():
    syms = declared_symbols()
    for name in ("mwsht_forward_z", "mwsht_inverse_z", "mwsht_forward_real_d",
                 "mwsht_inverse_real_d", "mwsht_fmm_core", "mwsht_flm_core",
                 "mwsht_fmm_core_real", "mwsht_flm_core_real", "mwsht_plan_create"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    from paper_1110_6298_b200 import _lib
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) <= set(_lib.EXPORTED)


def test_status_strings_and_version():
    from paper_1110_6298_b200 import _lib
    lib = _lib.load()
    assert b"sm_100a" in lib.mwsht_version()
    assert lib.mwsht_status_string(2) == b"invalid spin"
    assert lib.mwsht_status_string(0) == b"ok"


def test_status_codes_map_to_reference_exceptions():
    import paper_1110_6298_b200 as mw
    from paper_1110_6298_b200 import _lib
    for rc, exc in [(1, mw.InvalidBandLimitError), (2, mw.InvalidSpinError),
                    (3, mw.ContractViolationError), (4, mw.SymmetryError), (5, ValueError),
                    (6, mw.DeviceError)]:
        with pytest.raises(exc):
            _lib.check(rc, "probe")


def test_plan_create_rejects_bad_band_limit_without_device():
    import ctypes
    from paper_1110_6298_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    assert lib.mwsht_plan_create(0, 0, 1, ctypes.byref(h)) == 1
    assert not h.value


def test_missing_library_fails_loudly(tmp_path):
    from paper_1110_6298_b200 import _lib
    with pytest.raises(_lib.DeviceError):
        saved = _lib._lib
        _lib._lib = None
        try:
            _lib.load(str(tmp_path / "nope.so"))
        finally:
            _lib._lib = saved
