"""Host-side semantics of the drop-in API that run without a GPU: container
validation, validation order and exception types (mw.py:46-126, 419-566)."""

import numpy as np
import pytest

import paper_1110_6298_b200 as mw


def test_container_validation():
    # test_mw.py:283-310
    with pytest.raises(mw.ContractViolationError):
        mw.HarmonicCoeffs(3, 0, np.zeros(8, dtype=np.complex128))
    with pytest.raises(mw.ContractViolationError):
        mw.MwSignal(3, 0, np.zeros((3, 6), dtype=np.complex128))
    values = np.ones(9, dtype=np.complex128)
    with pytest.raises(mw.ContractViolationError):
        mw.HarmonicCoeffs(3, 2, values)
    coeffs = mw.HarmonicCoeffs(3, 0, values)
    with pytest.raises(ValueError):
        coeffs.values[0] = 0.0
    with pytest.raises(mw.ContractViolationError):
        coeffs.value(3, 0)
    assert coeffs.value(2, -2) == coeffs.values[4]
    with pytest.raises(mw.InvalidBandLimitError):
        mw.HarmonicCoeffs(0, 0, np.zeros(0, dtype=np.complex128))


def test_errors_raised_before_any_device_work():
    # spin and recursion checks happen on the host, in the reference's order
    with pytest.raises(mw.InvalidSpinError):
        mw.inverse(mw.HarmonicCoeffs(4, 4, np.zeros(16, complex)))
    with pytest.raises(mw.InvalidSpinError):
        mw.forward(mw.MwSignal(4, -4, np.zeros((4, 7), complex)))
    with pytest.raises(ValueError):
        mw.forward(mw.MwSignal(3, 0, np.zeros((3, 5), complex)), recursion="fourier")
    with pytest.raises(mw.InvalidSpinError):
        mw.forward_real(mw.MwSignal(6, 1, np.zeros((6, 11))))
    with pytest.raises(mw.InvalidSpinError):
        mw.inverse_real(mw.HarmonicCoeffs(6, 1, np.zeros(36, complex)))
    with pytest.raises(mw.ContractViolationError):
        mw.forward_real(mw.MwSignal(5, 0, np.zeros((5, 9)) + 1e-3j))
    # spin error wins over recursion error (mw.py:371 before :311)
    with pytest.raises(mw.InvalidSpinError):
        mw.forward(mw.MwSignal(3, 5, np.zeros((3, 5), complex)), recursion="bad")
    # lead zeros are checked by the inverse itself too (mw.py:429-434)
    good = mw.HarmonicCoeffs(3, 1, np.zeros(9, complex))
    object.__setattr__(good, "values", np.ones(9, complex))
    with pytest.raises(mw.ContractViolationError):
        mw.inverse(good)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(mw.DeviceError):
        mw.inverse(mw.HarmonicCoeffs(4, 0, np.zeros(16, complex)))


def test_grid_matches_reference_formula():
    L = 7
    t = mw.mw_grid_thetas(L)
    assert t[-1] == pytest.approx(np.pi)
    assert np.allclose(t, np.pi * (2 * np.arange(L) + 1) / (2 * L - 1))
    assert np.allclose(mw.mw_grid_phis(L), 2 * np.pi * np.arange(2 * L - 1) / (2 * L - 1))
