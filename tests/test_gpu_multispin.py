"""Multi-spin batches sharing one Wigner recursion (the
paper's footnote PAPER.md:505): every map of a batch, whatever its spin, is
checked against the oracle (the reference's algorithm) for that spin, at the
north_star tolerance rel <= 1e-12."""

import numpy as np
import pytest

from helpers import max_abs, random_signal, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1110_6298_b200 as m
    return m


@pytest.fixture(scope="module")
def O():
    from oracle import mw_oracle
    return mw_oracle


@pytest.mark.parametrize("L,spins", [(96, [0, 2, -1, 3, 0, -2, 1]), (300, [2, -2]),
                                     (257, [0, 1, 5])])
def test_multi_spin_matches_oracle_per_spin(mw, O, L, spins):
    vals = np.stack([O.gaussian_coeffs(L, s, 30 + k) for k, s in enumerate(spins)])
    sig = mw.inverse_multi_spin(vals, L, spins)
    raw = np.stack([random_signal(L, s, 70 + k) for k, s in enumerate(spins)])
    fwd = mw.forward_multi_spin(raw, L, spins)
    back = mw.forward_multi_spin(sig, L, spins)
    for b, s in enumerate(spins):
        ref = O.inverse(vals[b], L, s, threads=8)
        assert rel(sig[b], ref) < 1e-12, (b, s)
        assert rel(fwd[b], O.forward(raw[b], L, s, threads=8)) < 1e-12, (b, s)
        assert max_abs(back[b], vals[b]) < 1e-12, (b, s)
        # and the single-spin transform of the same map
        one = mw.inverse(mw.HarmonicCoeffs(L, s, vals[b].copy())).samples
        assert rel(sig[b], one) < 1e-13, (b, s)


def test_multi_spin_more_maps_than_one_call(mw, O):
    L = 40
    spins = [k % 5 - 2 for k in range(19)]   # 19 maps: two native calls of <= 16
    vals = np.stack([O.gaussian_coeffs(L, s, k) for k, s in enumerate(spins)])
    sig = mw.inverse_multi_spin(vals, L, spins)
    back = mw.forward_multi_spin(sig, L, spins)
    for b, s in enumerate(spins):
        assert rel(sig[b], O.inverse(vals[b], L, s)) < 1e-12
        assert max_abs(back[b], vals[b]) < 1e-12


def test_multi_spin_validation(mw, O):
    L = 8
    v = np.stack([O.gaussian_coeffs(L, 0, 1), O.gaussian_coeffs(L, 0, 2)])
    with pytest.raises(mw.ContractViolationError):       # l < |s| entries must be zero
        mw.inverse_multi_spin(v, L, [0, 3])
    with pytest.raises(mw.InvalidSpinError):
        mw.inverse_multi_spin(v, L, [0, 8])
    with pytest.raises(mw.ContractViolationError):
        mw.forward_multi_spin(np.zeros((2, L, 2 * L - 1), complex), L, [0])
