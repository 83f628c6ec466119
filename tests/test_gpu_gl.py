"""Gauss-Legendre comparator on the GPU against the
reference's own outputs (tests/golden/gl.npz, made by make_gl_golden.py) and
the oracle's bit-identical restatement, plus the reference's GL test
semantics (test_gl.py: round trips, shared grids, gates, validation).

Tolerance: the kernels take 1/den_l from a per-degree table and fuse
multiply-adds where the reference divides per node, so they agree with the
reference to rounding: rel <= 1e-12 through L = 128 (the reference's own GL
round trips are only asserted to 1e-10, test_acceptance.py:235-243)."""

import os

import numpy as np
import pytest

from helpers import max_abs, random_signal, rel

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def mw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1110_6298_b200 as m
    return m


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(ROOT, "tests", "golden", "gl.npz"))


@pytest.mark.parametrize("L,spin", [(1, 0), (2, 0), (2, 1), (8, 0), (8, -3), (33, 2), (64, -1),
                                    (128, 0)])
def test_gl_matches_reference(mw, golden, L, spin):
    from oracle import mw_oracle as O
    k = f"L{L}_s{spin}"
    v = O.gaussian_coeffs(L, spin, 100 + L)
    sig = mw.gl_inverse(mw.HarmonicCoeffs(L, spin, v))
    assert isinstance(sig, np.ndarray) and sig.shape == (L, 2 * L - 1)
    assert rel(sig, golden[k + "_inverse"]) < 1e-12
    fwd = mw.gl_forward(random_signal(L, spin, 200 + L), spin).values
    assert rel(fwd, golden[k + "_forward"]) < 1e-12


@pytest.mark.parametrize("L,spin", [(200, 3), (301, 0)])
def test_gl_matches_oracle_larger(mw, L, spin):
    from oracle import mw_oracle as O
    g = mw.gl_nodes(L)
    v = O.gaussian_coeffs(L, spin, 5)
    sig = mw.gl_inverse(mw.HarmonicCoeffs(L, spin, v), grid=g)
    assert rel(sig, O.gl_inverse(v, L, spin, np.asarray(g.nodes))) < 1e-12
    raw = random_signal(L, spin, 6)
    fwd = mw.gl_forward(raw, spin, grid=g).values
    assert rel(fwd, O.gl_forward(raw, L, spin, np.asarray(g.nodes), np.asarray(g.weights))) < 1e-12


@pytest.mark.parametrize("L,spin", [(2, 0), (16, 1), (32, 2), (128, 0), (1024, 2)])
def test_gl_round_trip(mw, L, spin):
    from oracle import mw_oracle as O
    v = O.gaussian_coeffs(L, spin, L + spin)
    out = mw.gl_forward(mw.gl_inverse(mw.HarmonicCoeffs(L, spin, v)), spin).values
    # test_gl.py:52-60 (1e-11 to L=32), test_acceptance.py:235-243 (1e-10 to
    # L=128); at the stability gate L=1024 the reference's own round trip of
    # this input is 1.579e-10 (measured here), ours agrees to 4 digits
    bound = 1e-11 if L <= 32 else (1e-10 if L <= 128 else 2e-10)
    assert max_abs(out, v) < bound


def test_gl_cross_sampling_and_semantics(mw):
    from oracle import mw_oracle as O
    L = 16
    for spin in (0, 2):
        c = mw.HarmonicCoeffs(L, spin, O.gaussian_coeffs(L, spin, spin))
        via_mw = mw.forward(mw.inverse(c)).values
        via_gl = mw.gl_forward(mw.gl_inverse(c), spin).values
        assert max_abs(via_mw, via_gl) < 1e-11            # test_gl.py:77-86
    c = mw.HarmonicCoeffs(12, 2, O.gaussian_coeffs(12, 2, 0))
    grid = mw.gl_nodes(12)
    a = mw.gl_inverse(c, grid=grid)
    assert max_abs(a, mw.gl_inverse(c)) == 0.0            # shared grid: identical
    with pytest.raises(mw.ContractViolationError):
        mw.gl_inverse(c, spin=0)
    with pytest.raises(mw.ContractViolationError):
        mw.gl_inverse(c, grid=mw.gl_nodes(5))
    with pytest.raises(mw.ContractViolationError):
        mw.gl_forward(np.zeros((4, 8)), 0)
    big = mw.STABLE_BAND_LIMIT + 1
    with pytest.raises(mw.UnsupportedDegreeError):
        mw.gl_inverse(mw.HarmonicCoeffs(big, 0, np.zeros(big * big, complex)))
    with pytest.raises(mw.UnsupportedDegreeError):
        mw.gl_forward(np.zeros((big, 2 * big - 1)), 0)
