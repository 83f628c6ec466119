"""Paired inverse-core tiles (core_inverse.cu) against the
plain tiles and the oracle.

Paired tiles run each (m', m) chain with m' > m once and emit both T[m', m]
and the transpose T[m, m'] = (-1)^(m'-m) sum_l z W_l(m) g_l(m').  The
default pairs every spin-0 inverse; these tests compare it with the plain
tiles (mode 0) at sizes the oracle finishes in seconds.  Spin != 0 always runs
the plain kernel (mode 1 falls back to it; checked too).  Tolerance: rel 1e-12 against
the oracle (north_star), and the paired/plain difference stays at rounding.
"""

import numpy as np
import pytest

from helpers import max_abs, rel

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


def _with_mode(mw, L, mode, fn):
    plan = mw.get_plan(L)
    plan.set_paired(mode)
    try:
        return fn()
    finally:
        plan.set_paired(-1)


@pytest.mark.parametrize("L,spin", [(1, 0), (2, 0), (3, 0), (33, 0), (64, 0), (97, 0), (130, 0),
                                    (200, 0), (257, 0), (70, 3), (97, -2)])
def test_paired_fmm_core_matches_oracle(mw, O, L, spin):
    from paper_1110_6298_b200 import kernels
    rng = np.random.default_rng(L * 7 + spin)
    flm2d = rng.standard_normal((L, 2 * L - 1)) + 1j * rng.standard_normal((L, 2 * L - 1))
    cl = O.cl_table(L)
    ref = O.fmm_core(flm2d, cl, L, spin, True, threads=4)
    Tp = _with_mode(mw, L, 1, lambda: kernels.fmm_core(flm2d, cl, L, spin, True))
    Tq = _with_mode(mw, L, 0, lambda: kernels.fmm_core(flm2d, cl, L, spin, True))
    assert rel(Tp, ref) < 1e-12
    assert rel(Tp, Tq) < 1e-13
    if spin == 0:
        half = np.ascontiguousarray(flm2d[:, L - 1:])
        refh = O.fmm_core_real(half, cl, L, True)
        Th = _with_mode(mw, L, 1, lambda: kernels.fmm_core_real(half, cl, L, True))
        assert rel(Th, refh) < 1e-12


@pytest.mark.parametrize("L,spin", [(64, 0), (256, 2), (256, -2), (300, 0)])
def test_paired_inverse_transform_matches_oracle(mw, O, L, spin):
    v = O.gaussian_coeffs(L, spin, 5)
    sig = _with_mode(mw, L, 1,
                     lambda: mw.inverse(mw.HarmonicCoeffs(L, spin, v.copy())).samples)
    ref = O.inverse(v, L, spin, threads=8)
    assert rel(sig, ref) < 1e-12
    back = mw.forward(mw.MwSignal(L, spin, np.array(sig))).values
    assert max_abs(back, v) < 1e-11


def test_paired_real_transform_matches_oracle(mw, O):
    L = 192
    v = O.gaussian_real_coeffs(L, 4)
    sig = _with_mode(mw, L, 1,
                     lambda: mw.inverse_real(mw.HarmonicCoeffs(L, 0, v.copy())).samples)
    assert rel(sig, O.inverse_real(v, L)) < 1e-12


def test_paired_batched(mw, O):
    L, s, B = 96, 1, 3
    vals = np.stack([O.gaussian_coeffs(L, s, k) for k in range(B)])
    plan = mw.get_plan(L, max_batch=B)
    plan.set_paired(1)
    try:
        sig = mw.inverse_batch(vals, L, s)
    finally:
        plan.set_paired(-1)
    for b in range(B):
        assert rel(sig[b], O.inverse(vals[b], L, s, threads=8)) < 1e-12
