"""Band limits above 4096 (quarter-split FFT engine, up to the cap L = 8192).

The reference accepts every L >= 1 (grid.py:37-42).  Here, beyond L = 4096,
the FFT stages split each convolution into four quarter-convolutions (the
cores are the same code as below 4096).  Checks:
* the forward FFT stages against the oracle (the reference's numpy stages),
  on a subset of order rows (the oracle's full plane would need tens of GB);
* the inverse against closed-form spherical harmonics: unit coefficients at
  (l, 0) give sqrt((2l+1)/4pi) P_l(cos theta), and at (l, m) the normalised
  associated Legendre function times e^{i m phi}, evaluated by the standard
  stable recursions in numpy (convention pinned at L = 1024, where the GPU is
  pinned to the reference);
* round trips inverse -> forward for spin 0 and 2.
"""

import math

import numpy as np
import pytest

from helpers import random_signal, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mw():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1110_6298_b200 as m
    return m


def ylm_column(L, ell, m):
    """Normalised Y_lm(theta_t, 0) on the MW rings, l >= |m| >= 0 (Condon-Shortley
    sign as the reference; validated against the GPU at L = 1024 below).  The
    standard m-then-l recursions run in 80-bit long double: its exponent range
    holds sin^m(theta) near the poles (no underflow) and its precision keeps the
    reference's own rounding below the tolerance."""
    ld = np.longdouble
    theta = np.pi * (2 * np.arange(L, dtype=ld) + 1) / ld(2 * L - 1)
    x, s = np.cos(theta), np.sin(theta)
    am = abs(m)
    logc = ld(0.5) * (np.log(ld(2 * am + 1) / (4 * np.pi * ld(1))) +
                      np.sum(np.log((2 * np.arange(1, am + 1, dtype=ld) - 1) /
                                    (2 * np.arange(1, am + 1, dtype=ld)))))
    pmm = np.exp(logc + am * np.log(s)) * (ld(-1) ** am)
    if ell == am:
        p = pmm
    else:
        p_prev, p = pmm, x * np.sqrt(ld(2 * am + 3)) * pmm
        for ll in range(am + 2, ell + 1):
            a = np.sqrt(ld(4 * ll * ll - 1) / ld(ll * ll - am * am))
            b = np.sqrt(ld((ll - 1) ** 2 - am * am) / ld(4 * (ll - 1) ** 2 - 1))
            p_prev, p = p, a * (x * p - b * p_prev)
    if m < 0:
        p = p * (-1) ** am
    return p.astype(np.float64)


def _unit(L, ell, m):
    v = np.zeros(L * L, dtype=np.complex128)
    v[ell * (ell + 1) + m] = 1.0
    return v


@pytest.mark.parametrize("ell,m", [(900, 0), (900, 300), (1000, -7)])
def test_closed_form_convention_at_L1024(mw, ell, m):
    L = 1024
    sig = mw.inverse(mw.HarmonicCoeffs(L, 0, _unit(L, ell, m))).samples
    phi = 2 * math.pi * np.arange(2 * L - 1) / (2 * L - 1)
    ref = ylm_column(L, ell, m)[:, None] * np.exp(1j * m * phi)[None, :]
    assert rel(sig, ref) < 1e-11


@pytest.mark.parametrize("L,ell,m", [(4500, 4499, 0), (4500, 3000, 1200), (8192, 8191, 0),
                                     (8192, 6000, -2500)])
def test_inverse_matches_closed_form_above_4096(mw, L, ell, m):
    import torch
    v = torch.from_numpy(_unit(L, ell, m)).cuda()
    sig = mw.inverse(mw.HarmonicCoeffs(L, 0, v)).samples.cpu().numpy()
    phi = 2 * math.pi * np.arange(2 * L - 1) / (2 * L - 1)
    ref = ylm_column(L, ell, m)[:, None] * np.exp(1j * m * phi)[None, :]
    assert rel(sig, ref) < 5e-12  # the Q = 2 path at L = 4096 (pinned to the oracle) gives 1.7e-12


def _gfold_rows(samples, L, spin, ms):
    """Oracle forward stages (mw.py:149-285) restricted to order rows ms."""
    from oracle import mw_oracle as O
    G = O.phi_fft(samples, L)                         # (L, N), column L-1+m
    cols = [L - 1 + m for m in ms]
    g = G[:, cols]
    par = np.array([(-1.0) ** ((m + spin) % 2) for m in ms])
    ext = np.concatenate([g, g[L - 2::-1, :] * par[None, :]], axis=0) if L > 1 else g
    N = 2 * L - 1
    mp = np.arange(-(L - 1), L)
    F = np.fft.fftshift(np.fft.fft(ext, axis=0), axes=0)
    F *= (np.exp(-1j * mp * (math.pi / N)) / (2.0 * math.pi * N))[:, None]
    Gc = O.convolve_rows(F.T.copy(), L)                # (rows, N), columns m'
    fold = np.empty((len(ms), L), dtype=np.complex128)
    fold[:, 0] = Gc[:, L - 1]
    fold[:, 1:] = Gc[:, L:] + par[:, None] * Gc[:, L - 2::-1]
    return fold


@pytest.mark.parametrize("L,spin", [(4097, 0), (5000, 2), (8192, -1)])
def test_forward_stages_above_4096(mw, L, spin):
    from paper_1110_6298_b200 import kernels
    sig = random_signal(L, spin, 17)
    got = kernels.forward_stages(sig, L, spin)        # (N, L), row L-1+m
    rng = np.random.default_rng(L)
    ms = sorted(set(rng.integers(-(L - 1), L, 24).tolist()) | {0, L - 1, -(L - 1)})
    ref = _gfold_rows(sig, L, spin, ms)
    assert rel(got[[L - 1 + m for m in ms]], ref) < 1e-13


@pytest.mark.parametrize("L,spin", [(4500, 0), (4500, 2), (8192, 0)])
def test_round_trip_above_4096(mw, L, spin):
    import torch
    from oracle import mw_oracle as O
    v = torch.from_numpy(O.gaussian_coeffs(L, spin, 3)).cuda()
    sig = mw.inverse(mw.HarmonicCoeffs(L, spin, v)).samples
    back = mw.forward(mw.MwSignal(L, spin, sig)).values
    assert (back - v).abs().max().item() < 2e-11


def test_real_path_above_4096(mw):
    import torch
    from oracle import mw_oracle as O
    L = 5000
    v = torch.from_numpy(O.gaussian_real_coeffs(L, 1)).cuda()
    sig = mw.inverse_real(mw.HarmonicCoeffs(L, 0, v)).samples
    back = mw.forward_real(mw.MwSignal(L, 0, sig)).values
    assert (back - v).abs().max().item() < 2e-11


def test_mcolumn_sharding_above_4096(mw):
    # the m-column shard stages with the quarter-split FFTs (dense-layout
    # emulation of 2 ranks on one GPU) match the unsharded transform
    import torch
    from oracle import mw_oracle as O
    from paper_1110_6298_b200 import shard
    L, spin = 4500, 2
    v = torch.from_numpy(O.gaussian_coeffs(L, spin, 8)).cuda()
    samples, flm = shard.emulate_mcolumn(L, 2, spin, v)
    plan = mw.get_plan(L)
    plan.set_paired(0)
    try:
        ref = mw.inverse(mw.HarmonicCoeffs(L, spin, v)).samples
    finally:
        plan.set_paired(-1)
    assert (samples - ref).abs().max().item() == 0.0
    assert (flm - v).abs().max().item() < 2e-11
