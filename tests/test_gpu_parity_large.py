"""Parity at the sizes the headline runs (round 2).

* Forward of RAW (not band-limited) signals, which exercises the whole
  forward map rather than the round-trip subspace: full arrays against the
  oracle at L = 256 (s = +-2) and L = 1024 (complex and real), and against
  reference-generated golden vectors at L = 1100 (s = 2) and L = 2048 (Risbo,
  produced by torusht.forward itself).
* The forward FFT stages past the oracle's direct-matrix branch (L > 128:
  FFT convolution, reference mw.py:232-251).
* C5 itself (L = 4096, s = 0 and s = 2, the bench's headline config): inverse
  samples and raw-signal forward coefficients against oracle-Risbo golden
  vectors (tests/golden/make_golden_big.py).

Golden comparisons check a 65536-entry subsample entrywise and every row and
column checksum of the whole array (helpers.checksum_dev), so an error
anywhere in the array is caught.  Tolerances: rel <= 1e-12 for L <= 1024
(north_star), 2e-12 beyond (the reference Risbo's own error at L = 2048 is
~1.4e-12), checksums within 4x the per-entry tolerance after
the sqrt(n) scaling.
"""

import os

import numpy as np
import pytest

from helpers import checksum_dev, max_abs, random_signal, rel

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = max(1, min(32, os.cpu_count() or 1))


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


def _big(name):
    return np.load(os.path.join(ROOT, "tests", "golden", f"big_{name}.npz"))


# ------------------------------------------------ forward of raw signals

@pytest.mark.parametrize("L,spin", [(256, 2), (256, -2), (1024, 0), (777, 3)])
def test_forward_raw_signal_full_array(mw, O, L, spin):
    raw = random_signal(L, spin, 900 + L)
    got = mw.forward(mw.MwSignal(L, spin, raw)).values
    ref = O.forward(raw, L, spin, "trapani", threads=THREADS)
    assert rel(got, ref) < 1e-12


@pytest.mark.parametrize("L", [1024, 601, 513])  # 601, 513: odd row counts, padded rows (H = 2048)
def test_forward_real_raw_signal_full_array(mw, O, L):
    raw = random_signal(L, 0, 77).real.copy()
    got = mw.forward_real(mw.MwSignal(L, 0, raw)).values
    ref = O.forward_real(raw, L, "trapani", threads=THREADS)
    assert rel(got, ref) < 1e-12


@pytest.mark.parametrize("L,spin", [(129, 0), (256, -2), (1024, 1), (513, 0), (640, -1), (1025, 2)])
def test_forward_stages_fft_branch(mw, O, L, spin):
    # L > 128: the oracle (like mw.py:232-251) correlates by FFT, not by matrix
    from paper_1110_6298_b200 import kernels
    sig = random_signal(L, spin, 5)
    assert rel(kernels.forward_stages(sig, L, spin), O.gfold_of(sig, L, spin)) < 1e-13


# ------------------------------------------------ golden (reference / oracle Risbo)

def _check_samples(g, samples, L, tol):
    samples = np.asarray(samples)
    mx = float(g["samples_max"])
    sub = samples.reshape(-1)[g["samples_idx"]]
    r = max_abs(sub, g["samples_sub"]) / mx
    assert r < tol, ("samples subsample", r)
    d = checksum_dev(samples, g["samples_rowsum"], g["samples_colsum"], 1000 + L) / mx
    assert d < 4 * tol, ("samples checksums", d)
    return r, d


def _check_fwd(O, g, flm, L, tol):
    flm = np.asarray(flm)
    mx = float(g["fwd_max"])
    r = max_abs(flm[g["fwd_idx"]], g["fwd_sub"]) / mx
    assert r < tol, ("coefficient subsample", r)
    d = checksum_dev(O.from_flat(flm, L), g["fwd_rowsum"], g["fwd_colsum"], 2000 + L) / mx
    assert d < 4 * tol, ("coefficient checksums", d)
    return r, d


def test_golden_L1100_spin2_reference_risbo(mw, O):
    g = _big("L1100_s2_risbo")
    L, spin = 1100, 2
    assert str(g["producer"]) == "reference"
    v = O.gaussian_coeffs(L, spin, int(g["seed"]))
    sig = mw.inverse(mw.HarmonicCoeffs(L, spin, v), recursion="risbo").samples
    _check_samples(g, sig, L, 2e-12)
    raw = random_signal(L, spin, int(g["raw_seed"]))
    _check_fwd(O, g, mw.forward(mw.MwSignal(L, spin, raw), recursion="risbo").values, L, 2e-12)


def test_golden_L2048_raw_forward_reference_risbo(mw, O):
    g = _big("L2048_s0_risbo_raw")
    L = 2048
    assert str(g["producer"]) == "reference"
    raw = random_signal(L, 0, int(g["raw_seed"]))
    _check_fwd(O, g, mw.forward(mw.MwSignal(L, 0, raw), recursion="risbo").values, L, 2e-12)


@pytest.mark.parametrize("spin", [0, 2])
def test_golden_C5_L4096_oracle_risbo(mw, O, spin):
    import torch
    g = _big(f"L4096_s{spin}_risbo")
    L = 4096
    v = torch.from_numpy(O.gaussian_coeffs(L, spin, int(g["seed"]))).cuda()
    sig = mw.inverse(mw.HarmonicCoeffs(L, spin, v), recursion="risbo").samples
    _check_samples(g, sig.cpu().numpy(), L, 2e-12)
    del sig
    raw = torch.from_numpy(random_signal(L, spin, int(g["raw_seed"]))).cuda()
    flm = mw.forward(mw.MwSignal(L, spin, raw), recursion="risbo").values
    _check_fwd(O, g, flm.cpu().numpy(), L, 2e-12)


@pytest.mark.parametrize("L,spin,real", [(64, 0, False), (256, -2, False), (1024, 0, True),
                                         (1024, 2, False)])
def test_config_full_arrays_match_oracle(mw, O, L, spin, real):
    # C1-C3 (and C3's size at spin 2) compared on the WHOLE arrays, not a
    # subsample: the inverse of the seeded BASELINE coefficients and the forward
    # of those samples, against the oracle (the reference's algorithm)
    if real:
        v = O.gaussian_real_coeffs(L, 0)
        sig = mw.inverse_real(mw.HarmonicCoeffs(L, 0, v.copy())).samples
        ref = O.inverse_real(v, L, threads=THREADS)
        back = mw.forward_real(mw.MwSignal(L, 0, np.array(sig))).values
        ref_back = O.forward_real(ref, L, threads=THREADS)
    else:
        v = O.gaussian_coeffs(L, spin, 0)
        sig = mw.inverse(mw.HarmonicCoeffs(L, spin, v.copy())).samples
        ref = O.inverse(v, L, spin, threads=THREADS)
        back = mw.forward(mw.MwSignal(L, spin, np.array(sig))).values
        ref_back = O.forward(ref, L, spin, threads=THREADS)
    assert rel(sig, ref) < 1e-12
    assert rel(back, ref_back) < 1e-12
