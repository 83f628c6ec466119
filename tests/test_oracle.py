"""The oracle (oracle/, a CPU restatement of the reference) pinned against the
reference's own outputs in tests/golden/ (produced by make_golden.py from the
reference).  CPU only."""

import math

import numpy as np
import pytest

from conftest import golden_cfg
from helpers import SMALL_CASES, checksums, max_abs, random_signal

from oracle import mw_oracle as O


@pytest.mark.parametrize("rec", ["trapani", "risbo"])
@pytest.mark.parametrize("L,spin", SMALL_CASES)
def test_oracle_reproduces_reference_small(golden_small, L, spin, rec):
    key = f"L{L}_s{spin}_{rec}"
    v = O.gaussian_coeffs(L, spin, L + abs(spin))
    sig = O.inverse(v, L, spin, rec)
    assert max_abs(sig, golden_small[key + "_samples"]) == 0.0
    back = O.forward(sig, L, spin, rec)
    assert max_abs(back, golden_small[key + "_back"]) == 0.0
    raw = random_signal(L, spin, L + abs(spin))
    assert max_abs(O.forward(raw, L, spin, rec), golden_small[key + "_fwdraw"]) == 0.0


@pytest.mark.parametrize("spin", [0, 2, -1])
@pytest.mark.parametrize("rec", ["trapani", "risbo"])
def test_oracle_kernels_bit_identical(golden_small, spin, rec):
    L = 9
    key = f"k9_s{spin}_{rec}"
    cl = np.sqrt((2.0 * np.arange(L) + 1.0) / (4.0 * math.pi))
    tr = rec == "trapani"
    assert max_abs(O.fmm_core(golden_small[key + "_flm2d"], cl, L, spin, tr),
                   golden_small[key + "_fmm"]) == 0.0
    assert max_abs(O.flm_core(golden_small[key + "_gfold"], L, spin, tr),
                   golden_small[key + "_flm"]) == 0.0


def test_oracle_real_kernels(golden_small):
    cl = np.sqrt((2.0 * np.arange(8) + 1.0) / (4.0 * math.pi))
    assert max_abs(O.fmm_core_real(golden_small["k8real_in"], cl, 8, True),
                   golden_small["k8real_fmm"]) == 0.0
    assert max_abs(O.flm_core_real(golden_small["k8real_gf"], 8, True),
                   golden_small["k8real_flm"]) == 0.0


def test_oracle_real_path(golden_small):
    v = O.gaussian_real_coeffs(16, 6)
    sig = O.inverse_real(v, 16)
    assert max_abs(sig, golden_small["real16_samples"]) == 0.0
    assert max_abs(O.forward_real(sig, 16), golden_small["real16_back"]) == 0.0


@pytest.mark.parametrize("name", ["L64_s0_trapani", "L256_s2_trapani", "L256_s-2_trapani"])
def test_oracle_configs(name):
    g = golden_cfg(name)
    L, spin = int(g["L"]), int(g["spin"])
    v = O.gaussian_coeffs(L, spin, int(g["seed"]))
    np.testing.assert_allclose(checksums(v), g["input_checksums"], rtol=1e-14)
    sig = O.inverse(v, L, spin, threads=4)
    assert max_abs(sig.reshape(-1)[g["samples_idx"]], g["samples_sub"]) == 0.0
    back = O.forward(sig, L, spin, threads=4)
    assert max_abs(back[g["back_idx"]], g["back_sub"]) == 0.0


def test_oracle_threads_do_not_change_bits():
    L, s = 60, 1
    rng = np.random.default_rng(0)
    flm2d = rng.standard_normal((L, 2 * L - 1)) + 1j * rng.standard_normal((L, 2 * L - 1))
    gf = rng.standard_normal((2 * L - 1, L)) + 1j * rng.standard_normal((2 * L - 1, L))
    cl = O.cl_table(L)
    for rec in (True, False):
        a = O.fmm_core(flm2d, cl, L, s, rec, threads=1)
        b = O.fmm_core(flm2d, cl, L, s, rec, threads=5)
        assert max_abs(a, b) == 0.0
        assert max_abs(O.flm_core(gf, L, s, rec, threads=1),
                       O.flm_core(gf, L, s, rec, threads=3)) == 0.0


def test_golden_inputs_regenerate():
    # the config inputs are regenerated from seeds on the GPU box: pin the generator
    for name in ("L64_s0_trapani", "L256_s2_trapani", "L1024_s0_trapani_real",
                 "L1100_s0_risbo"):
        g = golden_cfg(name)
        L, spin = int(g["L"]), int(g["spin"])
        v = (O.gaussian_real_coeffs(L, int(g["seed"])) if bool(g["real"])
             else O.gaussian_coeffs(L, spin, int(g["seed"])))
        np.testing.assert_allclose(checksums(v), g["input_checksums"], rtol=1e-13)


def test_real_coefficients_are_real_symmetric():
    v = O.gaussian_real_coeffs(12, 3)
    worst, tol = O.reality_residual(v, 12)
    assert worst <= tol


@pytest.mark.parametrize("L,s", [(1, 0), (2, 1), (7, 0), (16, -2), (33, 3), (64, 0)])
def test_oracle_reduced_grid_and_quadrature_match_reference(L, s):
    import os
    from conftest import ROOT
    g = np.load(os.path.join(ROOT, "tests", "golden", "reduced.npz"))
    v = O.gaussian_coeffs(L, s, 100 + L)
    key = f"L{L}_s{s}"
    assert np.max(np.abs(O.synthesize_reduced(v, L, s) - g[key + "_reduced"])) == 0.0
    assert np.max(np.abs(O.ring_weights_v(L) - g[key + "_v"])) == 0.0
    q = O.quad_weights_q(L, s)
    assert np.max(np.abs(q - g[key + "_q"])) == 0.0
    assert O.integrate(g[key + "_reduced"], q) == complex(g[key + "_integral"])


def test_gl_oracle_matches_reference_golden():
    # oracle/'s restatement of gl_flm_core / gl_fm_core (_numba.py:191-268)
    # against the reference's own gl_inverse / gl_forward outputs
    import os
    import numpy as np
    from helpers import random_signal
    from oracle import mw_oracle as O
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "gl.npz"))
    for L, s in [(1, 0), (2, 0), (2, 1), (8, 0), (8, -3), (33, 2), (64, -1)]:
        k = f"L{L}_s{s}"
        inv = O.gl_inverse(O.gaussian_coeffs(L, s, 100 + L), L, s, g[k + "_nodes"])
        fwd = O.gl_forward(random_signal(L, s, 200 + L), L, s, g[k + "_nodes"], g[k + "_weights"])
        assert np.array_equal(inv, g[k + "_inverse"]), k
        assert np.array_equal(fwd, g[k + "_forward"]), k


def test_gl_nodes_match_reference_golden():
    import os
    import numpy as np
    from paper_1110_6298_b200.gl import gl_nodes
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "gl.npz"))
    for L, s in [(1, 0), (2, 0), (8, 0), (33, 2), (64, -1), (128, 0)]:
        grid = gl_nodes(L)
        assert np.array_equal(grid.nodes, g[f"L{L}_s{s}_nodes"])
        assert np.array_equal(grid.weights, g[f"L{L}_s{s}_weights"])
