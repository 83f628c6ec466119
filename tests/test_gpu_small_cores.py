"""One-thread-per-chain cores for small band limits (csrc/core_small.cu): the
default path below the crossovers (inverse L <= 160, forward L <= 320).  The
tiled and per-chain cores must agree to rounding and both match the oracle;
each runs in its own process because the crossovers are read once."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import json, sys, numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_1110_6298_b200 as mw
from paper_1110_6298_b200 import kernels
from oracle import mw_oracle as O
from helpers import rel, random_signal
out = {}
for L, s in [(1, 0), (2, 1), (17, -3), (64, 0), (100, 2), (160, -1)]:
    v = O.gaussian_coeffs(L, s, L)
    sig = mw.inverse(mw.HarmonicCoeffs(L, s, v.copy())).samples
    raw = random_signal(L, s, L)
    fwd = mw.forward(mw.MwSignal(L, s, raw)).values
    out[f"{L},{s}"] = [rel(sig, O.inverse(v, L, s, threads=8)), rel(fwd, O.forward(raw, L, s, threads=8))]
for L in (3, 64, 150):
    vr = O.gaussian_real_coeffs(L, 2)
    sr = mw.inverse_real(mw.HarmonicCoeffs(L, 0, vr.copy())).samples
    out[f"real{L}"] = [rel(sr, O.inverse_real(vr, L)),
                       rel(mw.forward_real(mw.MwSignal(L, 0, np.array(sr))).values, O.forward_real(sr, L))]
rng = np.random.default_rng(4)
L = 40
gf = rng.standard_normal((2 * L - 1, L)) + 1j * rng.standard_normal((2 * L - 1, L))
f2 = rng.standard_normal((L, 2 * L - 1)) + 1j * rng.standard_normal((L, 2 * L - 1))
cl = O.cl_table(L)
out["hooks"] = [rel(kernels.flm_core(gf, L, 2, True), O.flm_core(gf, L, 2, True)),
                rel(kernels.fmm_core(f2, cl, L, 2, True), O.fmm_core(f2, cl, L, 2, True))]
print(json.dumps(out))
''' % (ROOT, os.path.join(ROOT, "tests"))


@pytest.mark.parametrize("limits", [("0", "0"), ("100000", "100000")], ids=["tiled", "per_chain"])
def test_small_and_tiled_cores_match_oracle(limits):
    env = dict(os.environ, MWSHT_SMALL_INV=limits[0], MWSHT_SMALL_FWD=limits[1])
    res = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr[-2000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    for key, errs in out.items():
        assert max(errs) < 1e-12, (key, errs)
