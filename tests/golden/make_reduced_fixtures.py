"""Golden vectors for the reduced-grid synthesis and the quadrature weights,
produced by the REFERENCE (mw.py:449-466, quadrature.py:77-139).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_reduced_fixtures.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import torusht as ref  # noqa: E402
from torusht import quadrature as rq  # noqa: E402

from oracle.mw_oracle import gaussian_coeffs  # noqa: E402

out = {}
for L, s in [(1, 0), (2, 1), (7, 0), (16, -2), (33, 3), (64, 0)]:
    v = gaussian_coeffs(L, s, 100 + L)
    key = f"L{L}_s{s}"
    out[key + "_reduced"] = np.asarray(ref.synthesize_reduced(ref.HarmonicCoeffs(L, s, v)))
    w = rq.quad_weights(L, s)
    out[key + "_v"] = np.asarray(w.v)
    out[key + "_q"] = np.asarray(w.q)
    out[key + "_integral"] = np.array(rq.integrate(out[key + "_reduced"], w))
np.savez_compressed(os.path.join(HERE, "reduced.npz"), **out)
print("wrote", len(out), "arrays")
