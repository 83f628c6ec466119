"""Golden vectors of the reference's Gauss-Legendre comparator (gl.py,
kernels/_numba.py:191-268), produced by importing the reference here:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_gl_golden.py

For each (L, spin): the nodes and weights (gl_nodes), gl_inverse of the
seeded coefficients (oracle.mw_oracle.gaussian_coeffs) and gl_forward of a
seeded raw signal (tests/helpers.random_signal).  tests/test_oracle.py pins
oracle/'s GL restatement to these, tests/test_gpu_gl.py the CUDA kernels."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.abspath(os.path.join(HERE, "..", ".."))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torusht as ref  # noqa: E402

from helpers import random_signal  # noqa: E402
from oracle.mw_oracle import gaussian_coeffs  # noqa: E402

CASES = [(1, 0), (2, 0), (2, 1), (8, 0), (8, -3), (33, 2), (64, -1), (128, 0)]


def main():
    out = {}
    for L, s in CASES:
        g = ref.gl_nodes(L)
        v = gaussian_coeffs(L, s, 100 + L)
        sig = np.asarray(ref.gl_inverse(ref.HarmonicCoeffs(L, s, v.copy())))
        raw = random_signal(L, s, 200 + L)
        fwd = np.asarray(ref.gl_forward(raw, s).values)
        k = f"L{L}_s{s}"
        out[k + "_nodes"] = np.asarray(g.nodes)
        out[k + "_weights"] = np.asarray(g.weights)
        out[k + "_inverse"] = sig
        out[k + "_forward"] = fwd
    np.savez_compressed(os.path.join(HERE, "gl.npz"), **out)


if __name__ == "__main__":
    main()
