"""Small transforms for compute-sanitizer runs where the tool is available
(memcheck / racecheck / synccheck; it is disabled on the round-1 GPU pool):

    compute-sanitizer --tool memcheck python tools/sanitize.py
Covers the paired and plain inverse cores, the batched (two maps per CTA)
cores, the real path and every FFT stage, at band limits the tools finish fast.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1110_6298_b200 as mw  # noqa: E402
from oracle.mw_oracle import gaussian_coeffs, gaussian_real_coeffs  # noqa: E402

L = int(os.environ.get("SAN_L", "72"))
for spin in (0, 2):
    v = gaussian_coeffs(L, spin, 1)
    sig = mw.inverse(mw.HarmonicCoeffs(L, spin, v)).samples
    back = mw.forward(mw.MwSignal(L, spin, sig)).values
    assert np.max(np.abs(back - v)) < 1e-11
vals = np.stack([gaussian_coeffs(L, 0, k) for k in range(3)])
b = mw.forward_batch(mw.inverse_batch(vals, L, 0), L, 0)
assert np.max(np.abs(b - vals)) < 1e-11
vr = gaussian_real_coeffs(L, 2)
r = mw.forward_real(mw.inverse_real(mw.HarmonicCoeffs(L, 0, vr))).values
assert np.max(np.abs(r - vr)) < 1e-11
print("sanitize workload ok, L =", L)
