"""Small transforms for compute-sanitizer runs where the tool is available
(memcheck / racecheck / synccheck).  compute-sanitizer is closed on this
build's GPU pool (round 2 re-checked: "closed on this pool and stays closed"),
so bounds and races are covered by the oracle comparisons, the bitwise
repeatability test and the small/tiled core cross-checks instead:

    compute-sanitizer --tool memcheck python tools/sanitize.py
Covers the paired and plain inverse cores, the batched (two maps per CTA)
cores, the multi-spin cores, the real path, every FFT stage and the GL
kernels, at band limits the tools finish fast.  Run it once with the default
small-L per-chain cores and once with MWSHT_SMALL_INV=0 MWSHT_SMALL_FWD=0
(tiled cores).
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
ms = [0, 2, -1]
mv = np.stack([gaussian_coeffs(L, s, k) for k, s in enumerate(ms)])
m2 = mw.forward_multi_spin(mw.inverse_multi_spin(mv, L, ms), L, ms)
assert np.max(np.abs(m2 - mv)) < 1e-11
g = mw.gl_forward(mw.gl_inverse(mw.HarmonicCoeffs(L, 2, gaussian_coeffs(L, 2, 3))), 2).values
assert np.max(np.abs(g - gaussian_coeffs(L, 2, 3))) < 1e-10
print("sanitize workload ok, L =", L, "small-core limits",
      os.environ.get("MWSHT_SMALL_INV", "default"), os.environ.get("MWSHT_SMALL_FWD", "default"))
