import numpy as np, sys
sys.path.insert(0, '.')
import paper_1110_6298_b200 as mw
from oracle import mw_oracle as O
for L, s, B in [(96, 1, 3), (96, 0, 3), (96, 1, 2), (64, 1, 2), (96, 1, 1)]:
    vals = np.stack([O.gaussian_coeffs(L, s, k) for k in range(B)])
    sig = mw.inverse_batch(vals, L, s)
    errs = []
    for b in range(B):
        ref = O.inverse(vals[b], L, s, threads=8)
        one = mw.inverse(mw.HarmonicCoeffs(L, s, vals[b].copy())).samples
        errs.append((np.max(np.abs(sig[b] - ref)) / np.max(np.abs(ref)), np.max(np.abs(one - ref)) / np.max(np.abs(ref))))
    print(L, s, B, errs)
