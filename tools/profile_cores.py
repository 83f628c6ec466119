"""Run a few inverse+forward transforms at one config (for ncu captures).

    python tools/profile_cores.py --L 2048 --spin 0 [--real] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1110_6298_b200 as mw  # noqa: E402
from oracle.mw_oracle import gaussian_coeffs, gaussian_real_coeffs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=2048)
ap.add_argument("--spin", type=int, default=0)
ap.add_argument("--real", action="store_true")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--paired", type=int, default=-1)
a = ap.parse_args()
L, s = a.L, a.spin
v = gaussian_real_coeffs(L, 0) if a.real else gaussian_coeffs(L, s, 0)
f = torch.from_numpy(v).cuda()
mw.get_plan(L).set_paired(a.paired)
for _ in range(a.reps):
    if a.real:
        sig = mw.inverse_real(mw.HarmonicCoeffs(L, 0, f))
        back = mw.forward_real(sig)
    else:
        sig = mw.inverse(mw.HarmonicCoeffs(L, s, f))
        back = mw.forward(sig)
torch.cuda.synchronize()
print("roundtrip max abs err", float((back.values - f).abs().max()))
