"""Core times of the tiled vs one-thread-per-chain cores over band limits
(run on the GPU box): python tools/small_sweep.py  -> table on stdout.
Each configuration runs in a fresh process (the limits are read once)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1110_6298_b200 as mw
from paper_1110_6298_b200 import _lib
from oracle.mw_oracle import gaussian_coeffs
L, s = int(sys.argv[1]), int(sys.argv[2])
v = torch.from_numpy(gaussian_coeffs(L, s, 0)).cuda()
p = mw.get_plan(L); lib = _lib.load()
lib.mwsht_plan_set_timing(p.handle, 1)
inv, fwd = [], []
for k in range(25):
    sig = mw.inverse(mw.HarmonicCoeffs(L, s, v)).samples
    back = mw.forward(mw.MwSignal(L, s, sig)).values
    torch.cuda.synchronize()
    c, st = _lib.ctypes.c_float(), _lib.ctypes.c_float()
    lib.mwsht_plan_last_timing(p.handle, 1, _lib.ctypes.byref(c), _lib.ctypes.byref(st)); a = c.value
    lib.mwsht_plan_last_timing(p.handle, 0, _lib.ctypes.byref(c), _lib.ctypes.byref(st)); b = c.value
    if k >= 5: inv.append(a); fwd.append(b)
print(json.dumps({"inv": float(np.median(inv)), "fwd": float(np.median(fwd)),
                  "err": float((back - v).abs().max())}))
''' % ROOT

for L in (64, 96, 128, 192, 256, 384, 512):
    row = [L]
    for lim in (0, 100000):
        env = dict(os.environ, MWSHT_SMALL_INV=str(lim), MWSHT_SMALL_FWD=str(lim))
        out = subprocess.run([sys.executable, "-c", CHILD, str(L), "2"], env=env,
                             capture_output=True, text=True).stdout.strip().splitlines()[-1]
        d = json.loads(out)
        row += [d["inv"], d["fwd"], d["err"]]
    print("L=%4d  tiled inv %.4f fwd %.4f (err %.1e) | per-chain inv %.4f fwd %.4f (err %.1e) ms"
          % tuple(row), flush=True)
