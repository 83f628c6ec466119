"""Time the transform stages at one config with CUDA events (A/B tool).

    MWSHT_LIB=/path/variant.so python tools/stage_time.py --L 4096 [--spin 0] [--reps 5]
Prints forward FFT stages, forward core, inverse core and whole inverse/forward (ms).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1110_6298_b200 as mw  # noqa: E402
from paper_1110_6298_b200 import _lib  # noqa: E402
from oracle.mw_oracle import gaussian_coeffs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=4096)
ap.add_argument("--spin", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--real", action="store_true")
ap.add_argument("--paired", type=int, default=-1)
a = ap.parse_args()
L, s = a.L, a.spin
lib = _lib.load()
plan = mw.get_plan(L, 0)
plan.set_paired(a.paired)
lib.mwsht_plan_set_timing(plan.handle, 1)
from oracle.mw_oracle import gaussian_real_coeffs  # noqa: E402
f = torch.from_numpy(gaussian_real_coeffs(L, 0) if a.real else gaussian_coeffs(L, s, 0)).cuda()
sig = torch.empty((L, 2 * L - 1), dtype=torch.float64 if a.real else torch.complex128,
                  device="cuda")
back = torch.empty_like(f)
st = _lib._P(torch.cuda.current_stream().cuda_stream)
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
rows = []
for r in range(a.reps + 1):
    e[0].record()
    if a.real:
        _lib.check(lib.mwsht_inverse_real_d(plan.handle, f.data_ptr(), sig.data_ptr(), 0, st))
    else:
        _lib.check(lib.mwsht_inverse_z(plan.handle, f.data_ptr(), sig.data_ptr(), s, 0, st))
    e[1].record()
    if a.real:
        _lib.check(lib.mwsht_forward_real_d(plan.handle, sig.data_ptr(), back.data_ptr(), 0, st))
    else:
        _lib.check(lib.mwsht_forward_z(plan.handle, sig.data_ptr(), back.data_ptr(), s, 0, st))
    e[2].record()
    torch.cuda.synchronize()
    c, g = _lib.ctypes.c_float(), _lib.ctypes.c_float()
    lib.mwsht_plan_last_timing(plan.handle, 1, _lib.ctypes.byref(c), _lib.ctypes.byref(g))
    inv_core = c.value
    lib.mwsht_plan_last_timing(plan.handle, 0, _lib.ctypes.byref(c), _lib.ctypes.byref(g))
    if r:
        rows.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2]), inv_core, c.value, g.value))
m = np.median(np.array(rows), axis=0)
err = float((back - f).abs().max())
print(f"L={L} s={s} real={a.real} paired={a.paired} {os.environ.get('MWSHT_LIB', 'in-tree')}: inverse {m[0]:.2f} ms (core {m[2]:.2f}, stages "
      f"{m[0]-m[2]:.2f}) | forward {m[1]:.2f} ms (stages {m[4]:.2f}, core {m[3]:.2f}) | "
      f"pair {m[0]+m[1]:.2f} ms | err {err:.1e}")
