import ctypes, os, sys
sys.path.insert(0, '.')
os.environ['MWSHT_LIB'] = 'tools/runs/libmwsht_prof.so'
import numpy as np, torch
import paper_1110_6298_b200 as mw
from paper_1110_6298_b200 import _lib
from oracle.mw_oracle import gaussian_coeffs
lib = _lib.load()
lib.mwsht_debug_prof.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
for L in (1024, 2048, 4096):
    plan = mw.get_plan(L, 0)
    plan.set_paired(0)
    f = torch.from_numpy(gaussian_coeffs(L, 0, 0)).cuda()
    sig = mw.inverse(mw.HarmonicCoeffs(L, 0, f)).samples
    buf = (ctypes.c_ulonglong * 8)()
    lib.mwsht_debug_prof(buf, 1)
    sig = mw.inverse(mw.HarmonicCoeffs(L, 0, f)).samples
    torch.cuda.synchronize()
    lib.mwsht_debug_prof(buf, 1)
    w, t, first, n, seed, ramp, _, _ = list(buf)
    print(f"L={L}: warps {n}, wait(k>0) {w/t:.3f} of consumer cycles, first-chunk wait {first/t:.3f}, avg warp cycles {t/n:.0f}, prologue {seed/t:.3f}, ramp {ramp/t:.3f}")
