"""A/B of the batched inverse (C4: 8 maps, L=2048) with paired vs plain tiles.

    python tools/batch_ab.py
"""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1110_6298_b200 as mw
from paper_1110_6298_b200 import _lib
from oracle.mw_oracle import gaussian_coeffs
L, B = 2048, 8
for spin in (0, 2):
    vals = torch.from_numpy(np.stack([gaussian_coeffs(L, spin, k) for k in range(B)])).cuda()
    plan = mw.get_plan(L, 0, max_batch=B)
    lib = _lib.load()
    for mode in (1, 0):
        plan.set_paired(mode)
        for _ in range(2):
            sig = mw.inverse_batch(vals, L, spin)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            sig = mw.inverse_batch(vals, L, spin)
        e1.record(); torch.cuda.synchronize()
        back = mw.forward_batch(sig, L, spin)
        print(f"spin {spin} paired={mode}: inverse batch of {B} {e0.elapsed_time(e1)/3:.2f} ms, roundtrip {float((back-vals).abs().max()):.2e}")
    plan.set_paired(-1)
