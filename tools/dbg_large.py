import sys, math, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1110_6298_b200 as mw
from test_gpu_large_L import ylm_column, _unit
from helpers import rel
for L, ell, m in [(1024, 1023, 0), (2048, 2047, 0), (4096, 4095, 0), (4096, 3000, 1200), (4500, 4499, 0), (4500, 3000, 1200)]:
    v = torch.from_numpy(_unit(L, ell, m)).cuda()
    sig = mw.inverse(mw.HarmonicCoeffs(L, 0, v)).samples
    back = mw.forward(mw.MwSignal(L, 0, sig)).values
    s = sig.cpu().numpy()
    phi = 2 * math.pi * np.arange(2 * L - 1) / (2 * L - 1)
    ref = ylm_column(L, ell, m)[:, None] * np.exp(1j * m * phi)[None, :]
    d = np.abs(s - ref)
    i = np.unravel_index(np.argmax(d), d.shape)
    print(L, ell, m, 'rel', rel(s, ref), 'worst at ring', i[0], 'max', np.abs(ref).max(), 'rt', float((back - v).abs().max()))
