import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_1110_6298_b200 as mw
from paper_1110_6298_b200 import kernels
from oracle import mw_oracle as O
from helpers import random_signal, rel
for L in (1024, 1100, 2048):
    sig = random_signal(L, 0, 3)
    g = kernels.forward_stages(sig, L, 0)
    ref = O.gfold_of(sig, L, 0)
    print(L, 'stages rel', rel(g, ref))
    # phi stage only: compare AT rows via a trick: spin-0 band-limited?
