"""m-column sharding on one GPU: the shard stage entry points
run as k virtual ranks must reproduce the unsharded transforms.

The shards run the plain inverse-core tiles (paired tiles would emit orders
outside the shard), so the bit-exact comparison is against the unsharded
transform with plain tiles; the default (paired for spin 0) agrees to rounding."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,spin,world", [(256, 2, 2), (256, 0, 3), (300, -1, 4), (96, 0, 2)])
def test_mcolumn_emulation_matches_unsharded(L, spin, world):
    import torch
    import paper_1110_6298_b200 as mw
    from paper_1110_6298_b200 import shard
    from oracle import mw_oracle as O
    v = torch.from_numpy(O.gaussian_coeffs(L, spin, 5)).cuda()
    samples, flm = shard.emulate_mcolumn(L, world, spin, v)
    plan = mw.get_plan(L)
    plan.set_paired(0)
    try:
        ref_s = mw.inverse(mw.HarmonicCoeffs(L, spin, v)).samples
    finally:
        plan.set_paired(-1)
    assert (samples - ref_s).abs().max().item() == 0.0
    dflt = mw.inverse(mw.HarmonicCoeffs(L, spin, v)).samples
    assert (samples - dflt).abs().max().item() <= 1e-12 * dflt.abs().max().item()
    ref_f = mw.forward(mw.MwSignal(L, spin, ref_s)).values
    assert (flm - ref_f).abs().max().item() == 0.0
    assert (flm - v).abs().max().item() < 1e-11
