"""m-column sharding on one GPU: the shard stage entry points
run as k virtual ranks must reproduce the unsharded transforms.

The shards run the plain inverse-core tiles (paired tiles would emit orders
outside the shard), so the bit-exact comparison is against the unsharded
transform with plain tiles; the default (paired for spin 0) agrees to rounding."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("L,spin,world", [(256, 2, 2), (256, 0, 3), (300, -1, 4), (96, 0, 2),
                                            (600, 1, 2), (1100, 0, 3)])  # H >= 2048: decoupled theta stage
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


def _live_worker(rank, world, port, L, spin, q):
    # one process per rank, all on cuda:0 (the exchange is host-staged gloo, so
    # no rank's kernels wait on another's): the real MColumnSharding data path
    import os
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1110_6298_b200 as mw
        from paper_1110_6298_b200 import shard
        from oracle import mw_oracle as O
        torch.cuda.set_device(0)
        v = torch.from_numpy(O.gaussian_coeffs(L, spin, 9)).cuda()
        sh = shard.MColumnSharding(L, world, rank, 0)
        rings = sh.inverse(v, spin)
        flm = sh.forward(rings, spin)
        torch.cuda.synchronize()
        parts = [torch.empty((sh.tb[r + 1] - sh.tb[r], 2 * L - 1), dtype=torch.complex128)
                 for r in range(world)]
        dist.all_gather(parts, rings.cpu())
        samples = torch.cat(parts, 0)
        plan = mw.get_plan(L)
        plan.set_paired(0)   # the shards run plain inverse tiles
        ref_s = mw.inverse(mw.HarmonicCoeffs(L, spin, v)).samples.cpu()
        ref_f = mw.forward(mw.MwSignal(L, spin, samples.cuda())).values.cpu()
        q.put((rank, float((samples - ref_s).abs().max()), float((flm.cpu() - ref_f).abs().max()),
               float((flm - v).abs().max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("L,spin,world", [(256, 2, 2), (300, 0, 3), (600, 1, 2)])  # 600: H = 2048
def test_mcolumn_live_ranks_match_unsharded(L, spin, world):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.spawn(_live_worker, args=(world, port, L, spin, q), nprocs=world, join=True)
    res = [q.get() for _ in range(world)]
    for rank, ds, df, rt in res:
        assert ds == 0.0, (rank, ds)      # bit-identical to the unsharded inverse
        assert df == 0.0, (rank, df)      # and forward
        assert rt < 1e-11, (rank, rt)
