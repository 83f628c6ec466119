"""Multi-rank host logic of SURVEY.md §8e on CPU: work-balanced order splits,
the all-to-all ring <-> order transposes, and map sharding, with world_size-2
gloo process groups (127.0.0.1)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1110_6298_b200 import shard


def test_balanced_splits_equalize_core_work():
    for L, parts in [(4096, 2), (4096, 4), (4096, 8), (2048, 8), (256, 2), (1024, 3)]:
        b = shard.balanced_m_splits(L, parts)
        assert b[0] == 0 and b[-1] == L and len(b) == parts + 1
        assert all(x % 32 == 0 for x in b[:-1])
        assert all(y > x for x, y in zip(b, b[1:]))
        w = shard.column_work(L)
        per = np.array([w[b0:b1].sum() for b0, b1 in zip(b, b[1:])])
        # rounding to 32-wide tiles leaves at most a few percent imbalance
        assert per.max() / per.mean() < 1.0 + 0.05 * parts * 64 / L * 16
    # SURVEY.md §8e split at L=4096 over 2 GPUs is |m| = 1422 (before tile rounding)
    assert abs(shard.balanced_m_splits(4096, 2)[1] - 1422) <= 32


def test_order_bins_partition_all_rows():
    L, N = 100, 199
    for parts in (1, 2, 3):
        b = shard.balanced_m_splits(L, parts, align=32) if parts > 1 else [0, L]
        rows = sum((shard.order_bins(L, b0, b1) for b0, b1 in zip(b, b[1:])), [])
        assert sorted(rows) == list(range(N))


def test_shard_maps_cover_batch():
    for n, w in [(8, 1), (8, 2), (8, 3), (8, 8), (5, 4)]:
        got = sum((shard.shard_maps(n, w, r) for r in range(w)), [])
        assert got == list(range(n))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = fn(rank, world)
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, fn, out), nprocs=world, join=True)
    return dict(out)


def _full_AT(L):
    N = 2 * L - 1
    k = torch.arange(N, dtype=torch.float64)[:, None]
    t = torch.arange(L, dtype=torch.float64)[None, :]
    return (k * 1000 + t) + 1j * (k - 0.5 * t)


def _exchange_fwd(rank, world):
    L = 70
    b = shard.balanced_m_splits(L, world, align=32)
    tb = shard.ring_splits(L, world)
    full = _full_AT(L)
    AT = torch.full_like(full, complex("nan"))
    AT[:, tb[rank]:tb[rank + 1]] = full[:, tb[rank]:tb[rank + 1]]   # own rings only
    shard.exchange_rings_to_orders(AT, b, tb, rank)
    rows = shard.order_bins(L, b[rank], b[rank + 1])
    return bool(torch.equal(AT[rows], full[rows]))


def _exchange_inv(rank, world):
    L = 70
    b = shard.balanced_m_splits(L, world, align=32)
    tb = shard.ring_splits(L, world)
    full = _full_AT(L).T.contiguous()   # (L, N)
    OUT = torch.full_like(full, complex("nan"))
    cols = shard.order_bins(L, b[rank], b[rank + 1])
    OUT[:, cols] = full[:, cols]        # own orders only
    shard.exchange_orders_to_rings(OUT, b, tb, rank)
    return bool(torch.equal(OUT[tb[rank]:tb[rank + 1]], full[tb[rank]:tb[rank + 1]]))


def test_all_to_all_transposes_gloo():
    assert all(_run(_exchange_fwd).values())
    assert all(_run(_exchange_inv).values())


def _maps(rank, world):
    from oracle import mw_oracle as O
    L, s, n = 12, 1, 5
    vals = np.stack([O.gaussian_coeffs(L, s, k) for k in range(n)])
    mine = shard.shard_maps(n, world, rank)
    local = torch.from_numpy(np.stack([O.inverse(vals[k], L, s) for k in mine]))
    ms = shard.MapSharding(L, n, world, rank, "cpu")
    full = ms.gather(local).numpy()
    ref = np.stack([O.inverse(vals[k], L, s) for k in range(n)])
    return float(np.max(np.abs(full - ref)))


def test_map_sharding_gather_gloo():
    assert max(_run(_maps).values()) == 0.0


def test_balanced_splits_stay_on_tile_grid_or_refuse():
    # every interior bound must be a multiple of the tile width (the shard entry
    # points reject anything else); too small L for the rank count is refused
    for L, parts in [(250, 7), (256, 8), (300, 4), (97, 3), (4096, 8), (1000, 5)]:
        b = shard.balanced_m_splits(L, parts)
        assert all(x % 32 == 0 for x in b[1:-1]), (L, parts, b)
        assert all(y - x >= 32 for x, y in zip(b, b[1:]))
    with pytest.raises(ValueError):
        shard.balanced_m_splits(250, 8)
