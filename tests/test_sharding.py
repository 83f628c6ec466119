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


def _spec(k, t):
    """Synthetic spectrum value of bin k at ring t (distinct per pair)."""
    return (k * 1000.0 + t) + 1j * (k - 0.5 * t)


def _exchange_roundtrip(rank, world, L=200):
    """Both all-to-all transposes through ExchangeLayout on real gloo ranks,
    with numpy standing in for the stage kernels' table addressing
    (include/mwsht.h): what the forward theta stage reads must be the phi
    spectra of its orders for every ring, and what the inverse phi stage reads
    must be every order's synthesis of its rings."""
    N = 2 * L - 1
    b = shard.balanced_m_splits(L, world, align=32)
    tb = shard.ring_splits(L, world)
    lay = shard.ExchangeLayout(L, b, tb, rank)
    t0, t1 = tb[rank], tb[rank + 1]
    rows = shard.order_bins(L, b[rank], b[rank + 1])
    # forward: k_phi_fwd writes bin k, ring t at send[row_off[k] + t - t0]
    send = torch.full((sum(lay.fsend_counts),), complex("nan"), dtype=torch.complex128)
    for k in range(N):
        for t in range(t0, t1):
            send[lay.fphi_row_off[k] + t - t0] = _spec(k, t)
    recv = torch.full((sum(lay.frecv_counts),), complex("nan"), dtype=torch.complex128)
    shard.all_to_all_flat(send, lay.fsend_counts, recv, lay.frecv_counts)
    ok = True
    for i, k in enumerate(rows):   # k_theta_fwd reads row i, ring t
        got = [recv[lay.ftheta_col_off[t] + i * lay.ftheta_col_stride[t]].item() for t in range(L)]
        ok &= got == [_spec(k, t) for t in range(L)]
    # inverse: k_theta_inv writes ring t of row i at send[row_off[t] + i]
    isend = torch.full((sum(lay.isend_counts),), complex("nan"), dtype=torch.complex128)
    for i, k in enumerate(rows):
        for t in range(L):
            isend[lay.itheta_row_off[t] + i] = _spec(k, t)
    irecv = torch.full((sum(lay.irecv_counts),), complex("nan"), dtype=torch.complex128)
    shard.all_to_all_flat(isend, lay.isend_counts, irecv, lay.irecv_counts)
    for t in range(t0, t1):        # k_phi_inv reads ring t, bin n
        got = [irecv[lay.iphi_col_off[n] + (t - t0) * lay.iphi_col_stride[n]].item()
               for n in range(N)]
        ok &= got == [_spec(n, t) for n in range(N)]
    return bool(ok)


def _flm_gather(rank, world, L=150):
    """Packed coefficient blocks (forward core out_mode 2) all-gathered and
    unpacked (k_flm_unpack's index math, mirrored) rebuild the flat flm."""
    b = shard.balanced_m_splits(L, world, align=32)
    lay = shard.ExchangeLayout(L, b, shard.ring_splits(L, world), rank)
    full = np.arange(L * L) * (1.0 + 0.5j)
    m0, m1 = b[rank], b[rank + 1]
    block = torch.zeros(lay.flm_maxlen, dtype=torch.complex128)
    n = 0
    for l in range(L):
        for m in range(-l, l + 1):
            if m0 <= abs(m) < m1:
                block[int(shard.shard_flm_index(l, m, m0, m1))] = complex(full[l * (l + 1) + m])
                n += 1
    assert n == lay.flm_len[rank]
    gathered = torch.empty(world * lay.flm_maxlen, dtype=torch.complex128)
    shard.all_gather_flat(block, gathered)
    out = np.empty(L * L, complex)
    for l in range(L):
        for m in range(-l, l + 1):
            r = int(np.searchsorted(b, abs(m), side="right") - 1)
            out[l * (l + 1) + m] = gathered[r * lay.flm_maxlen +
                                            int(shard.shard_flm_index(l, m, b[r], b[r + 1]))]
    return bool(np.array_equal(out, full))


def test_exchange_layout_all_to_all_gloo():
    assert all(_run(_exchange_roundtrip, world=2).values())
    assert all(_run(_exchange_roundtrip, world=3).values())


def test_flm_blocks_all_gather_gloo():
    assert all(_run(_flm_gather, world=2).values())
    assert all(_run(_flm_gather, world=3).values())


def test_flm_block_index_is_a_bijection():
    for L, parts in [(150, 3), (97, 2), (64, 2), (33, 1)]:
        b = shard.balanced_m_splits(L, parts) if parts > 1 else [0, L]
        for q in range(parts):
            m0, m1 = b[q], b[q + 1]
            idx = [int(shard.shard_flm_index(l, m, m0, m1)) for l in range(L)
                   for m in range(-l, l + 1) if m0 <= abs(m) < m1]
            assert sorted(idx) == list(range(int(shard.shard_flm_base(L, m0, m1))))


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
