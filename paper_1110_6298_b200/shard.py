"""Multi-GPU sharding of the MW transforms.

Two ways the path shards:

* Independent maps (config C4): ``shard_maps`` hands rank r a contiguous block
  of the batch and ``MapSharding`` runs the batched transforms on it.  No
  data-path collective is needed; ``gather`` is optional.  The reference's
  callers loop over maps one by one (cli.py:159-224).

* m-column sharding of one map (config C5): ``MColumnSharding``.  For every
  order m the O(L^3) core is an independent matvec
  (kernels/_numba.py:75-105, 131-166).  The GPU recursions are also
  independent per chain (l-recursion per (m', m), Trapani column per (l, m)),
  so a rank owning orders m0 <= |m| < m1 needs no Delta halo.  Ranks split
  the |m| range so that core work is equal (``balanced_m_splits``) and the
  rings evenly.  The only exchange is one all-to-all transpose of the ring
  spectra per transform (t-sharded <-> m-sharded), done on NCCL with
  ``dist.all_to_all`` (gloo: pairwise send/recv).
  * Forward: phi DFT of own rings, all-to-all, theta stage + core for own
    orders, all-reduce of the (disjoint) coefficient blocks.
  * Inverse: core + theta synthesis for own orders, all-to-all, phi
    synthesis of own rings.
"""

import numpy as np
import torch
import torch.distributed as dist

from . import _lib


# ------------------------------------------------------------ partitions

def column_work(L):
    """Core work per order |m| (chain steps of both cores, +-m counted twice)."""
    m = np.arange(L, dtype=np.float64)
    inv = m * (L - m) + (L - m) * (L - m + 1) / 2.0   # sum_{m'} (L - max(m', m))
    fwd = (L * (L + 1) - m * (m + 1)) / 2.0           # sum_{l >= m} (l + 1)
    w = inv + fwd
    w[1:] *= 2.0
    return w


def balanced_m_splits(L, parts, align=32):
    """Boundaries 0 = b_0 < ... < b_parts = L of |m| with equal core work,
    rounded to multiples of `align` (the core's tile width)."""
    if parts <= 1:
        return [0, L]
    if L < align * parts:
        raise ValueError(f"cannot split L={L} into {parts} order ranges of width >= {align} "
                         f"(needs L >= {align * parts})")
    w = np.cumsum(column_work(L))
    total = w[-1]
    bounds = [0]
    for k in range(1, parts):
        target = total * k / parts
        b = int(np.searchsorted(w, target)) + 1
        b = int(round(b / align)) * align
        # the last ranges each need >= align columns; interior bounds stay on the
        # align grid (the shard entry points require it, plan.cu check_range)
        hi = (L - align * (parts - k)) // align * align
        b = min(max(b, bounds[-1] + align), hi)
        bounds.append(b)
    bounds.append(L)
    if any(b1 <= b0 for b0, b1 in zip(bounds, bounds[1:])):
        raise ValueError(f"cannot split L={L} into {parts} order ranges of width >= {align}")
    return bounds


def ring_splits(L, parts):
    return [L * k // parts for k in range(parts + 1)]


def order_bins(L, m0, m1):
    """Rows bin(m) = m mod N of the orders m0 <= |m| < m1, in the kernels'
    row order (+m ascending, then -m)."""
    N = 2 * L - 1
    pos = list(range(m0, m1))
    neg = [N - m for m in range(max(m0, 1), m1)]
    return pos + neg


def shard_maps(n, world, rank):
    """Contiguous block of map indices for `rank` (C4: maps sharded over ranks)."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return list(range(lo, hi))


# -------------------------------------------------------------- exchange

def _is_nccl(group=None):
    return dist.is_initialized() and dist.get_backend(group) == "nccl"


def all_to_all(send, recv_shapes, dtype, device, group=None):
    """send[q] -> rank q; returns recv[r] (shape recv_shapes[r]) from rank r."""
    if not dist.is_initialized():
        return [send[0].contiguous()]
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    recv = [torch.empty(shp, dtype=dtype, device=device) for shp in recv_shapes]
    if _is_nccl(group):
        dist.all_to_all(recv, [s.contiguous() for s in send], group=group)
        return recv
    reqs = []
    for k in range(1, world):
        dst = (rank + k) % world
        src = (rank - k) % world
        reqs.append(dist.isend(send[dst].contiguous(), dst, group=group))
        reqs.append(dist.irecv(recv[src], src, group=group))
    recv[rank].copy_(send[rank])
    for r in reqs:
        r.wait()
    return recv


def exchange_rings_to_orders(AT, bounds, tb, rank, group=None):
    """Forward transpose.  AT (N, L): this rank filled columns tb[rank]:tb[rank+1]
    for every bin; afterwards rows of this rank's orders hold all columns."""
    L = AT.shape[1]
    world = len(bounds) - 1
    t0, t1 = tb[rank], tb[rank + 1]
    rows = [torch.as_tensor(order_bins(L, bounds[q], bounds[q + 1]), device=AT.device)
            for q in range(world)]
    send = [AT.index_select(0, rows[q])[:, t0:t1] for q in range(world)]
    shapes = [(rows[rank].numel(), tb[r + 1] - tb[r]) for r in range(world)]
    recv = all_to_all(send, shapes, AT.dtype, AT.device, group)
    for r in range(world):
        AT[rows[rank], tb[r]:tb[r + 1]] = recv[r]
    return AT


def exchange_orders_to_rings(OUT, bounds, tb, rank, group=None):
    """Inverse transpose.  OUT (L, N): this rank filled the columns of its
    orders for every ring; afterwards its rings hold every column."""
    L = OUT.shape[0]
    world = len(bounds) - 1
    cols = [torch.as_tensor(order_bins(L, bounds[q], bounds[q + 1]), device=OUT.device)
            for q in range(world)]
    send = [OUT[tb[q]:tb[q + 1]].index_select(1, cols[rank]) for q in range(world)]
    shapes = [(tb[rank + 1] - tb[rank], cols[r].numel()) for r in range(world)]
    recv = all_to_all(send, shapes, OUT.dtype, OUT.device, group)
    t0, t1 = tb[rank], tb[rank + 1]
    for r in range(world):
        OUT[t0:t1, cols[r]] = recv[r]
    return OUT


# ----------------------------------------------------- GPU shard drivers

class MColumnSharding:
    """One complex map split over `world` ranks by order columns and rings."""

    def __init__(self, L, world, rank, device, group=None):
        from .mw import get_plan
        self.L, self.N = L, 2 * L - 1
        self.world, self.rank, self.group = world, rank, group
        self.device = torch.device(device)
        self.bounds = balanced_m_splits(L, world)
        self.tb = ring_splits(L, world)
        self.m0, self.m1 = self.bounds[rank], self.bounds[rank + 1]
        self.t0, self.t1 = self.tb[rank], self.tb[rank + 1]
        self.plan = get_plan(L, self.device.index)
        self.lib = _lib.load()
        self.AT = torch.empty((self.N, L), dtype=torch.complex128, device=self.device)
        self.OUT = torch.empty((L, self.N), dtype=torch.complex128, device=self.device)

    def _st(self):
        return _lib._P(torch.cuda.current_stream(self.device).cuda_stream)

    def forward_local(self, samples_rows, AT=None):
        AT = self.AT if AT is None else AT
        _lib.check(self.lib.mwsht_shard_forward_phi(self.plan.handle, samples_rows.data_ptr(),
                                                    self.t0, self.t1, AT.data_ptr(), self._st()),
                   "shard_forward_phi")
        return AT

    def forward_rest(self, spin, AT=None, flm=None):
        AT = self.AT if AT is None else AT
        if flm is None:
            flm = torch.zeros(self.L * self.L, dtype=torch.complex128, device=self.device)
        _lib.check(self.lib.mwsht_shard_forward_rest(self.plan.handle, AT.data_ptr(), self.m0,
                                                     self.m1, int(spin), flm.data_ptr(),
                                                     self._st()), "shard_forward_rest")
        return flm

    def forward(self, samples_rows, spin):
        """samples_rows: this rank's rings (t1-t0, N) -> full flm on every rank."""
        self.forward_local(samples_rows)
        exchange_rings_to_orders(self.AT, self.bounds, self.tb, self.rank, self.group)
        flm = self.forward_rest(spin)
        if self.world > 1:
            dist.all_reduce(flm, group=self.group)
        return flm

    def inverse_front(self, flm, spin, OUT=None):
        OUT = self.OUT if OUT is None else OUT
        _lib.check(self.lib.mwsht_shard_inverse_front(self.plan.handle, flm.data_ptr(), self.m0,
                                                      self.m1, int(spin), OUT.data_ptr(),
                                                      self._st()), "shard_inverse_front")
        return OUT

    def inverse_rings(self, OUT=None, out=None):
        OUT = self.OUT if OUT is None else OUT
        if out is None:
            out = torch.empty((self.t1 - self.t0, self.N), dtype=torch.complex128,
                              device=self.device)
        _lib.check(self.lib.mwsht_shard_inverse_phi(self.plan.handle, OUT.data_ptr(), self.t0,
                                                    self.t1, out.data_ptr(), self._st()),
                   "shard_inverse_phi")
        return out

    def inverse(self, flm, spin):
        """flm (L^2,) on every rank -> this rank's rings (t1-t0, N)."""
        self.inverse_front(flm, spin)
        exchange_orders_to_rings(self.OUT, self.bounds, self.tb, self.rank, self.group)
        return self.inverse_rings()


def emulate_mcolumn(L, world, spin, flm, device=0):
    """Run the m-column-sharded inverse and forward of one map as `world`
    virtual ranks in one process (exchange by direct copies).  Validates
    the range logic of the shard stages on a single GPU."""
    shards = [MColumnSharding(L, world, r, device) for r in range(world)]
    N = 2 * L - 1
    OUT = torch.empty((L, N), dtype=torch.complex128, device=f"cuda:{device}")
    for sh in shards:  # each writes its own order columns of the shared OUT
        sh.inverse_front(flm, spin, OUT=OUT)
    rings = [sh.inverse_rings(OUT=OUT) for sh in shards]
    samples = torch.cat(rings, 0)
    AT = torch.empty((N, L), dtype=torch.complex128, device=f"cuda:{device}")
    for sh in shards:
        sh.forward_local(samples[sh.t0:sh.t1].contiguous(), AT=AT)
    flm_out = torch.zeros(L * L, dtype=torch.complex128, device=f"cuda:{device}")
    for sh in shards:
        flm_out += sh.forward_rest(spin, AT=AT)
    return samples, flm_out


class MapSharding:
    """Independent maps sharded over ranks (C4); no data-path collective."""

    def __init__(self, L, n_maps, world, rank, device):
        self.L, self.n, self.world, self.rank = L, n_maps, world, rank
        self.mine = shard_maps(n_maps, world, rank)
        self.device = device

    def inverse(self, values_local, spin):
        from .mw import inverse_batch
        return inverse_batch(values_local, self.L, spin)

    def forward(self, samples_local, spin):
        from .mw import forward_batch
        return forward_batch(samples_local, self.L, spin)

    def gather(self, local, group=None):
        """All-gather the per-rank blocks into the full batch (optional)."""
        if self.world == 1:
            return local
        sizes = [len(shard_maps(self.n, self.world, r)) for r in range(self.world)]
        out = [torch.empty((s,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
               for s in sizes]
        if _is_nccl(group):
            dist.all_gather(out, local.contiguous(), group=group)
        else:
            for r in range(self.world):
                buf = local.contiguous() if r == self.rank else out[r]
                dist.broadcast(buf, r, group=group)
                if r == self.rank:
                    out[r] = local
        return torch.cat(out, 0)
