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
    orders, all-gather of the (disjoint) packed coefficient blocks.
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


def order_owner(L, bounds, k):
    """Rank owning bin k (order m = k for k < L, k - N otherwise)."""
    N = 2 * L - 1
    am = k if k < L else N - k
    return int(np.searchsorted(bounds, am, side="right") - 1)


def shard_flm_base(l, m0, m1):
    """Offset of degree l in an order-range shard's packed coefficient block
    (numpy mirror of common.cuh shard_flm_base); l = L gives the block size."""
    k = np.clip(np.asarray(l) - m0, 0, m1 - m0)
    s1 = k * (k + 1) // 2 + (m1 - m0) * np.maximum(np.asarray(l) - m1, 0)
    return 2 * s1 - (np.asarray(l) if m0 == 0 else 0)


def shard_flm_index(l, m, m0, m1):
    """Position of (l, m) in the packed block (common.cuh shard_flm_index)."""
    l, m = np.asarray(l), np.asarray(m)
    hi = np.minimum(l, m1 - 1)
    mn = max(m0, 1)
    b = shard_flm_base(l, m0, m1)
    return np.where(m < 0, b + (m + hi), b + (hi - mn + 1) + (m - m0))


class ExchangeLayout:
    """Offset tables of the all-to-all buffers of one rank (include/mwsht.h,
    m-column / ring sharding).  Every buffer is shard-sized: the send and
    receive blocks of each peer are contiguous, and the stage kernels read
    and write them in place (no gather/scatter pass around the collective).

    forward:  send block to q = q's order rows x my rings   (row-major, nt[me] wide)
              recv block from r = my order rows x r's rings (row-major, nt[r] wide)
    inverse:  send block to q = q's rings x my order rows   (ring-major, nrow[me] wide)
              recv block from r = my rings x r's order rows (ring-major, nrow[r] wide)
    """

    def __init__(self, L, bounds, tb, rank):
        N = 2 * L - 1
        world = len(bounds) - 1
        self.L, self.N, self.world, self.rank = L, N, world, rank
        rows = [order_bins(L, bounds[q], bounds[q + 1]) for q in range(world)]
        nrow = [len(r) for r in rows]
        nt = [tb[q + 1] - tb[q] for q in range(world)]
        local = np.empty(N, dtype=np.int64)    # bin -> local row index in its owner's order
        owner = np.empty(N, dtype=np.int64)
        for q in range(world):
            local[rows[q]] = np.arange(nrow[q])
            owner[rows[q]] = q
        ring_owner = np.concatenate([np.full(nt[q], q) for q in range(world)])
        me = rank

        def offsets(counts):
            return [int(x) for x in np.concatenate([[0], np.cumsum(counts)[:-1]])]

        self.fsend_counts = [nrow[q] * nt[me] for q in range(world)]
        self.frecv_counts = [nrow[me] * nt[r] for r in range(world)]
        self.isend_counts = [nt[q] * nrow[me] for q in range(world)]
        self.irecv_counts = [nt[me] * nrow[r] for r in range(world)]
        fso, fro = offsets(self.fsend_counts), offsets(self.frecv_counts)
        iso, iro = offsets(self.isend_counts), offsets(self.irecv_counts)
        t = np.arange(L)
        n = np.arange(N)
        # forward phi (send): bin k, my ring t -> fso[q(k)] + i(k) * nt[me] + (t - t0)
        self.fphi_row_off = np.array([fso[q] for q in owner], dtype=np.int64) + local * nt[me]
        # forward theta (recv): my row i, ring t -> fro[r(t)] + (t - tb[r]) + i * nt[r(t)]
        self.ftheta_col_off = (np.array([fro[r] for r in ring_owner], dtype=np.int64)
                               + t - np.array([tb[r] for r in ring_owner]))
        self.ftheta_col_stride = np.array([nt[r] for r in ring_owner], dtype=np.int32)
        # inverse theta (send): ring t, my row i -> iso[q(t)] + (t - tb[q]) * nrow[me] + i
        self.itheta_row_off = (np.array([iso[q] for q in ring_owner], dtype=np.int64)
                               + (t - np.array([tb[q] for q in ring_owner])) * nrow[me])
        # inverse phi (recv): my ring t, bin n -> iro[r(n)] + j(n) + (t - t0) * nrow[r(n)]
        self.iphi_col_off = np.array([iro[r] for r in owner], dtype=np.int64) + local[n]
        self.iphi_col_stride = np.array([nrow[r] for r in owner], dtype=np.int32)
        self.flm_len = [int(shard_flm_base(L, bounds[q], bounds[q + 1])) for q in range(world)]
        self.flm_maxlen = max(self.flm_len)


# -------------------------------------------------------------- exchange

def _is_nccl(group=None):
    return dist.is_initialized() and dist.get_backend(group) == "nccl"


def all_to_all_flat(send, send_counts, recv, recv_counts, group=None):
    """Variable-size all-to-all of contiguous blocks of 1-D complex buffers:
    send[sum(send_counts[:q]) : +send_counts[q]] goes to rank q.  NCCL works on
    device buffers directly (complex128 as float64 pairs); gloo stages through
    host memory with pairwise send/recv."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        recv.copy_(send)
        return recv
    if _is_nccl(group):
        dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send),
                               output_split_sizes=list(recv_counts),
                               input_split_sizes=list(send_counts), group=group)
        return recv
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    hs = torch.view_as_real(send).cpu()
    hr = torch.empty((recv.numel(), 2), dtype=torch.float64)
    so = np.concatenate([[0], np.cumsum(send_counts)]).astype(int)
    ro = np.concatenate([[0], np.cumsum(recv_counts)]).astype(int)
    reqs = []
    for k in range(1, world):
        dst, src = (rank + k) % world, (rank - k) % world
        reqs.append(dist.isend(hs[so[dst]:so[dst + 1]].contiguous(), dst, group=group))
        reqs.append(dist.irecv(hr[ro[src]:ro[src + 1]], src, group=group))
    hr[ro[rank]:ro[rank + 1]] = hs[so[rank]:so[rank + 1]]
    for r in reqs:
        r.wait()
    torch.view_as_real(recv).copy_(hr)
    return recv


def all_gather_flat(block, out, group=None):
    """out (world * len(block),) <- every rank's block (complex 1-D)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        out.copy_(block)
        return out
    if _is_nccl(group):
        dist.all_gather_into_tensor(torch.view_as_real(out), torch.view_as_real(block),
                                    group=group)
        return out
    world = dist.get_world_size(group)
    parts = [torch.empty((block.numel(), 2), dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.view_as_real(block).cpu().contiguous(), group=group)
    torch.view_as_real(out).copy_(torch.cat(parts, 0))
    return out


# ----------------------------------------------------- GPU shard drivers

class MColumnSharding:
    """One complex map split over `world` ranks by order columns and rings.

    forward(samples_rows, spin): this rank's rings (t1-t0, N) -> full flm (L^2,)
    on every rank.  inverse(flm, spin): full flm on every rank -> this rank's
    rings.  Per transform: the stage kernels write/read the shard-sized
    all-to-all buffers in place (ExchangeLayout), one all-to-all, and for the
    forward an all-gather of the packed coefficient blocks (each rank owns
    disjoint orders) unpacked by one kernel."""

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
        lay = self.layout = ExchangeLayout(L, self.bounds, self.tb, rank)
        dev = self.device

        def t(x):
            return torch.from_numpy(np.ascontiguousarray(x)).to(dev)

        self.fphi_row_off = t(lay.fphi_row_off)
        self.ftheta_col_off, self.ftheta_col_stride = t(lay.ftheta_col_off), t(lay.ftheta_col_stride)
        self.itheta_row_off = t(lay.itheta_row_off)
        self.iphi_col_off, self.iphi_col_stride = t(lay.iphi_col_off), t(lay.iphi_col_stride)
        self.bounds_dev = t(np.array(self.bounds, dtype=np.int32))
        c128 = dict(dtype=torch.complex128, device=dev)
        self.fsend = torch.empty(sum(lay.fsend_counts), **c128)
        self.frecv = torch.empty(sum(lay.frecv_counts), **c128)
        self.isend = torch.empty(sum(lay.isend_counts), **c128)
        self.irecv = torch.empty(sum(lay.irecv_counts), **c128)
        self.block = torch.zeros(lay.flm_maxlen, **c128)
        self.gathered = torch.empty(world * lay.flm_maxlen, **c128)
        self.launches = 0

    def _st(self):
        return _lib._P(torch.cuda.current_stream(self.device).cuda_stream)

    def _count(self):
        self.launches += self.plan.last_launches()

    def forward(self, samples_rows, spin):
        P = self.plan.handle
        _lib.check(self.lib.mwsht_shard_forward_phi(
            P, samples_rows.data_ptr(), self.t0, self.t1, self.fphi_row_off.data_ptr(),
            self.fsend.data_ptr(), self._st()), "shard_forward_phi")
        self._count()
        all_to_all_flat(self.fsend, self.layout.fsend_counts, self.frecv,
                        self.layout.frecv_counts, self.group)
        _lib.check(self.lib.mwsht_shard_forward_rest(
            P, self.frecv.data_ptr(), self.m0, self.m1, self.ftheta_col_off.data_ptr(),
            self.ftheta_col_stride.data_ptr(), int(spin), self.block.data_ptr(), 1, self._st()),
            "shard_forward_rest")
        self._count()
        all_gather_flat(self.block, self.gathered, self.group)
        flm = torch.empty(self.L * self.L, dtype=torch.complex128, device=self.device)
        _lib.check(self.lib.mwsht_shard_unpack_flm(
            P, self.gathered.data_ptr(), self.layout.flm_maxlen, self.bounds_dev.data_ptr(),
            self.world, flm.data_ptr(), self._st()), "shard_unpack_flm")
        self._count()
        return flm

    def inverse(self, flm, spin):
        P = self.plan.handle
        _lib.check(self.lib.mwsht_shard_inverse_front(
            P, flm.data_ptr(), self.m0, self.m1, int(spin), self.itheta_row_off.data_ptr(),
            self.isend.data_ptr(), self._st()), "shard_inverse_front")
        self._count()
        all_to_all_flat(self.isend, self.layout.isend_counts, self.irecv,
                        self.layout.irecv_counts, self.group)
        out = torch.empty((self.t1 - self.t0, self.N), dtype=torch.complex128, device=self.device)
        _lib.check(self.lib.mwsht_shard_inverse_phi(
            P, self.irecv.data_ptr(), self.t0, self.t1, self.iphi_col_off.data_ptr(),
            self.iphi_col_stride.data_ptr(), out.data_ptr(), self._st()), "shard_inverse_phi")
        self._count()
        return out


def emulate_mcolumn(L, world, spin, flm, device=0):
    """Run the m-column-sharded inverse and forward of one map as `world`
    virtual ranks in one process, with the dense single-GPU layouts (NULL
    offset tables: AT (N+1) x L in bin pairs, OUT L x N) shared by the virtual ranks instead of
    an exchange.  Validates the order/ring range logic of the shard stages."""
    from .mw import get_plan
    lib = _lib.load()
    plan = get_plan(L, device)
    st = _lib._P(torch.cuda.current_stream(device).cuda_stream)
    bounds, tb = balanced_m_splits(L, world), ring_splits(L, world)
    N = 2 * L - 1
    dev = f"cuda:{device}"
    OUT = torch.empty((L, N), dtype=torch.complex128, device=dev)
    for r in range(world):  # each writes its own order columns of the shared OUT
        _lib.check(lib.mwsht_shard_inverse_front(plan.handle, flm.data_ptr(), bounds[r],
                                                 bounds[r + 1], int(spin), None, OUT.data_ptr(),
                                                 st), "shard_inverse_front")
    samples = torch.empty((L, N), dtype=torch.complex128, device=dev)
    for r in range(world):
        _lib.check(lib.mwsht_shard_inverse_phi(plan.handle, OUT.data_ptr(), tb[r], tb[r + 1],
                                               None, None, samples[tb[r]].data_ptr(), st),
                   "shard_inverse_phi")
    AT = torch.empty((N + 1, L), dtype=torch.complex128, device=dev)  # bins in pairs (mwsht.h)
    for r in range(world):
        rows = samples[tb[r]:tb[r + 1]].contiguous()
        _lib.check(lib.mwsht_shard_forward_phi(plan.handle, rows.data_ptr(), tb[r], tb[r + 1],
                                               None, AT.data_ptr(), st), "shard_forward_phi")
    flm_out = torch.zeros(L * L, dtype=torch.complex128, device=dev)
    for r in range(world):
        part = torch.zeros(L * L, dtype=torch.complex128, device=dev)
        _lib.check(lib.mwsht_shard_forward_rest(plan.handle, AT.data_ptr(), bounds[r],
                                                bounds[r + 1], None, None, int(spin),
                                                part.data_ptr(), 0, st), "shard_forward_rest")
        flm_out += part
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
