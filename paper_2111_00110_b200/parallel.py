"""Data-parallel sharding of the FC2T2 layers across GPUs.

Sources, queries and rays are independent units: each rank owns a shard of
the sources (p, w) and of the targets (queries q, or rays).  The one exchange
step is the finest coefficient grid.  For every expansion (the forward's and
the backward's), with the finest grid split into x-slabs (x is the slowest
grid axis, so a slab is contiguous; res / world cells each):

    M_r     = P2M(p_r, w_r)                      full-size partial moments
    M[slab] = reduce_scatter_r M_r               in place: rank r's slab summed
    halo    = 3 planes either side from the      the finest M2L reach
              neighbouring ranks (send/recv)     (ref kernel.py:39), overlapped
                                                 with the M2M chain below
    up      : M2M chain on the slab only; every coarse M level all-gathered
              in place (1/7 of the finest grid in total)
    down    : M2L + L2L on the slab at every level (tcgen05 / separable /
              FFMA kernels restricted to x-slabs), finest L on the slab
    L       = all_gather_r L[slab]               in place
    then every rank evaluates its own queries / rays / sources (no exchange).

No cascade level is replicated when the slab maps to whole cells at every
level (fc2t2_expand_slab_split); otherwise the cascade falls back to one
all-reduce of M and the slab cascade with full coarse levels (still no
replicated finest M2L).  Multi-GPU results differ from one GPU only by the
reassociation of the moment sums.

Two entry points:
  * ``sharded(engine, group)`` -- a context under which every layer of
    layers.py (explicit, depth / surface-gradient, line integral, radiance)
    called on this rank's shards runs its expansions through the sharded
    cascade and raises DomainError on every rank when any rank saw an
    out-of-domain point (the flag is max-reduced);
  * ``explicit_forward_sharded / explicit_jvp_sharded`` -- the explicit layer
    against any backend (tests/test_parallel_gloo.py plugs the CPU oracle in).

Collectives run over NCCL (NVLink) for CUDA tensors; a gloo group (CPU tests,
or several processes sharing one GPU) stages device tensors through the host.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib

REACH = 3   # finest-level M2L reach in cells (ref kernel.py:39, FAR_REACH)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of n units for a rank."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def slab_range(res: int, rank: int, world: int) -> tuple[int, int] | None:
    """This rank's x-slab [x0, x1) of the finest grid, or None when res does
    not split into equal multiples of 4 cells."""
    if res % 4 or (res // 4) % world:
        return None
    width = res // world
    return rank * width, (rank + 1) * width


# ------------------------------------------------------------ collectives ---

class Comm:
    """The collectives of the sharded cascade on one process group.  NCCL
    groups work in place on device tensors; gloo groups stage CUDA tensors
    through host memory (correctness path for CPU tests / shared GPUs)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def _host(self, t: torch.Tensor) -> bool:
        return (not self.nccl) and t.is_cuda

    def all_reduce(self, t: torch.Tensor, op=dist.ReduceOp.SUM) -> torch.Tensor:
        if self._host(t):
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)
        return t

    def reduce_scatter_slab(self, t: torch.Tensor) -> None:
        """t[slab_r] <- sum over ranks of t[slab_r] (the rest of t keeps this
        rank's own partial values)."""
        w = t.shape[0] // self.world
        mine = t[self.rank * w:(self.rank + 1) * w]
        if self._host(t):
            out = torch.empty(mine.shape, dtype=t.dtype)
            dist.reduce_scatter_tensor(out, t.cpu(), group=self.group)
            mine.copy_(out)
        elif self.nccl:
            dist.reduce_scatter_tensor(mine, t, group=self.group)     # in place
        else:
            out = torch.empty_like(mine)
            dist.reduce_scatter_tensor(out, t, group=self.group)
            mine.copy_(out)

    def all_gather_slabs(self, t: torch.Tensor) -> None:
        """t's first axis in `world` equal slabs; every rank fills in the others'."""
        w = t.shape[0] // self.world
        mine = t[self.rank * w:(self.rank + 1) * w]
        if self._host(t):
            full = torch.empty(t.shape, dtype=t.dtype)
            dist.all_gather_into_tensor(full, mine.cpu(), group=self.group)
            t.copy_(full)
        elif self.nccl:
            dist.all_gather_into_tensor(t, mine, group=self.group)     # in place
        else:
            dist.all_gather_into_tensor(t, mine.clone(), group=self.group)

    def halo(self, t: torch.Tensor, x0: int, x1: int, reach: int):
        """Start the exchange of `reach` planes with the x-neighbours: receive
        t[x0-reach:x0] and t[x1:x1+reach]; returns a handle for ``wait``."""
        res = t.shape[0]
        ops, posts = [], []
        host = self._host(t)

        def buf(view):
            return view.cpu() if host else view.contiguous()
        if x0 > 0:
            lo = max(0, x0 - reach)
            r = torch.empty(t[lo:x0].shape, dtype=t.dtype, device="cpu" if host else t.device)
            ops.append(dist.P2POp(dist.isend, buf(t[x0:x0 + (x0 - lo)]), self._peer(-1),
                                  self.group))
            ops.append(dist.P2POp(dist.irecv, r, self._peer(-1), self.group))
            posts.append((lo, x0, r))
        if x1 < res:
            hi = min(res, x1 + reach)
            r = torch.empty(t[x1:hi].shape, dtype=t.dtype, device="cpu" if host else t.device)
            ops.append(dist.P2POp(dist.isend, buf(t[x1 - (hi - x1):x1]), self._peer(1),
                                  self.group))
            ops.append(dist.P2POp(dist.irecv, r, self._peer(1), self.group))
            posts.append((x1, hi, r))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return reqs, posts, t

    def _peer(self, d: int) -> int:
        r = self.rank + d
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    @staticmethod
    def wait(handle) -> None:
        reqs, posts, t = handle
        for r in reqs:
            r.wait()
        for lo, hi, r in posts:
            t[lo:hi].copy_(r)


# --------------------------------------------------------- sharded cascade ---

def sharded_cascade(be, m: torch.Tensor, comm: Comm) -> torch.Tensor:
    """Finest L on every rank from this rank's partial finest moments m (full
    size; overwritten).  ``be`` provides cascade(m, x_range), slab_split_ok(x0,
    x1), cascade_up(m, x_range) -> ws, coarse_views(ws) -> [(level, grid
    view)] and cascade_down(m, ws, x_range) -> L (DeviceBackend below; the CPU
    tests plug an oracle adapter in)."""
    if comm.world == 1:
        return be.cascade(m)
    res = int(m.shape[0])
    sl = slab_range(res, comm.rank, comm.world)
    if sl is None:
        return be.cascade(comm.all_reduce(m))            # replicated (res not divisible)
    x0, x1 = sl
    if not be.slab_split_ok(x0, x1):
        L = be.cascade(comm.all_reduce(m), sl)
        comm.all_gather_slabs(L)
        return L
    comm.reduce_scatter_slab(m)
    h = comm.halo(m, x0, x1, REACH)
    ws = be.cascade_up(m, sl)                             # overlaps the halo traffic
    for _lvl, view in be.coarse_views(ws):
        comm.all_gather_slabs(view)
    comm.wait(h)
    L = be.cascade_down(m, ws, sl)
    comm.all_gather_slabs(L)
    return L


class DeviceBackend:
    """The B200 engine as a sharding backend (grids are device tensors)."""

    def __init__(self, engine):
        self.engine = engine
        self.levels = engine.levels

    # -- cascade pieces (C ABI fc2t2_expand_slab / _up / _down) --
    def cascade(self, m: torch.Tensor, x_range=None) -> torch.Tensor:
        return self.engine._cascade_raw(m, x_range)

    def slab_split_ok(self, x0: int, x1: int) -> bool:
        return bool(_lib.lib().fc2t2_expand_slab_split(self.engine.handle, x0, x1))

    def cascade_up(self, m: torch.Tensor, x_range):
        return self.engine.cascade_up(m, x_range)

    def coarse_views(self, ws):
        return self.engine.coarse_views(ws)

    def cascade_down(self, m: torch.Tensor, ws, x_range) -> torch.Tensor:
        return self.engine.cascade_down(m, ws, x_range)

    # -- the explicit layer's point stages --
    def p2m_grid(self, p: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        return self.engine.p2m_device(p, w).storage

    def evaluate_value_grad(self, L: torch.Tensor, pts: torch.Tensor):
        out = self._acc(L).eval_device(pts, _lib.L2P_VALUE | _lib.L2P_GRAD)
        return out["value"], out["grad"]

    def weighted_grad(self, grad: torch.Tensor, wts: torch.Tensor) -> torch.Tensor:
        from .layers import _weighted_grad
        return _weighted_grad(grad, wts.reshape(grad.shape[0], -1))

    def evaluate(self, L: torch.Tensor, pts: torch.Tensor, wts: torch.Tensor | None, value: bool):
        mode = (_lib.L2P_VALUE if value else 0) | (_lib.L2P_WGRAD if wts is not None else 0)
        out = self._acc(L).eval_device(pts, mode, wts=wts)
        return out["value"], out["wgrad"]

    def raise_if_set(self, what: str, group=None) -> None:
        """DomainError on every rank when any rank's point kernels flagged an
        out-of-domain point (the flag is max-reduced over the ranks)."""
        flag = self.engine.flag
        prev = flag.reduce_hook
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            flag.reduce_hook = _flag_reducer(flag, Comm(group), group)
        try:
            flag.raise_if_set(what)
        finally:
            flag.reduce_hook = prev

    def _acc(self, L):
        from .expansion import Accessor, ExpansionGrid
        eng = self.engine
        return Accessor(ExpansionGrid(eng.levels, "L", L, eng.rho), eng.table, eng.flops,
                        flag=eng.flag)


def _flag_reducer(flag, comm: Comm, group):
    def reduce_flag(v: int) -> int:
        t = torch.tensor([int(v)], dtype=torch.int32, device=flag.t.device if comm.nccl else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return int(t.item())
    return reduce_flag


@contextmanager
def sharded(engine, group=None):
    """Run the layers of layers.py on this rank's shards: every expansion goes
    through ``sharded_cascade`` and the domain flag is max-reduced over the
    ranks before it is read (all ranks raise together).  Every rank must make
    the same sequence of layer calls (SPMD)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        yield engine
        return
    comm = Comm(group)
    be = DeviceBackend(engine)
    _ = engine.handle
    prev = (engine._cascade_hook, engine.flag.reduce_hook)
    engine._cascade_hook = lambda m: sharded_cascade(be, m, comm)
    engine.flag.reduce_hook = _flag_reducer(engine.flag, comm, group)
    try:
        yield engine
    finally:
        engine._cascade_hook, engine.flag.reduce_hook = prev


# ------------------------------------------- explicit layer, generic backend ---

@dataclass
class ShardedExplicitResult:
    values: torch.Tensor     # (M_r, C) this rank's queries
    L: torch.Tensor
    q: torch.Tensor
    p: torch.Tensor
    w: torch.Tensor
    q_grad: torch.Tensor = None     # grad f(q_r), when the backend recycles it


def _cascade(backend, m: torch.Tensor, group) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        return sharded_cascade(backend, m, Comm(group))
    return backend.cascade(m)


def explicit_forward_sharded(backend, p, w, q, group=None) -> ShardedExplicitResult:
    """Forward of the explicit layer on this rank's shards (see module doc)."""
    L = _cascade(backend, backend.p2m_grid(p, w), group)
    q_grad = None
    if hasattr(backend, "evaluate_value_grad"):
        values, q_grad = backend.evaluate_value_grad(L, q)
    else:
        values, _ = backend.evaluate(L, q, None, True)
    if hasattr(backend, "raise_if_set"):
        backend.raise_if_set("source/query", group)
    return ShardedExplicitResult(values=values, L=L, q=q, p=p, w=w, q_grad=q_grad)


def explicit_jvp_sharded(backend, y_bar, res: ShardedExplicitResult, group=None):
    """(w_bar_r, p_bar_r, q_bar_r) for this rank's shards."""
    if res.q_grad is not None:
        q_bar = backend.weighted_grad(res.q_grad, y_bar)
    else:
        _, q_bar = backend.evaluate(res.L, res.q, y_bar, False)
    G = _cascade(backend, backend.p2m_grid(res.q, y_bar), group)
    w_bar, p_bar = backend.evaluate(G, res.p, res.w, True)
    if hasattr(backend, "raise_if_set"):
        backend.raise_if_set("source/query", group)
    return w_bar, p_bar, q_bar
