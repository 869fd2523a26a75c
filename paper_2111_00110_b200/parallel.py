"""Data-parallel sharding of the explicit layer across GPUs.

Sources and queries are independent units: each rank owns a shard of the
sources (p, w) and of the queries (q, y_bar).  Per expansion there are two
exchange steps on the finest grids (NCCL over NVLink on B200s; gloo in the CPU
tests):

    M   = allreduce_r P2M(p_r, w_r)             full finest moments on every rank
    L_r = cascade(M) on the x-slab r             coarse levels replicated (cheap),
                                                 finest M2L only for x in slab r
    L   = allgather_r L_r                        slabs are contiguous (x is the
                                                 slowest grid axis)
    f(q_r), and in the backward the same with (q_r, y_r), then G(p_r), grad G(p_r)

The finest-level M2L is thus divided among the ranks instead of replicated;
the all-reduce provides every rank with the halo planes its slab's M2L reads.
Slabs are multiples of 4 cells (for the dense tensor-core kernel, two class
lattice planes; the separable form restricts its passes to the slab plus the
3-cell halo); when the grid does not split evenly the cascade falls back to
replication.  The compute backend is
any object with ``p2m_grid``, ``cascade_grid(m, x_range=None)``, ``evaluate``
(the device Engine adapter below; tests/test_parallel_gloo.py plugs the CPU
oracle in to check the sharding logic on CPU with world size 2).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of n units for a rank."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class DeviceBackend:
    """The B200 engine as a sharding backend (grids are device tensors).  Beyond
    the three methods every backend has, it offers the single-GPU layer's
    shortcuts (layers.py): the query cell sort started on the engine's aux
    stream in the forward, and q_bar recycled from the forward's grad f(q)."""

    def __init__(self, engine):
        self.engine = engine

    def p2m_grid(self, p: torch.Tensor, w: torch.Tensor, sort=None) -> torch.Tensor:
        return self.engine.p2m_device(p, w, sort).storage

    def early_sort(self, q: torch.Tensor):
        from .layers import EARLY_QUERY_SORT, _early_sort
        return _early_sort(self.engine, q) if EARLY_QUERY_SORT else (None, None)

    def evaluate_value_grad(self, L: torch.Tensor, pts: torch.Tensor):
        from .expansion import Accessor, ExpansionGrid
        eng = self.engine
        acc = Accessor(ExpansionGrid(eng.levels, "L", L, eng.rho), eng.table, eng.flops,
                       flag=eng.flag)
        out = acc.eval_device(pts, _lib.L2P_VALUE | _lib.L2P_GRAD)
        return out["value"], out["grad"]

    def weighted_grad(self, grad: torch.Tensor, wts: torch.Tensor) -> torch.Tensor:
        from .layers import _weighted_grad
        return _weighted_grad(grad, wts.reshape(grad.shape[0], -1))

    def cascade_grid(self, m: torch.Tensor, x_range: tuple | None = None) -> torch.Tensor:
        return self.engine.cascade_device(m, x_range)

    def evaluate(self, L: torch.Tensor, pts: torch.Tensor, wts: torch.Tensor | None, value: bool):
        from .expansion import Accessor, ExpansionGrid
        eng = self.engine
        acc = Accessor(ExpansionGrid(eng.levels, "L", L, eng.rho), eng.table, eng.flops,
                       flag=eng.flag)
        mode = (_lib.L2P_VALUE if value else 0) | (_lib.L2P_WGRAD if wts is not None else 0)
        out = acc.eval_device(pts, mode, wts=wts)
        return out["value"], out["wgrad"]


@dataclass
class ShardedExplicitResult:
    values: torch.Tensor     # (M_r, C) this rank's queries
    L: torch.Tensor
    q: torch.Tensor
    p: torch.Tensor
    w: torch.Tensor
    q_grad: torch.Tensor = None     # grad f(q_r), when the backend recycles it
    q_sort: object = None           # (CellSort, ready event) of q_r from the aux stream


def _allreduce(t: torch.Tensor, group) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def slab_range(res: int, rank: int, world: int) -> tuple[int, int] | None:
    """This rank's x-slab [x0, x1) of the finest grid, or None when res does
    not split into equal multiples of 4 cells."""
    if res % 4 or (res // 4) % world:
        return None
    width = res // world
    return rank * width, (rank + 1) * width


def _cascade(backend, m: torch.Tensor, group) -> torch.Tensor:
    """Finest L on every rank: each rank computes its x-slab, one all-gather."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return backend.cascade_grid(m)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    sl = slab_range(int(m.shape[0]), rank, world)
    if sl is None:
        return backend.cascade_grid(m)
    L = backend.cascade_grid(m, sl)
    mine = L[sl[0]:sl[1]]
    if dist.get_backend(group) != "nccl":
        mine = mine.clone()     # NCCL gathers in place; gloo wants a separate input
    dist.all_gather_into_tensor(L, mine, group=group)
    return L


def explicit_forward_sharded(backend, p, w, q, group=None) -> ShardedExplicitResult:
    """Forward of the explicit layer on this rank's shards (see module doc)."""
    q_sort = backend.early_sort(q) if hasattr(backend, "early_sort") else None
    m = _allreduce(backend.p2m_grid(p, w), group)
    L = _cascade(backend, m, group)
    q_grad = None
    if hasattr(backend, "evaluate_value_grad"):
        values, q_grad = backend.evaluate_value_grad(L, q)
    else:
        values, _ = backend.evaluate(L, q, None, True)
    return ShardedExplicitResult(values=values, L=L, q=q, p=p, w=w, q_grad=q_grad, q_sort=q_sort)


def explicit_jvp_sharded(backend, y_bar, res: ShardedExplicitResult, group=None):
    """(w_bar_r, p_bar_r, q_bar_r) for this rank's shards."""
    if res.q_grad is not None:
        q_bar = backend.weighted_grad(res.q_grad, y_bar)
    else:
        _, q_bar = backend.evaluate(res.L, res.q, y_bar, False)
    srt = None
    if res.q_sort is not None and res.q_sort[0] is not None:
        srt, ready = res.q_sort
        torch.cuda.current_stream().wait_event(ready)
    b = _allreduce(backend.p2m_grid(res.q, y_bar, srt) if srt is not None
                   else backend.p2m_grid(res.q, y_bar), group)
    G = _cascade(backend, b, group)
    w_bar, p_bar = backend.evaluate(G, res.p, res.w, True)
    return w_bar, p_bar, q_bar
