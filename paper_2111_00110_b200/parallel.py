"""Data-parallel sharding of the explicit layer across GPUs.

Sources and queries are independent units: each rank owns a shard of the
sources (p, w) and of the queries (q, y_bar).  The only exchange step is the
finest moment grid -- each rank's P2M of its shard is summed with one
all-reduce (NCCL over NVLink on B200s; gloo in the CPU tests) -- after which
every rank holds the global field and evaluates its own queries / sources with
no further communication:

    forward   M_r = P2M(p_r, w_r);  M = allreduce(M_r);  L = cascade(M);  f(q_r)
    backward  B_r = P2M(q_r, y_r);  B = allreduce(B_r);  G = cascade(B);
              w_bar_r = G(p_r),  p_bar_r = w_r grad G(p_r),  q_bar_r = y_r grad f(q_r)

The cascade is replicated (per-GPU work constant under weak scaling; the
all-reduce of 37.7 MB at config 2 costs ~0.1 ms over NVLink).  The compute
backend is any object with ``p2m_grid``, ``cascade_grid``, ``evaluate`` (the
device Engine adapter below; tests/test_parallel_gloo.py plugs the CPU oracle
in to check the sharding logic on CPU with world size 2).
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
    """The B200 engine as a sharding backend (grids are device tensors)."""

    def __init__(self, engine):
        self.engine = engine

    def p2m_grid(self, p: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
        return self.engine.p2m_device(p, w).storage

    def cascade_grid(self, m: torch.Tensor) -> torch.Tensor:
        return self.engine.cascade_device(m)

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


def _allreduce(t: torch.Tensor, group) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def explicit_forward_sharded(backend, p, w, q, group=None) -> ShardedExplicitResult:
    """Forward of the explicit layer on this rank's shards (see module doc)."""
    m = _allreduce(backend.p2m_grid(p, w), group)
    L = backend.cascade_grid(m)
    values, _ = backend.evaluate(L, q, None, True)
    return ShardedExplicitResult(values=values, L=L, q=q, p=p, w=w)


def explicit_jvp_sharded(backend, y_bar, res: ShardedExplicitResult, group=None):
    """(w_bar_r, p_bar_r, q_bar_r) for this rank's shards."""
    _, q_bar = backend.evaluate(res.L, res.q, y_bar, False)
    b = _allreduce(backend.p2m_grid(res.q, y_bar), group)
    G = backend.cascade_grid(b)
    w_bar, p_bar = backend.evaluate(G, res.p, res.w, True)
    return w_bar, p_bar, q_bar
