"""CUDA-graph replay of a layer step (the B200 answer to launch-bound small
configurations, e.g. BASELINE config 1: ~45 kernels for 8192 points).

The explicit layer's forward + JVP (layers.explicit_forward / explicit_jvp,
reference layers.py:167-188) is captured once for fixed shapes on device
tensors and replayed: inputs are copied into the graph's static buffers, the
whole kernel sequence -- sorts, P2M, the cascade with its side-stream fork/join,
L2P -- replays as one graph launch, and the domain flag (zeroed inside the
graph) is read once per replay, raising DomainError like the eager path.
Replays are bit-identical to eager calls (same kernels, same inputs).
"""

from __future__ import annotations

import torch

from .expansion import DomainError, Engine, SourceSet
from .layers import explicit_forward, explicit_jvp


class GraphedExplicit:
    """Replayable explicit-layer step for fixed (N, M, C).

    step = GraphedExplicit(engine, p, w, q, y_bar)   # captures (device tensors)
    values, w_bar, p_bar, q_bar = step(p, w, q, y_bar)

    Outputs are the graph's static tensors: clone them to keep a result past
    the next replay.  Engine counters (expansion_count, flops) advance once at
    capture, not per replay.
    """

    def __init__(self, engine: Engine, p: torch.Tensor, w: torch.Tensor, q: torch.Tensor,
                 y_bar: torch.Tensor, warmup: int = 2):
        for t in (p, w, q, y_bar):
            if not (isinstance(t, torch.Tensor) and t.is_cuda):
                raise TypeError("GraphedExplicit captures device tensors")
        self.engine = engine
        self.p = p.detach().clone().contiguous()
        self.w = w.detach().clone().reshape(p.shape[0], -1).contiguous()
        self.q = q.detach().clone().contiguous()
        self.y = y_bar.detach().clone().reshape(q.shape[0], -1).contiguous()
        _ = engine.handle          # uploads the tables and creates the domain flag
        flag = engine.flag
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side), flag.deferred():
            for _ in range(warmup):          # allocator warm-up outside the graph
                self._step()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        flag.t.zero_()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph), flag.deferred():
            flag.t.zero_()
            self.out = self._step()
        torch.cuda.synchronize()

    def _step(self):
        res = explicit_forward(self.engine, SourceSet(self.p, self.w), self.q)
        g = explicit_jvp(self.y, res)
        return res.values, g.w_bar, g.p_bar, g.q_bar

    def __call__(self, p=None, w=None, q=None, y_bar=None, check: bool = True):
        """Copy new inputs (any may be omitted to keep the previous ones),
        replay, and return (values, w_bar, p_bar, q_bar)."""
        for dst, src in ((self.p, p), (self.w, w), (self.q, q), (self.y, y_bar)):
            if src is not None:
                dst.copy_(src.reshape(dst.shape), non_blocking=True)
        self.graph.replay()
        if check:
            self.engine.flag.raise_if_set("source/query")
        return self.out
