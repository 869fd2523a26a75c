"""Differentiable layers on the device engine: drop-in for ``fc2t2.layers``.

Every backward pass is exactly one extra expansion (reference
layers.py:1-22): the output tangent becomes an insertion over the target
geometry, one cascade smooths it, and w_bar = B(p), p_bar = w * grad B(p).
The pipeline is self-adjoint (K_l2l = K_m2m^T, A(-o) = A(o)^T), so the
backward reuses the forward kernels (SURVEY.md section 8(a) note 8).

Explicit layer (reference layers.py:158-188):
    forward   values = L2P(expand(p, w), q)
    jvp       q_bar = sum_c y_bar_c grad f_c(q)     (forward accessor, fused WGRAD L2P)
              B     = expand(q, y_bar)
              w_bar = B(p), p_bar = sum_c w_c grad B_c(p)   (one fused VALUE|WGRAD L2P)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .expansion import (Accessor, Engine, HostIO, SourceSet, _host_domain_check,
                        is_host_tensor, like_input, to_device)


@dataclass
class LayerGradients:
    """Parameter tangents of a layer JVP (reference layers.py:43-50)."""

    w_bar: object
    p_bar: object = None
    q_bar: object = None
    diagnostics: dict = field(default_factory=dict)


@dataclass
class ExplicitResult:
    """Reference layers.py:158-164; ``q`` is the caller's query array."""

    values: object
    accessor: Accessor
    q: object
    sources: SourceSet
    engine: Engine
    q_dev: torch.Tensor = None


def explicit_forward(engine: Engine, sources: SourceSet, q) -> ExplicitResult:
    _host_domain_check(q, "query")
    if is_host_tensor(q):
        # host tensors: the query upload overlaps the source expansion
        qd, q_ready = HostIO.h2d(q, 3)
        acc = engine.expand_device(sources.p, sources.w)
        torch.cuda.current_stream().wait_event(q_ready)
        vals = acc.eval_device(qd, _lib.L2P_VALUE)["value"]
        out = HostIO.d2h(vals)
        HostIO.finish()
        engine.flag.raise_if_set("source/query")
        return ExplicitResult(values=out, accessor=acc, q=q, sources=sources, engine=engine,
                              q_dev=qd)
    qd = to_device(q, 3, points=True)
    acc = engine.expand_device(sources.p, sources.w)
    vals = acc.eval_device(qd, _lib.L2P_VALUE)["value"]
    engine.flag.raise_if_set("source/query")
    return ExplicitResult(values=like_input(vals, q), accessor=acc, q=q, sources=sources,
                          engine=engine, q_dev=qd)


def explicit_jvp(y_bar, res: ExplicitResult) -> LayerGradients:
    eng = res.engine
    qd = res.q_dev
    src = res.sources
    if is_host_tensor(y_bar):
        # host tensors: q_bar's download overlaps the backward expansion
        yb, y_ready = HostIO.h2d(y_bar)
        torch.cuda.current_stream().wait_event(y_ready)
        yb = yb.reshape(qd.shape[0], -1)
        q_bar = res.accessor.eval_device(qd, _lib.L2P_WGRAD, wts=yb)["wgrad"]
        q_bar_h = HostIO.d2h(q_bar)
        back = eng.expand_device(qd, yb)
        out = back.eval_device(src.p, _lib.L2P_VALUE | _lib.L2P_WGRAD, wts=src.w)
        w_bar_h, p_bar_h = HostIO.d2h(out["value"]), HostIO.d2h(out["wgrad"])
        HostIO.finish()
        eng.flag.raise_if_set("source/query")
        return LayerGradients(w_bar=w_bar_h, p_bar=p_bar_h, q_bar=q_bar_h)
    yb = to_device(y_bar).reshape(qd.shape[0], -1).contiguous()
    q_bar = res.accessor.eval_device(qd, _lib.L2P_WGRAD, wts=yb)["wgrad"]
    back = eng.expand_device(qd, yb)
    out = back.eval_device(src.p, _lib.L2P_VALUE | _lib.L2P_WGRAD, wts=src.w)
    eng.flag.raise_if_set("source/query")
    ref = y_bar
    return LayerGradients(w_bar=like_input(out["value"], ref), p_bar=like_input(out["wgrad"], ref),
                          q_bar=like_input(q_bar, ref))
