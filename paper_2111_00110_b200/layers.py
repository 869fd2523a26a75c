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
from .expansion import (Accessor, Engine, ExpansionGrid, HostIO, SourceSet, _host_domain_check,
                        _ptr, _stream, is_host_tensor, like_input, to_device)
from .kernel import level_resolution
from .multiindex import ROOT_MAX_ORDER, OrderError
from .ray import RayBundle, segment_offsets


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
    q_grad: torch.Tensor = None   # (M, C, 3) grad f at q, stored for the backward
    q_ready: object = None        # event: q_dev valid (the backward partitions q early)


# q_bar recycling ("expansion recycling"): the forward L2P at q
# also returns grad f(q) -- the same cell-row gather, 12 B more per point and
# channel written -- so explicit_jvp forms q_bar = sum_c y_bar_c grad f_c
# (fc2t2_weighted_grad, bit-identical to an L2P_WGRAD pass) instead of
# gathering every query's cell row a second time.

def _weighted_grad(grad: torch.Tensor, wts: torch.Tensor, out: torch.Tensor | None = None
                   ) -> torch.Tensor:
    n, C = int(grad.shape[0]), int(grad.shape[1])
    if out is None:
        out = torch.empty((n, 3), dtype=torch.float32, device=grad.device)
    _lib.call("fc2t2_weighted_grad", _ptr(grad), _ptr(wts.contiguous()), n, C, _ptr(out), _stream())
    return out


def _expand_checked(engine: Engine, p: torch.Tensor, w: torch.Tensor) -> tuple:
    """(accessor, mark): P2M of (p, w) -- whose partition pass checks p's
    domain -- then the flag mark, then the cascade, so raise_if_set(mark)
    waits only for the checking kernels and the host can enqueue the rest."""
    m = engine.p2m_device(p, w)
    checked = engine.flag.mark()
    return engine.accessor_from_moments(m.storage), checked


# Host-tensor callers: the per-point streams (q, y_bar up; values, q_bar down)
# move in HOST_CHUNKS row chunks so PCIe uploads, downloads (separate streams,
# both directions at once) and the L2P of finished chunks overlap each other
# and the expansions.
HOST_CHUNKS = 8


def _explicit_forward_host(engine: Engine, sources: SourceSet, q) -> ExplicitResult:
    qd, chunks = HostIO.h2d(q, 3, chunks=HOST_CHUNKS)
    acc = engine.expand_device(sources.p, sources.w)
    cs = torch.cuda.current_stream()
    out = torch.empty((qd.shape[0], acc.channels), dtype=torch.float32, pin_memory=True)
    q_grad = torch.empty((qd.shape[0], acc.channels, 3), dtype=torch.float32, device=qd.device)
    for a, b, ev in chunks:
        cs.wait_event(ev)
        if b > a:
            r = acc.eval_device(qd[a:b], _lib.L2P_VALUE | _lib.L2P_GRAD, outs={"grad": q_grad[a:b]})
            HostIO.d2h(r["value"], out[a:b])
    HostIO.finish()
    engine.flag.raise_if_set("source/query")
    return ExplicitResult(values=out, accessor=acc, q=q, sources=sources, engine=engine, q_dev=qd,
                          q_grad=q_grad)


def _recycled_qbar_host(y_bar, res: ExplicitResult):
    """Upload y_bar chunk by chunk and, right behind each chunk, form and
    download its q_bar rows from the stored gradient -- the first download
    starts as soon as the first chunk lands (the PCIe-bound backward's
    critical path is upload chunk 1 -> download of all of q_bar)."""
    cs = torch.cuda.current_stream()
    up, _ = HostIO._pair()
    C = res.accessor.channels
    src = y_bar if y_bar.is_pinned() else y_bar.pin_memory()
    src = src.reshape(-1, C)
    n = int(src.shape[0])
    yb = torch.empty((n, C), dtype=torch.float32, device=res.q_dev.device)
    qb_dev = torch.empty((n, 3), dtype=torch.float32, device=res.q_dev.device)
    q_bar = torch.empty((n, 3), dtype=torch.float32, pin_memory=True)
    k = max(1, min(HOST_CHUNKS, n)) if n else 1
    bounds = [(n * i) // k for i in range(k + 1)]
    for a, b in zip(bounds[:-1], bounds[1:]):
        if b <= a:
            continue
        with torch.cuda.stream(up):
            yb[a:b].copy_(src[a:b], non_blocking=True)
            ev = up.record_event()
        cs.wait_event(ev)
        HostIO.d2h(_weighted_grad(res.q_grad[a:b], yb[a:b], out=qb_dev[a:b]), q_bar[a:b])
    yb.record_stream(up)
    return yb, q_bar


def _explicit_jvp_host(y_bar, res: ExplicitResult) -> LayerGradients:
    eng, qd, src = res.engine, res.q_dev, res.sources
    yb, q_bar = _recycled_qbar_host(y_bar, res)
    back = eng.expand_device(qd, yb)
    out = back.eval_device(src.p, _lib.L2P_VALUE | _lib.L2P_WGRAD, wts=src.w)
    w_bar, p_bar = HostIO.d2h(out["value"]), HostIO.d2h(out["wgrad"])
    HostIO.finish()
    eng.flag.raise_if_set("source/query")
    return LayerGradients(w_bar=w_bar, p_bar=p_bar, q_bar=q_bar)


def explicit_forward(engine: Engine, sources: SourceSet, q) -> ExplicitResult:
    _host_domain_check(q, "query")
    if is_host_tensor(q):
        return _explicit_forward_host(engine, sources, q)
    qd = to_device(q, 3, points=True)
    # the query domain check overlaps the source P2M (aux stream); the
    # caller's stream joins it before the flag mark
    cs = torch.cuda.current_stream()
    aux = engine.aux_stream()
    aux.wait_stream(cs)
    q_ready = cs.record_event()
    with torch.cuda.stream(aux):
        engine.flag.check_points(qd)
    m = engine.p2m_device(sources.p, sources.w)
    cs.wait_stream(aux)
    checked = engine.flag.mark()
    acc = engine.accessor_from_moments(m.storage)
    r = acc.eval_device(qd, _lib.L2P_VALUE | _lib.L2P_GRAD)
    engine.flag.raise_if_set("source/query", checked)
    return ExplicitResult(values=like_input(r["value"], q), accessor=acc, q=q, sources=sources,
                          engine=engine, q_dev=qd, q_grad=r["grad"], q_ready=q_ready)


def explicit_jvp(y_bar, res: ExplicitResult) -> LayerGradients:
    if is_host_tensor(y_bar):
        return _explicit_jvp_host(y_bar, res)
    eng, qd, src = res.engine, res.q_dev, res.sources
    checked = eng.flag.mark()           # p and q were checked by the forward
    yb = to_device(y_bar).reshape(qd.shape[0], -1).contiguous()
    # On the aux stream, beside the tail of the forward still running on the
    # caller's stream: the brick partition of q (it needs only q, valid since
    # the forward's start), then q_bar from the stored gradient; the caller's
    # stream waits for the partition before the query P2M's second phase and
    # joins the aux stream before returning
    cs = torch.cuda.current_stream()
    aux = eng.aux_stream()
    y_ready = cs.record_event()
    prep = None
    with torch.cuda.stream(aux):
        if res.q_ready is not None:
            aux.wait_event(res.q_ready)
            prep = eng.p2m_prepare(qd, int(yb.shape[1]))
            prep_done = aux.record_event()
        aux.wait_event(y_ready)
        q_bar = _weighted_grad(res.q_grad, yb)
    q_bar.record_stream(cs)             # the caller uses it on its stream
    if prep is not None:
        prep["ws"].record_stream(cs)
        cs.wait_event(prep_done)
    back = eng.accessor_from_moments(eng.p2m_device(qd, yb, prepared=prep).storage)
    out = back.eval_device(src.p, _lib.L2P_VALUE | _lib.L2P_WGRAD, wts=src.w)
    cs.wait_stream(aux)
    eng.flag.raise_if_set("source/query", checked)
    ref = y_bar
    return LayerGradients(w_bar=like_input(out["value"], ref), p_bar=like_input(out["wgrad"], ref),
                          q_bar=like_input(q_bar, ref))


# ---------------------------------------------------------------- insertion ---

def insert_and_expand(engine: Engine, keys: torch.Tensor, payload: torch.Tensor,
                      channels: int, records: int | None = None) -> Accessor:
    """_insert_moments (reference layers.py:144-153): stable sort of the item
    cell keys, per-cell sums of the payload rows in sorted order (no atomics,
    deterministic), then one cascade -- the one extra expansion of a JVP.
    With ``records`` (= colours) the items are radiance segment records,
    expanded to rows inside the per-cell sum (fc2t2_vol_insert)."""
    n = int(keys.shape[0])
    lv = engine.levels
    R3 = level_resolution(lv) ** 3
    dev = keys.device
    ws_b = int(_lib.lib().fc2t2_key_sort_workspace_size(lv, n))
    ws = torch.empty(max(ws_b, 4), dtype=torch.uint8, device=dev)
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    start = torch.empty(R3 + 1, dtype=torch.int32, device=dev)
    _lib.call("fc2t2_key_sort", lv, _ptr(keys), n, _ptr(order), _ptr(start), _ptr(ws), ws_b,
              _stream())
    m = engine._empty_grid(lv, channels, "M")
    if records is not None:   # segment records expanded while summing (radiance layer)
        _lib.call("fc2t2_vol_insert", engine.rho, lv, records, _ptr(payload), _ptr(order),
                  _ptr(start), _ptr(m.storage), _stream())
    else:
        _lib.call("fc2t2_insert", engine.rho, lv, channels, _ptr(payload), _ptr(order),
                  _ptr(start), _ptr(m.storage), _stream())
    out = engine.cascade_device(m.storage)
    grid = ExpansionGrid(level=lv, kind="L", storage=out, rho=engine.rho)
    return Accessor(grid, engine.table, engine.flops, flag=engine.flag)


def _source_adjoints(back: Accessor, sources: SourceSet):
    """w_bar = B(p), p_bar = sum_c w_c grad B_c(p) (reference layers.py:8-12)."""
    out = back.eval_device(sources.p, _lib.L2P_VALUE | _lib.L2P_WGRAD, wts=sources.w)
    return out["value"], out["wgrad"]


def _like(t: torch.Tensor, ref):
    if isinstance(ref, torch.Tensor):
        return t if ref.is_cuda else t.cpu()
    a = t.detach().cpu().numpy()
    return a.astype(np.float64) if a.dtype != np.bool_ else a


def _tangent(y, n: int, cols: int) -> torch.Tensor:
    t = to_device(y).reshape(n, cols) if cols > 1 else to_device(y).reshape(n)
    return t.contiguous()


# ------------------------------------------------------------ root layers ---

@dataclass
class RootResult:
    """Reference layers.py:193-205; device tensors kept in ``dev`` for the JVPs."""

    lengths: object
    hit: object
    points: object
    grads: object
    denom: object
    accessor: Accessor
    bundle: RayBundle
    sources: SourceSet
    engine: Engine
    bias: float
    diagnostics: dict
    dev: dict = field(default_factory=dict, repr=False)


def depth_forward(engine: Engine, sources: SourceSet, bundle: RayBundle, bias: float = 0.05,
                  trav=None) -> RootResult:
    """First root of f = sum w psi + bias along each ray (reference layers.py:244-272):
    one expansion, then one fused walker per ray (traversal, line2poly, 5-sample
    screen, closed-form roots, hit point, gradient and Hessian at the hit)."""
    if sources.channels != 1:
        raise ValueError("root layers expect a single-channel field")
    if engine.rho > ROOT_MAX_ORDER:
        raise OrderError(f"root layers need rho <= {ROOT_MAX_ORDER}")
    acc, checked = _expand_checked(engine, sources.p, sources.w)
    org, dirs = bundle.dev()
    R = bundle.count
    dev = org.device
    lengths = torch.empty(R, dtype=torch.float64, device=dev)
    hit = torch.empty(R, dtype=torch.uint8, device=dev)
    points = torch.empty((R, 3), dtype=torch.float64, device=dev)
    grads = torch.empty((R, 3), dtype=torch.float32, device=dev)
    hess = torch.empty((R, 6), dtype=torch.float32, device=dev)
    denom = torch.empty(R, dtype=torch.float32, device=dev)
    st = acc.grid.storage
    _lib.call("fc2t2_depth_forward", engine.rho, engine.levels, _ptr(st), _ptr(org), _ptr(dirs), R,
              float(bias), _ptr(lengths), _ptr(hit), _ptr(points), _ptr(grads), _ptr(hess),
              _ptr(denom), _stream())
    engine.flag.raise_if_set("source", checked)
    hitb = hit.bool()
    ref = bundle.origins
    diag = Diagnostics(dead_pixels=R - hit.sum(dtype=torch.int64), ift_clamped=0)
    return RootResult(lengths=_like(lengths, ref), hit=_like(hitb, ref), points=_like(points, ref),
                      grads=_like(grads, ref), denom=_like(denom, ref), accessor=acc,
                      bundle=bundle, sources=sources, engine=engine, bias=bias,
                      diagnostics=diag,
                      dev={"hit": hit, "points": points, "grads": grads, "hess": hess,
                           "denom": denom})


class Diagnostics(dict):
    """The reference's diagnostics dict ({"dead_pixels": int, "ift_clamped":
    int}); counts produced on the device stay device scalars until a value is
    first read, so a layer call does not stall the stream for them."""

    def _get(self, k):
        v = dict.__getitem__(self, k)
        if isinstance(v, torch.Tensor):
            v = int(v.item())
            dict.__setitem__(self, k, v)
        return v

    def __getitem__(self, k):
        return self._get(k)

    def get(self, k, default=None):
        return self._get(k) if k in self else default

    def items(self):
        return [(k, self._get(k)) for k in list(self.keys())]

    def values(self):
        return [self._get(k) for k in list(self.keys())]

    def resolved(self) -> dict:
        return dict(self.items())

    def __eq__(self, other):
        return self.resolved() == (other.resolved() if isinstance(other, Diagnostics) else other)

    __hash__ = None

    def __repr__(self):
        return repr(self.resolved())


def _root_jvp(res: RootResult, y_len, y_grad) -> LayerGradients:
    eng, src, R = res.engine, res.sources, res.bundle.count
    grads = LayerGradients(w_bar=None, p_bar=None, diagnostics=Diagnostics(res.diagnostics))
    ref = y_len if y_len is not None else y_grad
    checked = eng.flag.mark()           # p and the rays were checked by the forward
    yl = _tangent(y_len, R, 1) if y_len is not None else None
    yg = _tangent(y_grad, R, 3) if y_grad is not None else None
    PP = eng.PP
    keys = torch.empty(R, dtype=torch.int32, device=src.p.device)
    payload = torch.empty((R, 1, PP), dtype=torch.float32, device=src.p.device)
    nclamp = torch.zeros(1, dtype=torch.int32, device=src.p.device)
    d = res.dev
    _, dirs = res.bundle.dev()
    _lib.call("fc2t2_root_payload", eng.rho, eng.levels, _ptr(dirs), R, _ptr(d["hit"]),
              _ptr(d["points"]), _ptr(d["grads"]), _ptr(d["hess"]), _ptr(d["denom"]),
              _ptr(yl), _ptr(yg), _ptr(keys), _ptr(payload), _ptr(nclamp), _stream())
    back = insert_and_expand(eng, keys, payload, 1)
    w_bar, p_bar = _source_adjoints(back, src)
    eng.flag.raise_if_set("source", checked)
    grads.diagnostics["ift_clamped"] = nclamp[0]
    grads.w_bar, grads.p_bar = _like(w_bar, ref), _like(p_bar, ref)
    return grads


def depth_jvp(y_bar, res: RootResult) -> LayerGradients:
    """Ray-length adjoints via the IFT projection (reference layers.py:285-303)."""
    return _root_jvp(res, y_bar, None)


def surface_gradient_forward(engine: Engine, sources: SourceSet, bundle: RayBundle,
                             bias: float = 0.05, trav=None) -> RootResult:
    """Same roots; the output is grad f at the hit (reference layers.py:306-310)."""
    return depth_forward(engine, sources, bundle, bias=bias, trav=trav)


def surface_gradient_jvp(y_bar, res: RootResult) -> LayerGradients:
    """Monopole mu = -sum y_i kappa_i plus dipoles y_a, one expansion
    (reference layers.py:313-356)."""
    return _root_jvp(res, None, y_bar)


def depth_surface_jvp(y_len, y_grad, res: RootResult) -> LayerGradients:
    """depth_jvp + surface_gradient_jvp in ONE insertion and one expansion
    (the payloads add)."""
    return _root_jvp(res, y_len, y_grad)


@dataclass
class RGBDResult:
    """RGBD composition: depth = first root of the SDF field,
    rgb = colour field at the hit point (0 where the ray misses)."""

    depth: object
    hit: object
    rgb: object
    root: RootResult
    color: ExplicitResult


def rgbd_forward(engine: Engine, sdf: SourceSet, color: SourceSet, bundle: RayBundle,
                 bias: float = 0.05) -> RGBDResult:
    """Composed, not bespoke: depth_forward supplies the roots and
    explicit_forward evaluates the colour channels at the hit points.  Missed
    rays query the domain centre and are masked, so no compaction (and no
    extra host sync) is needed."""
    root = depth_forward(engine, sdf, bundle, bias=bias)
    hit = root.dev["hit"].bool()
    q = torch.where(hit[:, None], root.dev["points"], 0.0).to(torch.float32).contiguous()
    col = explicit_forward(engine, color, q)
    rgb = torch.where(hit[:, None], col.values, 0.0)
    lengths = root.lengths if isinstance(root.lengths, torch.Tensor) else to_device(root.lengths)
    depth = torch.where(hit, lengths.to(torch.float64), 0.0)
    ref = bundle.origins
    return RGBDResult(depth=_like(depth, ref), hit=_like(hit, ref), rgb=_like(rgb, ref), root=root,
                      color=col)


def rgbd_jvp(y_depth, y_rgb, res: RGBDResult) -> tuple[LayerGradients, LayerGradients]:
    """(SDF-source gradients, colour-source gradients).  The colour layer's
    JVP also yields q_bar at the hit point x = o + t r, which moves the root:
    dL/dt += q_bar . r, so the depth tangent handed to depth_jvp is
    y_depth + q_bar . r on hit rays -- two insertions, two expansions."""
    hit = res.root.dev["hit"].bool()
    R = hit.shape[0]
    C = int(res.color.values.shape[1])
    yr = torch.where(hit[:, None], to_device(y_rgb).reshape(R, C), 0.0)
    gc = explicit_jvp(yr.contiguous(), res.color)
    q_bar = gc.q_bar if isinstance(gc.q_bar, torch.Tensor) else to_device(gc.q_bar)
    _, dirs = res.root.bundle.dev()
    dt = (q_bar.to(torch.float64) * dirs).sum(1)
    yd = _tangent(y_depth, R, 1).reshape(R).to(torch.float64) if y_depth is not None else 0.0
    tangent = torch.where(hit, yd + dt, 0.0).to(torch.float32).contiguous()
    gd = _root_jvp(res.root, tangent, None)
    ref = y_rgb
    for g in (gc, gd):
        g.w_bar, g.p_bar = _like(to_device(g.w_bar), ref), _like(to_device(g.p_bar), ref)
    return gd, gc


# -------------------------------------------------------- integral layers ---

@dataclass
class IntegralResult:
    """Reference layers.py:361-368."""

    values: object
    accessor: Accessor
    trav: object
    bundle: RayBundle
    sources: SourceSet
    engine: Engine


def line_integral_forward(engine: Engine, sources: SourceSet, bundle: RayBundle,
                          trav=None) -> IntegralResult:
    """Exact integral of the field along every ray (reference layers.py:371-386)."""
    acc = engine.expand_device(sources.p, sources.w)
    org, dirs = bundle.dev()
    R, C = bundle.count, sources.channels
    vals = torch.empty((R, C), dtype=torch.float32, device=org.device)
    _lib.call("fc2t2_line_integral", engine.rho, engine.levels, C, _ptr(acc.grid.storage),
              _ptr(org), _ptr(dirs), R, _ptr(vals), _stream())
    engine.flag.raise_if_set("source")
    return IntegralResult(values=_like(vals, bundle.origins), accessor=acc, trav=trav,
                          bundle=bundle, sources=sources, engine=engine)


_GAUSS: dict = {}


def _gauss_dev(G: int, dev):
    if G not in _GAUSS:
        x, w = np.polynomial.legendre.leggauss(G)
        _GAUSS[G] = (torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev))
    return _GAUSS[G]


def line_integral_jvp(y_bar, res: IntegralResult) -> LayerGradients:
    """Closed-form weighted-segment insertion, one expansion (reference layers.py:389-402)."""
    eng, src, bundle = res.engine, res.sources, res.bundle
    org, dirs = bundle.dev()
    R, C = bundle.count, src.channels
    yb = to_device(y_bar).reshape(R, C).contiguous()
    offs, S = segment_offsets(bundle, eng.levels)
    G = eng.rho // 2 + 1
    gx, gw = _gauss_dev(G, org.device)
    keys = torch.empty(max(S, 1), dtype=torch.int32, device=org.device)
    payload = torch.empty((max(S, 1), C, eng.PP), dtype=torch.float32, device=org.device)
    _lib.call("fc2t2_line_payload", eng.rho, eng.levels, C, _ptr(org), _ptr(dirs), R, _ptr(offs),
              _ptr(yb), _ptr(gx), _ptr(gw), G, _ptr(keys), _ptr(payload), _stream())
    back = insert_and_expand(eng, keys[:S], payload[:S], C)
    w_bar, p_bar = _source_adjoints(back, src)
    eng.flag.raise_if_set("source")
    return LayerGradients(w_bar=_like(w_bar, y_bar), p_bar=_like(p_bar, y_bar))


# ------------------------------------------------------------ radiance layer ---

EXP_CUTOFF = 4.5      # reference poly1d.py:22
EXP_FIT_RANGE = 5.0   # reference poly1d.py:23


def fit_exp_poly() -> np.ndarray:
    """Degree-4 fit of exp(-x) over 64 Chebyshev nodes on [0, 5] with the value
    1 at 0 (reference poly1d.py:224-242); host constant."""
    k = np.arange(64)
    x = 2.5 + 2.5 * np.cos((2 * k + 1) * np.pi / 128)
    V = x[:, None] ** np.arange(1, 5)[None, :]
    tail, *_ = np.linalg.lstsq(V, np.exp(-x) - 1.0, rcond=None)
    return np.concatenate([[1.0], tail])


@dataclass
class RenderResult:
    """Reference layers.py:405-424.  The per-segment caches of the reference
    (sigma/colour/transmittance polynomials, depth0, anti) are recomputed by the
    backward walker instead of stored; ``alive`` is materialised on access."""

    rgb: object
    accessor: Accessor
    trav: object
    bundle: RayBundle
    p: object
    w_sigma: object
    w_color: object
    background: object
    engine: Engine
    depth_final: object = None
    dev: dict = field(default_factory=dict, repr=False)

    @property
    def alive(self):
        """Per-segment alive flags in traversal order (depth0 <= 4.5, layers.py:453)."""
        if "alive" not in self.dev:
            eng, b = self.engine, self.bundle
            org, dirs = b.dev()
            offs, S = segment_offsets(b, eng.levels)
            flags = torch.empty(max(S, 1), dtype=torch.uint8, device=org.device)
            rgb = torch.empty((b.count, self.dev["colors"]), dtype=torch.float32, device=org.device)
            dfin = torch.empty(b.count, dtype=torch.float64, device=org.device)
            _lib.call("fc2t2_vol_forward", eng.rho, eng.levels, self.dev["colors"],
                      _ptr(self.accessor.grid.storage), _ptr(org), _ptr(dirs), b.count,
                      _ptr(self.dev["efit"]), _ptr(self.dev["bg"]), _ptr(rgb), _ptr(dfin),
                      _ptr(offs), _ptr(flags), _stream())
            self.dev["alive"] = flags[:S].bool()
        return _like(self.dev["alive"], self.bundle.origins)


def volumetric_forward(engine: Engine, p, w_sigma, w_color, bundle: RayBundle, background,
                       trav=None) -> RenderResult:
    """Emission/absorption rendering with closed-form per-segment algebra
    (reference layers.py:427-480): relu'd density weights, one 1+C channel
    expansion, then one walker thread per ray."""
    ws = to_device(w_sigma).reshape(-1, 1)
    wc = to_device(w_color)
    wc = wc.reshape(ws.shape[0], -1)
    C = int(wc.shape[1])
    src = SourceSet(p, torch.cat([ws.clamp(min=0.0), wc], dim=1))
    acc = engine.expand_device(src.p, src.w)
    org, dirs = bundle.dev()
    R = bundle.count
    efit = torch.from_numpy(fit_exp_poly()).to(org.device)
    bg = torch.as_tensor(np.asarray(background, dtype=np.float64) if not isinstance(
        background, torch.Tensor) else background, dtype=torch.float64).to(org.device).reshape(-1)
    rgb = torch.empty((R, C), dtype=torch.float32, device=org.device)
    dfin = torch.empty(R, dtype=torch.float64, device=org.device)
    # the walk also produces the backward's pass-A totals (one walk saved per JVP)
    n_alive = torch.zeros(R + 1, dtype=torch.int32, device=org.device)
    totals = torch.empty((R, C), dtype=torch.float64, device=org.device)
    _lib.call("fc2t2_vol_forward_ex", engine.rho, engine.levels, C, _ptr(acc.grid.storage),
              _ptr(org), _ptr(dirs), R, _ptr(efit), _ptr(bg), _ptr(rgb), _ptr(dfin),
              _ptr(n_alive), _ptr(totals), _stream())
    engine.flag.raise_if_set("source")
    ref = bundle.origins
    return RenderResult(rgb=_like(rgb, ref), accessor=acc, trav=trav, bundle=bundle, p=p,
                        w_sigma=w_sigma, w_color=w_color, background=background, engine=engine,
                        depth_final=_like(dfin, ref),
                        dev={"src": src, "ws": ws, "colors": C, "efit": efit, "bg": bg,
                             "n_alive": n_alive, "totals": totals, "dfin": dfin})


def volumetric_jvp(y_bar, res: RenderResult) -> LayerGradients:
    """Adjoint rendering via weighted-segment insertion, one expansion
    (reference layers.py:483-544).  Uses E' of the fitted quartic, so the JVP
    is exact for the implemented forward."""
    eng, b = res.engine, res.bundle
    org, dirs = b.dev()
    R, C = b.count, res.dev["colors"]
    dev = org.device
    yb = to_device(y_bar).reshape(R, C).contiguous()
    st = res.accessor.grid.storage
    efit, bg = res.dev["efit"], res.dev["bg"]
    if "totals" in res.dev:   # pass A came with the forward walk
        n_alive, totals, dfin = res.dev["n_alive"], res.dev["totals"], res.dev["dfin"]
    else:
        n_alive = torch.zeros(R + 1, dtype=torch.int32, device=dev)
        totals = torch.empty((R, C), dtype=torch.float64, device=dev)
        dfin = torch.empty(R, dtype=torch.float64, device=dev)
        _lib.call("fc2t2_vol_totals", eng.rho, eng.levels, C, _ptr(st), _ptr(org), _ptr(dirs), R,
                  _ptr(efit), _ptr(n_alive), _ptr(totals), _ptr(dfin), _stream())
    offs = torch.empty_like(n_alive)
    ws_b = int(_lib.lib().fc2t2_scan_workspace_size(R + 1))
    wsp = torch.empty(max(ws_b, 4), dtype=torch.uint8, device=dev)
    _lib.call("fc2t2_scan_u32", _ptr(n_alive), _ptr(offs), R + 1, _ptr(wsp), ws_b, _stream())
    A = int(offs[R].item())
    G = int(_lib.lib().fc2t2_vol_gauss_nodes(eng.rho))
    gx, gw = _gauss_dev(G, dev)
    keys = torch.empty(max(A, 1), dtype=torch.int32, device=dev)
    rec = torch.empty((max(A, 1), int(_lib.lib().fc2t2_vol_record_floats(C))),
                      dtype=torch.float32, device=dev)
    _lib.call("fc2t2_vol_payload", eng.rho, eng.levels, C, _ptr(st), _ptr(org), _ptr(dirs), R,
              _ptr(efit), _ptr(bg), _ptr(yb), _ptr(offs), _ptr(totals), _ptr(dfin), _ptr(gx),
              _ptr(gw), _ptr(keys), _ptr(rec), _stream())
    back = insert_and_expand(eng, keys[:A], rec[:A], 1 + C, records=C)
    src = res.dev["src"]
    val, p_bar = _source_adjoints(back, src)
    w_bar = val.clone()
    w_bar[:, 0] = torch.where(res.dev["ws"][:, 0] > 0.0, val[:, 0], torch.zeros_like(val[:, 0]))
    eng.flag.raise_if_set("source")
    return LayerGradients(w_bar=_like(w_bar, y_bar), p_bar=_like(p_bar, y_bar))
