"""Device-resident FC2T2 engine: the drop-in for ``fc2t2.expansion``.

Same names, arguments, dataclass fields and exceptions as the reference
(``pkg/src/fc2t2/expansion.py``); the arrays live in HBM as float32 torch
tensors and every stage runs through the C ABI (``include/fc2t2_b200.h``):

    SourceSet            reference :31-54   (p, w) on the device
    ExpansionGrid        reference :57-76   ``storage`` is (res,res,res,C,PP);
                                            ``data`` is the (res,res,res,C,P) view
    find_box/box_centers reference :79-93   bit-exact cell indices (fp64 on device)
    Engine.p2m           reference :186-198 stable sort by cell + segmented sum
    Engine.m2m/l2l/m2l   reference :200-264
    Engine.expand*       reference :268-285 one fused cascade call
    Accessor             reference :296-398 L2P value / partials / partials2

Inputs may be numpy arrays (converted to float32 and uploaded) or torch
tensors; results come back in the caller's kind (numpy in -> numpy out,
torch in -> torch CUDA out), so reference-style numpy user code keeps working.
``Engine.flops`` and ``Engine.expansion_count`` follow the reference's
counting rules exactly (they are host-side tallies, pinned by tests).
"""

from __future__ import annotations

from dataclasses import dataclass
import os

import numpy as np
import torch

from . import _lib, flops
from .kernel import (COARSEST_LEVEL, KernelModel, M2LTable, fit_m2l_tables,
                     separable_eligible, separable_factors, separable_far_eligible,
                     level_box_width, level_resolution)
from .multiindex import MultiIndexTable


class DomainError(ValueError):
    """A location lies on or outside the boundary of (-1, 1)^3 (reference :23-24)."""


class StageError(ValueError):
    """A grid of the wrong kind/level was fed to a stage (reference :27-28)."""


# ------------------------------------------------------------- plumbing ---

def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the FC2T2 B200 engine needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return ct_void(torch.cuda.current_stream().cuda_stream)


def ct_void(v):
    import ctypes
    return ctypes.c_void_p(int(v))


def _ptr(t: torch.Tensor | None):
    import ctypes
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


_ONE_BELOW = np.float32(np.nextafter(np.float32(1.0), np.float32(0.0)))


def to_device(x, cols: int | None = None, points: bool = False) -> torch.Tensor:
    """float32 contiguous CUDA tensor from numpy / torch input.

    ``points=True`` keeps coordinates strictly inside (-1, 1) after the
    float32 rounding (a float64 value just below 1 can round to 1.0f); the
    domain check itself happened on the float64 input.
    """
    if isinstance(x, torch.Tensor):
        t = x.to(device=_device(), dtype=torch.float32)
    else:
        a = np.asarray(x, dtype=np.float64)
        a32 = a.astype(np.float32)
        if points and a32.size:
            a32 = np.clip(a32, -_ONE_BELOW, _ONE_BELOW)
        t = torch.from_numpy(a32).to(_device())
    if cols is not None:
        t = t.reshape(-1, cols)
    return t.contiguous()


class HostIO:
    """Host <-> device staging for host-tensor callers.  Uploads run on an
    "up" stream and downloads on a "down" stream, so the two PCIe directions
    overlap each other and the compute stream; results land in pinned buffers
    (torch's caching host allocator).  ``h2d(..., chunks=k)`` splits an upload
    by rows with one ready event per chunk, letting per-chunk consumers start
    while the rest is in flight."""

    _streams: dict = {}
    _aux: dict = {}

    @classmethod
    def aux(cls) -> torch.cuda.Stream:
        """A second compute stream for work that overlaps the main one."""
        dev = torch.cuda.current_device()
        if dev not in cls._aux:
            cls._aux[dev] = torch.cuda.Stream(device=dev)
        return cls._aux[dev]

    @classmethod
    def _pair(cls):
        dev = torch.cuda.current_device()
        if dev not in cls._streams:
            cls._streams[dev] = (torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev))
        return cls._streams[dev]

    @classmethod
    def h2d(cls, x: torch.Tensor, cols: int | None = None, chunks: int = 1):
        """Async upload of a host tensor.  Returns (device tensor, ready event)
        for chunks == 1, else (device tensor, [(row0, row1, event), ...])."""
        cs = torch.cuda.current_stream()
        up, _ = cls._pair()
        src = x if x.is_pinned() else x.pin_memory()
        if cols is not None:
            src = src.reshape(-1, cols)
        n = int(src.shape[0]) if src.dim() else 1
        k = max(1, min(int(chunks), n)) if n else 1
        bounds = [(n * i) // k for i in range(k + 1)]
        with torch.cuda.stream(up):
            t = torch.empty(tuple(src.shape), dtype=torch.float32, device=_device())
            evs = []
            for a, b in zip(bounds[:-1], bounds[1:]):
                if b > a:
                    t[a:b].copy_(src[a:b], non_blocking=True)
                evs.append((a, b, up.record_event()))
        t.record_stream(cs)
        if chunks == 1:
            return t, evs[-1][2]
        return t, evs

    @classmethod
    def d2h(cls, t: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Start an async download of ``t`` after the current stream's work
        (into ``out`` if given, else a new pinned tensor); call finish()
        before the host reads the result."""
        cs = torch.cuda.current_stream()
        _, down = cls._pair()
        down.wait_stream(cs)
        if out is None:
            out = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
        with torch.cuda.stream(down):
            out.copy_(t, non_blocking=True)
        t.record_stream(down)
        return out

    @classmethod
    def finish(cls) -> None:
        up, down = cls._pair()
        down.synchronize()
        up.synchronize()


def is_host_tensor(x) -> bool:
    return isinstance(x, torch.Tensor) and not x.is_cuda


def like_input(t: torch.Tensor, ref):
    """Return ``t`` in the caller's kind: CUDA tensor for CUDA input, a
    (pinned) host tensor for host-tensor input, float64 numpy for numpy."""
    if isinstance(ref, torch.Tensor):
        if ref.is_cuda:
            return t
        out = t.to("cpu", non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    return t.detach().cpu().numpy().astype(np.float64)


def _host_domain_check(a, what: str) -> None:
    if isinstance(a, torch.Tensor):
        return
    a = np.asarray(a, dtype=np.float64)
    if a.size and np.max(np.abs(a)) >= 1.0:
        raise DomainError(f"{what} locations must lie strictly inside (-1, 1)^3")


class DomainFlag:
    """Device int32 accumulating FLAG_* bits; read once per public call.

    A layer whose inputs are checked by early kernels calls ``mark()`` right
    after them; ``raise_if_set`` then copies the flag on a side stream that
    waits only for that point, so the main stream is not drained (its later
    kernels keep running while the host decides).  Without a mark the read is
    stream-ordered after everything enqueued.  ``deferred()`` suspends the
    read (CUDA-graph capture: a host sync cannot be captured; graphs.py checks
    the flag once after each replay)."""

    def __init__(self):
        self.t = torch.zeros(1, dtype=torch.int32, device=_device())
        self._defer = 0
        self.reduce_hook = None     # parallel.sharded: max of the flag over the ranks
        self._host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._side = None
        self._mark = None
        self._done = None

    class _Deferred:
        def __init__(self, flag):
            self.flag = flag

        def __enter__(self):
            self.flag._defer += 1

        def __exit__(self, *a):
            self.flag._defer -= 1

    def deferred(self):
        return DomainFlag._Deferred(self)

    def mark(self, stream=None):
        """Every kernel that checks this call's inputs has been enqueued (on
        ``stream``, default the current one); returns the token the same call
        passes to ``raise_if_set``."""
        if self._defer:
            return None
        if self._side is None:
            self._side = torch.cuda.Stream(device=self.t.device)
            self._mark = torch.cuda.Event()
            self._done = torch.cuda.Event()
        self._mark.record(stream if stream is not None else torch.cuda.current_stream(self.t.device))
        return self._mark

    def raise_if_set(self, what: str, mark=None) -> None:
        if self._defer:
            return
        if mark is not None:
            with torch.cuda.stream(self._side):
                self._side.wait_event(self._mark)
                self._host.copy_(self.t, non_blocking=True)
                self._done.record(self._side)
            self._done.synchronize()
            v = int(self._host[0])
        else:
            v = int(self.t.item())
        if self.reduce_hook is not None:
            v = self.reduce_hook(v)
        if v & _lib.FLAG_DOMAIN:
            self.t.zero_()      # stream-ordered: after the call's trailing kernels too
            raise DomainError(f"{what} locations must lie strictly inside (-1, 1)^3")

    def check_points(self, pts: torch.Tensor) -> None:
        """Enqueue a stand-alone domain check of pts (n, 3) float32."""
        n = int(pts.shape[0])
        if n:
            _lib.call("fc2t2_domain_check", _ptr(pts), n, _ptr(self.t), _stream())


# ------------------------------------------------------------ datatypes ---

@dataclass
class SourceSet:
    """Source locations and per-channel weights, device resident (reference :31-54)."""

    p: object    # (N, 3)
    w: object    # (N, C)

    def __post_init__(self):
        self._numpy_input = not isinstance(self.p, torch.Tensor)
        p_np = None if isinstance(self.p, torch.Tensor) else np.atleast_2d(
            np.asarray(self.p, dtype=np.float64))
        w_in = self.w
        if not isinstance(w_in, torch.Tensor):
            w_in = np.asarray(w_in, dtype=np.float64)
            if w_in.ndim == 1:
                w_in = w_in[:, None]
        elif w_in.dim() == 1:
            w_in = w_in[:, None]
        n_p = p_np.shape[0] if p_np is not None else self.p.reshape(-1, 3).shape[0]
        if n_p != w_in.shape[0]:
            raise ValueError("p and w disagree on the number of sources")
        if p_np is not None:
            _host_domain_check(p_np, "source")
        if (isinstance(self.p, torch.Tensor) and isinstance(w_in, torch.Tensor)
                and not self.p.is_cuda and not w_in.is_cuda and self.p.is_pinned()
                and w_in.is_pinned() and self.p.dtype == torch.float32
                and w_in.dtype == torch.float32):
            # pinned host tensors: asynchronous upload on the copy stream (the
            # compute stream waits on it), torch's non_blocking convention --
            # every layer call returns only after its results are downloaded,
            # so the copies have completed by the time the caller regains
            # control from one
            self.p, _ = HostIO.h2d(self.p, 3)
            self.w, ev = HostIO.h2d(w_in.reshape(self.p.shape[0], -1))
            torch.cuda.current_stream().wait_event(ev)
            return
        self.p = to_device(p_np if p_np is not None else self.p, 3, points=True)
        self.w = to_device(w_in).reshape(self.p.shape[0], int(w_in.shape[1]))

    @property
    def n(self) -> int:
        return int(self.p.shape[0])

    @property
    def channels(self) -> int:
        return int(self.w.shape[1])


@dataclass
class ExpansionGrid:
    """Per-level grid of coefficient rows (reference :57-76).

    ``storage`` is the padded device tensor (res, res, res, C, PP); ``data``
    is its (res, res, res, C, P) view in graded-lex order.
    """

    level: int
    kind: str
    storage: torch.Tensor
    rho: int

    @property
    def data(self) -> torch.Tensor:
        from .multiindex import index_count
        return self.storage[..., :index_count(self.rho)]

    @property
    def res(self) -> int:
        return int(self.storage.shape[0])

    @property
    def channels(self) -> int:
        return int(self.storage.shape[3])

    @property
    def box_width(self) -> float:
        return level_box_width(self.level)


def box_centers(level: int, idx) -> np.ndarray:
    """Centres of boxes with index triples ``idx`` (reference :79-82)."""
    w = level_box_width(level)
    return -1.0 + (np.asarray(idx, dtype=np.float64) + 0.5) * w


def find_box(level: int, q):
    """Box index triples, bit-exact with the reference (:85-93), computed by
    the device kernel (float64 arithmetic on the float32 coordinates)."""
    pts = to_device(q, 3)
    out = torch.empty((pts.shape[0], 3), dtype=torch.int32, device=pts.device)
    _lib.call("fc2t2_find_box", int(level), _ptr(pts), int(pts.shape[0]), _ptr(out),
              _ptr(None), _stream())
    if isinstance(q, torch.Tensor):
        return out
    return out.cpu().numpy().astype(np.int64).reshape(np.shape(q))


def axis_points(n: int, a: float = -1.0, b: float = 1.0) -> np.ndarray:
    """linspace with bare domain endpoints nudged inward (reference :288-293)."""
    lo = np.nextafter(-1.0, 0.0) if a <= -1.0 else a
    hi = np.nextafter(1.0, 0.0) if b >= 1.0 else b
    return np.linspace(lo, hi, n)


def _axis_target_count(res: int, delta: int, parity) -> int:
    """Number of targets one stencil offset touches along an axis (the
    slice bounds of reference _axis_slices, :135-151)."""
    lo, hi = max(0, -delta), min(res - 1, res - 1 - delta)
    if parity is not None:
        if lo % 2 != parity:
            lo += 1
        if hi % 2 != parity:
            hi -= 1
        return 0 if lo > hi else (hi - lo) // 2 + 1
    return max(0, hi - lo + 1)


def m2l_pairs(table: M2LTable) -> int:
    """(target, offset) pairs one M2L pass over ``table`` touches; times
    C*P*P*2 this is the reference's FLOP count (expansion.py:262)."""
    res = level_resolution(table.level)
    parity_stencil = not table.nearfield and table.level != COARSEST_LEVEL
    total = 0
    for off, act in zip(table.offsets, table.active):
        if not act:
            continue
        cnt = 1
        for a in range(3):
            d = int(off[a])
            parity = (1 if d == -3 else 0) if (parity_stencil and abs(d) == 3) else None
            cnt *= _axis_target_count(res, d, parity)
        total += cnt
    return total


# --------------------------------------------------------------- engine ---

class _Handle:
    def __init__(self, rho: int, levels: int):
        import ctypes
        self.lib = _lib.lib()
        h = ctypes.c_void_p()
        _lib.check(self.lib.fc2t2_engine_create(rho, levels, ctypes.byref(h)), "engine_create")
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.lib.fc2t2_engine_destroy(self.h)
        except Exception:
            pass


class Engine:
    """A configured transform (reference expansion.py:154-285)."""

    def __init__(self, kernel: KernelModel, levels: int, lsq: bool = True,
                 nodes_per_axis: int = 6, admissibility_tol: float = 1e-3,
                 check_admissibility: bool = True, *, separable: bool | None = None):
        if levels < COARSEST_LEVEL:
            raise StageError(f"levels must be >= {COARSEST_LEVEL}")
        self.kernel = kernel
        self.levels = levels
        self.rho = kernel.rho
        self.table: MultiIndexTable = kernel.table
        self.lsq = lsq
        self.m2l_tables = fit_m2l_tables(
            kernel, levels, lsq=lsq, nodes_per_axis=nodes_per_axis,
            admissibility_tol=admissibility_tol, check=check_admissibility)
        self.flops = flops.FlopCounter()
        self.expansion_count = 0
        self.P = self.table.size
        self.PP = self.table.padded_size
        self._pairs = {("far", l): m2l_pairs(t) for l, t in self.m2l_tables["far"].items()}
        self._pairs[("near", levels)] = m2l_pairs(self.m2l_tables["near"])
        self._h = None
        self._flag = None
        self._cascade_hook = None    # parallel.sharded: the multi-GPU cascade
        # finest far + near M2L through the per-axis factors of its tables
        # (kernel.separable_factors, csrc/m2l_sep.cu) when they factor;
        # separable=False or FC2T2_M2L_DENSE=1 keeps the dense tcgen05 path
        if separable is None:
            separable = os.environ.get("FC2T2_M2L_DENSE", "0") != "1"
        self.separable = bool(separable) and separable_eligible(
            self.m2l_tables, levels, self.rho, lsq, nodes_per_axis)
        self._sep = (separable_factors(kernel, levels, lsq, nodes_per_axis)
                     if self.separable else None)
        # coarse levels' far tables through their own per-axis factors (the
        # parity box minus the hole as three disjoint separable pieces)
        self._sep_far = {l: separable_factors(kernel, l, lsq, nodes_per_axis)
                         for l in range(COARSEST_LEVEL + 1, levels)
                         if separable and separable_far_eligible(
                             self.m2l_tables, l, levels, self.rho, lsq, nodes_per_axis)}

    # the device side is created lazily so the host tables can be built
    # (and pinned by CPU tests) without a GPU
    @property
    def handle(self):
        if self._h is None:
            h = _Handle(self.rho, self.levels)
            tabs = list(self.m2l_tables["far"].values()) + [self.m2l_tables["near"]]
            for t in tabs:
                off = np.ascontiguousarray(t.offsets, dtype=np.int64)
                act = np.ascontiguousarray(t.active, dtype=np.uint8)
                co = np.ascontiguousarray(t.coeffs, dtype=np.float64)
                _lib.check(h.lib.fc2t2_engine_set_table(
                    h.h, int(t.level), int(bool(t.nearfield)), int(off.shape[0]),
                    off.ctypes.data, act.ctypes.data, co.ctypes.data), "engine_set_table")
            _lib.check(h.lib.fc2t2_engine_upload(h.h, _stream()), "engine_upload")
            if self._sep is not None:
                f = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in self._sep.items()}
                _lib.check(h.lib.fc2t2_engine_set_separable(
                    h.h, f["pre"].ctypes.data, f["post"].ctypes.data, f["conv"].ctypes.data),
                    "engine_set_separable")
            for lvl, fac in self._sep_far.items():
                f = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in fac.items()}
                _lib.check(h.lib.fc2t2_engine_set_separable_far(
                    h.h, int(lvl), f["pre"].ctypes.data, f["post"].ctypes.data,
                    f["conv"].ctypes.data), "engine_set_separable_far")
            self._h = h
            self._flag = DomainFlag()
        return self._h.h

    @property
    def flag(self) -> DomainFlag:
        """The engine's device domain flag (created with the device side)."""
        if self._flag is None:
            _ = self.handle
        return self._flag

    def aux_stream(self) -> torch.cuda.Stream:
        """A second stream for short kernels that only depend on a layer's
        inputs (the forward's query domain check, the backward's recycled
        q_bar): they overlap the P2M on the caller's stream, which joins the
        aux stream before anything reads their results."""
        if getattr(self, "_aux", None) is None:
            self._aux = torch.cuda.Stream(device=_device())
        return self._aux

    def interaction_list(self, level: int, table: int = _lib.TABLE_FAR):
        """Device interaction list of one level: (entries (n,4) {dx,dy,dz,slot},
        class starts (ncls+1,)) -- exposed for the bit-exactness tests."""
        n = _lib.lib().fc2t2_engine_list_entries(self.handle, level, table)
        if n < 0:
            _lib.check(_lib.ESTAGE, "engine_list_entries")
        ent = np.zeros((max(n, 1), 4), dtype=np.int32)
        starts = np.zeros(9, dtype=np.int32)
        ncls = _lib.lib().fc2t2_engine_get_list(self.handle, level, table, ent.ctypes.data,
                                                starts.ctypes.data)
        return ent[:n], starts[:ncls + 1]

    # -- grids --------------------------------------------------------------

    def zero_grid(self, level: int, channels: int, kind: str) -> ExpansionGrid:
        res = level_resolution(level)
        st = torch.zeros((res, res, res, channels, self.PP), dtype=torch.float32,
                         device=_device())
        return ExpansionGrid(level=level, kind=kind, storage=st, rho=self.rho)

    def finest_grid_bytes(self, channels: int) -> int:
        return level_resolution(self.levels) ** 3 * channels * self.PP * 4

    def _empty_grid(self, level: int, channels: int, kind: str) -> ExpansionGrid:
        res = level_resolution(level)
        st = torch.empty((res, res, res, channels, self.PP), dtype=torch.float32,
                         device=_device())
        return ExpansionGrid(level=level, kind=kind, storage=st, rho=self.rho)

    # -- stages -------------------------------------------------------------

    def sort_points(self, pts: torch.Tensor) -> tuple:
        """Stable sort by finest cell: (order (n,), cell_start (res^3+1,)) --
        the np.add.at key order of expansion.py:195 (diagnostics and tests;
        P2M partitions the points itself, see p2m_device)."""
        n = int(pts.shape[0])
        R = level_resolution(self.levels) ** 3
        ws_bytes = _lib.lib().fc2t2_cell_sort_workspace_size(self.levels, n)
        ws = torch.empty(int(ws_bytes), dtype=torch.uint8, device=pts.device)
        order = torch.empty(max(n, 1), dtype=torch.int32, device=pts.device)
        start = torch.empty(R + 1, dtype=torch.int32, device=pts.device)
        _ = self.handle
        _lib.call("fc2t2_cell_sort", self.levels, _ptr(pts), n, _ptr(order), _ptr(start),
                  _ptr(self.flag.t), _ptr(ws), int(ws_bytes), _stream())
        return order, start

    def p2m_prepare(self, pts: torch.Tensor, channels: int) -> dict:
        """Phase 1 of P2M on the current stream: the brick partition of the
        points (reads only pts; sets the domain flag).  The returned handle
        goes to ``p2m_device(pts, w, prepared=...)`` for the same points."""
        n = int(pts.shape[0])
        h = self.handle
        ws_bytes = int(_lib.lib().fc2t2_p2m_points_workspace_size(h, channels, n))
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=pts.device)
        _lib.call("fc2t2_p2m_points_phase", h, channels, _ptr(pts), _ptr(None), n, _ptr(None),
                  _ptr(self.flag.t), _ptr(ws), ws_bytes, 1, _stream())
        return {"ws": ws, "n": n, "C": int(channels)}

    def p2m_device(self, pts: torch.Tensor, w: torch.Tensor, prepared: dict | None = None
                   ) -> ExpansionGrid:
        """P2M straight from the caller's point order (fc2t2_p2m_points: a
        deterministic brick partition + per-cell sums in index order); sets
        the domain flag for points outside (-1, 1)^3.  With ``prepared``
        (p2m_prepare of the same points) only phase 2 runs."""
        C = int(w.shape[1])
        n = int(pts.shape[0])
        grid = self._empty_grid(self.levels, C, "M")
        h = self.handle
        if prepared is not None and prepared["n"] == n and prepared["C"] == C:
            ws = prepared["ws"]
            _lib.call("fc2t2_p2m_points_phase", h, C, _ptr(pts), _ptr(w), n, _ptr(grid.storage),
                      _ptr(self.flag.t), _ptr(ws), int(ws.numel()), 2, _stream())
        else:
            ws_bytes = int(_lib.lib().fc2t2_p2m_points_workspace_size(h, C, n))
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=pts.device)
            _lib.call("fc2t2_p2m_points", h, C, _ptr(pts), _ptr(w), n, _ptr(grid.storage),
                      _ptr(self.flag.t), _ptr(ws), ws_bytes, _stream())
        self.flops.add("p2m", flops.p2m_flops(n, self.rho, self.P))
        return grid

    def p2m(self, sources: SourceSet) -> ExpansionGrid:
        grid = self.p2m_device(sources.p, sources.w)
        self.flag.raise_if_set("source")
        return grid

    def m2m(self, fine: ExpansionGrid) -> ExpansionGrid:
        if fine.kind != "M":
            raise StageError("m2m expects an M grid")
        if fine.level <= COARSEST_LEVEL:
            raise StageError("already at the coarsest level")
        coarse = self._empty_grid(fine.level - 1, fine.channels, "M")
        _lib.call("fc2t2_m2m", self.handle, fine.channels, fine.level,
                  _ptr(fine.storage.contiguous()), _ptr(coarse.storage), _stream())
        self.flops.add("m2m", flops.translate_flops(coarse.res, self.P))
        return coarse

    def l2l(self, coarse: ExpansionGrid) -> ExpansionGrid:
        if coarse.kind != "L":
            raise StageError("l2l expects an L grid")
        fine = self._empty_grid(coarse.level + 1, coarse.channels, "L")
        _lib.call("fc2t2_l2l", self.handle, coarse.channels, coarse.level,
                  _ptr(coarse.storage.contiguous()), _ptr(fine.storage), 0, _stream())
        self.flops.add("l2l", flops.translate_flops(coarse.res, self.P))
        return fine

    def m2l(self, m: ExpansionGrid, table: M2LTable) -> ExpansionGrid:
        if m.kind != "M":
            raise StageError("m2l expects an M grid")
        if m.level != table.level:
            raise StageError(f"grid level {m.level} != table level {table.level}")
        kind = _lib.TABLE_NEAR if table.nearfield else _lib.TABLE_FAR
        out = self._empty_grid(m.level, m.channels, "L")
        ws_bytes = int(_lib.lib().fc2t2_m2l_workspace_size(self.handle, m.channels, m.level, kind))
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=out.storage.device)
        _lib.call("fc2t2_m2l", self.handle, m.channels, m.level, kind,
                  _ptr(m.storage.contiguous()), _ptr(out.storage), 0, _ptr(ws), ws_bytes,
                  _stream())
        key = ("near" if table.nearfield else "far", table.level)
        self.flops.add("m2l", self._pairs[key] * m.channels * self.P * self.P * 2)
        return out

    # -- orchestration ------------------------------------------------------

    def _tally_cascade(self, channels: int) -> None:
        """Reference FLOP bookkeeping of expand_from_moments (:268-281)."""
        P = self.P
        for level in range(self.levels, COARSEST_LEVEL, -1):
            self.flops.add("m2m", flops.translate_flops(level_resolution(level - 1), P))
        for level in range(COARSEST_LEVEL, self.levels + 1):
            self.flops.add("m2l", self._pairs[("far", level)] * channels * P * P * 2)
            if level > COARSEST_LEVEL:
                self.flops.add("l2l", flops.translate_flops(level_resolution(level - 1), P))
        self.flops.add("m2l", self._pairs[("near", self.levels)] * channels * P * P * 2)

    def cascade_device(self, m_finest: torch.Tensor, x_range: tuple | None = None) -> torch.Tensor:
        """M2M / M2L / L2L in one C-ABI call; returns the finest L storage.
        ``x_range=(x0, x1)`` (multiples of 4) computes only the finest cells
        with x in [x0, x1) -- one rank's slab; the rest of the returned grid
        is unspecified.  Inside ``parallel.sharded`` the whole-grid cascade of
        a rank's partial moments goes through the sharded cascade instead
        (m_finest is then overwritten)."""
        C = int(m_finest.shape[3])
        self.expansion_count += 1
        self._tally_cascade(C)
        if x_range is None and self._cascade_hook is not None:
            return self._cascade_hook(m_finest)
        return self._cascade_raw(m_finest, x_range)

    def _expand_ws(self, C: int, dev) -> torch.Tensor:
        ws_bytes = int(_lib.lib().fc2t2_expand_workspace_size(self.handle, C))
        return torch.empty(ws_bytes, dtype=torch.uint8, device=dev)

    def _cascade_raw(self, m_finest: torch.Tensor, x_range: tuple | None = None) -> torch.Tensor:
        C = int(m_finest.shape[3])
        out = torch.empty_like(m_finest)
        ws = self._expand_ws(C, m_finest.device)
        x0, x1 = (0, -1) if x_range is None else (int(x_range[0]), int(x_range[1]))
        _lib.call("fc2t2_expand_slab", self.handle, C, _ptr(m_finest), _ptr(out), x0, x1,
                  _ptr(ws), int(ws.numel()), _stream())
        return out

    # the two-phase slab cascade of the multi-GPU path (parallel.sharded_cascade)
    def cascade_up(self, m_finest: torch.Tensor, x_range: tuple) -> tuple:
        """M2M chain on the x-slab (m_finest valid on the slab); returns the
        state (workspace, channels) whose coarse M grids the caller all-gathers."""
        C = int(m_finest.shape[3])
        ws = self._expand_ws(C, m_finest.device)
        _lib.call("fc2t2_expand_up", self.handle, C, _ptr(m_finest), int(x_range[0]),
                  int(x_range[1]), _ptr(ws), int(ws.numel()), _stream())
        return ws, C

    def coarse_views(self, state: tuple) -> list:
        """[(level, (res, res, res, C, PP) view into the workspace)] of the
        coarse M grids the slab cascade reads, levels lowest .. levels-1."""
        ws, C = state
        lib = _lib.lib()
        out = []
        for lvl in range(lib.fc2t2_expand_lowest(self.handle), self.levels):
            off = int(lib.fc2t2_expand_grid_offset(self.handle, C, lvl))
            res = level_resolution(lvl)
            n = res ** 3 * C * self.PP * 4
            out.append((lvl, ws[off:off + n].view(torch.float32).view(res, res, res, C, self.PP)))
        return out

    def cascade_down(self, m_finest: torch.Tensor, state: tuple, x_range: tuple) -> torch.Tensor:
        """Coarse M2L + L2L and the finest M2L on the slab (m_finest valid on
        the slab plus 3 planes either side); returns the finest L storage."""
        ws, C = state
        out = torch.empty_like(m_finest)
        _lib.call("fc2t2_expand_down", self.handle, C, _ptr(m_finest), _ptr(out), int(x_range[0]),
                  int(x_range[1]), _ptr(ws), int(ws.numel()), _stream())
        return out

    def expand_from_moments(self, m_finest: ExpansionGrid) -> "Accessor":
        if m_finest.kind != "M" or m_finest.level != self.levels:
            raise StageError("expand_from_moments expects the finest M grid")
        out = self.cascade_device(m_finest.storage.contiguous())
        grid = ExpansionGrid(level=self.levels, kind="L", storage=out, rho=self.rho)
        return Accessor(grid, self.table, self.flops)

    def accessor_from_moments(self, m_finest: torch.Tensor) -> "Accessor":
        """Cascade of device moments -> Accessor sharing the engine's flag."""
        out = self.cascade_device(m_finest)
        grid = ExpansionGrid(level=self.levels, kind="L", storage=out, rho=self.rho)
        return Accessor(grid, self.table, self.flops, flag=self.flag)

    def expand_device(self, pts: torch.Tensor, w: torch.Tensor) -> "Accessor":
        """expand() on device tensors without the per-call domain sync."""
        return self.accessor_from_moments(self.p2m_device(pts, w).storage)

    def expand(self, sources: SourceSet) -> "Accessor":
        acc = self.expand_device(sources.p, sources.w)
        self.flag.raise_if_set("source")
        return acc


# ------------------------------------------------------------- accessor ---

class Accessor:
    """Value / derivative queries against an L grid (reference :296-398)."""

    def __init__(self, grid: ExpansionGrid, table: MultiIndexTable,
                 counter: flops.FlopCounter | None = None, flag: DomainFlag | None = None):
        if grid.kind != "L":
            raise StageError("accessor requires an L grid")
        self.grid = grid
        self.table = table
        self._counter = counter
        self._flag = flag

    @property
    def channels(self) -> int:
        return self.grid.channels

    def _flagobj(self) -> DomainFlag:
        if self._flag is None:
            self._flag = DomainFlag()
        return self._flag

    def eval_device(self, q: torch.Tensor, mode: int, wts: torch.Tensor | None = None,
                    order: torch.Tensor | None = None, outs: dict | None = None):
        """One L2P launch; returns dict of the requested device outputs.  With a
        cell-sorted ``order`` the points are evaluated in that order (L1 reuse
        of the cell rows); outputs stay indexed by point.  ``outs`` may supply
        contiguous output tensors (e.g. row slices of a larger buffer)."""
        n, C = int(q.shape[0]), self.channels
        dev = q.device
        out = {}
        outs = outs or {}
        value = torch.empty((n, C), dtype=torch.float32, device=dev) if mode & _lib.L2P_VALUE else None
        grad = (outs.get("grad") if "grad" in outs else
                torch.empty((n, C, 3), dtype=torch.float32, device=dev)) if mode & _lib.L2P_GRAD else None
        hess = torch.empty((n, C, 6), dtype=torch.float32, device=dev) if mode & _lib.L2P_HESS else None
        wgrad = torch.empty((n, 3), dtype=torch.float32, device=dev) if mode & _lib.L2P_WGRAD else None
        st = self.grid.storage if self.grid.storage.is_contiguous() else self.grid.storage.contiguous()
        _lib.call("fc2t2_l2p", self.table.rho, self.grid.level, C, _ptr(st), _ptr(q), n, mode,
                  _ptr(order), _ptr(wts), _ptr(value), _ptr(grad), _ptr(hess), _ptr(wgrad),
                  _ptr(self._flagobj().t), _stream())
        if self._counter is not None and mode & _lib.L2P_VALUE:
            self._counter.add("l2p", flops.l2p_flops(n, self.table.rho, self.table.size))
        out.update(value=value, grad=grad, hess=hess, wgrad=wgrad)
        return out

    def _query(self, q, mode: int, key: str):
        _host_domain_check(q, "query")
        qd = to_device(q, 3, points=True)
        r = self.eval_device(qd, mode)[key]
        self._flagobj().raise_if_set("query")
        return like_input(r, q)

    def box_coeffs(self, q):
        """(coeffs (M, C, P), d (M, 3)) of the query boxes (reference :340-346)."""
        _host_domain_check(q, "query")
        qd = to_device(q, 3, points=True)
        b = find_box(self.grid.level, qd).long()
        res = self.grid.res
        lin = (b[:, 0] * res + b[:, 1]) * res + b[:, 2]
        coeffs = self.grid.data.reshape(res ** 3, self.channels, -1)[lin]
        w = level_box_width(self.grid.level)
        d = qd.double() - (-1.0 + (b.double() + 0.5) * w)
        return like_input(coeffs, q), like_input(d, q)

    def value(self, q):
        return self._query(q, _lib.L2P_VALUE, "value")

    def partials(self, q):
        return self._query(q, _lib.L2P_GRAD, "grad")

    def partials2(self, q):
        return self._query(q, _lib.L2P_HESS, "hess")

    def _vol_points(self, xs, ys, zs):
        xs, ys, zs = (np.atleast_1d(np.asarray(a, dtype=np.float64)) for a in (xs, ys, zs))
        gx, gy, gz = np.meshgrid(xs, ys, zs, indexing="ij")
        pts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
        return pts, (xs.size, ys.size, zs.size)

    def value_vol(self, xs, ys, zs):
        pts, shape = self._vol_points(xs, ys, zs)
        v = self.value(pts)
        return np.moveaxis(v.reshape(*shape, self.channels), 3, 0)

    def partials_vol(self, xs, ys, zs):
        pts, shape = self._vol_points(xs, ys, zs)
        v = self.partials(pts)
        return np.moveaxis(v.reshape(*shape, self.channels, 3), 3, 0)

    def partials2_vol(self, xs, ys, zs):
        pts, shape = self._vol_points(xs, ys, zs)
        v = self.partials2(pts)
        return np.moveaxis(v.reshape(*shape, self.channels, 6), 3, 0)
