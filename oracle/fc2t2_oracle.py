"""CPU oracle for the FC2T2 hot path -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference algorithm
(/root/reference/pkg/src/fc2t2) used as the
parity checker for the CUDA path.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg may import it; the
product package never does.

Pinned: tests/test_oracle_golden.py checks every function here against golden
vectors produced by the reference itself (tests/golden/make_golden.py, run in
the build container where /root/reference is importable).

Each function cites the reference file:line it restates.  The arithmetic
follows the reference's float64 order where that matters for integer outputs
(cell indices, interaction masks); elsewhere it is an independent
re-expression with the same semantics.
"""

from __future__ import annotations

import math
from itertools import product

import numpy as np

COARSEST = 2          # kernel.py:38
REACH = 3             # kernel.py:39
PRUNE = 1e-16         # kernel.py:260 (prune_tol default)


# ------------------------------------------------------------ multiindex ---

def mi_entries(rho: int) -> np.ndarray:
    """Graded-lex multi-indices |n| <= rho (multiindex.py:74-96, key :84)."""
    e = sorted((t for t in product(range(rho + 1), repeat=3) if sum(t) <= rho),
               key=lambda t: (sum(t), t))
    return np.array(e, dtype=np.int64)


def mi_fact(e: np.ndarray) -> np.ndarray:
    """n1! n2! n3! per entry (multiindex.py:66-71)."""
    return np.array([math.factorial(a) * math.factorial(b) * math.factorial(c)
                     for a, b, c in e], dtype=np.float64)


def mi_lookup(e: np.ndarray) -> dict:
    return {tuple(int(v) for v in row): i for i, row in enumerate(e)}


# ---------------------------------------------------------------- kernel ---

def res_of(level: int) -> int:
    return 2 ** (level + 1)            # kernel.py:62-64


def width_of(level: int) -> float:
    return 2.0 / res_of(level)         # kernel.py:67-69


def monos(e: np.ndarray, d: np.ndarray) -> np.ndarray:
    """Rows d^n/n! (expansion.py:96-113): (m, 3) -> (m, P), from per-axis power
    tables by repeated multiplication (the reference's own scheme; ``**`` is
    several times slower and would understate the CPU baseline)."""
    d = np.atleast_2d(np.asarray(d, dtype=np.float64))
    rho = int(e.max()) if e.size else 0
    pows = np.empty((3, d.shape[0], rho + 1))
    pows[:, :, 0] = 1.0
    for k in range(1, rho + 1):
        pows[:, :, k] = pows[:, :, k - 1] * d.T
    out = pows[0][:, e[:, 0]]
    out *= pows[1][:, e[:, 1]]
    out *= pows[2][:, e[:, 2]]
    out /= mi_fact(e)[None, :]
    return out


def monos_pow(e: np.ndarray, d: np.ndarray) -> np.ndarray:
    """The LSQ basis rows d^n/n! exactly as kernel.py:147-153 builds them
    (generic ``**``; the table fit's pinv amplifies rounding differences)."""
    d = np.atleast_2d(d)
    return (d[:, None, :] ** e[None, :, :]).prod(axis=2) / mi_fact(e)[None, :]


def stencil(reach: int) -> np.ndarray:
    """meshgrid-'ij' offsets (kernel.py:207-210)."""
    r = np.arange(-reach, reach + 1)
    ox, oy, oz = np.meshgrid(r, r, r, indexing="ij")
    return np.stack([ox.ravel(), oy.ravel(), oz.ravel()], axis=1)


def active_mask(alpha: float, offsets: np.ndarray, width: float, hole: np.ndarray) -> np.ndarray:
    """Interaction list: outside the hole and psi(gap) > 1e-16 (kernel.py:213-217, :275)."""
    gap = np.maximum(np.abs(offsets) - 1, 0) * width
    peak = np.exp(-alpha * np.sum(gap * gap, axis=-1))
    return ~hole & (peak > PRUNE)


_LSQ_CACHE: dict = {}


def lsq_matrix(alpha: float, e: np.ndarray, width: float, off, nodes: int = 6) -> np.ndarray:
    """Joint LSQ fit A = pinv(V) Psi pinv(V)^T, returned as [k, n]
    (kernel.py:180-204), dense and literal."""
    key = (e.shape[0], width, nodes)
    if key not in _LSQ_CACHE:
        k = np.arange(nodes)
        x1 = np.cos((2 * k + 1) * np.pi / (2 * nodes)) * (width / 2.0)
        g = np.stack(np.meshgrid(x1, x1, x1, indexing="ij"), axis=-1).reshape(-1, 3)
        _LSQ_CACHE[key] = (g, np.linalg.pinv(monos_pow(e, g)))
    g, Pi = _LSQ_CACHE[key]
    c = np.asarray(off, dtype=np.float64) * width
    diff = c[None, None, :] + g[:, None, :] - g[None, :, :]        # p-node, q-node
    Psi = np.exp(-alpha * np.sum(diff * diff, axis=-1))
    return (Pi @ Psi @ Pi.T).T


def taylor_matrix(alpha: float, e: np.ndarray, rho: int, width: float, off) -> np.ndarray:
    """Pure Taylor entries (-1)^|k| d^(k+n) psi (kernel.py:168-178) as [k, n]."""
    c = np.asarray(off, dtype=np.float64) * width
    H = []
    for a in range(3):
        h = np.empty(2 * rho + 1)
        h[0] = math.exp(-alpha * c[a] ** 2)
        h[1] = -2.0 * alpha * c[a] * h[0]
        for n in range(1, 2 * rho):
            h[n + 1] = -2.0 * alpha * (c[a] * h[n] + n * h[n - 1])
        H.append(h)
    P = e.shape[0]
    out = np.zeros((P, P))
    for i in range(P):
        for j in range(P):
            s = e[i] + e[j]
            if np.all(s <= rho):
                out[i, j] = (-1.0) ** int(e[i].sum()) * H[0][s[0]] * H[1][s[1]] * H[2][s[2]]
    return out


def fit_tables(alpha: float, rho: int, levels: int, lsq: bool = True) -> dict:
    """{"far": {level: dict}, "near": dict} like fit_m2l_tables (kernel.py:257-300),
    without the admissibility probe."""
    e = mi_entries(rho)
    P = e.shape[0]

    def build(level, offsets, hole, near):
        w = width_of(level)
        act = active_mask(alpha, offsets, w, hole)
        co = np.zeros((offsets.shape[0], P, P))
        for i in np.flatnonzero(act):
            co[i] = lsq_matrix(alpha, e, w, offsets[i]) if lsq else \
                taylor_matrix(alpha, e, rho, w, offsets[i])
        return {"level": level, "near": near, "offsets": offsets, "hole": hole,
                "active": act, "coeffs": co}

    far = {}
    for level in range(COARSEST, levels + 1):
        off = stencil(res_of(level) - 1 if level == COARSEST else REACH)
        far[level] = build(level, off, np.all(np.abs(off) <= 1, axis=1), False)
    off = stencil(1)
    return {"far": far, "near": build(levels, off, np.zeros(27, bool), True)}


# ------------------------------------------------------------- expansion ---

def find_box(level: int, q) -> np.ndarray:
    """floor((q + 1) res / 2) clipped (expansion.py:85-93)."""
    res = res_of(level)
    b = np.floor((np.asarray(q, dtype=np.float64) + 1.0) * (res / 2.0)).astype(np.int64)
    return np.clip(b, 0, res - 1)


def box_centers(level: int, b) -> np.ndarray:
    return -1.0 + (np.asarray(b, dtype=np.float64) + 0.5) * width_of(level)   # :79-82


class Oracle:
    """The FC2T2 pipeline in float64 (expansion.py:154-285, layers.py:158-188)."""

    def __init__(self, alpha: float, rho: int, levels: int, lsq: bool = True, tables=None):
        self.alpha, self.rho, self.levels = float(alpha), int(rho), int(levels)
        self.e = mi_entries(rho)
        self.P = self.e.shape[0]
        self.fact = mi_fact(self.e)
        self.lookup = mi_lookup(self.e)
        self.tables = tables if tables is not None else fit_tables(alpha, rho, levels, lsq)
        self.expansions = 0

    # P2M (expansion.py:186-198)
    def p2m(self, p: np.ndarray, w: np.ndarray) -> np.ndarray:
        p = np.asarray(p, dtype=np.float64).reshape(-1, 3)
        w = np.asarray(w, dtype=np.float64)
        w = w.reshape(p.shape[0], w.shape[-1] if w.ndim > 1 else 1)
        res = res_of(self.levels)
        grid = np.zeros((res ** 3, w.shape[1], self.P))
        if p.shape[0]:
            b = find_box(self.levels, p)
            mono = monos(self.e, p - box_centers(self.levels, b))
            key = (b[:, 0] * res + b[:, 1]) * res + b[:, 2]
            np.add.at(grid, key, w[:, :, None] * mono[:, None, :])
        return grid.reshape(res, res, res, w.shape[1], self.P)

    def insert(self, boxes: np.ndarray, payload: np.ndarray) -> np.ndarray:
        """Scatter per-item (C, P) payloads (layers.py:144-153)."""
        res = res_of(self.levels)
        grid = np.zeros((res ** 3, payload.shape[1], self.P))
        key = (boxes[:, 0] * res + boxes[:, 1]) * res + boxes[:, 2]
        np.add.at(grid, key, payload)
        return grid.reshape(res, res, res, payload.shape[1], self.P)

    def shift(self, d: np.ndarray, up: bool) -> np.ndarray:
        """Binomial re-centering K (expansion.py:116-132); up = m2m."""
        P = self.P
        K = np.zeros((P, P))
        for i in range(P):
            for j in range(P):
                diff = self.e[i] - self.e[j] if up else self.e[j] - self.e[i]
                if np.all(diff >= 0):
                    K[i, j] = np.prod(d ** diff) / np.prod([math.factorial(int(x)) for x in diff])
        return K

    def m2m(self, fine: np.ndarray, fine_level: int) -> np.ndarray:
        """expansion.py:200-213."""
        r = fine.shape[0] // 2
        coarse = np.zeros((r, r, r) + fine.shape[3:])
        wf = width_of(fine_level)
        for c in product((0, 1), repeat=3):
            K = self.shift((np.array(c) - 0.5) * wf, True)
            coarse += fine[c[0]::2, c[1]::2, c[2]::2] @ K.T
        return coarse

    def l2l(self, coarse: np.ndarray, coarse_level: int) -> np.ndarray:
        """expansion.py:215-225 (assigns; the caller adds)."""
        r = coarse.shape[0] * 2
        fine = np.zeros((r, r, r) + coarse.shape[3:])
        wf = width_of(coarse_level + 1)
        for c in product((0, 1), repeat=3):
            K = self.shift((np.array(c) - 0.5) * wf, False)
            fine[c[0]::2, c[1]::2, c[2]::2] = coarse @ K.T
        return fine

    @staticmethod
    def _slices(res: int, delta: int, parity):
        """Target/source index ranges for one axis (expansion.py:135-151)."""
        step = 1 if parity is None else 2
        lo, hi = max(0, -delta), min(res - 1, res - 1 - delta)
        if parity is not None:
            lo += (lo % 2 != parity)
            hi -= (hi % 2 != parity)
        if lo > hi:
            return None
        return slice(lo, hi + 1, step), slice(lo + delta, hi + delta + 1, step)

    def m2l(self, m: np.ndarray, tab: dict) -> np.ndarray:
        """expansion.py:227-264, per active offset a strided slab matmul."""
        out = np.zeros_like(m)
        res = m.shape[0]
        par_st = (not tab["near"]) and tab["level"] != COARSEST
        for i in np.flatnonzero(tab["active"]):
            off = tab["offsets"][i]
            sl = []
            for a in range(3):
                d = int(off[a])
                par = (1 if d == -3 else 0) if (par_st and abs(d) == 3) else None
                s = self._slices(res, d, par)
                if s is None:
                    break
                sl.append(s)
            else:
                tgt = tuple(s[0] for s in sl)
                src = tuple(s[1] for s in sl)
                # one contiguous 2-D GEMM per offset, as expansion.py:251-253
                block = np.ascontiguousarray(m[src])
                prod = block.reshape(-1, block.shape[-1]) @ tab["coeffs"][i].T
                out[tgt] += prod.reshape(block.shape)
        return out

    def cascade(self, m_fine: np.ndarray) -> np.ndarray:
        """expand_from_moments (expansion.py:268-281): finest L grid."""
        self.expansions += 1
        M = {self.levels: m_fine}
        for l in range(self.levels, COARSEST, -1):
            M[l - 1] = self.m2m(M[l], l)
        L = self.m2l(M[COARSEST], self.tables["far"][COARSEST])
        for l in range(COARSEST + 1, self.levels + 1):
            L = self.m2l(M[l], self.tables["far"][l]) + self.l2l(L, l - 1)
        return L + self.m2l(M[self.levels], self.tables["near"])

    def expand(self, p, w) -> np.ndarray:
        return self.cascade(self.p2m(p, w))

    # L2P (expansion.py:335-373)
    def shift_map(self, s) -> np.ndarray:
        return np.array([self.lookup.get((int(n[0] + s[0]), int(n[1] + s[1]), int(n[2] + s[2])), -1)
                         for n in self.e])

    def evaluate(self, L: np.ndarray, q, level: int | None = None, what: str = "value"):
        level = self.levels if level is None else level
        q = np.atleast_2d(np.asarray(q, dtype=np.float64))
        b = find_box(level, q)
        co = L[b[:, 0], b[:, 1], b[:, 2]]                       # (m, C, P)
        mono = monos(self.e, q - box_centers(level, b))
        if what == "value":
            return np.einsum("mcp,mp->mc", co, mono)
        shifts = ([(1, 0, 0), (0, 1, 0), (0, 0, 1)] if what == "grad" else
                  [(2, 0, 0), (0, 2, 0), (0, 0, 2), (1, 1, 0), (1, 0, 1), (0, 1, 1)])
        out = np.zeros(co.shape[:2] + (len(shifts),))
        for k, s in enumerate(shifts):
            idx = self.shift_map(s)
            ok = idx >= 0
            out[:, :, k] = np.einsum("mcp,mp->mc", co[:, :, idx[ok]], mono[:, ok])
        return out

    # explicit layer (layers.py:167-188)
    def explicit(self, p, w, q, y_bar):
        """Forward values and (w_bar, p_bar, q_bar) of the explicit layer."""
        p = np.atleast_2d(np.asarray(p, dtype=np.float64))
        w = np.asarray(w, dtype=np.float64).reshape(p.shape[0], -1)
        q = np.atleast_2d(np.asarray(q, dtype=np.float64))
        yb = np.asarray(y_bar, dtype=np.float64).reshape(q.shape[0], -1)
        L = self.expand(p, w)
        values = self.evaluate(L, q)
        q_bar = np.einsum("mc,mca->ma", yb, self.evaluate(L, q, what="grad"))
        B = self.expand(q, yb)
        w_bar = self.evaluate(B, p)
        p_bar = np.einsum("nc,nca->na", w, self.evaluate(B, p, what="grad"))
        return values, w_bar, p_bar, q_bar


# --------------------------------------------------------------- brute force ---

def naive_sum(alpha: float, p, w, q) -> np.ndarray:
    """Direct O(NM) sum (oracle.py:20-34)."""
    p, q = np.atleast_2d(p), np.atleast_2d(q)
    w = np.asarray(w, dtype=np.float64).reshape(p.shape[0], -1)
    out = np.empty((q.shape[0], w.shape[1]))
    for lo in range(0, q.shape[0], 2048):
        d = q[lo:lo + 2048, None, :] - p[None, :, :]
        out[lo:lo + 2048] = np.exp(-alpha * np.sum(d * d, axis=2)) @ w
    return out


def naive_grads(alpha: float, p, w, q) -> np.ndarray:
    """Direct gradient sum (oracle.py:37-55)."""
    p, q = np.atleast_2d(p), np.atleast_2d(q)
    w = np.asarray(w, dtype=np.float64).reshape(p.shape[0], -1)
    out = np.empty((q.shape[0], w.shape[1], 3))
    for lo in range(0, q.shape[0], 2048):
        d = q[lo:lo + 2048, None, :] - p[None, :, :]
        k = np.exp(-alpha * np.sum(d * d, axis=2))
        out[lo:lo + 2048] = np.einsum("mna,nc->mca", -2.0 * alpha * d * k[:, :, None], w)
    return out


def rel_l2(fast, exact) -> float:
    """OracleReport.compare's rel-L2 (oracle.py:281-297)."""
    fast = np.asarray(fast, dtype=np.float64)
    exact = np.asarray(exact, dtype=np.float64)
    den = float(np.linalg.norm(exact))
    num = float(np.linalg.norm(fast - exact))
    return num / den if den > 0 else num
