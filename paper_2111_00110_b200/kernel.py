"""Kernel model and per-level M2L tables (host precompute, float64).

Restates the reference's table construction (``pkg/src/fc2t2/kernel.py``) in
its own vectorised form; the *integer* outputs (offsets, hole, active mask =
the interaction lists) are bit-exact with the reference and the fitted
coefficients agree to ~1e-12 (tests/test_tables.py pins both against golden
vectors generated from the reference).

* Gaussian kernel psi(x) = exp(-alpha |x|^2) with per-axis Hermite-recurrence
  derivatives (reference kernel.py:72-121).
* Level geometry: res = 2^(level+1) boxes per axis on (-1, 1)^3
  (reference kernel.py:62-69).
* Tables: the coarsest level (2) uses the full reach res-1 stencil, finer far
  levels reach 3 with the |off|_inf <= 1 hole; the finest level additionally
  owns a hole-less 3x3x3 near table (reference kernel.py:257-300).  An
  offset is active iff it is outside the hole and the peak box-pair
  interaction psi(max(|off|-1, 0) * width) exceeds 1e-16 (kernel.py:213-217,
  :275).
* LSQ coefficients: A = pinv(V) Psi pinv(V)^T over a 6^3 Chebyshev tensor grid
  per box (reference kernel.py:180-204), stored transposed [k_local,
  n_moment].  Psi is a Kronecker product of per-axis node-pair kernels, so the
  two-sided product is evaluated one axis at a time instead of forming the
  216 x 216 pair matrix.

On a GPU the LSQ fit itself runs on the device (``_lsq_tables_device`` ->
``fc2t2_fit_tables``, csrc/tables.cu: one CTA per offset, float64, SURVEY
8(f)3); only pinv(V) -- one small SVD per level -- stays on the host.
``FC2T2_HOST_TABLES=1`` (or a machine without CUDA) selects the numpy fit
above, which the same golden tests pin.

Everything here runs once per Engine.  The device copy (fp32, padded, grouped
into per-parity interaction lists) is made by ``expansion.Engine``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .multiindex import MultiIndexTable, build_table

COARSEST_LEVEL = 2
FAR_REACH = 3
DEFAULT_ALPHA = {2: 12.0, 3: 50.0, 4: 200.0, 5: 1000.0, 6: 4000.0}
PRUNE_TOL = 1e-16


class KernelConfigError(ValueError):
    """Unsupported kernel configuration (reference kernel.py:46-47)."""


class AdmissibilityError(RuntimeError):
    """Kernel too sharp for the grid hierarchy (reference kernel.py:50-59)."""

    def __init__(self, level: int, worst: float, tol: float):
        self.level = level
        self.worst = worst
        super().__init__(f"kernel fails admissibility at level {level}: worst probe "
                         f"error {worst:.3e} exceeds tolerance {tol:.3e}")


def level_resolution(level: int) -> int:
    return 1 << (level + 1)


def level_box_width(level: int) -> float:
    return 2.0 / level_resolution(level)


@dataclass(frozen=True)
class KernelModel:
    """Gaussian difference kernel with analytic partials (reference kernel.py:72-121)."""

    family: str
    alpha: float
    rho: int
    table: MultiIndexTable = field(repr=False, default=None)

    def __post_init__(self):
        if self.family != "gaussian":
            raise KernelConfigError(f"unsupported kernel family: {self.family!r}")
        if not self.alpha > 0:
            raise KernelConfigError("alpha must be positive")
        if self.table is None:
            object.__setattr__(self, "table", build_table(self.rho))

    def psi(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        return np.exp(-self.alpha * np.sum(x * x, axis=-1))

    def axis_derivatives(self, max_order: int, coords) -> np.ndarray:
        """Rows n = 0..max_order of d^n/dx^n exp(-alpha x^2)."""
        x = np.atleast_1d(np.asarray(coords, dtype=np.float64))
        h = np.empty((max_order + 1, x.size))
        h[0] = np.exp(-self.alpha * x ** 2)
        two_a = -2.0 * self.alpha
        if max_order >= 1:
            h[1] = two_a * x * h[0]
        for n in range(1, max_order):
            h[n + 1] = two_a * (x * h[n] + n * h[n - 1])
        return h

    def partial(self, order, x) -> np.ndarray:
        order = tuple(int(o) for o in order)
        if sum(order) > 2 * self.rho:
            raise KernelConfigError(
                f"partial order {order} exceeds supported total order {2 * self.rho}")
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        top = max(order)
        out = np.ones(x.shape[0])
        for a in range(3):
            out = out * self.axis_derivatives(top, x[:, a])[order[a]]
        return out


@dataclass
class M2LTable:
    """One level's stencil (field layout of reference kernel.py:124-141)."""

    level: int
    nearfield: bool
    offsets: np.ndarray        # (K, 3) int64, source index - target index
    coeffs: np.ndarray         # (K, P, P) float64, [k_local, n_moment]
    hole: np.ndarray           # (K,) bool
    active: np.ndarray         # (K,) bool
    fit_residual: float
    box_width: float


def stencil_offsets(reach: int) -> np.ndarray:
    """All integer offsets in [-reach, reach]^3, x slowest (meshgrid 'ij')."""
    r = np.arange(-reach, reach + 1)
    return np.stack(np.meshgrid(r, r, r, indexing="ij"), axis=-1).reshape(-1, 3)


def interaction_mask(kernel: KernelModel, offsets: np.ndarray, width: float,
                     hole: np.ndarray, prune_tol: float = PRUNE_TOL) -> np.ndarray:
    """Active offsets: outside the hole and peak interaction above prune_tol.
    Same float64 expression as reference kernel.py:213-217 / :275 so the mask
    is bit-exact."""
    gap = np.maximum(np.abs(offsets) - 1, 0) * width
    return ~hole & (kernel.psi(gap) > prune_tol)


def _cheb(n: int) -> np.ndarray:
    return np.cos((2 * np.arange(n) + 1) * np.pi / (2 * n))


def monomial_rows(table: MultiIndexTable, pts: np.ndarray) -> np.ndarray:
    """(G, P) rows of d^n / n! at points (G, 3)."""
    e = table.entries
    return np.prod(pts[:, None, :] ** e[None, :, :], axis=2) / table.entry_factorial()


def _lsq_tables(kernel: KernelModel, width: float, offsets: np.ndarray,
                nodes: int) -> tuple[np.ndarray, float]:
    t = kernel.table
    P, G = t.size, nodes
    x1 = _cheb(G) * (width / 2.0)
    grid = np.stack(np.meshgrid(x1, x1, x1, indexing="ij"), axis=-1).reshape(-1, 3)
    V = monomial_rows(t, grid)                                  # (G^3, P)
    Pv = np.linalg.pinv(V).reshape(P, G, G, G)                  # (P, gx, gy, gz)
    diff = x1[:, None] - x1[None, :]                            # d_p - d_q
    axis_vals = {int(d): np.exp(-kernel.alpha * (d * width + diff) ** 2)
                 for d in np.unique(offsets)}
    out = np.empty((offsets.shape[0], P, P))
    resid = 0.0
    chunk = 256
    for lo in range(0, offsets.shape[0], chunk):
        off = offsets[lo:lo + chunk]
        ex = np.stack([axis_vals[int(o)] for o in off[:, 0]])   # (B, G, G) [p_node, q_node]
        ey = np.stack([axis_vals[int(o)] for o in off[:, 1]])
        ez = np.stack([axis_vals[int(o)] for o in off[:, 2]])
        # (Psi Pv^T)[b, (a,b,c), k] one axis at a time over the q-side nodes
        w = np.einsum("kxyz,Bcz->Bkxyc", Pv, ez)
        w = np.einsum("Bkxyc,Bby->Bkxbc", w, ey)
        w = np.einsum("Bkxbc,Bax->Bkabc", w, ex)                 # (B, k, a, b, c)
        A = np.einsum("nabc,Bkabc->Bnk", Pv, w)                  # A[n_moment, k_local]
        out[lo:lo + chunk] = np.swapaxes(A, 1, 2)
        # fit residual max |V A V^T - Psi| (reference kernel.py:202)
        fit = V[None] @ A @ V.T[None]
        psi = (ex[:, :, None, None, :, None, None] * ey[:, None, :, None, None, :, None]
               * ez[:, None, None, :, None, None, :]).reshape(off.shape[0], G ** 3, G ** 3)
        resid = max(resid, float(np.max(np.abs(fit - psi))))
    return out, resid


def _lsq_tables_device(kernel: KernelModel, width: float, offsets: np.ndarray,
                       nodes: int) -> tuple[np.ndarray, float]:
    """_lsq_tables on the device (csrc/tables.cu): same float64 arithmetic per
    offset, summed in a different order (agrees to ~1e-13 relative)."""
    import torch

    from . import _lib
    t = kernel.table
    P, G = t.size, nodes
    x1 = _cheb(G) * (width / 2.0)
    grid = np.stack(np.meshgrid(x1, x1, x1, indexing="ij"), axis=-1).reshape(-1, 3)
    V = monomial_rows(t, grid)                                  # (G^3, P)
    Pv = np.linalg.pinv(V)                                      # (P, G^3)
    dev = torch.device("cuda", torch.cuda.current_device())
    d_pv = torch.from_numpy(np.ascontiguousarray(Pv)).to(dev)
    d_v = torch.from_numpy(np.ascontiguousarray(V)).to(dev)
    d_x = torch.from_numpy(x1).to(dev)
    d_off = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int32)).to(dev)
    K = int(offsets.shape[0])
    d_c = torch.empty((K, P, P), dtype=torch.float64, device=dev)
    d_r = torch.empty(max(K, 1), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    _lib.call("fc2t2_fit_tables", t.rho, G, d_pv.data_ptr(), d_v.data_ptr(), d_x.data_ptr(),
              float(kernel.alpha), float(width), d_off.data_ptr(), K, d_c.data_ptr(),
              d_r.data_ptr(), s)
    return d_c.cpu().numpy(), float(d_r[:K].max().item()) if K else 0.0


def _device_fit_available(nodes: int) -> bool:
    import os
    if os.environ.get("FC2T2_HOST_TABLES", "0") == "1" or nodes != 6:
        return False
    try:
        import torch
        return torch.cuda.is_available()
    except ImportError:
        return False


def _taylor_tables(kernel: KernelModel, width: float, offsets: np.ndarray) -> np.ndarray:
    """Pure Taylor re-expansion (reference kernel.py:168-178): entry [k, n] is
    (-1)^|k| d^(k+n) psi(off * width), kept only where k_a + n_a <= rho."""
    t = kernel.table
    e, rho = t.entries, t.rho
    nk = e[:, None, :] + e[None, :, :]                          # (P_k, P_n, 3)
    keep = np.all(nk <= rho, axis=2)
    sign = np.where(t.norms % 2 == 1, -1.0, 1.0)
    out = np.empty((offsets.shape[0], t.size, t.size))
    for i, off in enumerate(offsets):
        c = off * width
        h = [kernel.axis_derivatives(2 * rho, np.array([c[a]]))[:, 0] for a in range(3)]
        full = h[0][nk[..., 0]] * h[1][nk[..., 1]] * h[2][nk[..., 2]]
        out[i] = sign[:, None] * np.where(keep, full, 0.0)
    return out


def _probe_error(kernel: KernelModel, table: M2LTable, idx: int, rng) -> float:
    """Worst reproduction error over the target box of a unit source at the
    centre of the box at stencil offset idx (reference kernel.py:220-229)."""
    t = kernel.table
    w = table.box_width
    c = table.offsets[idx] * w
    local = table.coeffs[idx][:, 0]
    probes = rng.uniform(-w / 2, w / 2, size=(64, 3))
    pred = monomial_rows(t, probes) @ local
    return float(np.max(np.abs(pred - kernel.psi(c[None, :] - probes))))


def _check_admissibility(kernel, table: M2LTable, tol: float, rng) -> None:
    """Probe one table entry against the kernel (reference kernel.py:232-254):
    the near table at its self offset (0, 0, 0), with a 20x looser limit; a
    far table at its closest active offset (Chebyshev distance), if any."""
    if table.nearfield:
        probe, limit = int(np.argmax(~table.offsets.any(axis=1))), 20.0 * tol
    elif table.active.any():
        cheb = np.where(table.active, np.abs(table.offsets).max(axis=1), np.iinfo(np.int64).max)
        probe, limit = int(np.argmin(cheb)), tol
    else:
        return                      # nothing resolved at this level
    err = _probe_error(kernel, table, probe, rng)
    if err > limit:
        raise AdmissibilityError(table.level, err, limit)


def fit_m2l_tables(kernel: KernelModel, levels: int, lsq: bool = True,
                   nodes_per_axis: int = 6, admissibility_tol: float = 1e-3,
                   check: bool = True, prune_tol: float = PRUNE_TOL,
                   device: bool | None = None) -> dict:
    """``{"far": {level: M2LTable}, "near": M2LTable}`` (reference kernel.py:257-300).
    ``device`` (default: when a GPU is present) fits the LSQ tables on it."""
    if device is None:
        device = lsq and _device_fit_available(nodes_per_axis)
    lsq_fit = _lsq_tables_device if device else _lsq_tables
    if levels < COARSEST_LEVEL:
        raise KernelConfigError(f"levels must be >= {COARSEST_LEVEL}")
    rng = np.random.default_rng(0)
    P = kernel.table.size

    def build(level, offsets, hole, nearfield):
        width = level_box_width(level)
        active = interaction_mask(kernel, offsets, width, hole, prune_tol)
        coeffs = np.zeros((offsets.shape[0], P, P))
        resid = 0.0
        if active.any():
            if lsq:
                coeffs[active], resid = lsq_fit(kernel, width, offsets[active],
                                                nodes_per_axis)
            else:
                coeffs[active] = _taylor_tables(kernel, width, offsets[active])
        return M2LTable(level, nearfield, offsets, coeffs, hole, active, resid, width)

    far = {}
    for level in range(COARSEST_LEVEL, levels + 1):
        reach = level_resolution(level) - 1 if level == COARSEST_LEVEL else FAR_REACH
        offsets = stencil_offsets(reach)
        hole = np.all(np.abs(offsets) <= 1, axis=1)
        tab = build(level, offsets, hole, False)
        if check:
            _check_admissibility(kernel, tab, admissibility_tol, rng)
        far[level] = tab
    near_off = stencil_offsets(1)
    near = build(levels, near_off, np.zeros(near_off.shape[0], bool), True)
    if check:
        _check_admissibility(kernel, near, admissibility_tol, rng)
    return {"far": far, "near": near}


# ------------------------------------------------- separable finest M2L ---
#
# The Gaussian is a product over axes, and so is every finest-level table:
#   LSQ (reference kernel.py:180-204): A(o) = pinv(V) Psi(o) pinv(V)^T with
#     Psi(o) = Psi_x(o_x) (x) Psi_y(o_y) (x) Psi_z(o_z) over the 6^3 Chebyshev
#     tensor nodes and V = (V1 (x) V1 (x) V1) S, V1 the (6, rho+1) per-axis
#     rows x^m/m!, S the selection of the total-degree <= rho entries.  With
#     V1 = Q R (thin QR, R upper triangular) the total-degree subspace is
#     invariant under R (x) R (x) R, hence V = (Q (x) Q (x) Q) S R_S with
#     R_S = S^T (R (x) R (x) R) S and orthonormal (Q (x) Q (x) Q) S, so
#       coeffs(o) = A(o)^T = R_S^{-1} S^T (K(o_x) (x) K(o_y) (x) K(o_z)) S R_S^{-T},
#       K(d) = (Q^T Psi_1(d) Q)^T                     ((rho+1) x (rho+1) each);
#   Taylor (reference kernel.py:169-177): coeffs(o)[k, n] = prod_a (-1)^{k_a}
#     h(o_a w)[n_a + k_a] [n_a + k_a <= rho]  -- K(d) directly, no transforms.
# At the finest level the far (parity stencil, reference expansion.py:246-249)
# and near tables together cover, per target, the 6 x 6 x 6 box of source
# offsets {-2..3} (even target index) or {-3..2} (odd) on every axis whenever
# every stencil offset is active, so the whole finest M2L is three 1-D
# convolutions with the 7 matrices K(-3..3) between two per-axis triangular
# transforms -- ~4e3 instead of 2.6e5 multiply-adds per cell at rho = 4.  The
# orthonormal middle keeps float32 rounding at the level of the inputs
# (measured 1.3e-7 rel-L2 per coefficient vs the float64 tables; the
# monomial-basis form inv(H) (x) K (x) inv(H) loses 2e-3).

def separable_far_eligible(tables: dict, level: int, levels: int, rho: int, lsq: bool = True,
                           nodes_per_axis: int = 6) -> bool:
    """A coarse level's far table (parity stencil minus the hole, reference
    expansion.py:246-249) runs separably (three disjoint per-axis pieces,
    csrc/m2l_sep.cu) when the grid is at least 16 cells wide, the per-axis fit
    is full rank and the level has work.  Offsets the reference prunes have a
    peak interaction below PRUNE_TOL (interaction_mask); the separable form
    includes them, a change below 1e-16 of the kernel peak per unit weight."""
    if not (COARSEST_LEVEL < level < levels) or level_resolution(level) < 16:
        return False
    if lsq and rho + 1 > nodes_per_axis:
        return False
    if rho > 5:
        return False
    far = tables["far"][level]
    hole = np.abs(far.offsets).max(axis=1) <= 1
    return bool(far.active.any() and np.array_equal(far.hole, hole)
                and not (far.active & far.hole).any()
                and np.abs(far.offsets).max() == FAR_REACH)


def separable_factors(kernel: KernelModel, level: int, lsq: bool = True,
                      nodes_per_axis: int = 6) -> dict:
    """Per-axis factors of the finest-level tables: ``pre`` (R^{-T}, lower
    triangular), ``post`` (R^{-1}, upper triangular) and ``conv`` (7, rho+1,
    rho+1) = K(d) for d = -3..3, all as [out][in] float64."""
    rho = kernel.rho
    R1 = rho + 1
    width = level_box_width(level)
    if not lsq:
        conv = np.zeros((7, R1, R1))
        for i, d in enumerate(range(-3, 4)):
            h = kernel.axis_derivatives(2 * rho, np.array([d * width]))[:, 0]
            for k in range(R1):
                for n in range(R1 - k):
                    conv[i, k, n] = (-1.0) ** k * h[n + k]
        eye = np.eye(R1)
        return {"pre": eye, "post": eye.copy(), "conv": conv}
    x1 = _cheb(nodes_per_axis) * (width / 2.0)
    fact = np.array([float(np.prod(np.arange(1, m + 1))) for m in range(R1)])
    V1 = x1[:, None] ** np.arange(R1)[None, :] / fact[None, :]
    Q, R = np.linalg.qr(V1)
    sgn = np.sign(np.diag(R))
    Q, R = Q * sgn[None, :], sgn[:, None] * R
    Rinv = np.linalg.inv(R)
    pair = x1[:, None] - x1[None, :]
    conv = np.empty((7, R1, R1))
    for i, d in enumerate(range(-3, 4)):
        psi1 = kernel.axis_derivatives(0, (d * width + pair).ravel())[0].reshape(pair.shape)
        conv[i] = (Q.T @ psi1 @ Q).T
    return {"pre": Rinv.T.copy(), "post": Rinv, "conv": conv}


def separable_dense(factors: dict, table: MultiIndexTable, offset) -> np.ndarray:
    """The (P, P) [k][n] table one offset's factors represent (for tests):
    post_S @ conv_S(o) @ pre_S with X_S = S^T (X (x) X (x) X) S."""
    e = table.entries

    def kron_s(mats):
        out = np.ones((e.shape[0], e.shape[0]))
        for a in range(3):
            out = out * mats[a][e[:, a][:, None], e[:, a][None, :]]
        return out

    pre = kron_s([factors["pre"]] * 3)
    post = kron_s([factors["post"]] * 3)
    mid = kron_s([factors["conv"][int(o) + 3] for o in offset])
    return post @ mid @ pre


def separable_eligible(tables: dict, levels: int, rho: int, lsq: bool = True,
                       nodes_per_axis: int = 6) -> bool:
    """True when the finest far table activates every offset of its parity
    stencil outside the hole and the near table all 27, i.e. each finest
    target sees the full 6^3 source box; the grid is at least 32 cells wide
    (the kernels' tile); and, for LSQ tables, the per-axis fit is not rank
    deficient (rho + 1 <= nodes per axis: at rho = 6 with 6 nodes the pure
    degree-6 column is dependent on the nodes and pinv's minimum-norm
    solution does not factor per axis, so those engines keep the dense M2L)."""
    if levels <= COARSEST_LEVEL or level_resolution(levels) < 32:
        return False
    if lsq and rho + 1 > nodes_per_axis:
        return False
    far, near = tables["far"][levels], tables["near"]
    return bool(np.array_equal(far.active, ~far.hole) and near.active.all()
                and np.abs(far.offsets).max() == FAR_REACH)


