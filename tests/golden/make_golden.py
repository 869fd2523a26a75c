"""Generate golden vectors from the REFERENCE implementation.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [part ...]

Writes small compressed .npz fixtures next to this script.  Inputs are drawn
in float64, quantised to float32 (the device dtype) and fed to the reference
as float64, per the parity protocol in SURVEY.md section 8(c).  Nothing at
test time imports the reference; the GPU box only sees these files.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import fc2t2.multiindex as rmi  # noqa: E402

rmi.MAX_ORDER = 6  # harness-only patch for config 5 (rho = 6), SURVEY.md 8(c)

from fc2t2.expansion import Engine, SourceSet, find_box  # noqa: E402
from fc2t2.kernel import KernelModel, fit_m2l_tables  # noqa: E402
from fc2t2.layers import explicit_forward, explicit_jvp  # noqa: E402
from fc2t2.multiindex import build_table  # noqa: E402


def q32(a):
    """float32 quantisation kept strictly inside (-1, 1)."""
    a = np.asarray(a, dtype=np.float64).astype(np.float32)
    one = np.nextafter(np.float32(1), np.float32(0))
    return np.clip(a, -one, one).astype(np.float64)


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    size = os.path.getsize(OUT / f"{name}.npz")
    print(f"  {name}.npz  {size / 1024:.1f} KiB", flush=True)


def part_multiindex():
    out = {f"entries_rho{r}": build_table(r).entries for r in range(1, 7)}
    save("multiindex", **out)


def part_find_box():
    rng = np.random.default_rng(11)
    special = np.array([-0.999, 0.0, 0.999, -1e-40, 1e-40, -0.0, 0.5, -0.5, 0.25, -0.25,
                        np.nextafter(np.float32(1), np.float32(0)),
                        -np.nextafter(np.float32(1), np.float32(0)),
                        np.nextafter(np.float32(0.5), np.float32(0)),
                        np.nextafter(np.float32(-0.5), np.float32(0)),
                        1.0 / 64, -1.0 / 64, 3.0 / 128, -3.0 / 128], dtype=np.float32)
    # values one float32 ulp around every plane of the level-6 grid
    planes = (-1.0 + np.arange(1, 128) * (2.0 / 128)).astype(np.float32)
    near = np.concatenate([planes, np.nextafter(planes, np.float32(2)),
                           np.nextafter(planes, np.float32(-2))])
    rnd = rng.uniform(-1, 1, 3000).astype(np.float32)
    vals = np.concatenate([special, near, rnd]).astype(np.float32)
    vals = vals[np.abs(vals) < 1]
    n = vals.size // 3 * 3
    pts = vals[:n].reshape(-1, 3).astype(np.float64)
    # also every special value on every axis
    sp = np.stack(np.meshgrid(special, special, special[:4], indexing="ij"), -1).reshape(-1, 3)
    pts = np.concatenate([pts, sp.astype(np.float64)])
    out = {"pts": pts.astype(np.float32)}
    for level in range(2, 8):
        out[f"box_l{level}"] = find_box(level, pts).astype(np.int32)
    out["known"] = find_box(2, np.array([[-0.999, 0.0, 0.999]]))  # test_expansion.py:24-30
    save("find_box", **out)


CFG_TABLES = {
    "cfg1": (200.0, 4, 4),    # config 1 (level 4, alpha 200)
    "cfg2": (1000.0, 5, 4),   # configs 2-4 (level 5, alpha 1000)
    "cfg5": (4000.0, 6, 6),   # config 5 (level 6, alpha 4000, rho 6)
    "small": (50.0, 3, 4),    # the reference's layer-test engine
}


def part_tables():
    for name, (alpha, levels, rho) in CFG_TABLES.items():
        t0 = time.time()
        tabs = fit_m2l_tables(KernelModel("gaussian", alpha, rho), levels, lsq=True, check=False)
        out = {"alpha": alpha, "levels": levels, "rho": rho}
        rng = np.random.default_rng(3)
        for key, t in list(("far%d" % l, t) for l, t in tabs["far"].items()) + [("near", tabs["near"])]:
            out[f"{key}_offsets"] = t.offsets.astype(np.int8)
            out[f"{key}_hole"] = t.hole
            out[f"{key}_active"] = t.active
            out[f"{key}_coef_sum"] = t.coeffs.sum(axis=(1, 2))
            out[f"{key}_coef_absmax"] = np.abs(t.coeffs).max(axis=(1, 2))
            act = np.flatnonzero(t.active)
            if act.size:
                pick = np.unique(np.concatenate([act[:1], act[-1:], rng.choice(act, 3)]))
                out[f"{key}_sample_idx"] = pick
                out[f"{key}_sample_coef"] = t.coeffs[pick]
            out[f"{key}_fit_residual"] = t.fit_residual
        save(f"tables_{name}", **out)
        print(f"    ({time.time() - t0:.1f}s)")


def part_expansion():
    """Stage outputs of the reference engine (test_expansion.py fixture shape)."""
    rng = np.random.default_rng(7)
    eng = Engine(KernelModel("gaussian", 200.0, 4), 4, lsq=True, check_admissibility=False)
    p = q32(rng.uniform(-0.95, 0.95, (1000, 3)))
    w = q32(rng.normal(size=(1000, 2)))
    q = q32(rng.uniform(-0.95, 0.95, (1000, 3)))
    acc = eng.expand(SourceSet(p, w))
    m = eng.p2m(SourceSet(p[:60], w[:60]))
    occ = np.argwhere(np.abs(m.data).sum(axis=(3, 4)) > 0)
    save("expansion_l4", p=p.astype(np.float32), w=w.astype(np.float32), q=q.astype(np.float32),
         value=acc.value(q), partials=acc.partials(q), partials2=acc.partials2(q),
         p2m_cells=occ.astype(np.int32), p2m_moments=m.data[occ[:, 0], occ[:, 1], occ[:, 2]],
         flops_p2m=eng.flops.stages["p2m"], flops_m2l=eng.flops.stages["m2l"],
         flops_m2m=eng.flops.stages["m2m"], flops_l2l=eng.flops.stages["l2l"])
    # L2L / M2M on a random coarse grid at level 3 (values at points)
    g = eng.zero_grid(3, 1, "L")
    g.data[:] = q32(rng.normal(size=g.data.shape))
    fine = eng.l2l(g)
    qq = q32(rng.uniform(-0.999, 0.999, (300, 3)))
    from fc2t2.expansion import Accessor
    save("l2l_l3", coarse=g.data.astype(np.float32), q=qq.astype(np.float32),
         fine_value=Accessor(fine, eng.table).value(qq))


def part_explicit_cfg1():
    """BASELINE config 1: 2D points lifted to z = 0.03125."""
    rng = np.random.default_rng(2021)
    n = m = 4096
    xy = rng.uniform(-1, 1, (n, 2))
    p = q32(np.concatenate([xy, np.full((n, 1), 0.03125)], axis=1))
    w = q32(rng.normal(size=(n, 1)))
    qxy = rng.uniform(-1, 1, (m, 2))
    q = q32(np.concatenate([qxy, np.full((m, 1), 0.03125)], axis=1))
    yb = q32(rng.normal(size=(m, 1)))
    t0 = time.time()
    eng = Engine(KernelModel("gaussian", 200.0, 4), 4, lsq=True, check_admissibility=False)
    t1 = time.time()
    res = explicit_forward(eng, SourceSet(p, w), q)
    g = explicit_jvp(yb, res)
    t2 = time.time()
    save("explicit_cfg1", p=p.astype(np.float32), w=w.astype(np.float32),
         q=q.astype(np.float32), y_bar=yb.astype(np.float32), values=res.values,
         w_bar=g.w_bar, p_bar=g.p_bar, q_bar=g.q_bar, t_engine=t1 - t0, t_layer=t2 - t1)


def _explicit_at_geometry(name, seed, alpha, levels, rho, n, m, q_sub):
    """Explicit layer fwd + jvp at a BASELINE config's own geometry (level,
    alpha, rho), reduced N and M.  Stores values, w_bar, p_bar, q_bar and the
    device-comparable interaction lists (ref layers.py:167-188,
    expansion.py:268-281)."""
    rng = np.random.default_rng(seed)
    p = q32(rng.uniform(-1, 1, (n, 3)))
    w = q32(rng.normal(0.0, 0.1, (n, 1)))
    q = q32(rng.uniform(-1, 1, (m, 3)))
    yb = q32(rng.normal(size=(m, 1)))
    t0 = time.time()
    eng = Engine(KernelModel("gaussian", alpha, rho), levels, lsq=True, check_admissibility=False)
    t1 = time.time()
    res = explicit_forward(eng, SourceSet(p, w), q)
    t2 = time.time()
    g = explicit_jvp(yb, res)
    t3 = time.time()
    print(f"    engine {t1 - t0:.1f}s fwd {t2 - t1:.1f}s jvp {t3 - t2:.1f}s", flush=True)
    # the forward's finest L grid sampled at q_sub cells (checks the cascade
    # itself, not only through L2P)
    data = res.accessor.grid.data
    cells = rng.integers(0, data.shape[0], (q_sub, 3))
    out = dict(p=p.astype(np.float32), w=w.astype(np.float32), q=q.astype(np.float32),
               y_bar=yb.astype(np.float32), values=res.values, w_bar=g.w_bar, p_bar=g.p_bar,
               q_bar=g.q_bar, L_cells=cells.astype(np.int32),
               L_rows=data[cells[:, 0], cells[:, 1], cells[:, 2]],
               alpha=alpha, levels=levels, rho=rho, t_engine=t1 - t0, t_fwd=t2 - t1,
               t_jvp=t3 - t2, expansion_count=eng.expansion_count)
    for lvl, t in eng.m2l_tables["far"].items():
        out[f"far{lvl}_active"] = t.active
        out[f"far{lvl}_offsets"] = t.offsets.astype(np.int8)
    out["near_active"] = eng.m2l_tables["near"].active
    # large float64 outputs stored as float32 (adds <= 6e-8 relative, far
    # below the 1e-5 gate) to keep the fixture small
    for k in ("values", "w_bar", "p_bar", "q_bar"):
        out[k] = out[k].astype(np.float32)
    save(name, **out)


def part_explicit_cfg2():
    """BASELINE config 2 geometry: level 5 (64^3), alpha 1000, rho 4; 2^16 + 2^16 points."""
    _explicit_at_geometry("explicit_cfg2", 2022, 1000.0, 5, 4, 1 << 16, 1 << 16, 512)


def part_explicit_cfg5():
    """BASELINE config 5 geometry: level 6 (128^3), alpha 4000, rho 6 (P = 84);
    2^16 sources, 4096 queries (rho = 6 needs the MAX_ORDER patch above)."""
    _explicit_at_geometry("explicit_cfg5", 2025, 4000.0, 6, 6, 1 << 16, 4096, 256)


PARTS = {
    "explicit_cfg2": part_explicit_cfg2,
    "explicit_cfg5": part_explicit_cfg5,
    "multiindex": part_multiindex,
    "find_box": part_find_box,
    "tables": part_tables,
    "expansion": part_expansion,
    "explicit_cfg1": part_explicit_cfg1,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(PARTS)
    for nm in names:
        print(nm, flush=True)
        PARTS[nm]()
