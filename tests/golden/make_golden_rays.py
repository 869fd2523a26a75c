"""Golden vectors for the ray layers from the REFERENCE implementation.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_rays.py [part ...]

Scenes follow the reference's own layer tests (tests/test_layers.py fixtures)
at larger camera sizes, plus reduced-size stand-ins for BASELINE configs 3
and 4 (same level, alpha, camera geometry and value distributions; fewer
sources and rays so the float64 reference finishes in about a minute).
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from fc2t2.expansion import Engine, SourceSet  # noqa: E402
from fc2t2.kernel import KernelModel  # noqa: E402
from fc2t2.layers import (depth_forward, depth_jvp, line_integral_forward,  # noqa: E402
                          line_integral_jvp, surface_gradient_jvp,
                          volumetric_forward, volumetric_jvp)
from fc2t2.poly1d import fit_exp_poly, quartic_roots  # noqa: E402
from fc2t2.ray import (Camera, generate_rays, line2poly, line2taylor_h,  # noqa: E402
                       segment_geometry, traverse)


def q32(a):
    a = np.asarray(a, dtype=np.float64).astype(np.float32)
    one = np.nextafter(np.float32(1), np.float32(0))
    return np.clip(a, -one, one).astype(np.float64)


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"  {name}.npz  {os.path.getsize(OUT / f'{name}.npz') / 1024:.1f} KiB", flush=True)


def seeded_direction(rng):
    """Unit vector, rejecting near-vertical ones (SURVEY 8(d) camera rule)."""
    while True:
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        if abs(u[1]) <= 0.99:
            return u


def part_poly():
    rng = np.random.default_rng(42)
    coeffs = rng.normal(size=(1000, 5))
    roots = np.full((1000, 4), np.nan)
    for i in range(1000):
        r = quartic_roots(coeffs[i])
        roots[i, :r.size] = r
    special = np.array([[24.0, -50.0, 35.0, -10.0, 1.0], [1.0, 0, 0, 0, 1.0],
                        [-1.0, 1.0, 0.0, 0.0, 1e-15], [4.0, -4.0, 5.0, -4.0, 1.0],
                        [4.0, 0.0, -5.0, 0.0, 1.0]])
    sroots = np.full((5, 4), np.nan)
    for i in range(5):
        r = quartic_roots(special[i])
        sroots[i, :r.size] = r
    save("poly1d", coeffs=coeffs, roots=roots, special=special, special_roots=sroots,
         mexp_coeffs=fit_exp_poly())


def small_scene():
    rng = np.random.default_rng(7)
    p = q32(rng.uniform(-0.6, 0.6, (40, 3)))
    w = q32(-(np.abs(rng.normal(size=(40, 1))) * 0.5 + 0.3))
    return p, w


def part_layers_small():
    """Reference layer-test scene (test_layers.py:17-35) with a 24x24 camera."""
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, lsq=True, check_admissibility=False)
    p, w = small_scene()
    cam = Camera(position=np.array([0.0, 0.0, -2.5]), look_at=np.zeros(3),
                 up=np.array([0.0, 1.0, 0.0]), fov_deg=30.0, width=24, height=24)
    b = generate_rays(cam)
    trav = traverse(b, 3)
    d, r, s = segment_geometry(trav, b, 3)
    rng = np.random.default_rng(3)
    res = depth_forward(eng, SourceSet(p, w), b, bias=0.3)
    yl = rng.normal(size=b.count)
    yg = rng.normal(size=(b.count, 3))
    gd = depth_jvp(yl, res)
    gs = surface_gradient_jvp(yg, res)
    li = line_integral_forward(eng, SourceSet(p, w), b)
    yi = rng.normal(size=(b.count, 1))
    gi = line_integral_jvp(yi, li)
    rng2 = np.random.default_rng(8)
    w_sigma = -w
    w_sigma[::7] *= -1.0
    w_color = q32(rng2.uniform(0.2, 1.0, (40, 2)))
    bg = np.array([0.4, 0.8])
    vr = volumetric_forward(eng, p, w_sigma, w_color, b, bg)
    yv = rng.normal(size=(b.count, 2))
    gv = volumetric_jvp(yv, vr)
    coeffs = res.accessor.grid.data[trav.box[:, 0], trav.box[:, 1], trav.box[:, 2]]
    polys = line2poly(coeffs, d, r, 4)
    h = rng.normal(size=(d.shape[0], 3))
    mom = line2taylor_h(d, r, s, h, 4)
    save("rays_small", p=p, w=w, origins=b.origins, directions=b.directions,
         ray_id=trav.ray_id, t0=trav.t0, t1=trav.t1, box=trav.box, offsets=trav.offsets,
         t_enter=trav.t_enter, seg_d=d[:1500], polys=polys[:1500], h=h[:1500],
         moments=mom[:1500],
         lengths=res.lengths, hit=res.hit, points=res.points, grads=res.grads, denom=res.denom,
         y_len=yl, y_grad=yg, depth_w_bar=gd.w_bar, depth_p_bar=gd.p_bar,
         surf_w_bar=gs.w_bar, surf_p_bar=gs.p_bar,
         li_values=li.values, y_li=yi, li_w_bar=gi.w_bar, li_p_bar=gi.p_bar,
         w_sigma=w_sigma, w_color=w_color, bg=bg, rgb=vr.rgb, alive=vr.alive,
         y_vol=yv, vol_w_bar=gv.w_bar, vol_p_bar=gv.p_bar)


def part_cfg3_small():
    """Config 3 geometry (level 5, alpha 1000, radius 2, fov 60, bias +0.05) with
    N = 2^14 sources and a 48x48 camera."""
    rng = np.random.default_rng(33)
    n = 1 << 14
    p = q32(rng.uniform(-1, 1, (n, 3)))
    w = q32(rng.normal(0.0, 0.1, (n, 1)))
    pos = 2.0 * seeded_direction(rng)
    cam = Camera(position=pos, look_at=np.zeros(3), up=np.array([0.0, 1.0, 0.0]),
                 fov_deg=60.0, width=48, height=48)
    b = generate_rays(cam)
    t0 = time.time()
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, lsq=True, check_admissibility=False)
    res = depth_forward(eng, SourceSet(p, w), b, bias=0.05)
    yl = rng.normal(size=b.count)
    yg = rng.normal(size=(b.count, 3))
    gd = depth_jvp(yl, res)
    gs = surface_gradient_jvp(yg, res)
    print(f"    cfg3 small: {time.time() - t0:.1f}s, hit fraction {res.hit.mean():.3f}")
    # conditioning floor: the reference's own change under a 2^-24 relative
    # perturbation of the weights (the IFT weights -y/<r, grad f> are large and
    # of both signs, so w_bar = sum_r u_r psi(p - x_r) cancels)
    pr = np.random.default_rng(0)
    wp = w * (1 + pr.normal(size=w.shape) * 2.0 ** -24)
    rp = depth_forward(eng, SourceSet(p, wp), b, bias=0.05)
    dp, sp = depth_jvp(yl, rp), surface_gradient_jvp(yg, rp)

    def rl(a, c):
        return float(np.linalg.norm(a - c) / np.linalg.norm(c))
    sens = np.array([rl(dp.w_bar, gd.w_bar), rl(dp.p_bar, gd.p_bar), rl(sp.w_bar, gs.w_bar),
                     rl(sp.p_bar, gs.p_bar)])
    print(f"    self-sensitivity (depth w,p / surface w,p): {sens}")
    # float32 floor: the reference's own adjoints when the ONLY change is
    # rounding its float64 finest L grid to float32 in the forward (the roots,
    # gradients and Hessians then come from a correctly rounded float32 field)
    orig = Engine.expand

    def rounded_expand(self, src):
        acc = orig(self, src)
        acc.grid.data[...] = acc.grid.data.astype(np.float32).astype(np.float64)
        return acc
    Engine.expand = rounded_expand
    try:
        rr = depth_forward(eng, SourceSet(p, w), b, bias=0.05)
    finally:
        Engine.expand = orig
    dr, sr = depth_jvp(yl, rr), surface_gradient_jvp(yg, rr)
    floor = np.array([rl(dr.w_bar, gd.w_bar), rl(dr.p_bar, gd.p_bar), rl(sr.w_bar, gs.w_bar),
                      rl(sr.p_bar, gs.p_bar)])
    both = rr.hit & res.hit
    floor_denom = rl(rr.denom[both], res.denom[both])      # the mediator: <r, grad f> at the hit
    print(f"    float32-grid floor (depth w,p / surface w,p): {floor}, "
          f"hit flips {int((rr.hit != res.hit).sum())}, denominators moved {floor_denom:.3e}")
    # the reference's own hit points and Hessians (rows xx yy zz xy xz yz) at
    # them: the backward can be checked on identical roots
    hess = np.zeros((b.count, 6))
    hess[res.hit] = res.accessor.partials2(res.points[res.hit])[:, 0, :]
    save("rays_cfg3", p=p, w=w, origins=b.origins, directions=b.directions, bias=0.05,
         sensitivity=sens, floor_fp32_grid=floor, floor_denom=floor_denom,
         n_segments=res.hit.size, lengths=res.lengths, hit=res.hit, grads=res.grads,
         denom=res.denom, points=res.points, hess=hess, y_len=yl, y_grad=yg,
         depth_w_bar=gd.w_bar, depth_p_bar=gd.p_bar,
         surf_w_bar=gs.w_bar, surf_p_bar=gs.p_bar)


def part_cfg4_small():
    """Config 4 geometry (level 5, 4 channels, radius 2.5, fov 50, bg 1) with
    N = 2^14 sources and one 32x32 pose."""
    rng = np.random.default_rng(44)
    n = 1 << 14
    p = q32(rng.uniform(-1, 1, (n, 3)))
    ws = q32(np.abs(rng.normal(size=(n, 1))))
    wc = q32(rng.uniform(0, 1, (n, 3)))
    pos = 2.5 * seeded_direction(rng)
    cam = Camera(position=pos, look_at=np.zeros(3), up=np.array([0.0, 1.0, 0.0]),
                 fov_deg=50.0, width=32, height=32)
    b = generate_rays(cam)
    bg = np.ones(3)
    t0 = time.time()
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, lsq=True, check_admissibility=False)
    vr = volumetric_forward(eng, p, ws, wc, b, bg)
    target = rng.uniform(0, 1, (b.count, 3))
    yv = 2.0 * (vr.rgb - target) / vr.rgb.size
    gv = volumetric_jvp(yv, vr)
    print(f"    cfg4 small: {time.time() - t0:.1f}s, alive {vr.alive.mean():.3f}")
    save("rays_cfg4", p=p, w_sigma=ws, w_color=wc, origins=b.origins, directions=b.directions,
         bg=bg, rgb=vr.rgb, alive=vr.alive, y=yv, w_bar=gv.w_bar, p_bar=gv.p_bar)


PARTS = {"poly": part_poly, "small": part_layers_small, "cfg3": part_cfg3_small,
         "cfg4": part_cfg4_small}

if __name__ == "__main__":
    for nm in sys.argv[1:] or list(PARTS):
        print(nm, flush=True)
        PARTS[nm]()
