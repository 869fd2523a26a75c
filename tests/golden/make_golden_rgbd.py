"""Golden vectors for the RGBD composition: the REFERENCE's
depth_forward supplies the roots, its explicit_forward evaluates colour
channels at the hit points, and the backward composes explicit_jvp (whose
q_bar moves the hit point along the ray: dL/dt = q_bar . r) with depth_jvp.

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_rgbd.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from fc2t2.expansion import Engine, SourceSet  # noqa: E402
from fc2t2.kernel import KernelModel  # noqa: E402
from fc2t2.layers import depth_forward, depth_jvp, explicit_forward, explicit_jvp  # noqa: E402
from fc2t2.ray import Camera, generate_rays  # noqa: E402

OUT = Path(__file__).resolve().parent


def q32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def main():
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, lsq=True, check_admissibility=False)
    rng = np.random.default_rng(7)            # the layer-test scene of make_golden_rays.py
    p = q32(rng.uniform(-0.6, 0.6, (40, 3)))
    w = q32(-(np.abs(rng.normal(size=(40, 1))) * 0.5 + 0.3))
    rng = np.random.default_rng(12)
    pc = q32(rng.uniform(-0.8, 0.8, (60, 3)))
    wc = q32(rng.uniform(0.0, 0.5, (60, 3)))
    cam = Camera(position=np.array([0.4, 0.3, -2.5]), look_at=np.zeros(3),
                 up=np.array([0.0, 1.0, 0.0]), fov_deg=30.0, width=20, height=20)
    b = generate_rays(cam)
    bias = 0.3
    root = depth_forward(eng, SourceSet(p, w), b, bias=bias)
    hit = root.hit
    q = np.where(hit[:, None], root.points, 0.0)
    col = explicit_forward(eng, SourceSet(pc, wc), q)
    rgb = np.where(hit[:, None], col.values, 0.0)
    y_depth = rng.normal(size=b.count)
    y_rgb = rng.normal(size=(b.count, 3))
    gc = explicit_jvp(np.where(hit[:, None], y_rgb, 0.0), col)
    tangent = np.where(hit, y_depth + np.sum(gc.q_bar * b.directions, axis=1), 0.0)
    gd = depth_jvp(tangent, root)
    np.savez_compressed(OUT / "rgbd.npz", p=p, w=w, pc=pc, wc=wc, origins=b.origins,
                        directions=b.directions, bias=np.array(bias), hit=hit,
                        depth=np.where(hit, root.lengths, 0.0), rgb=rgb, y_depth=y_depth,
                        y_rgb=y_rgb, color_w_bar=gc.w_bar, color_p_bar=gc.p_bar,
                        sdf_w_bar=gd.w_bar, sdf_p_bar=gd.p_bar)
    print("hit fraction", hit.mean())


if __name__ == "__main__":
    main()
