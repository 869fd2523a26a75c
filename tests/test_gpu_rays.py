"""GPU parity of traversal and the root-implicit / line-integral layers.

Checkers: golden vectors from the reference (tests/golden/make_golden_rays.py)
and the pinned CPU oracle (oracle/rays.py).  Box lists and hit masks are
integer outputs (bit-exact / mismatch counts); floats rel-L2 against the
float64 reference on identical float32 inputs.
"""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle.fc2t2_oracle import Oracle, rel_l2
from oracle.rays import camera_rays, traverse as ora_traverse

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def small():
    return golden("rays_small")


@pytest.fixture(scope="module")
def eng3(cuda):
    from paper_2111_00110_b200 import Engine, KernelModel
    return Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)


def _bundle(g):
    from paper_2111_00110_b200.ray import RayBundle
    return RayBundle(g["origins"], g["directions"])


def test_traverse_bit_exact_vs_reference(small, cuda):
    from paper_2111_00110_b200.ray import traverse
    tr = traverse(_bundle(small), 3)
    assert np.array_equal(tr.ray_id.cpu().numpy(), small["ray_id"])
    assert np.array_equal(tr.box.cpu().numpy(), small["box"])
    assert np.array_equal(tr.t0.cpu().numpy(), small["t0"])
    assert np.array_equal(tr.t1.cpu().numpy(), small["t1"])
    assert np.array_equal(tr.offsets.cpu().numpy(), small["offsets"])


def test_traverse_bit_exact_config3_camera(cuda):
    """Config-3 geometry at level 5 (radius 2, fov 60), 128x128 rays, vs the oracle."""
    from paper_2111_00110_b200.ray import RayBundle, traverse
    rng = np.random.default_rng(3)
    u = rng.normal(size=3)
    u /= np.linalg.norm(u)
    o, d = camera_rays(2.0 * u, np.zeros(3), np.array([0.0, 1.0, 0.0]), 60.0, 128, 128)
    # add axis-parallel and grazing rays
    o = np.concatenate([o, [[-3.0, 0.001, 0.001], [0.3, -2.0, 0.5], [0.5, 0.5, -3.0]]])
    d = np.concatenate([d, [[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]])
    ref = ora_traverse(o, d, 5)
    tr = traverse(RayBundle(o, d), 5)
    for k in ("ray_id", "box", "t0", "t1", "offsets"):
        assert np.array_equal(getattr(tr, k).cpu().numpy(), ref[k]), k


def test_depth_forward_matches_reference(small, eng3):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.layers import depth_forward
    res = depth_forward(eng3, SourceSet(small["p"], small["w"]), _bundle(small), bias=0.3)
    assert np.array_equal(res.hit, small["hit"])
    h = res.hit
    assert rel_l2(res.lengths[h], small["lengths"][h]) < TOL
    assert rel_l2(res.grads, small["grads"]) < TOL
    assert rel_l2(res.denom, small["denom"]) < TOL
    assert np.all(np.isnan(res.lengths[~h]))
    assert res.diagnostics["dead_pixels"] == int((~h).sum())


def test_root_jvps_match_reference(small, eng3):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.layers import (depth_forward, depth_jvp, depth_surface_jvp,
                                              surface_gradient_jvp)
    res = depth_forward(eng3, SourceSet(small["p"], small["w"]), _bundle(small), bias=0.3)
    n0 = eng3.expansion_count
    gd = depth_jvp(small["y_len"], res)
    assert eng3.expansion_count == n0 + 1
    assert rel_l2(gd.w_bar, small["depth_w_bar"]) < TOL
    assert rel_l2(gd.p_bar, small["depth_p_bar"]) < TOL
    gs = surface_gradient_jvp(small["y_grad"], res)
    assert rel_l2(gs.w_bar, small["surf_w_bar"]) < TOL
    assert rel_l2(gs.p_bar, small["surf_p_bar"]) < TOL
    gf = depth_surface_jvp(small["y_len"], small["y_grad"], res)
    assert rel_l2(gf.w_bar, small["depth_w_bar"] + small["surf_w_bar"]) < TOL
    assert rel_l2(gf.p_bar, small["depth_p_bar"] + small["surf_p_bar"]) < TOL


def test_depth_invariants(small, eng3):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.layers import depth_forward, depth_jvp
    b = _bundle(small)
    s = SourceSet(small["p"], small["w"])
    dead = depth_forward(eng3, s, b, bias=-0.2)
    assert not dead.hit.any() and dead.diagnostics["dead_pixels"] == b.count
    zd = depth_jvp(np.ones(b.count), dead)          # no hits: exact zeros, no shortcut
    assert not np.any(zd.w_bar) and not np.any(zd.p_bar)
    assert zd.diagnostics == {"dead_pixels": b.count, "ift_clamped": 0}
    a = depth_forward(eng3, s, b, bias=0.3)
    c = depth_forward(eng3, SourceSet(small["p"], 3.0 * small["w"]), b, bias=0.9)
    assert np.array_equal(a.hit, c.hit)
    assert np.allclose(a.lengths[a.hit], c.lengths[c.hit], atol=1e-6)
    z = depth_jvp(np.zeros(b.count), a)
    assert not np.any(z.w_bar) and not np.any(z.p_bar)
    # hit points re-evaluate to ~0 (acceptance criterion 3)
    f = a.accessor.value(a.points[a.hit])[:, 0] + 0.3
    assert np.max(np.abs(f)) < 1e-5


def _backward_on_reference_roots(res, g, keep, y_len, y_grad):
    """Our device backward (payload + insertion + expansion + source adjoints)
    run on the REFERENCE's roots: its hit points, gradients, denominators and
    Hessians from the golden file, for the rays in ``keep``."""
    import dataclasses

    import torch
    from paper_2111_00110_b200.layers import _root_jvp
    dev = res.dev["hit"].device
    hit = torch.from_numpy((g["hit"] & keep).astype(np.uint8)).to(dev)
    pts = np.where(g["hit"][:, None], g["points"], 0.0)
    d = {"hit": hit, "points": torch.from_numpy(pts).to(dev),
         "grads": torch.from_numpy(np.nan_to_num(g["grads"]).astype(np.float32)).to(dev),
         "hess": torch.from_numpy(g["hess"].astype(np.float32)).to(dev),
         "denom": torch.from_numpy(np.nan_to_num(g["denom"]).astype(np.float32)).to(dev)}
    return _root_jvp(dataclasses.replace(res, dev=d), y_len, y_grad)


def test_config3_backward_on_reference_roots(cuda):
    """The root-layer backward alone, at config-3 geometry, on the reference's
    own roots: every float32 step after the root walk (IFT weights, dipole
    payloads, insertion, expansion, source adjoints) to 1e-5."""
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import depth_forward
    g = golden("rays_cfg3")
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    res = depth_forward(eng, SourceSet(g["p"], g["w"]), _bundle(g), bias=float(g["bias"]))
    allr = np.ones(g["hit"].size, bool)
    gd = _backward_on_reference_roots(res, g, allr, g["y_len"], None)
    gs = _backward_on_reference_roots(res, g, allr, None, g["y_grad"])
    errs = [rel_l2(gd.w_bar, g["depth_w_bar"]), rel_l2(gd.p_bar, g["depth_p_bar"]),
            rel_l2(gs.w_bar, g["surf_w_bar"]), rel_l2(gs.p_bar, g["surf_p_bar"])]
    print("backward on reference roots (depth w,p / surface w,p):", errs)
    assert max(errs) < TOL, errs


def test_config3_small_matches_reference(cuda):
    """Config-3 geometry at level 5 (reduced N and camera; golden from the reference).

    Forward: hit mask (flips counted, <= 0.2 %), lengths and gradients < 1e-5.
    Adjoints, always compared: tangents of rays whose hit status differs are
    zeroed on our side, and their reference contribution is removed from the
    golden by linearity (our backward on the reference's roots for those rays,
    pinned to 1e-5 by test_config3_backward_on_reference_roots).

    Tolerance: the root-layer adjoints are ill-conditioned in the IFT
    denominators <r, grad f> at the hits.  The reference's OWN adjoints move by
    ``floor_fp32_grid`` (1.6-1.9e-5, > 1e-5) when the only change is rounding
    its float64 L grid to float32, which moves its denominators by
    ``floor_denom``; so no float32 field can reach 1e-5.  Our field is a
    float32 cascade (denominators off by e_den), and the adjoint error must be
    what that conditioning predicts: <= 3 x floor x e_den / floor_denom."""
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import depth_forward, depth_jvp, surface_gradient_jvp
    g = golden("rays_cfg3")
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    res = depth_forward(eng, SourceSet(g["p"], g["w"]), _bundle(g), bias=float(g["bias"]))
    flip = res.hit != g["hit"]
    mism = int(flip.sum())
    print(f"config 3: {mism} hit flips of {flip.size} rays")
    assert mism <= max(2, int(0.002 * g["hit"].size)), mism
    both = res.hit & g["hit"]
    assert rel_l2(res.lengths[both], g["lengths"][both]) < TOL
    assert rel_l2(res.grads[both], g["grads"][both]) < TOL
    e_den = rel_l2(res.denom[both], g["denom"][both])
    yl = np.where(flip, 0.0, g["y_len"])
    yg = np.where(flip[:, None], 0.0, g["y_grad"])
    ref = {k: g[k].copy() for k in ("depth_w_bar", "depth_p_bar", "surf_w_bar", "surf_p_bar")}
    if mism:
        fd = _backward_on_reference_roots(res, g, flip, g["y_len"], None)
        fs = _backward_on_reference_roots(res, g, flip, None, g["y_grad"])
        ref["depth_w_bar"] -= fd.w_bar
        ref["depth_p_bar"] -= fd.p_bar
        ref["surf_w_bar"] -= fs.w_bar
        ref["surf_p_bar"] -= fs.p_bar
    gd = depth_jvp(yl, res)
    gs = surface_gradient_jvp(yg, res)
    errs = np.array([rel_l2(gd.w_bar, ref["depth_w_bar"]), rel_l2(gd.p_bar, ref["depth_p_bar"]),
                     rel_l2(gs.w_bar, ref["surf_w_bar"]), rel_l2(gs.p_bar, ref["surf_p_bar"])])
    bound = 3.0 * g["floor_fp32_grid"] * e_den / float(g["floor_denom"])
    print(f"config-3 adjoints (depth w,p / surface w,p) {errs}; denominators off by {e_den:.2e} "
          f"(reference float32-grid floor: {g['floor_fp32_grid']} at {float(g['floor_denom']):.2e}); "
          f"bound {bound}")
    assert np.all(errs <= bound), (errs, bound)


def test_line_integral_matches_reference(small, eng3):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.layers import line_integral_forward, line_integral_jvp
    res = line_integral_forward(eng3, SourceSet(small["p"], small["w"]), _bundle(small))
    assert rel_l2(res.values, small["li_values"]) < TOL
    n0 = eng3.expansion_count
    g = line_integral_jvp(small["y_li"], res)
    assert eng3.expansion_count == n0 + 1
    assert rel_l2(g.w_bar, small["li_w_bar"]) < TOL
    assert rel_l2(g.p_bar, small["li_p_bar"]) < TOL
    res2 = line_integral_forward(eng3, SourceSet(small["p"], 2.5 * small["w"]), _bundle(small))
    assert rel_l2(res2.values, 2.5 * res.values) < 1e-6


def test_volumetric_matches_reference(small, eng3):
    from paper_2111_00110_b200.layers import volumetric_forward, volumetric_jvp
    res = volumetric_forward(eng3, small["p"], small["w_sigma"], small["w_color"], _bundle(small),
                             small["bg"])
    assert rel_l2(res.rgb, small["rgb"]) < TOL
    assert np.array_equal(res.alive, small["alive"])
    n0 = eng3.expansion_count
    g = volumetric_jvp(small["y_vol"], res)
    assert eng3.expansion_count == n0 + 1
    assert rel_l2(g.w_bar, small["vol_w_bar"]) < TOL
    assert rel_l2(g.p_bar, small["vol_p_bar"]) < TOL
    # relu mask: clipped density weights get no density gradient (test_layers.py:266-272)
    neg = small["w_sigma"][:, 0] <= 0
    assert not np.any(g.w_bar[neg, 0])


def test_volumetric_zero_density_is_background(small, eng3):
    from paper_2111_00110_b200.layers import volumetric_forward
    res = volumetric_forward(eng3, small["p"], np.zeros_like(small["w_sigma"]), small["w_color"],
                             _bundle(small), small["bg"])
    assert np.allclose(res.rgb, np.broadcast_to(small["bg"], res.rgb.shape), atol=1e-7)


def test_volumetric_config4_small_matches_reference(cuda):
    """Config-4 geometry (level 5, 3 colours, radius 2.5, fov 50), reduced N and rays."""
    from paper_2111_00110_b200 import Engine, KernelModel
    from paper_2111_00110_b200.layers import volumetric_forward, volumetric_jvp
    g = golden("rays_cfg4")
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    res = volumetric_forward(eng, g["p"], g["w_sigma"], g["w_color"], _bundle(g), g["bg"])
    assert rel_l2(res.rgb, g["rgb"]) < TOL
    gr = volumetric_jvp(g["y"], res)
    assert rel_l2(gr.w_bar, g["w_bar"]) < TOL
    assert rel_l2(gr.p_bar, g["p_bar"]) < TOL


def test_forward_pass_a_bit_identical_to_vol_totals(small, eng3):
    """volumetric_forward's walk also returns the backward's pass-A outputs
    (fc2t2_vol_forward_ex); they equal fc2t2_vol_totals bit for bit."""
    import torch
    from paper_2111_00110_b200 import _lib
    from paper_2111_00110_b200.expansion import _ptr, _stream
    from paper_2111_00110_b200.layers import volumetric_forward
    res = volumetric_forward(eng3, small["p"], small["w_sigma"], small["w_color"], _bundle(small),
                             small["bg"])
    org, dirs = res.bundle.dev()
    R, C = res.bundle.count, res.dev["colors"]
    n_alive = torch.zeros(R + 1, dtype=torch.int32, device="cuda")
    totals = torch.empty((R, C), dtype=torch.float64, device="cuda")
    dfin = torch.empty(R, dtype=torch.float64, device="cuda")
    _lib.call("fc2t2_vol_totals", eng3.rho, eng3.levels, C, _ptr(res.accessor.grid.storage),
              _ptr(org), _ptr(dirs), R, _ptr(res.dev["efit"]), _ptr(n_alive), _ptr(totals),
              _ptr(dfin), _stream())
    assert torch.equal(n_alive, res.dev["n_alive"])
    assert torch.equal(totals, res.dev["totals"])
    assert torch.equal(dfin, res.dev["dfin"])
