"""Pin the ray-layer oracle (oracle/rays.py) against the reference's golden
vectors: traversal box lists bit-exact, closed-form roots, line restriction,
and every layer's forward and JVP."""

import numpy as np
import pytest

from conftest import golden
from oracle.fc2t2_oracle import Oracle, rel_l2
from oracle.rays import (RayOracle, exp_fit, line2poly, line2taylor_h, quartic_roots,
                         seg_geometry, traverse)


def test_quartic_roots_match_reference():
    g = golden("poly1d")
    for c, ref in zip(g["coeffs"], g["roots"]):
        got = quartic_roots(c)
        ref = ref[~np.isnan(ref)]
        assert got.shape == ref.shape and np.array_equal(got, ref)
    for c, ref in zip(g["special"], g["special_roots"]):
        ref = ref[~np.isnan(ref)]
        assert np.array_equal(quartic_roots(c), ref)
    assert np.array_equal(exp_fit(), g["mexp_coeffs"])


@pytest.fixture(scope="module")
def small():
    return golden("rays_small")


@pytest.fixture(scope="module")
def ro3():
    return RayOracle(Oracle(50.0, 4, 3))


def test_traversal_bit_exact(small):
    tr = traverse(small["origins"], small["directions"], 3)
    for k in ("ray_id", "box", "offsets"):
        assert np.array_equal(tr[k], small[k]), k
    assert np.array_equal(tr["t0"], small["t0"]) and np.array_equal(tr["t1"], small["t1"])
    d, r, s = seg_geometry(tr, small["origins"], small["directions"], 3)
    assert np.array_equal(d[:1500], small["seg_d"])


def test_line_kernels(small, ro3):
    d = small["seg_d"]
    r = small["directions"][small["ray_id"][:1500]]
    s = (small["t1"] - small["t0"])[:1500]
    L = ro3.o.expand(small["p"], small["w"])
    box = small["box"][:1500]
    co = L[box[:, 0], box[:, 1], box[:, 2]]
    assert rel_l2(line2poly(co, d, r, 4), small["polys"]) < 1e-12
    assert rel_l2(line2taylor_h(d, r, s, small["h"], 4), small["moments"]) < 1e-12


def test_depth_and_surface_layers(small, ro3):
    o, d = small["origins"], small["directions"]
    fw = ro3.depth_forward(small["p"], small["w"], o, d, 0.3)
    assert np.array_equal(fw["hit"], small["hit"])
    h = small["hit"]
    assert rel_l2(fw["lengths"][h], small["lengths"][h]) < 1e-12
    assert rel_l2(fw["grads"], small["grads"]) < 1e-12
    wb, pb = ro3.depth_jvp(small["y_len"], fw, small["p"], small["w"])
    assert rel_l2(wb, small["depth_w_bar"]) < 1e-11 and rel_l2(pb, small["depth_p_bar"]) < 1e-11
    wb, pb = ro3.surface_jvp(small["y_grad"], fw, small["p"], small["w"], d)
    assert rel_l2(wb, small["surf_w_bar"]) < 1e-11 and rel_l2(pb, small["surf_p_bar"]) < 1e-11


def test_line_integral_layer(small, ro3):
    o, d = small["origins"], small["directions"]
    vals, tr = ro3.line_integral(small["p"], small["w"], o, d)
    assert rel_l2(vals, small["li_values"]) < 1e-12
    wb, pb = ro3.line_integral_jvp(small["y_li"], tr, small["p"], small["w"], o, d)
    assert rel_l2(wb, small["li_w_bar"]) < 1e-11 and rel_l2(pb, small["li_p_bar"]) < 1e-11


def test_volumetric_layer(small, ro3):
    o, d = small["origins"], small["directions"]
    rgb, cache = ro3.volumetric(small["p"], small["w_sigma"], small["w_color"], o, d,
                                small["bg"])
    assert np.array_equal(cache["alive"], small["alive"])
    assert rel_l2(rgb, small["rgb"]) < 1e-12
    wb, pb = ro3.volumetric_jvp(small["y_vol"], cache, small["p"], o, d)
    assert rel_l2(wb, small["vol_w_bar"]) < 1e-11 and rel_l2(pb, small["vol_p_bar"]) < 1e-11
