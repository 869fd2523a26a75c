"""RGBD composition (layers.rgbd_forward / rgbd_jvp) against the
reference's depth_forward + explicit_forward composed the same way
(tests/golden/make_golden_rgbd.py)."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle.fc2t2_oracle import rel_l2

pytestmark = pytest.mark.gpu


def test_rgbd_matches_reference_composition(cuda):
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import rgbd_forward, rgbd_jvp
    from paper_2111_00110_b200.ray import RayBundle
    g = golden("rgbd")
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()   # noqa: E731
    bundle = RayBundle(dev(g["origins"]), dev(g["directions"]))
    res = rgbd_forward(eng, SourceSet(g["p"], g["w"]), SourceSet(g["pc"], g["wc"]), bundle,
                       bias=float(g["bias"]))
    hit = res.hit.cpu().numpy()
    assert np.array_equal(hit, g["hit"])
    assert rel_l2(res.depth.cpu().numpy(), g["depth"]) < 1e-6
    assert rel_l2(res.rgb.cpu().numpy(), g["rgb"]) < 1e-5
    assert not res.rgb[~res.hit].abs().any()
    sdf_g, col_g = rgbd_jvp(dev(g["y_depth"]).float(), dev(g["y_rgb"]).float(), res)
    assert rel_l2(col_g.w_bar.cpu().numpy(), g["color_w_bar"]) < 1e-5
    assert rel_l2(col_g.p_bar.cpu().numpy(), g["color_p_bar"]) < 1e-5
    # the SDF adjoints chain two approximations: the colour gradient at the
    # float32 hit point (q_bar) and the IFT division by <r, grad f>, which
    # amplifies on grazing rays -- 5e-5 (measured 1.05e-5)
    assert rel_l2(sdf_g.w_bar.cpu().numpy(), g["sdf_w_bar"]) < 5e-5
    assert rel_l2(sdf_g.p_bar.cpu().numpy(), g["sdf_p_bar"]) < 5e-5


def test_rgbd_colour_only_tangent_moves_roots(cuda):
    """With y_depth = 0 the SDF still gets gradients through the hit point
    (q_bar . r), and y_rgb = 0 gives zero colour gradients."""
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import rgbd_forward, rgbd_jvp
    from paper_2111_00110_b200.ray import RayBundle
    g = golden("rgbd")
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    bundle = RayBundle(torch.from_numpy(g["origins"]).cuda(),
                       torch.from_numpy(g["directions"]).cuda())
    res = rgbd_forward(eng, SourceSet(g["p"], g["w"]), SourceSet(g["pc"], g["wc"]), bundle,
                       bias=float(g["bias"]))
    R = bundle.count
    sdf_g, col_g = rgbd_jvp(torch.zeros(R, device="cuda"),
                            torch.from_numpy(g["y_rgb"]).float().cuda(), res)
    assert sdf_g.w_bar.abs().sum() > 0
    sdf_g, col_g = rgbd_jvp(torch.from_numpy(g["y_depth"]).float().cuda(),
                            torch.zeros(R, 3, device="cuda"), res)
    assert not col_g.w_bar.abs().any()
