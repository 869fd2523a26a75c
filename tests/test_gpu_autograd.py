"""torch.autograd wrappers (paper_2111_00110_b200/autograd.py): gradients from
loss.backward() equal the layers' JVP outputs bit for bit, and match the
reference's adjoints (golden vectors) where those exist."""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle.fc2t2_oracle import rel_l2

pytestmark = pytest.mark.gpu


def _t(a, grad=False):
    return torch.tensor(np.asarray(a), dtype=torch.float32, device="cuda", requires_grad=grad)


def test_explicit_autograd_equals_jvp(cuda):
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.autograd import explicit
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    eng = Engine(KernelModel("gaussian", 200.0, 4), 4, check_admissibility=False)
    rng = np.random.default_rng(3)
    p = _t(rng.uniform(-0.9, 0.9, (2000, 3)), True)
    w = _t(rng.normal(size=(2000, 2)), True)
    q = _t(rng.uniform(-0.9, 0.9, (3000, 3)), True)
    yb = _t(rng.normal(size=(3000, 2)))
    f = explicit(eng, p, w, q)
    (f * yb).sum().backward()
    res = explicit_forward(eng, SourceSet(p.detach(), w.detach()), q.detach())
    g = explicit_jvp(yb, res)
    assert torch.equal(f.detach(), res.values)
    assert torch.equal(p.grad, g.p_bar) and torch.equal(w.grad, g.w_bar)
    assert torch.equal(q.grad, g.q_bar)


def test_explicit_autograd_trains():
    """A few Adam steps through the autograd wrapper reduce an MSE fit."""
    from paper_2111_00110_b200 import Engine, KernelModel
    from paper_2111_00110_b200.autograd import explicit
    eng = Engine(KernelModel("gaussian", 200.0, 4), 4, check_admissibility=False)
    rng = np.random.default_rng(4)
    q = _t(rng.uniform(-0.9, 0.9, (4000, 3)))
    target = torch.sin(3 * q[:, :1]) * 0.1
    p = _t(rng.uniform(-0.9, 0.9, (1000, 3)), True)
    w = _t(rng.normal(0, 0.01, (1000, 1)), True)
    opt = torch.optim.Adam([w], lr=1e-2)
    losses = []
    for _ in range(20):
        opt.zero_grad()
        loss = ((explicit(eng, p, w, q) - target) ** 2).mean()
        loss.backward()
        opt.step()
        losses.append(float(loss.detach()))
    assert losses[-1] < 0.5 * losses[0]


def test_depth_normal_autograd_equals_jvp_and_reference():
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.autograd import depth_normal
    from paper_2111_00110_b200.layers import depth_forward, depth_surface_jvp
    from paper_2111_00110_b200.ray import RayBundle
    g = golden("rays_small")
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    p, w = _t(g["p"], True), _t(g["w"], True)
    org = torch.tensor(g["origins"], dtype=torch.float64, device="cuda")
    dirs = torch.tensor(g["directions"], dtype=torch.float64, device="cuda")
    yl = torch.tensor(g["y_len"], dtype=torch.float64, device="cuda")
    yg = torch.tensor(g["y_grad"], dtype=torch.float32, device="cuda")
    lengths, grads, hit = depth_normal(eng, p, w, org, dirs, 0.3)   # the golden scene's bias
    h = hit.bool()
    ((lengths[h] * yl[h]).sum() + (grads[h] * yg[h]).sum()).backward()
    res = depth_forward(eng, SourceSet(p.detach(), w.detach()), RayBundle(org, dirs), bias=0.3)
    jv = depth_surface_jvp(torch.where(res.hit, yl, 0.0), torch.where(res.hit[:, None], yg, 0.0), res)
    assert torch.equal(p.grad, jv.p_bar) and torch.equal(w.grad, jv.w_bar)
    # the reference's depth + surface adjoints add (one fused insertion)
    assert rel_l2(w.grad.cpu().numpy(), g["depth_w_bar"] + g["surf_w_bar"]) < 1e-5
    assert rel_l2(p.grad.cpu().numpy(), g["depth_p_bar"] + g["surf_p_bar"]) < 1e-5


def test_radiance_autograd_equals_jvp_and_reference():
    from paper_2111_00110_b200 import Engine, KernelModel
    from paper_2111_00110_b200.autograd import radiance
    from paper_2111_00110_b200.layers import volumetric_forward, volumetric_jvp
    from paper_2111_00110_b200.ray import RayBundle
    g = golden("rays_small")
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    p, ws, wc = _t(g["p"], True), _t(g["w_sigma"], True), _t(g["w_color"], True)
    org = torch.tensor(g["origins"], dtype=torch.float64, device="cuda")
    dirs = torch.tensor(g["directions"], dtype=torch.float64, device="cuda")
    yv = _t(g["y_vol"])
    rgb = radiance(eng, p, ws, wc, org, dirs, g["bg"])
    (rgb * yv).sum().backward()
    res = volumetric_forward(eng, p.detach(), ws.detach(), wc.detach(), RayBundle(org, dirs), g["bg"])
    jv = volumetric_jvp(yv, res)
    assert torch.equal(p.grad, jv.p_bar)
    assert torch.equal(ws.grad, jv.w_bar[:, :1]) and torch.equal(wc.grad, jv.w_bar[:, 1:])
    assert rel_l2(torch.cat([ws.grad, wc.grad], 1).cpu().numpy(), g["vol_w_bar"]) < 1e-5
    assert rel_l2(p.grad.cpu().numpy(), g["vol_p_bar"]) < 1e-5


def test_line_integral_autograd_matches_reference():
    from paper_2111_00110_b200 import Engine, KernelModel
    from paper_2111_00110_b200.autograd import line_integral
    g = golden("rays_small")
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    p, w = _t(g["p"], True), _t(g["w"], True)
    org = torch.tensor(g["origins"], dtype=torch.float64, device="cuda")
    dirs = torch.tensor(g["directions"], dtype=torch.float64, device="cuda")
    v = line_integral(eng, p, w, org, dirs)
    assert rel_l2(v.detach().cpu().numpy(), g["li_values"]) < 1e-5
    (v * _t(g["y_li"])).sum().backward()
    assert rel_l2(w.grad.cpu().numpy(), g["li_w_bar"]) < 1e-5
    assert rel_l2(p.grad.cpu().numpy(), g["li_p_bar"]) < 1e-5
