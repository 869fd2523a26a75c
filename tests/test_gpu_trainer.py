"""Device training glue (paper_2111_00110_b200/trainer.py, train.cu) against
the reference trainer's own outputs (tests/golden/trainer.npz)."""

import numpy as np
import pytest
import torch

from conftest import golden

pytestmark = pytest.mark.gpu

CASES = {"adam": dict(optimizer="adam", learning_rate=0.05),
         "sgd": dict(optimizer="sgd", learning_rate=0.1, lr_schedule=[(1, 0.05), (2, 0.02)]),
         "adam_frozen": dict(optimizer="adam", learning_rate=0.05, train_positions=False)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_optimizer_steps_match_reference(cuda, name):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.trainer import Optimizer, TrainConfig
    g = golden("trainer")
    opt = Optimizer(TrainConfig(**CASES[name]))
    src, bias = SourceSet(g["opt_p0"], g["opt_w0"]), 0.5
    for k in range(3):
        src, bias = opt.step(src, torch.from_numpy(g["opt_wg"][k]).float().cuda(),
                             torch.from_numpy(g["opt_pg"][k]).float().cuda(), k,
                             bias=bias, bias_bar=float(g["opt_bb"][k]))
        # float32 parameters and moments vs the reference's float64
        np.testing.assert_allclose(src.p.cpu().numpy(), g[f"opt_{name}_p"][k], atol=2e-7)
        np.testing.assert_allclose(src.w.cpu().numpy(), g[f"opt_{name}_w"][k], atol=2e-7)
        assert bias == pytest.approx(float(g[f"opt_{name}_bias"][k]), abs=1e-12)
    assert src.p.max().item() <= 1.0 - 1e-6 + 1e-7


def test_losses_and_l1_match_reference(cuda):
    from paper_2111_00110_b200.trainer import l1_term, loss_and_tangent
    g = golden("trainer")
    pred = torch.from_numpy(g["loss_pred"]).float().cuda()
    target = torch.from_numpy(g["loss_target"]).float().cuda()
    for kind in ("mae", "mse"):
        for m, tag in ((None, ""), (g["loss_mask"], "_masked")):
            v, t = loss_and_tangent(pred, target, kind, m)
            assert v == pytest.approx(float(g[f"loss_{kind}{tag}"]), rel=1e-12)
            np.testing.assert_allclose(t.cpu().numpy(), g[f"loss_{kind}{tag}_tangent"], rtol=1e-7)
        # numpy in -> numpy out
        v, t = loss_and_tangent(g["loss_pred"], g["loss_target"], kind)
        assert isinstance(t, np.ndarray) and t.shape == g["loss_pred"].shape
    v, t = l1_term(torch.from_numpy(g["opt_w0"]).float().cuda(), 0.25)
    assert v == pytest.approx(float(g["l1_value"]), rel=1e-6)
    np.testing.assert_array_equal(t.cpu().numpy(), g["l1_grad"])
    v, t = loss_and_tangent(pred, target, "mae", np.zeros(100, bool))   # empty valid set
    assert v == 0.0 and not t.abs().any()


def test_nonfinite_gradient_raises_without_update(cuda):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.trainer import Optimizer, TrainConfig
    src = SourceSet(np.zeros((2, 3)), np.ones((2, 1)))
    opt = Optimizer(TrainConfig(optimizer="sgd"))
    with pytest.raises(FloatingPointError):
        opt.step(src, torch.tensor([[float("nan")], [0.0]], device="cuda"), None, 0)
    assert opt.t == 0
    out, _ = opt.step(src, torch.ones(2, 1, device="cuda"), None, 0)
    assert torch.allclose(out.w, torch.full((2, 1), 0.99, device="cuda"))


def test_fit_sdf_epochs_match_reference(cuda):
    """Two epochs of the reference fit-sdf loop (cli.py:129-145): explicit layer,
    MAE loss + tangent, L1, JVP, SGD step with bias."""
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.trainer import Optimizer, TrainConfig, fit_sdf_epoch
    g = golden("trainer")
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    src, bias = SourceSet(g["fit_p0"], g["fit_w0"]), float(g["fit_bias0"])
    q = torch.from_numpy(g["fit_q"]).float().cuda()
    target = torch.from_numpy(g["fit_target"]).float().cuda()
    opt = Optimizer(TrainConfig(optimizer="sgd", learning_rate=0.2, l1_weight=1e-3, loss="mae"))
    for epoch in range(2):
        src, bias, loss, data_loss = fit_sdf_epoch(eng, src, bias, q, target, opt, epoch)
        assert loss == pytest.approx(float(g["fit_losses"][epoch][0]), rel=1e-5)
        assert data_loss == pytest.approx(float(g["fit_losses"][epoch][1]), rel=1e-5)
    rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)  # noqa: E731
    assert rel(src.p.cpu().numpy(), g["fit_p"]) < 1e-6
    assert rel(src.w.cpu().numpy(), g["fit_w"]) < 1e-5
    assert bias == pytest.approx(float(g["fit_bias"]), rel=1e-6)
