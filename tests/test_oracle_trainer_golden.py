"""The trainer oracle (oracle/trainer.py) against the reference's own outputs
(tests/golden/trainer.npz, made by tests/golden/make_golden_trainer.py)."""

import numpy as np
import pytest

from conftest import golden
from oracle.trainer import Optimizer, l1_term, loss_and_tangent

CASES = {"adam": dict(optimizer="adam", lr=0.05),
         "sgd": dict(optimizer="sgd", lr=0.1, schedule=[(1, 0.05), (2, 0.02)]),
         "adam_frozen": dict(optimizer="adam", lr=0.05, train_positions=False)}


@pytest.mark.parametrize("name", sorted(CASES))
def test_optimizer_oracle_matches_reference(name):
    g = golden("trainer")
    opt = Optimizer(**CASES[name])
    p, w, bias = g["opt_p0"], g["opt_w0"], 0.5
    for k in range(3):
        p, w, bias = opt.step(p, w, g["opt_wg"][k], g["opt_pg"][k], k, bias, float(g["opt_bb"][k]))
        np.testing.assert_allclose(p, g[f"opt_{name}_p"][k], rtol=0, atol=1e-15)
        np.testing.assert_allclose(w, g[f"opt_{name}_w"][k], rtol=0, atol=1e-15)
        assert bias == pytest.approx(float(g[f"opt_{name}_bias"][k]), abs=1e-15)


def test_loss_and_l1_oracle_match_reference():
    g = golden("trainer")
    for kind in ("mae", "mse"):
        for m, tag in ((None, ""), (g["loss_mask"], "_masked")):
            v, t = loss_and_tangent(g["loss_pred"], g["loss_target"], kind, m)
            assert v == pytest.approx(float(g[f"loss_{kind}{tag}"]), rel=1e-15)
            np.testing.assert_array_equal(t, g[f"loss_{kind}{tag}_tangent"])
    v, t = l1_term(g["opt_w0"], 0.25)
    assert v == pytest.approx(float(g["l1_value"]), rel=1e-15)
    np.testing.assert_array_equal(t, g["l1_grad"])


def test_nonfinite_gradient_raises():
    opt = Optimizer("sgd", 0.1)
    with pytest.raises(FloatingPointError):
        opt.step(np.zeros((2, 3)), np.zeros((2, 1)), np.array([[np.nan], [0.0]]), None, 0)
