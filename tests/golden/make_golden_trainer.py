"""Golden vectors for the training glue, produced by the REFERENCE trainer
(trainer.py) and its fit-sdf loop body (cli.py:129-145).

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_trainer.py

Writes trainer.npz next to this script.  Parameters and gradients are
float32-quantised before the reference sees them (the device dtype).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from fc2t2.expansion import Engine, SourceSet  # noqa: E402
from fc2t2.kernel import KernelModel  # noqa: E402
from fc2t2.layers import explicit_forward, explicit_jvp  # noqa: E402
from fc2t2.trainer import (Optimizer, TrainConfig, init_params, l1_term,  # noqa: E402
                           loss_and_tangent)


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def main():
    rng = np.random.default_rng(2024)
    g = {}
    # ---- optimizer steps with given gradients (Adam + SGD with schedule)
    n, c = 64, 2
    p0 = f32(rng.uniform(-0.95, 0.95, (n, 3)))
    p0[0] = [0.9999985, -0.9999985, 0.0]         # next to the clipping margin
    w0 = f32(rng.normal(0, 0.1, (n, c)))
    wg = [f32(rng.normal(0, 1.0, (n, c))) for _ in range(3)]
    pg = [f32(rng.normal(0, 1.0, (n, 3))) for _ in range(3)]
    pg[0][0] = [-50.0, 50.0, 0.0]                # pushes p0[0] through the clip
    bb = [0.3, -0.7, 0.2]
    g.update(opt_p0=p0, opt_w0=w0, opt_wg=np.stack(wg), opt_pg=np.stack(pg), opt_bb=np.array(bb))
    for name, tc in (("adam", TrainConfig(optimizer="adam", learning_rate=0.05)),
                     ("sgd", TrainConfig(optimizer="sgd", learning_rate=0.1,
                                         lr_schedule=[(1, 0.05), (2, 0.02)])),
                     ("adam_frozen", TrainConfig(optimizer="adam", learning_rate=0.05,
                                                 train_positions=False))):
        opt = Optimizer(tc)
        src, bias = SourceSet(p0.copy(), w0.copy()), 0.5
        ps, ws, bs = [], [], []
        for k in range(3):
            src, bias = opt.step(src, wg[k], pg[k], k, bias=bias, bias_bar=bb[k])
            ps.append(src.p.copy())
            ws.append(src.w.copy())
            bs.append(bias)
        g[f"opt_{name}_p"] = np.stack(ps)
        g[f"opt_{name}_w"] = np.stack(ws)
        g[f"opt_{name}_bias"] = np.array(bs)
    # ---- losses (masked and not)
    pred = f32(rng.normal(0, 1, (100, 3)))
    target = f32(rng.normal(0, 1, (100, 3)))
    mask = rng.uniform(0, 1, 100) < 0.7
    g.update(loss_pred=pred, loss_target=target, loss_mask=mask)
    for kind in ("mae", "mse"):
        for m, tag in ((None, ""), (mask, "_masked")):
            v, t = loss_and_tangent(pred, target, kind, m)
            g[f"loss_{kind}{tag}"] = np.array(v)
            g[f"loss_{kind}{tag}_tangent"] = t
    v, t = l1_term(w0, 0.25)
    g.update(l1_value=np.array(v), l1_grad=t)
    # ---- two fit-sdf epochs (cli.py:129-145) with SGD, L1 and MAE
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    src, _ = init_params(200, 1, "uniform", 0.05, seed=3)
    src = SourceSet(f32(src.p), f32(src.w))
    q = f32(rng.uniform(-0.95, 0.95, (400, 3)))
    target = f32(rng.normal(0, 0.1, (400, 1)))
    bias = float(np.mean(target))
    tc = TrainConfig(optimizer="sgd", learning_rate=0.2, l1_weight=1e-3, loss="mae")
    opt = Optimizer(tc)
    g.update(fit_p0=src.p, fit_w0=src.w, fit_q=q, fit_target=target, fit_bias0=np.array(bias))
    losses = []
    for epoch in range(2):
        res = explicit_forward(eng, src, q)
        pred = res.values + bias
        loss, tangent = loss_and_tangent(pred, target, tc.loss)
        reg, reg_grad = l1_term(src.w, tc.l1_weight)
        gr = explicit_jvp(tangent, res)
        bias_bar = float(np.sum(tangent))
        src, bias = opt.step(src, gr.w_bar + reg_grad, gr.p_bar, epoch, bias=bias,
                             bias_bar=bias_bar)
        losses.append([loss + reg, loss])
    g.update(fit_p=src.p, fit_w=src.w, fit_bias=np.array(bias), fit_losses=np.array(losses))
    np.savez_compressed(OUT / "trainer.npz", **g)
    print("wrote", OUT / "trainer.npz", sorted(g))


if __name__ == "__main__":
    main()
