"""Golden vectors for the remaining training loops of SURVEY 8(f)1, produced by
the REFERENCE modules replaying the reference's own loop bodies:

* CGLS on the (w, bias) sub-problem of fit-sdf (cli.py:173-224),
* fit-depth epochs (cli.py:288-306),
* fit-radiance epochs with pooled minibatches (cli.py:363-382).

Run in the build container only (needs /root/reference, read-only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_training.py

Writes training.npz next to this script.  Inputs are float32-quantised first
(the device dtype).  The loop bodies below restate those cli.py lines against
the reference's public layer and trainer API; nothing is copied into the
package.
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
from fc2t2.layers import (depth_forward, depth_jvp, volumetric_forward,  # noqa: E402
                          volumetric_jvp)
from fc2t2.ray import Camera, RayBundle, generate_rays  # noqa: E402
from fc2t2.trainer import (Optimizer, TrainConfig, init_params, l1_term,  # noqa: E402
                           loss_and_tangent)


def f32(a):
    return np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)


def _cgls_run(eng, p, q, d, iters, noise=0.0, seed=0):
    """The reference CGLS loop (cli.py:173-224) verbatim in its arithmetic;
    ``noise`` multiplies every operator output by (1 + noise * N(0,1)) to
    measure how sensitive the iterates themselves are to operator rounding."""
    nrng = np.random.default_rng(seed)

    def nz(x):
        return x * (1.0 + noise * nrng.standard_normal(x.shape)) if noise else x

    def a_fwd(w, b):
        return nz(eng.expand(SourceSet(p, w[:, None])).value(q)[:, 0]) + b

    def a_adj(r):
        return nz(eng.expand(SourceSet(q, r[:, None])).value(p)[:, 0]), float(np.sum(r))

    w, bias = np.zeros(p.shape[0]), 0.0
    r = d - a_fwd(w, bias)
    s_w, s_b = a_adj(r)
    pk_w, pk_b = s_w.copy(), s_b
    gamma = float(s_w @ s_w + s_b * s_b)
    ws, bs, maes = [], [], []
    for _ in range(iters):
        qk = a_fwd(pk_w, pk_b)
        alpha = gamma / float(qk @ qk)
        w = w + alpha * pk_w
        bias += alpha * pk_b
        r = r - alpha * qk
        s_w, s_b = a_adj(r)
        gamma_new = float(s_w @ s_w + s_b * s_b)
        beta = gamma_new / gamma
        pk_w, pk_b = s_w + beta * pk_w, s_b + beta * pk_b
        gamma = gamma_new
        ws.append(w.copy())
        bs.append(bias)
        maes.append(float(np.mean(np.abs(r))))
    final = float(np.mean(np.abs(a_fwd(w, bias) - d)))
    return np.stack(ws), np.array(bs), np.array(maes), final


def cgls(g):
    """CGLS iterates are sensitive to operator rounding once the residual
    plateaus (the Gram matrix of Gaussian columns has tiny singular values),
    so the golden also stores the reference's own spread when every product
    is perturbed by 1e-7 relative noise (fp32-sized); the test's per-iteration
    tolerances derive from it."""
    eng = Engine(KernelModel("gaussian", 12.0, 4), 3, check_admissibility=False)
    rng = np.random.default_rng(41)
    g1 = np.linspace(-0.5, 0.5, 3)
    lat = np.stack(np.meshgrid(g1, g1, g1, indexing="ij"), -1).reshape(-1, 3)
    p = f32(lat + rng.uniform(-0.03, 0.03, lat.shape))
    q = f32(rng.uniform(-0.95, 0.95, (2000, 3)))
    d = f32(0.3 + np.sin(2.0 * q[:, 0]) * 0.2 + q[:, 1] * 0.1 + rng.normal(0, 0.01, 2000))
    ws, bs, maes, final = _cgls_run(eng, p, q, d, 4)
    sw, sb, sm = np.zeros(4), np.zeros(4), np.zeros(4)
    for seed in range(4):
        nw, nb, nm, _ = _cgls_run(eng, p, q, d, 4, noise=1e-7, seed=seed)
        sw = np.maximum(sw, np.linalg.norm(nw - ws, axis=1) / np.linalg.norm(ws, axis=1))
        sb = np.maximum(sb, np.abs(nb - bs) / np.abs(bs))
        sm = np.maximum(sm, np.abs(nm - maes) / maes)
    g.update(cgls_p=p, cgls_q=q, cgls_d=d, cgls_w=ws, cgls_bias=bs, cgls_mae=maes,
             cgls_final_mae=np.array(final), cgls_sens_w=sw, cgls_sens_bias=sb,
             cgls_sens_mae=sm)


def fit_depth(g, eng):
    rng = np.random.default_rng(42)
    p = f32(rng.uniform(-0.6, 0.6, (40, 3)))
    w = f32(-(np.abs(rng.normal(size=(40, 1))) * 0.5 + 0.3))
    cam = Camera(position=np.array([0.0, 0.0, -2.5]), look_at=np.zeros(3),
                 up=np.array([0.0, 1.0, 0.0]), fov_deg=30.0, width=24, height=24)
    b = generate_rays(cam)
    bias = 0.3
    r0 = depth_forward(eng, SourceSet(p, w), b, bias=bias)
    target = np.where(r0.hit, r0.lengths, 2.3) + 0.05 * np.cos(np.arange(b.count))
    target[::9] = np.nan                                   # invalid target pixels
    target = f32(target)
    valid = np.isfinite(target)
    tc = TrainConfig(optimizer="sgd", learning_rate=0.05, l1_weight=1e-4, loss="mae")
    opt = Optimizer(tc)
    src = SourceSet(p, w)
    g.update(depth_p0=p, depth_w0=w, depth_bias0=np.array(bias), depth_origins=b.origins,
             depth_directions=b.directions, depth_target=target)
    ps, wws, bs, losses, misses = [], [], [], [], []
    for epoch in range(2):
        res = depth_forward(eng, src, b, bias=bias)
        mask = res.hit & valid
        loss, tangent = loss_and_tangent(np.where(mask, res.lengths, 0.0),
                                         np.where(mask, target, 0.0), tc.loss, mask=mask)
        miss = float(np.mean(~mask))
        gr = depth_jvp(tangent, res)
        reg, reg_grad = l1_term(src.w, tc.l1_weight)
        src, bias = opt.step(src, gr.w_bar + reg_grad, gr.p_bar, epoch, bias=bias,
                             bias_bar=0.1 * miss)
        ps.append(src.p.copy())
        wws.append(src.w.copy())
        bs.append(bias)
        losses.append(loss)
        misses.append(miss)
    g.update(depth_p=np.stack(ps), depth_w=np.stack(wws), depth_bias=np.array(bs),
             depth_loss=np.array(losses), depth_miss=np.array(misses))


def fit_radiance(g, eng):
    rng = np.random.default_rng(43)
    tc = TrainConfig(optimizer="adam", learning_rate=0.01, l1_weight=1e-4, loss="mse")
    src, _ = init_params(60, 4, "uniform", 0.8, seed=7)
    p = f32(src.p * 0.7)
    w_sigma = f32(np.abs(src.w[:, :1]))
    w_color = f32(np.abs(src.w[:, 1:]))
    bg = np.array([1.0, 1.0, 1.0])
    pool_o, pool_d, pool_t = [], [], []
    for k in range(2):
        ang = 0.7 * k
        cam = Camera(position=2.5 * np.array([np.sin(ang), 0.2, -np.cos(ang)]),
                     look_at=np.zeros(3), up=np.array([0.0, 1.0, 0.0]), fov_deg=40.0,
                     width=12, height=12)
        b = generate_rays(cam)
        pool_o.append(b.origins)
        pool_d.append(b.directions)
        pool_t.append(f32(rng.uniform(0, 1, (b.count, 3))))
    pool_o, pool_d, pool_t = (np.concatenate(a) for a in (pool_o, pool_d, pool_t))
    g.update(rad_p0=p, rad_ws0=w_sigma, rad_wc0=w_color, rad_origins=pool_o,
             rad_directions=pool_d, rad_target=pool_t)
    opt = Optimizer(tc)
    idxs, ps, wss, wcs, losses = [], [], [], [], []
    for epoch in range(2):
        idx = rng.choice(pool_o.shape[0], size=100, replace=False)
        mb = RayBundle(origins=pool_o[idx], directions=pool_d[idx])
        res = volumetric_forward(eng, p, w_sigma, w_color, mb, bg)
        loss, tangent = loss_and_tangent(res.rgb, pool_t[idx], tc.loss)
        gr = volumetric_jvp(tangent, res)
        packed = SourceSet(p, np.concatenate([w_sigma, w_color], axis=1))
        reg, reg_grad = l1_term(packed.w, tc.l1_weight)
        packed, _ = opt.step(packed, gr.w_bar + reg_grad, gr.p_bar, epoch)
        p, w_sigma, w_color = packed.p, packed.w[:, :1], packed.w[:, 1:]
        idxs.append(idx)
        ps.append(p.copy())
        wss.append(w_sigma.copy())
        wcs.append(w_color.copy())
        losses.append(loss)
    g.update(rad_idx=np.stack(idxs), rad_p=np.stack(ps), rad_ws=np.stack(wss),
             rad_wc=np.stack(wcs), rad_loss=np.array(losses))


def main():
    eng = Engine(KernelModel("gaussian", 50.0, 4), 3, check_admissibility=False)
    g = {}
    cgls(g)
    fit_depth(g, eng)
    fit_radiance(g, eng)
    np.savez_compressed(OUT / "training.npz", **g)
    print("wrote", OUT / "training.npz", sorted(g))
    print("cgls mae", g["cgls_mae"], "final", g["cgls_final_mae"])
    print("cgls sensitivity w", g["cgls_sens_w"], "bias", g["cgls_sens_bias"], "mae",
          g["cgls_sens_mae"])
    print("depth loss", g["depth_loss"], "miss", g["depth_miss"])
    print("radiance loss", g["rad_loss"])


if __name__ == "__main__":
    main()
