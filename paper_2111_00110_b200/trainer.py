"""Training glue on the device: drop-in for ``fc2t2.trainer``.

Same names and semantics as the reference (trainer.py:1-152): TrainConfig,
init_params, loss_and_tangent, l1_term and Optimizer (SGD / Adam over
(w, p, bias) with domain clipping of p), plus the loop bodies of the
reference CLI's fitting commands: ``fit_sdf_epoch`` (cli.py:129-145),
``cgls_sdf`` (the CGLS solver, cli.py:173-224), ``fit_depth_epoch``
(cli.py:288-306) and ``fit_radiance_epoch`` (cli.py:363-382).  Tensors stay on the GPU: the
loss and its tangent come from one fused CUDA pass (train.cu, deterministic
float64 reductions), each parameter step is one fused kernel (gradient + L1
subgradient, Adam moments, clipping), and the non-finite check is a device
flag read once per step.  numpy inputs are accepted and answered in kind.

Differences from the reference are representational only: parameters and
Adam moments are float32 device tensors (the reference keeps float64 numpy);
the scalar bias and its Adam state stay float64 on the host.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .expansion import Engine, SourceSet, _device, _ptr, _stream, to_device
from .layers import (depth_forward, depth_jvp, explicit_forward, explicit_jvp,
                     volumetric_forward, volumetric_jvp)

DOMAIN_MARGIN = 1e-6  # sources are clipped back to (-1+eps, 1-eps)


@dataclass
class TrainConfig:
    """Reference trainer.py:21-51 (fields, validation and schedule)."""

    optimizer: str = "adam"
    learning_rate: float = 1e-2
    lr_schedule: list[tuple[int, float]] = field(default_factory=list)
    epochs: int = 100
    l1_weight: float = 0.0
    init_scheme: str = "uniform"
    init_scale: float = 1e-2
    seed: int = 0
    loss: str = "mae"
    train_positions: bool = True

    def __post_init__(self):
        if self.learning_rate <= 0:
            raise ValueError("learning rate must be positive")
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")
        if self.loss not in ("mae", "mse"):
            raise ValueError(f"unknown loss {self.loss!r}")
        if self.optimizer not in ("sgd", "adam"):
            raise ValueError(f"unknown optimizer {self.optimizer!r}")

    def lr_at(self, epoch: int) -> float:
        lr = self.learning_rate
        for start, value in sorted(self.lr_schedule):
            if epoch >= start:
                lr = value
        return lr


def init_params(n_sources: int, channels: int, scheme: str = "uniform",
                scale: float = 1e-2, seed: int = 0) -> tuple[SourceSet, float]:
    """Reference trainer.py:54-67: the same seeded float64 draws, uploaded."""
    rng = np.random.default_rng(seed)
    p = rng.uniform(-1.0 + DOMAIN_MARGIN, 1.0 - DOMAIN_MARGIN, (n_sources, 3))
    if scheme == "uniform":
        w = rng.uniform(-scale, scale, (n_sources, channels))
    elif scheme == "zeros":
        w = np.zeros((n_sources, channels))
    else:
        raise ValueError(f"unknown init scheme {scheme!r}")
    return SourceSet(p, w), 0.0


def _as_cols(x: torch.Tensor) -> torch.Tensor:
    return x.reshape(x.shape[0], -1) if x.dim() > 1 else x.reshape(-1, 1)


def _loss_device(pred, target, loss: str, mask=None, bias: float = 0.0):
    """(stats (3,) float64 device [count, loss, sum tangent], tangent) for
    device tensors; the fused train.cu pass."""
    pr = _as_cols(to_device(pred).contiguous())
    tg = _as_cols(to_device(target).contiguous()).reshape(pr.shape)
    n, cols = int(pr.shape[0]), int(pr.shape[1])
    m = None
    if mask is not None:
        m = torch.as_tensor(mask, device=_device()).reshape(n).to(torch.uint8).contiguous()
    tangent = torch.empty_like(pr)
    stats = torch.empty(3, dtype=torch.float64, device=_device())
    ws_b = int(_lib.lib().fc2t2_loss_workspace_size(n, cols))
    ws = torch.empty(max(ws_b, 1), dtype=torch.uint8, device=_device())
    _lib.call("fc2t2_loss", _ptr(pr), _ptr(tg), _ptr(m), n, cols, float(bias),
              1 if loss == "mse" else 0, _ptr(tangent), _ptr(stats), _ptr(ws), ws_b, _stream())
    return stats, tangent


def loss_and_tangent(pred, target, loss: str, mask=None):
    """Reference trainer.py:70-105: (loss over valid entries, d loss/d pred);
    an empty valid set gives (0, zeros)."""
    if loss not in ("mae", "mse"):
        raise ValueError(f"unknown loss {loss!r}")
    stats, tangent = _loss_device(pred, target, loss, mask)
    value = float(stats[1].item())
    ref = pred
    if isinstance(ref, torch.Tensor) and ref.is_cuda:
        return value, tangent.reshape(ref.shape)
    shape = np.shape(ref)
    return value, tangent.reshape(shape).cpu().numpy().astype(np.float64)


def l1_term(w, lam: float):
    """Reference trainer.py:108-112: lam * sum|w| and its subgradient."""
    if isinstance(w, torch.Tensor):
        if lam == 0.0:
            return 0.0, torch.zeros_like(w)
        return lam * float(w.abs().double().sum().item()), lam * torch.sign(w)
    w = np.asarray(w, dtype=np.float64)
    if lam == 0.0:
        return 0.0, np.zeros_like(w)
    return lam * float(np.sum(np.abs(w))), lam * np.sign(w)


class Optimizer:
    """SGD or Adam over (w, p, bias) with domain clipping of p (reference
    trainer.py:115-152); one fused kernel per parameter tensor."""

    def __init__(self, config: TrainConfig):
        self.config = config
        self.t = 0
        self._state: dict[str, tuple[torch.Tensor, torch.Tensor]] = {}
        self._bias_m = 0.0
        self._bias_v = 0.0
        self._flag = None

    def _moments(self, name: str, like: torch.Tensor):
        st = self._state.get(name)
        if st is None or st[0].shape != like.shape:
            st = (torch.zeros_like(like), torch.zeros_like(like))
            self._state[name] = st
        return st

    def _update(self, name: str, x: torch.Tensor, grad: torch.Tensor, lr: float, clip: bool,
                l1: float = 0.0) -> torch.Tensor:
        adam = self.config.optimizer == "adam"
        out = x.detach().clone().contiguous()
        g = to_device(grad).reshape(out.shape).contiguous()
        m, v = self._moments(name, out) if adam else (None, None)
        _lib.call("fc2t2_opt_step", _ptr(out), _ptr(g), _ptr(m), _ptr(v), int(out.numel()),
                  1 if adam else 0, float(lr), int(self.t), float(l1), 1 if clip else 0,
                  _ptr(self._flag), _stream())
        return out

    def step(self, sources: SourceSet, w_bar, p_bar, epoch: int, bias: float = 0.0,
             bias_bar: float | None = None, l1_weight: float = 0.0):
        """Returns (new SourceSet, bias).  ``l1_weight`` optionally fuses the
        L1 subgradient of w (the reference adds l1_term's gradient to w_bar
        before calling; both ways are supported)."""
        if self._flag is None:
            self._flag = torch.zeros(1, dtype=torch.int32, device=_device())
        self._flag.zero_()
        wb = to_device(w_bar).contiguous()
        _lib.call("fc2t2_nonfinite", _ptr(wb), int(wb.numel()), _ptr(self._flag), _stream())
        pb = None
        if p_bar is not None:
            pb = to_device(p_bar).contiguous()
            _lib.call("fc2t2_nonfinite", _ptr(pb), int(pb.numel()), _ptr(self._flag), _stream())
        if int(self._flag.item()) or (bias_bar is not None and not np.isfinite(bias_bar)):
            raise FloatingPointError("non-finite gradient in optimizer step")
        self.t += 1
        lr = self.config.lr_at(epoch)
        w = self._update("w", sources.w, wb, lr, False, l1_weight)
        p = sources.p
        if pb is not None and self.config.train_positions:
            p = self._update("p", sources.p, pb, lr, True)
        if bias_bar is not None:
            g = float(bias_bar)
            if self.config.optimizer == "adam":
                self._bias_m += 0.1 * (g - self._bias_m)
                self._bias_v += 0.001 * (g * g - self._bias_v)
                mhat = self._bias_m / (1 - 0.9 ** self.t)
                vhat = self._bias_v / (1 - 0.999 ** self.t)
                g = mhat / (np.sqrt(vhat) + 1e-8)
            bias = bias - lr * g
        return SourceSet(p, w), bias


def fit_sdf_epoch(engine: Engine, sources: SourceSet, bias: float, q, target,
                  opt: Optimizer, epoch: int):
    """One epoch of the reference fit-sdf loop (cli.py:129-145) on the device:
    explicit layer forward at q, loss + tangent of values + bias (fused),
    L1 term, JVP, optimizer step.  Returns (sources, bias, loss, data_loss)
    with loss = data_loss + L1 value, as the reference's metrics rows."""
    tc = opt.config
    res = explicit_forward(engine, sources, q)
    stats, tangent = _loss_device(res.values, target, tc.loss, bias=bias)
    g = explicit_jvp(tangent, res)
    reg = 0.0
    if tc.l1_weight:
        reg = tc.l1_weight * float(sources.w.abs().double().sum().item())
    st = stats.cpu().numpy()
    sources, bias = opt.step(sources, g.w_bar, g.p_bar, epoch, bias=bias,
                             bias_bar=float(st[2]), l1_weight=tc.l1_weight)
    return sources, bias, float(st[1]) + reg, float(st[1])


def cgls_sdf(engine: Engine, p, q, target, iterations: int) -> dict:
    """Conjugate-gradient least squares on the (w, bias) sub-problem of fit-sdf
    (reference cli.py:173-224): positions stay fixed, each iteration is one
    forward product (expand the sources, evaluate at the samples) and one
    adjoint product (expand the residual at the samples, evaluate at the
    sources).  The CG vectors and scalars are float64 device tensors; the
    products run through the fp32 engine; nothing is read back until the end.

    Returns {"w": (N, 1), "bias": float, "mae": [per iteration], "final_mae"}.
    """
    pd = to_device(p, 3, points=True)
    qd = to_device(q, 3, points=True)
    d = to_device(target).reshape(-1).double()
    value = _lib.L2P_VALUE

    def a_fwd(w, b):
        acc = engine.expand_device(pd, w.float().reshape(-1, 1).contiguous())
        return acc.eval_device(qd, value)["value"].reshape(-1).double() + b

    def a_adj(r):
        acc = engine.expand_device(qd, r.float().reshape(-1, 1).contiguous())
        return acc.eval_device(pd, value)["value"].reshape(-1).double(), r.sum()

    with engine.flag.deferred():
        w = torch.zeros(pd.shape[0], dtype=torch.float64, device=pd.device)
        bias = torch.zeros((), dtype=torch.float64, device=pd.device)
        r = d - a_fwd(w, bias)
        s_w, s_b = a_adj(r)
        pk_w, pk_b = s_w.clone(), s_b.clone()
        gamma = s_w @ s_w + s_b * s_b
        maes = []
        for _ in range(iterations):
            qk = a_fwd(pk_w, pk_b)
            alpha = gamma / (qk @ qk)
            w += alpha * pk_w
            bias += alpha * pk_b
            r -= alpha * qk
            s_w, s_b = a_adj(r)
            gamma_new = s_w @ s_w + s_b * s_b
            beta = gamma_new / gamma
            pk_w = s_w + beta * pk_w
            pk_b = s_b + beta * pk_b
            gamma = gamma_new
            maes.append(r.abs().mean())
        final = (a_fwd(w, bias) - d).abs().mean()
    engine.flag.raise_if_set("source/query")
    host = torch.stack(maes + [final, bias]).cpu().numpy() if maes else \
        torch.stack([final, bias]).cpu().numpy()
    return {"w": w.float().reshape(-1, 1), "bias": float(host[-1]),
            "mae": [float(v) for v in host[:-2]], "final_mae": float(host[-2])}


def fit_depth_epoch(engine: Engine, sources: SourceSet, bias: float, bundle, target,
                    opt: Optimizer, epoch: int, miss_penalty: float = 0.1):
    """One epoch of the reference fit-depth loop (cli.py:288-306): depth layer,
    masked loss over rays that hit and have a finite target, JVP, L1, step;
    the bias is pushed by miss_penalty * miss fraction.  ``target`` holds NaN
    where there is no valid depth.  Returns (sources, bias, loss, miss_fraction)."""
    tc = opt.config
    res = depth_forward(engine, sources, bundle, bias=bias)
    tgt = to_device(target).reshape(-1)
    valid = torch.isfinite(tgt)
    mask = res.dev["hit"].bool() & valid
    lengths = res.lengths if isinstance(res.lengths, torch.Tensor) else to_device(res.lengths)
    pred = torch.where(mask, lengths.to(torch.float32), 0.0)
    tg = torch.where(mask, tgt.to(torch.float32), 0.0)
    stats, tangent = _loss_device(pred, tg, tc.loss, mask=mask)
    g = depth_jvp(tangent.reshape(-1), res)
    miss = (~mask).sum()
    host = torch.cat([stats, miss.double().reshape(1)]).cpu().numpy()
    miss_frac = float(host[3]) / mask.numel()
    sources, bias = opt.step(sources, g.w_bar, g.p_bar, epoch, bias=bias,
                             bias_bar=miss_penalty * miss_frac, l1_weight=tc.l1_weight)
    return sources, bias, float(host[1]), miss_frac


def fit_radiance_epoch(engine: Engine, p, w_sigma, w_color, bundle, target, background,
                       opt: Optimizer, epoch: int):
    """One epoch of the reference fit-radiance loop (cli.py:363-382) on one
    minibatch of rays: volumetric forward, loss + tangent of rgb (fused),
    volumetric JVP, L1 on the packed weights, one step over (p, [w_sigma |
    w_color]).  The minibatch draw stays the caller's (the reference draws it
    on the host).  Returns (p, w_sigma, w_color, loss)."""
    tc = opt.config
    res = volumetric_forward(engine, p, w_sigma, w_color, bundle, background)
    rgb = res.rgb if isinstance(res.rgb, torch.Tensor) else to_device(res.rgb)
    stats, tangent = _loss_device(rgb, target, tc.loss)
    g = volumetric_jvp(tangent.reshape(rgb.shape), res)
    ws, wc = to_device(w_sigma), to_device(w_color)
    packed = SourceSet(to_device(p, 3, points=True),
                       torch.cat([ws.reshape(ws.shape[0], -1), wc.reshape(wc.shape[0], -1)], 1))
    packed, _ = opt.step(packed, g.w_bar, g.p_bar, epoch, l1_weight=tc.l1_weight)
    return packed.p, packed.w[:, :1], packed.w[:, 1:], float(stats[1].item())
