"""torch.autograd wrappers of the layers (optional
``torch.autograd.Function`` entry points for explicit(q, p, w),
depth + normal(p, w, bias, rays) and radiance(p, w_sigma, w_colour, rays, bg);
plus the line integral).

Each backward is the layer's own JVP -- one insertion and one expansion, the
self-adjoint pipeline of the reference (layers.py:1-22) -- so gradients equal
the ``*_jvp`` outputs exactly; the wrappers only route them to the inputs.
Inputs are CUDA float32 tensors; the Engine is passed through (no gradient).
"""

from __future__ import annotations

import torch

from .expansion import Engine, SourceSet
from .layers import (depth_forward, depth_surface_jvp, explicit_forward, explicit_jvp,
                     line_integral_forward, line_integral_jvp, volumetric_forward, volumetric_jvp)
from .ray import RayBundle


class _Explicit(torch.autograd.Function):
    @staticmethod
    def forward(ctx, engine: Engine, p, w, q):
        res = explicit_forward(engine, SourceSet(p.detach(), w.detach()), q.detach())
        ctx.res, ctx.w_shape = res, w.shape
        return res.values

    @staticmethod
    def backward(ctx, y_bar):
        g = explicit_jvp(y_bar.contiguous(), ctx.res)
        return None, g.p_bar, g.w_bar.reshape(ctx.w_shape), g.q_bar


def explicit(engine: Engine, p: torch.Tensor, w: torch.Tensor, q: torch.Tensor) -> torch.Tensor:
    """f(q) = sum_i w_i psi(q - p_i) (reference explicit_forward, layers.py:167-173)
    with gradients to p, w and q (explicit_jvp, layers.py:176-188)."""
    return _Explicit.apply(engine, p, w, q)


class _DepthNormal(torch.autograd.Function):
    @staticmethod
    def forward(ctx, engine: Engine, p, w, origins, directions, bias):
        res = depth_forward(engine, SourceSet(p.detach(), w.detach()),
                            RayBundle(origins.detach(), directions.detach()), bias=float(bias))
        ctx.res, ctx.w_shape = res, w.shape
        ctx.mark_non_differentiable(res.hit)
        return res.lengths, res.grads, res.hit

    @staticmethod
    def backward(ctx, y_len, y_grad, _y_hit):
        g = depth_surface_jvp(y_len, y_grad, ctx.res)
        return None, g.p_bar, g.w_bar.reshape(ctx.w_shape), None, None, None


def depth_normal(engine: Engine, p: torch.Tensor, w: torch.Tensor, origins: torch.Tensor,
                 directions: torch.Tensor, bias: float = 0.05):
    """(ray lengths to the first root of f + bias (NaN on a miss), the field
    gradient there (unnormalised surface normal), hit mask); gradients to p and
    w through one fused depth + normal insertion (layers.py:285-356).  Losses
    must mask missed rays (their lengths are NaN)."""
    return _DepthNormal.apply(engine, p, w, origins, directions, bias)


class _Radiance(torch.autograd.Function):
    @staticmethod
    def forward(ctx, engine: Engine, p, w_sigma, w_color, origins, directions, background):
        res = volumetric_forward(engine, p.detach(), w_sigma.detach(), w_color.detach(),
                                 RayBundle(origins.detach(), directions.detach()), background)
        ctx.res = res
        ctx.shapes = (w_sigma.shape, w_color.shape)
        return res.rgb

    @staticmethod
    def backward(ctx, y_bar):
        g = volumetric_jvp(y_bar.contiguous(), ctx.res)
        ws, wc = ctx.shapes
        return (None, g.p_bar, g.w_bar[:, :1].reshape(ws), g.w_bar[:, 1:].reshape(wc), None,
                None, None)


def radiance(engine: Engine, p: torch.Tensor, w_sigma: torch.Tensor, w_color: torch.Tensor,
             origins: torch.Tensor, directions: torch.Tensor, background) -> torch.Tensor:
    """Emission/absorption rendering (reference volumetric_forward, layers.py:427-480)
    with gradients to p, the density and the colour weights (volumetric_jvp,
    layers.py:483-544)."""
    return _Radiance.apply(engine, p, w_sigma, w_color, origins, directions, background)


class _LineIntegral(torch.autograd.Function):
    @staticmethod
    def forward(ctx, engine: Engine, p, w, origins, directions):
        res = line_integral_forward(engine, SourceSet(p.detach(), w.detach()),
                                    RayBundle(origins.detach(), directions.detach()))
        ctx.res, ctx.w_shape = res, w.shape
        return res.values

    @staticmethod
    def backward(ctx, y_bar):
        g = line_integral_jvp(y_bar.contiguous(), ctx.res)
        return None, g.p_bar, g.w_bar.reshape(ctx.w_shape), None, None


def line_integral(engine: Engine, p: torch.Tensor, w: torch.Tensor, origins: torch.Tensor,
                  directions: torch.Tensor) -> torch.Tensor:
    """Integral of the field along each ray through the domain (reference
    line_integral_forward / _jvp, layers.py:371-402) with gradients to p, w."""
    return _LineIntegral.apply(engine, p, w, origins, directions)
