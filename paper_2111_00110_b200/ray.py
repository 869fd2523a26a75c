"""Cameras, ray bundles and grid traversal: drop-in for ``fc2t2.ray``.

Camera / generate_rays build the ray bundle exactly as the reference
(ray.py:26-77, float64, pixel centres, row-major) -- this is input
preparation; the bundle is uploaded once as (R, 3) float64 device tensors.
``traverse`` (ray.py:123-157) runs on the device: a count pass, an exclusive
scan and a fill pass of the per-ray walker in csrc/rays.cu, bit-exact with the
reference's box lists.  The layers never materialise the traversal; they walk
rays on the fly (csrc/rays.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .expansion import _device, _ptr, _stream
from .kernel import level_resolution

MIN_SEGMENT = 1e-12


@dataclass
class Camera:
    """Pinhole camera; rays go through pixel centres (reference ray.py:26-48)."""

    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray
    fov_deg: float
    width: int
    height: int

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.look_at = np.asarray(self.look_at, dtype=np.float64)
        self.up = np.asarray(self.up, dtype=np.float64)

    def basis(self):
        fwd = self.look_at - self.position
        fwd = fwd / np.linalg.norm(fwd)
        right = np.cross(fwd, self.up)
        right = right / np.linalg.norm(right)
        return fwd, right, np.cross(fwd, right)


@dataclass
class RayBundle:
    """Origins and unit directions, one row per ray (reference ray.py:51-60).

    ``origins`` / ``directions`` keep the caller's arrays; ``dev()`` returns
    the float64 device copies (uploaded once)."""

    origins: object
    directions: object

    def __post_init__(self):
        self._dev = None

    @property
    def count(self) -> int:
        return int(self.origins.shape[0])

    def dev(self):
        if self._dev is None:
            def up(a):
                if isinstance(a, torch.Tensor):
                    return a.to(device=_device(), dtype=torch.float64).reshape(-1, 3).contiguous()
                return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).reshape(-1, 3)
                                        ).to(_device())
            self._dev = (up(self.origins), up(self.directions))
        return self._dev


def generate_rays(camera: Camera) -> RayBundle:
    """One ray per pixel, row-major over (height, width) (reference ray.py:63-77)."""
    fwd, right, down = camera.basis()
    tan = np.tan(np.radians(camera.fov_deg) / 2.0)
    aspect = camera.width / camera.height
    xs = (np.arange(camera.width) + 0.5) / camera.width * 2.0 - 1.0
    ys = (np.arange(camera.height) + 0.5) / camera.height * 2.0 - 1.0
    gy, gx = np.meshgrid(ys, xs, indexing="ij")
    dirs = (fwd[None, :] + gx.reshape(-1, 1) * (tan * aspect) * right[None, :]
            + gy.reshape(-1, 1) * tan * down[None, :])
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return RayBundle(origins=np.broadcast_to(camera.position, dirs.shape).copy(), directions=dirs)


@dataclass
class Traversal:
    """Per-segment view of a bundle walked through a level (reference ray.py:80-98).
    Device tensors: ray_id (S,) int32, t0/t1 (S,) float64, box (S, 3) int32,
    offsets (R+1,) int64."""

    level: int
    ray_id: torch.Tensor
    t0: torch.Tensor
    t1: torch.Tensor
    box: torch.Tensor
    offsets: torch.Tensor

    @property
    def count(self) -> int:
        return int(self.ray_id.shape[0])


def segment_offsets(bundle: RayBundle, level: int):
    """Per-ray segment counts -> (offsets uint32 (R+1,), total S)."""
    org, dirs = bundle.dev()
    R = bundle.count
    counts = torch.zeros(R + 1, dtype=torch.int32, device=org.device)
    _lib.call("fc2t2_traverse_count", level, _ptr(org), _ptr(dirs), R, _ptr(counts), _stream())
    offs = torch.empty_like(counts)
    ws_b = int(_lib.lib().fc2t2_scan_workspace_size(R + 1))
    ws = torch.empty(max(ws_b, 4), dtype=torch.uint8, device=org.device)
    _lib.call("fc2t2_scan_u32", _ptr(counts), _ptr(offs), R + 1, _ptr(ws), ws_b, _stream())
    return offs, int(offs[R].item())


def traverse(bundle: RayBundle, level: int) -> Traversal:
    """Split each ray into per-box segments (reference ray.py:123-157), on the device."""
    org, dirs = bundle.dev()
    R = bundle.count
    offs, S = segment_offsets(bundle, level)
    dev = org.device
    ray_id = torch.empty(max(S, 1), dtype=torch.int32, device=dev)
    t0 = torch.empty(max(S, 1), dtype=torch.float64, device=dev)
    t1 = torch.empty(max(S, 1), dtype=torch.float64, device=dev)
    box = torch.empty((max(S, 1), 3), dtype=torch.int32, device=dev)
    _lib.call("fc2t2_traverse_fill", level, _ptr(org), _ptr(dirs), R, _ptr(offs), _ptr(ray_id),
              _ptr(t0), _ptr(t1), _ptr(box), _stream())
    return Traversal(level, ray_id[:S], t0[:S], t1[:S], box[:S], offs.long())


def domain_span(bundle: RayBundle):
    """Entry / exit parameters against (-1, 1)^3 (reference ray.py:101-120)."""
    o, d = bundle.dev()
    with np.errstate(divide="ignore", invalid="ignore"):
        lo = (-1.0 - o) / d
        hi = (1.0 - o) / d
    near = torch.where(torch.isnan(lo), torch.full_like(lo, -np.inf), torch.minimum(lo, hi))
    far = torch.where(torch.isnan(hi), torch.full_like(hi, np.inf), torch.maximum(lo, hi))
    par = d == 0.0
    inside = o.abs() < 1.0
    inf = torch.full_like(near, np.inf)
    near = torch.where(par, torch.where(inside, -inf, inf), near)
    far = torch.where(par, torch.where(inside, inf, -inf), far)
    return near.max(dim=1).values.clamp(min=0.0), far.min(dim=1).values


def segment_geometry(trav: Traversal, bundle: RayBundle, level: int):
    """Per-segment (d, r, s) (reference ray.py:249-258), float64 on the device."""
    o, dirs = bundle.dev()
    rid = trav.ray_id.long()
    oo, rr = o[rid], dirs[rid]
    base = oo + trav.t0[:, None] * rr
    w = 2.0 / level_resolution(level)
    centre = -1.0 + (trav.box.double() + 0.5) * w
    return base - centre, rr, trav.t1 - trav.t0
