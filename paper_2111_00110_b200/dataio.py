"""Data formats: drop-in for the reference ``fc2t2.dataio``.

Same names, byte formats and errors as the reference (dataio.py:1-314), so
files written by either side load in the other:

* FCPT points  ``b"FCPT" | version u32 | M u64 | C u32 | M x (x, y, z, v1..vC) f64``
  (little-endian), or CSV with an ``x,y,z,v1..`` header;
* FCCK checkpoints ``b"FCCK" | version u32 | levels u32 | rho u32 |
  kernel u32 | alpha f64 | N u64 | C u32 | bias f64 | p (N x 3 f64) |
  w (N x C f64) | has_opt u32``;
* camera JSON frames ``{eye, gaze, up, fov_y, width, height, image?}``;
* binary PPM (P6, 8-bit, round-half-up) images.

The host functions keep float64 numpy (the reference's representation).  The
device loaders are what feeds the GPU path: ``load_points_device`` and
``load_checkpoint_device`` stream the float64 payload through two pinned
staging buffers (disk read of chunk k+1 overlaps the H2D copy of chunk k)
and one fused kernel (csrc/io.cu, ``fc2t2_unpack_rows``) de-interleaves the
rows into float32 ``p`` / values columns and finds the first point outside
(-1, 1)^3 -- the check ``PointSampleSet`` makes -- with a single flag read.
"""

from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field

import numpy as np

from .ray import Camera

POINTS_MAGIC = b"FCPT"
CHECKPOINT_MAGIC = b"FCCK"
POINTS_VERSION = 1
CHECKPOINT_VERSION = 1
_KERNEL_CODES = {"gaussian": 0}
_KERNEL_NAMES = {code: name for name, code in _KERNEL_CODES.items()}
_POINTS_HEAD = struct.Struct("<IQI")        # version, M, C
_CKPT_HEAD = struct.Struct("<IIIId")        # version, levels, rho, kernel, alpha
_CKPT_SIZES = struct.Struct("<QId")         # N, C, bias
_CAMERA_FIELDS = ("eye", "gaze", "up", "fov_y", "width", "height")
STAGE_BYTES = 64 << 20                      # pinned staging chunk of the device loaders


class FormatError(ValueError):
    """Malformed or unsupported file contents (reference dataio.py:36-37)."""


def _first_outside(loc: np.ndarray) -> int:
    bad = np.flatnonzero(~np.all(np.abs(loc) < 1.0, axis=1))
    return int(bad[0]) if bad.size else -1


@dataclass
class PointSampleSet:
    """Locations (M, 3) with per-point values (M, C), float64 (reference
    dataio.py:40-63); every location must lie strictly inside (-1, 1)^3."""

    locations: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.locations = np.atleast_2d(np.asarray(_host(self.locations), dtype=np.float64))
        vals = np.asarray(_host(self.values), dtype=np.float64)
        self.values = vals.reshape(-1, 1) if vals.ndim == 1 else vals
        bad = _first_outside(self.locations)
        if bad >= 0:
            raise FormatError(f"point {bad} lies outside (-1, 1)^3")

    @property
    def count(self) -> int:
        return int(self.locations.shape[0])

    @property
    def channels(self) -> int:
        return int(self.values.shape[1])


def _host(x):
    """numpy view of x (device tensors are copied back)."""
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().double().numpy()
    except ImportError:
        pass
    return x


def normalize_locations(raw, margin: float = 0.05):
    """Affine map into (-1, 1)^3 with a relative margin; returns
    (mapped, (scale, offset)) with mapped = (raw - offset) * scale
    (reference dataio.py:66-79)."""
    raw = np.atleast_2d(np.asarray(raw, dtype=np.float64))
    lo, hi = raw.min(axis=0), raw.max(axis=0)
    offset = 0.5 * (lo + hi)
    scale = 1.0 / (np.maximum(0.5 * (hi - lo), 1e-12) * (1.0 + margin))
    return (raw - offset) * scale, (scale, offset)


# ------------------------------------------------------------------ points ---

def _points_fmt(path, fmt):
    return fmt or ("csv" if str(path).endswith(".csv") else "binary")


def save_points(path: str, points: PointSampleSet, fmt: str | None = None) -> None:
    """CSV (17 significant digits, exact round trip) or FCPT binary
    (reference dataio.py:84-98)."""
    rows = np.concatenate([points.locations, points.values], axis=1)
    if _points_fmt(path, fmt) == "csv":
        head = ",".join(["x", "y", "z"] + [f"v{i + 1}" for i in range(points.channels)])
        np.savetxt(path, rows, delimiter=",", header=head, comments="", fmt="%.17g")
        return
    with open(path, "wb") as f:
        f.write(POINTS_MAGIC + _POINTS_HEAD.pack(POINTS_VERSION, points.count, points.channels))
        f.write(np.ascontiguousarray(rows, dtype="<f8").tobytes())


def _load_csv_rows(path) -> np.ndarray:
    """Blank lines are skipped; errors name the row as the reference counts it
    (header = 1, first data row = 2, among non-blank lines)."""
    with open(path) as f:
        lines = [ln.strip() for ln in f if ln.strip()]
    if not lines:
        raise FormatError(f"{path}: empty points file")
    cols = lines[0].split(",")
    if cols[:3] != ["x", "y", "z"]:
        raise FormatError(f"{path}:1: expected header starting x,y,z")
    out = np.empty((len(lines) - 1, len(cols)))
    for r, ln in enumerate(lines[1:]):
        parts = ln.split(",")
        if len(parts) != len(cols):
            raise FormatError(f"{path}:{r + 2}: expected {len(cols)} columns")
        try:
            out[r] = [float(x) for x in parts]
        except ValueError as exc:
            raise FormatError(f"{path}:{r + 2}: {exc}") from None
    return out


def _points_header(f, path) -> tuple[int, int]:
    magic = f.read(4)
    if magic != POINTS_MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    head = f.read(_POINTS_HEAD.size)
    if len(head) != _POINTS_HEAD.size:
        raise FormatError(f"{path}: truncated header")
    version, m, c = _POINTS_HEAD.unpack(head)
    if version > POINTS_VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    return m, c


def load_points(path: str, fmt: str | None = None) -> PointSampleSet:
    """Reference dataio.py:101-130 (host float64)."""
    if _points_fmt(path, fmt) == "csv":
        data = _load_csv_rows(path)
    else:
        with open(path, "rb") as f:
            m, c = _points_header(f, path)
            nbytes = m * (3 + c) * 8
            buf = f.read(nbytes)
            if len(buf) != nbytes:
                raise FormatError(f"{path}: truncated payload")
        data = np.frombuffer(buf, dtype="<f8").reshape(m, 3 + c).copy()
    return PointSampleSet(locations=data[:, :3], values=data[:, 3:])


# ----------------------------------------------------------------- cameras ---

def load_cameras(path: str) -> list[tuple[Camera, str | None]]:
    """JSON frames -> [(Camera, image path or None)]; gaze and up are
    normalised (reference dataio.py:140-162)."""
    with open(path) as f:
        frames = json.load(f)
    out = []
    for i, fr in enumerate(frames):
        missing = [k for k in _CAMERA_FIELDS if k not in fr]
        if missing:
            raise FormatError(f"{path}[{i}]: missing field {missing[0]!r}")
        eye = np.asarray(fr["eye"], dtype=np.float64)
        unit = {}
        for name in ("gaze", "up"):
            v = np.asarray(fr[name], dtype=np.float64)
            n = float(np.linalg.norm(v))
            if not np.isfinite(n) or n == 0.0:
                raise FormatError(f"{path}[{i}]: {name} is not normalizable")
            unit[name] = v / n
        cam = Camera(position=eye, look_at=eye + unit["gaze"], up=unit["up"],
                     fov_deg=float(fr["fov_y"]), width=int(fr["width"]),
                     height=int(fr["height"]))
        out.append((cam, fr.get("image")))
    return out


def save_cameras(path: str, frames) -> None:
    """Reference dataio.py:165-175."""
    rows = []
    for cam, image in frames:
        row = {"eye": [float(x) for x in cam.position],
               "gaze": [float(x) for x in cam.look_at - cam.position],
               "up": [float(x) for x in cam.up], "fov_y": cam.fov_deg,
               "width": cam.width, "height": cam.height}
        if image:
            row["image"] = image
        rows.append(row)
    with open(path, "w") as f:
        json.dump(rows, f, indent=1)


# ------------------------------------------------------------------ images ---

def _quantize(pixels) -> np.ndarray:
    """[0, 1] -> u8, round half up (reference dataio.py:180-182)."""
    return np.floor(np.clip(pixels, 0.0, 1.0) * 255.0 + 0.5).astype(np.uint8)


def save_image(path: str, pixels) -> None:
    """H x W (grey) or H x W x 3 reals in [0, 1] -> binary PPM, or PNG by
    extension (reference dataio.py:185-199)."""
    px = np.asarray(_host(pixels), dtype=np.float64)
    if px.ndim == 2:
        px = np.repeat(px[:, :, None], 3, axis=2)
    q = _quantize(px)
    if str(path).endswith(".png"):
        import matplotlib.image
        matplotlib.image.imsave(path, q)
        return
    h, w = q.shape[:2]
    with open(path, "wb") as f:
        f.write(b"P6\n%d %d\n255\n" % (w, h))
        f.write(q.tobytes())


def load_image(path: str) -> np.ndarray:
    """Image -> H x W x 3 floats in [0, 1] (reference dataio.py:202-223)."""
    if str(path).endswith(".png"):
        import matplotlib.image
        return np.asarray(matplotlib.image.imread(path), dtype=np.float64)[:, :, :3]
    data = open(path, "rb").read()
    if data[:2] != b"P6":
        raise FormatError(f"{path}: not a P6 PPM")
    # header: width, height and maxval as whitespace-separated integers after
    # the magic, '#' starting a comment that runs to the end of its line
    pos, hdr = 2, []
    while len(hdr) < 3:
        eol = data.find(b"\n", pos)
        if pos >= len(data):
            raise FormatError(f"{path}: truncated header")
        line = data[pos:] if eol < 0 else data[pos:eol + 1]
        pos += len(line)
        hdr.extend(int(t) for t in line.partition(b"#")[0].split())
    w, h, maxval = hdr[:3]
    if maxval != 255:
        raise FormatError(f"{path}: only 8-bit PPM supported")
    npix = 3 * w * h
    if len(data) - pos < npix:
        raise FormatError(f"{path}: truncated pixel data")
    return np.frombuffer(data, dtype=np.uint8, count=npix, offset=pos).reshape(h, w, 3) / 255.0


# ------------------------------------------------------------- checkpoints ---

@dataclass
class Checkpoint:
    """Reference dataio.py:228-238."""

    levels: int
    rho: int
    kernel: str
    alpha: float
    p: np.ndarray
    w: np.ndarray
    bias: float = 0.0
    version: int = CHECKPOINT_VERSION
    extra: dict = field(default_factory=dict)


def save_checkpoint(path: str, ckpt: Checkpoint) -> None:
    """Byte-identical for identical inputs (reference dataio.py:241-252);
    device tensors are accepted and written as float64."""
    p = np.ascontiguousarray(_host(ckpt.p), dtype="<f8")
    w = np.ascontiguousarray(_host(ckpt.w), dtype="<f8")
    if w.ndim == 1:
        w = w.reshape(-1, 1)
    n, c = w.shape
    with open(path, "wb") as f:
        f.write(CHECKPOINT_MAGIC)
        f.write(_CKPT_HEAD.pack(CHECKPOINT_VERSION, ckpt.levels, ckpt.rho,
                                _KERNEL_CODES[ckpt.kernel], float(ckpt.alpha)))
        f.write(_CKPT_SIZES.pack(n, c, float(ckpt.bias)))
        f.write(p.tobytes())
        f.write(w.tobytes())
        f.write(struct.pack("<I", 0))          # has_opt: no optimizer state


def _ckpt_header(f, path):
    magic = f.read(4)
    if magic != CHECKPOINT_MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    head = f.read(_CKPT_HEAD.size + _CKPT_SIZES.size)
    if len(head) != _CKPT_HEAD.size + _CKPT_SIZES.size:
        raise FormatError(f"{path}: truncated header")
    version, levels, rho, kcode, alpha = _CKPT_HEAD.unpack(head[:_CKPT_HEAD.size])
    if version > CHECKPOINT_VERSION:
        raise FormatError(f"{path}: unsupported version {version}")
    if kcode not in _KERNEL_NAMES:
        raise FormatError(f"{path}: unknown kernel code {kcode}")
    n, c, bias = _CKPT_SIZES.unpack(head[_CKPT_HEAD.size:])
    return version, levels, rho, _KERNEL_NAMES[kcode], alpha, n, c, bias


def load_checkpoint(path: str) -> Checkpoint:
    """Reference dataio.py:255-273 (host float64)."""
    with open(path, "rb") as f:
        version, levels, rho, kernel, alpha, n, c, bias = _ckpt_header(f, path)
        pb, wb = f.read(n * 24), f.read(n * c * 8)
    if len(pb) != n * 24 or len(wb) != n * c * 8:
        raise FormatError(f"{path}: truncated parameter block")
    return Checkpoint(levels=levels, rho=rho, kernel=kernel, alpha=alpha,
                      p=np.frombuffer(pb, "<f8").reshape(n, 3).copy(),
                      w=np.frombuffer(wb, "<f8").reshape(n, c).copy(), bias=bias,
                      version=version)


# ------------------------------------------------------------ device loads ---

def _stream_rows_to_device(f, path, m: int, width: int, dev):
    """Read m rows of `width` float64 from f into one device buffer through
    two pinned staging chunks (read of chunk k+1 overlaps the copy of k)."""
    import torch
    nbytes = m * width * 8
    out = torch.empty(m * width, dtype=torch.float64, device=dev)
    if nbytes == 0:
        return out
    raw = out.view(torch.uint8)
    step = max(width * 8, (STAGE_BYTES // (width * 8)) * width * 8)
    stage = [torch.empty(min(step, nbytes), dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    done = [None, None]
    stream = torch.cuda.current_stream(dev)
    for k, off in enumerate(range(0, nbytes, step)):
        b = k & 1
        if done[b] is not None:
            done[b].synchronize()            # the copy out of this buffer has finished
        n = min(step, nbytes - off)
        got = f.readinto(memoryview(stage[b].numpy())[:n])
        if got != n:
            raise FormatError(f"{path}: truncated payload")
        raw[off:off + n].copy_(stage[b][:n], non_blocking=True)
        done[b] = torch.cuda.Event()
        done[b].record(stream)
    for e in done:
        if e is not None:
            e.synchronize()                  # staging buffers are reused/freed after return
    return out


def _unpack(rows, m: int, c: int, dev, check: bool):
    import torch

    from . import _lib
    from .expansion import _ptr
    p = torch.empty((m, 3), dtype=torch.float32, device=dev)
    v = torch.empty((m, c), dtype=torch.float32, device=dev) if c else None
    bad = torch.full((1,), -1, dtype=torch.int64, device=dev) if check else None   # UINT64_MAX
    s = torch.cuda.current_stream(dev).cuda_stream
    _lib.call("fc2t2_unpack_rows", _ptr(rows), m, c, _ptr(p), _ptr(v), _ptr(bad), s)
    return p, v, bad


def load_points_device(path: str, device=None):
    """FCPT file -> (locations (M, 3), values (M, C)) float32 tensors on the
    GPU, with the PointSampleSet domain check (same FormatError, same first
    point named).  CSV files are parsed on the host and uploaded."""
    import torch
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    if _points_fmt(path, None) == "csv":
        ps = load_points(path)
        return (torch.from_numpy(ps.locations).float().to(dev),
                torch.from_numpy(ps.values).float().to(dev))
    with open(path, "rb") as f:
        m, c = _points_header(f, path)
        rows = _stream_rows_to_device(f, path, m, 3 + c, dev)
    p, v, bad = _unpack(rows, m, c, dev, True)
    first = int(bad.item())
    if first != -1:
        raise FormatError(f"point {first} lies outside (-1, 1)^3")
    return p, (v if v is not None else torch.empty((m, 0), dtype=torch.float32, device=dev))


def load_checkpoint_device(path: str, device=None) -> Checkpoint:
    """FCCK file -> Checkpoint whose p (N, 3) and w (N, C) are float32 GPU
    tensors (the SourceSet the layers take)."""
    import torch
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    with open(path, "rb") as f:
        version, levels, rho, kernel, alpha, n, c, bias = _ckpt_header(f, path)
        try:
            prow = _stream_rows_to_device(f, path, n, 3, dev)
            wrow = _stream_rows_to_device(f, path, n * c, 1, dev)
        except FormatError:
            raise FormatError(f"{path}: truncated parameter block") from None
    p, _, _ = _unpack(prow, n, 0, dev, False)
    w = wrow.to(torch.float32).reshape(n, c)
    return Checkpoint(levels=levels, rho=rho, kernel=kernel, alpha=alpha, p=p, w=w, bias=bias,
                      version=version)


# ------------------------------------------------------ analytic SDF sets ---

def sdf_sphere(center, radius: float):
    c = np.asarray(center, dtype=np.float64)
    return lambda q: np.linalg.norm(q - c, axis=-1) - radius


def sdf_box(center, half):
    c = np.asarray(center, dtype=np.float64)
    h = np.asarray(half, dtype=np.float64)

    def f(q):
        d = np.abs(q - c) - h
        return np.linalg.norm(np.maximum(d, 0.0), axis=-1) + np.minimum(d.max(axis=-1), 0.0)
    return f


def sdf_torus(center, major: float, minor: float):
    c = np.asarray(center, dtype=np.float64)

    def f(q):
        d = q - c
        return np.hypot(np.hypot(d[..., 0], d[..., 2]) - major, d[..., 1]) - minor
    return f


def sdf_union(*fs):
    return lambda q: np.minimum.reduce([f(q) for f in fs])


def sample_sdf(sdf, count: int, seed: int = 0, margin: float = 0.05) -> PointSampleSet:
    """Seeded uniform samples inside the domain with their SDF values
    (reference dataio.py:303-309)."""
    rng = np.random.default_rng(seed)
    q = rng.uniform(-1.0 + margin, 1.0 - margin, (count, 3))
    return PointSampleSet(locations=q, values=sdf(q))
