"""Device loaders of dataio (pinned staging + csrc/io.cu unpack kernel)."""

import struct
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2111_00110_b200 import dataio

pytestmark = pytest.mark.gpu
IO = Path(__file__).resolve().parent / "golden" / "io"


def _write_raw_points(path, rows):
    m, w = rows.shape
    with open(path, "wb") as f:
        f.write(b"FCPT" + struct.pack("<IQI", 1, m, w - 3))
        f.write(np.ascontiguousarray(rows, dtype="<f8").tobytes())


def test_load_points_device_matches_host(cuda):
    host = dataio.load_points(str(IO / "points.fcpt"))
    p, v = dataio.load_points_device(str(IO / "points.fcpt"))
    assert p.is_cuda and p.dtype == torch.float32 and v.shape == (50, 2)
    assert np.array_equal(p.cpu().numpy(), host.locations.astype(np.float32))
    assert np.array_equal(v.cpu().numpy(), host.values.astype(np.float32))
    p2, v2 = dataio.load_points_device(str(IO / "points.csv"))
    assert torch.equal(p, p2) and torch.equal(v, v2)


@pytest.mark.parametrize("stage", [40, 4096, 64 << 20])
def test_load_points_device_chunked_and_domain(cuda, tmp_path, monkeypatch, stage):
    """Many staging chunks (row-aligned, odd width) and the first bad row."""
    monkeypatch.setattr(dataio, "STAGE_BYTES", stage)
    rng = np.random.default_rng(9)
    rows = np.concatenate([rng.uniform(-0.99, 0.99, (3001, 3)), rng.normal(size=(3001, 4))], 1)
    _write_raw_points(tmp_path / "a.fcpt", rows)
    p, v = dataio.load_points_device(str(tmp_path / "a.fcpt"))
    assert np.array_equal(p.cpu().numpy(), rows[:, :3].astype(np.float32))
    assert np.array_equal(v.cpu().numpy(), rows[:, 3:].astype(np.float32))
    rows[2500, 1] = 1.0
    rows[1700, 2] = -1.5
    rows[2900, 0] = np.nan
    _write_raw_points(tmp_path / "b.fcpt", rows)
    with pytest.raises(dataio.FormatError, match="point 1700 "):
        dataio.load_points_device(str(tmp_path / "b.fcpt"))
    raw = (tmp_path / "a.fcpt").read_bytes()
    (tmp_path / "t.fcpt").write_bytes(raw[:-8])
    with pytest.raises(dataio.FormatError, match="truncated"):
        dataio.load_points_device(str(tmp_path / "t.fcpt"))


def test_load_points_device_empty_and_zero_channels(cuda, tmp_path):
    _write_raw_points(tmp_path / "e.fcpt", np.zeros((0, 3)))
    p, v = dataio.load_points_device(str(tmp_path / "e.fcpt"))
    assert p.shape == (0, 3) and v.shape == (0, 0)
    _write_raw_points(tmp_path / "z.fcpt", np.full((5, 3), 0.25))
    p, v = dataio.load_points_device(str(tmp_path / "z.fcpt"))
    assert v.shape == (5, 0) and bool((p == 0.25).all())


def test_load_checkpoint_device(cuda, tmp_path):
    host = dataio.load_checkpoint(str(IO / "sdf.ckpt"))
    dev = dataio.load_checkpoint_device(str(IO / "sdf.ckpt"))
    assert (dev.levels, dev.rho, dev.kernel, dev.alpha, dev.bias) == \
        (host.levels, host.rho, host.kernel, host.alpha, host.bias)
    assert np.array_equal(dev.p.cpu().numpy(), host.p.astype(np.float32))
    assert np.array_equal(dev.w.cpu().numpy(), host.w.astype(np.float32))
    # device tensors save back as float64 (exact for float32 values)
    dataio.save_checkpoint(str(tmp_path / "r.ckpt"), dev)
    again = dataio.load_checkpoint(str(tmp_path / "r.ckpt"))
    assert np.array_equal(again.p, host.p.astype(np.float32).astype(np.float64))
    (tmp_path / "t.ckpt").write_bytes((IO / "sdf.ckpt").read_bytes()[:-20])
    with pytest.raises(dataio.FormatError, match="truncated"):
        dataio.load_checkpoint_device(str(tmp_path / "t.ckpt"))
