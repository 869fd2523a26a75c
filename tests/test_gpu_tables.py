"""On-device M2L table fitting (csrc/tables.cu) against the
reference's golden tables and the host float64 fit."""

import time

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _items(tabs):
    out = [(f"far{l}", t) for l, t in tabs["far"].items()]
    return out + [("near", tabs["near"])]


@pytest.mark.parametrize("name", ["small", "cfg1", "cfg2", "cfg5"])
def test_device_fit_matches_reference(cuda, name):
    from paper_2111_00110_b200.kernel import KernelModel, fit_m2l_tables
    g = golden(f"tables_{name}")
    k = KernelModel("gaussian", float(g["alpha"]), int(g["rho"]))
    t0 = time.perf_counter()
    dev = fit_m2l_tables(k, int(g["levels"]), check=False, device=True)
    t_dev = time.perf_counter() - t0
    for key, t in _items(dev):
        assert np.array_equal(t.offsets, g[f"{key}_offsets"]), key
        assert np.array_equal(t.active, g[f"{key}_active"]), key
        scale = max(float(np.max(g[f"{key}_coef_absmax"])), 1e-300)
        if f"{key}_sample_idx" in g:
            idx = g[f"{key}_sample_idx"]
            err = np.max(np.abs(t.coeffs[idx] - g[f"{key}_sample_coef"])) / scale
            assert err < 1e-11, (key, err)
        amax = np.abs(t.coeffs).max(axis=(1, 2))
        assert np.max(np.abs(amax - g[f"{key}_coef_absmax"])) <= 1e-11 * scale, key
        ref_res = float(g[f"{key}_fit_residual"])
        # a max of float64 rounding-level differences: same order of magnitude
        assert t.fit_residual <= max(4.0 * ref_res, 1e-14), (key, t.fit_residual, ref_res)
    print(f"{name}: device fit {t_dev:.3f} s")


def test_device_fit_matches_host_fit(cuda):
    from paper_2111_00110_b200.kernel import KernelModel, fit_m2l_tables
    k = KernelModel("gaussian", 1000.0, 4)
    dev = fit_m2l_tables(k, 5, check=True, device=True)
    host = fit_m2l_tables(k, 5, check=True, device=False)
    for (key, a), (_, b) in zip(_items(dev), _items(host)):
        scale = max(float(np.abs(b.coeffs).max()), 1e-300)
        assert np.max(np.abs(a.coeffs - b.coeffs)) <= 1e-12 * scale, key
        assert np.array_equal(a.active, b.active)


def test_engine_uses_device_fit(cuda):
    """Engine construction on a GPU fits on the device; the expansion it
    drives is unchanged (bit-identical values vs the host-fitted engine)."""
    import torch

    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import explicit_forward
    rng = np.random.default_rng(5)
    p = torch.from_numpy(rng.uniform(-0.9, 0.9, (2000, 3)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.normal(0, 1, (2000, 1)).astype(np.float32)).cuda()
    q = torch.from_numpy(rng.uniform(-0.9, 0.9, (3000, 3)).astype(np.float32)).cuda()
    import os
    e_dev = Engine(KernelModel("gaussian", 200.0, 4), 4, check_admissibility=False)
    os.environ["FC2T2_HOST_TABLES"] = "1"
    try:
        e_host = Engine(KernelModel("gaussian", 200.0, 4), 4, check_admissibility=False)
    finally:
        del os.environ["FC2T2_HOST_TABLES"]
    a = explicit_forward(e_dev, SourceSet(p, w), q).values
    b = explicit_forward(e_host, SourceSet(p, w), q).values
    rel = float((a - b).norm() / b.norm())
    assert rel < 1e-6, rel
