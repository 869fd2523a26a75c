"""rho = 6 (P = 84, config 5's expansion order) through the whole device cascade,
including the tcgen05 M2L at TILES = 1 / N = 96, against the float64 oracle.
(The reference caps rho at 4; its golden tables for rho = 6 come from the
harness-patched reference, tests/golden/tables_cfg5.npz.)"""

import numpy as np
import pytest

from conftest import golden
from oracle.fc2t2_oracle import Oracle, rel_l2

pytestmark = pytest.mark.gpu


def test_rho6_tables_match_patched_reference(cuda):
    from paper_2111_00110_b200.kernel import KernelModel, fit_m2l_tables
    g = golden("tables_cfg5")
    tabs = fit_m2l_tables(KernelModel("gaussian", 4000.0, 6), 6, check=False)
    for lv in range(2, 7):
        t = tabs["far"][lv]
        assert np.array_equal(t.active, g[f"far{lv}_active"])
        if f"far{lv}_sample_idx" in g:
            idx = g[f"far{lv}_sample_idx"]
            scale = np.abs(g[f"far{lv}_sample_coef"]).max()
            assert np.max(np.abs(t.coeffs[idx] - g[f"far{lv}_sample_coef"])) < 1e-10 * scale


def test_rho6_cascade_matches_oracle(cuda):
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    eng = Engine(KernelModel("gaussian", 200.0, 6), 4, check_admissibility=False)
    ora = Oracle(200.0, 6, 4)
    rng = np.random.default_rng(66)
    p = rng.uniform(-1, 1, (6000, 3)).astype(np.float32).astype(np.float64)
    w = rng.normal(size=(6000, 1)).astype(np.float32).astype(np.float64)
    q = rng.uniform(-1, 1, (3000, 3)).astype(np.float32).astype(np.float64)
    acc = eng.expand(SourceSet(p, w))
    L = ora.expand(p, w)
    assert rel_l2(acc.grid.data.cpu().numpy().astype(np.float64), L) < 1e-5
    assert rel_l2(acc.value(q), ora.evaluate(L, q)) < 1e-5
    assert rel_l2(acc.partials(q), ora.evaluate(L, q, what="grad")) < 1e-5
