"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/fc2t2_oracle.py) is the checker of every GPU parity test;
these CPU tests are what make it trustworthy (parity pinned, not assumed).
"""

import numpy as np
import pytest

from conftest import golden
from oracle.fc2t2_oracle import Oracle, find_box, naive_grads, naive_sum, rel_l2


@pytest.mark.parametrize("level", range(2, 8))
def test_find_box_bit_exact(level):
    g = golden("find_box")
    pts = g["pts"].astype(np.float64)
    assert np.array_equal(find_box(level, pts), g[f"box_l{level}"])


def test_find_box_known_answer():
    assert tuple(find_box(2, np.array([[-0.999, 0.0, 0.999]]))[0]) == (0, 4, 7)
    assert tuple(golden("find_box")["known"][0]) == (0, 4, 7)


@pytest.fixture(scope="module")
def oracle_l4():
    return Oracle(200.0, 4, 4)


def test_oracle_expansion_matches_reference(oracle_l4):
    g = golden("expansion_l4")
    p, w, q = (g[k].astype(np.float64) for k in ("p", "w", "q"))
    L = oracle_l4.expand(p, w)
    assert rel_l2(oracle_l4.evaluate(L, q), g["value"]) < 1e-12
    assert rel_l2(oracle_l4.evaluate(L, q, what="grad"), g["partials"]) < 1e-12
    assert rel_l2(oracle_l4.evaluate(L, q, what="hess"), g["partials2"]) < 1e-12
    m = oracle_l4.p2m(p[:60], w[:60])
    c = g["p2m_cells"]
    assert np.allclose(m[c[:, 0], c[:, 1], c[:, 2]], g["p2m_moments"], rtol=1e-13, atol=0)
    assert np.count_nonzero(np.abs(m).sum(axis=(3, 4))) == c.shape[0]


def test_oracle_l2l_matches_reference(oracle_l4):
    g = golden("l2l_l3")
    fine = oracle_l4.l2l(g["coarse"].astype(np.float64), 3)
    v = oracle_l4.evaluate(fine, g["q"].astype(np.float64), level=4)
    assert rel_l2(v, g["fine_value"]) < 1e-13


def test_oracle_explicit_cfg1_matches_reference(oracle_l4):
    g = golden("explicit_cfg1")
    args = [g[k].astype(np.float64) for k in ("p", "w", "q", "y_bar")]
    values, w_bar, p_bar, q_bar = oracle_l4.explicit(*args)
    for got, key in ((values, "values"), (w_bar, "w_bar"), (p_bar, "p_bar"), (q_bar, "q_bar")):
        assert rel_l2(got, g[key]) < 1e-12, key


def test_reference_cfg1_against_direct_sum():
    """The reference's own bounds (test_expansion.py:127, :142) on config 1."""
    g = golden("explicit_cfg1")
    p, w, q, yb = (g[k].astype(np.float64) for k in ("p", "w", "q", "y_bar"))
    assert rel_l2(g["values"], naive_sum(200.0, p, w, q)) <= 1e-2
    assert rel_l2(g["w_bar"], naive_sum(200.0, q, yb, p)) <= 1e-2
    pb = np.einsum("nc,nca->na", w, naive_grads(200.0, q, yb, p))
    assert rel_l2(g["p_bar"], pb) <= 5e-2
