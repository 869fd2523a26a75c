"""Host precompute pinned against the reference's golden vectors (CPU).

Integer outputs -- coefficient order, offsets, hole and active masks (the
interaction lists) -- must be bit-exact; fitted coefficients agree to 1e-11
relative (reference kernel.py:257-300, multiindex.py:74-96).
"""

import numpy as np
import pytest

from conftest import golden
from paper_2111_00110_b200.expansion import Engine, m2l_pairs
from paper_2111_00110_b200.kernel import (AdmissibilityError, KernelModel, fit_m2l_tables,
                                          level_box_width, level_resolution)
from paper_2111_00110_b200.multiindex import OrderError, build_table, index_count
from oracle.fc2t2_oracle import fit_tables, mi_entries

TABLE_CFGS = ["cfg1", "cfg2", "small"]


@pytest.mark.parametrize("rho", range(1, 7))
def test_multiindex_matches_reference(rho):
    g = golden("multiindex")[f"entries_rho{rho}"]
    assert np.array_equal(build_table(rho).entries, g)
    assert np.array_equal(mi_entries(rho), g)
    assert build_table(rho).size == index_count(rho)


def test_multiindex_lookup_and_limits():
    t = build_table(4)
    for i, row in enumerate(t.entries):
        assert t.index_of(tuple(row)) == i
    assert t.index_of((4, 0, 0)) == 34
    with pytest.raises(OrderError):
        t.index_of((3, 1, 1))
    for bad in (0, 7, -1):
        with pytest.raises(OrderError):
            build_table(bad)
    assert np.array_equal(build_table(4).entries[:10], build_table(2).entries)
    assert t.padded_size == 36 and build_table(6).padded_size == 84


def _tables_of(name, impl):
    g = golden(f"tables_{name}")
    alpha, levels, rho = float(g["alpha"]), int(g["levels"]), int(g["rho"])
    if impl == "product":
        tabs = fit_m2l_tables(KernelModel("gaussian", alpha, rho), levels, check=False)
        items = [(f"far{l}", t.offsets, t.hole, t.active, t.coeffs) for l, t in tabs["far"].items()]
        n = tabs["near"]
        items.append(("near", n.offsets, n.hole, n.active, n.coeffs))
    else:
        tabs = fit_tables(alpha, rho, levels)
        items = [(f"far{l}", t["offsets"], t["hole"], t["active"], t["coeffs"])
                 for l, t in tabs["far"].items()]
        n = tabs["near"]
        items.append(("near", n["offsets"], n["hole"], n["active"], n["coeffs"]))
    return g, items


@pytest.mark.parametrize("impl", ["product", "oracle"])
@pytest.mark.parametrize("name", TABLE_CFGS)
def test_interaction_lists_bit_exact(name, impl):
    g, items = _tables_of(name, impl)
    for key, off, hole, act, coeffs in items:
        assert np.array_equal(off, g[f"{key}_offsets"]), key
        assert np.array_equal(hole, g[f"{key}_hole"]), key
        assert np.array_equal(act, g[f"{key}_active"]), key
        scale = max(float(np.max(g[f"{key}_coef_absmax"])), 1e-300)
        if f"{key}_sample_idx" in g:
            idx = g[f"{key}_sample_idx"]
            err = np.max(np.abs(coeffs[idx] - g[f"{key}_sample_coef"])) / scale
            assert err < 1e-11, (key, err)
        assert np.max(np.abs(np.abs(coeffs).max(axis=(1, 2)) - g[f"{key}_coef_absmax"])) <= 1e-11 * scale


def test_cfg5_rho6_interaction_lists_bit_exact():
    """Config 5 masks (level 6, alpha 4000, rho 6): only the integer lists are
    recomputed here (the rho-6 LSQ fit is pinned by its samples on the GPU box)."""
    from paper_2111_00110_b200.kernel import interaction_mask, stencil_offsets
    g = golden("tables_cfg5")
    k = KernelModel("gaussian", 4000.0, 6)
    for level in range(2, 7):
        reach = level_resolution(level) - 1 if level == 2 else 3
        off = stencil_offsets(reach)
        hole = np.all(np.abs(off) <= 1, axis=1)
        act = interaction_mask(k, off, level_box_width(level), hole)
        assert np.array_equal(off, g[f"far{level}_offsets"])
        assert np.array_equal(act, g[f"far{level}_active"])
    off = stencil_offsets(1)
    act = interaction_mask(k, off, level_box_width(6), np.zeros(27, bool))
    assert np.array_equal(act, g["near_active"])


def test_flop_tallies_match_reference():
    """Engine.flops follows the reference counting rules (flops.py, expansion.py:262)."""
    g = golden("expansion_l4")
    eng = Engine(KernelModel("gaussian", 200.0, 4), 4, check_admissibility=False)
    eng._tally_cascade(2)
    assert eng.flops.stages["m2l"] == int(g["flops_m2l"])
    assert eng.flops.stages["m2m"] == int(g["flops_m2m"])
    assert eng.flops.stages["l2l"] == int(g["flops_l2l"])
    from paper_2111_00110_b200 import flops
    assert flops.p2m_flops(10, 4, 35) == 10 * 106 and flops.l2p_flops(7, 4, 35) == 7 * 176


def test_m2l_flops_config2():
    """144.10 GFLOP per expansion per channel at cfg2."""
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    eng._tally_cascade(1)
    assert abs(eng.flops.stages["m2l"] / 1e9 - 144.10) < 0.01


def test_admissibility_failure_raises():
    k = KernelModel("gaussian", 4000.0, 4)
    with pytest.raises(AdmissibilityError) as exc:
        fit_m2l_tables(k, 2, lsq=True, admissibility_tol=1e-3)
    assert exc.value.level == 2


def test_taylor_tables_zeroth_column():
    """lsq=False: the n=0 column is the Taylor expansion of psi about the target
    centre (reference test_kernel.py:125-142)."""
    k = KernelModel("gaussian", 20.0, 3)
    tab = fit_m2l_tables(k, 3, lsq=False, check=False)["far"][3]
    idx = int(np.flatnonzero((tab.offsets == [0, 2, 0]).all(axis=1))[0])
    c = np.array([0, 2, 0]) * level_box_width(3)
    for j, kk in enumerate(k.table.entries):
        expect = (-1.0) ** int(kk.sum()) * k.partial(tuple(kk), c[None, :])[0]
        assert tab.coeffs[idx][j, 0] == pytest.approx(expect, rel=1e-10, abs=1e-12)


def test_polynomial_kernel_fit_exact():
    tabs = fit_m2l_tables(KernelModel("gaussian", 1e-4, 4), 4, lsq=True, check=False)
    assert tabs["near"].fit_residual < 1e-12


@pytest.mark.parametrize("alpha,rho,level,lsq", [(200.0, 4, 4, True), (1000.0, 4, 5, True),
                                                 (1000.0, 4, 5, False), (200.0, 3, 4, True),
                                                 (50.0, 2, 3, True), (4000.0, 6, 6, False),
                                                 (300.0, 1, 4, True)])
def test_separable_factors_reproduce_finest_tables(alpha, rho, level, lsq):
    """kernel.separable_factors: post_S (K(o_x) (x) K(o_y) (x) K(o_z))_S pre_S
    equals every active finest far and near table (float64).  The LSQ
    residual (~5e-8) is the reference pinv's own conditioning (cond V up to
    4.6e9 at level 5); Taylor tables factor exactly."""
    from paper_2111_00110_b200.kernel import separable_dense, separable_factors
    k = KernelModel("gaussian", alpha, rho)
    tabs = fit_m2l_tables(k, level, lsq=lsq, check=False, device=False)
    f = separable_factors(k, level, lsq)
    tol = 2e-7 if lsq else 1e-14
    for t in (tabs["far"][level], tabs["near"]):
        for i in np.flatnonzero(t.active):
            d = separable_dense(f, k.table, t.offsets[i])
            assert np.abs(d - t.coeffs[i]).max() <= tol * np.abs(t.coeffs[i]).max()


def test_separable_eligibility():
    """The separable path needs the full 6^3 finest box (every stencil offset
    active), a >= 32-cell grid and a full-rank per-axis LSQ fit."""
    from paper_2111_00110_b200.kernel import separable_eligible
    t = fit_m2l_tables(KernelModel("gaussian", 1000.0, 4), 5, check=False, device=False)
    assert separable_eligible(t, 5, 4)
    assert not separable_eligible(t, 5, 6)                     # rank-deficient LSQ at 6 nodes
    assert separable_eligible(t, 5, 6, lsq=False)
    t3 = fit_m2l_tables(KernelModel("gaussian", 50.0, 2), 3, check=False, device=False)
    assert not separable_eligible(t3, 3, 2)                    # 16-cell grid
    pruned = fit_m2l_tables(KernelModel("gaussian", 12000.0, 2), 4, check=False, device=False)
    assert not pruned["far"][4].active[~pruned["far"][4].hole].all()
    assert not separable_eligible(pruned, 4, 2)


@pytest.mark.parametrize("alpha,rho,levels,level", [(1000.0, 4, 5, 4), (1000.0, 4, 5, 3),
                                                    (200.0, 4, 4, 3), (60.0, 3, 5, 4)])
def test_separable_far_pieces_reproduce_coarse_tables(alpha, rho, levels, level):
    """Coarse-level far tables through their own per-axis factors: every
    active table equals its factored form (float64), the offsets the reference
    prunes (peak interaction < 1e-16, kernel.py:275) have negligible factored
    tables, and the three disjoint pieces F x A x A + N x F x A + N x N x F of
    csrc/m2l_sep.cu cover each parity stencil minus the hole exactly once."""
    from paper_2111_00110_b200.kernel import (separable_dense, separable_factors,
                                              separable_far_eligible)
    k = KernelModel("gaussian", alpha, rho)
    tabs = fit_m2l_tables(k, levels, check=False, device=False)
    assert separable_far_eligible(tabs, level, levels, rho)
    assert not separable_far_eligible(tabs, levels, levels, rho)      # the finest level
    assert not separable_far_eligible(tabs, 2, levels, rho)           # the coarsest stencil
    t = tabs["far"][level]
    f = separable_factors(k, level)
    peak = max(np.abs(t.coeffs[i]).max() for i in np.flatnonzero(t.active))
    for i in range(t.offsets.shape[0]):
        if t.hole[i]:
            continue
        d = separable_dense(f, k.table, t.offsets[i])
        if t.active[i]:
            assert np.abs(d - t.coeffs[i]).max() <= 2e-7 * np.abs(t.coeffs[i]).max()
        else:
            assert np.abs(d).max() <= 1e-12 * peak
    # the pieces: per parity, count how often each offset of the box is applied
    far_taps, near_taps = {-3, -2, 2, 3}, {-1, 0, 1}
    for par in range(2):
        box = set(range(-2 - par, 4 - par))
        F, N, A = box & far_taps, box & near_taps, box
        cover = {}
        for xs, ys, zs in ((F, A, A), (N, F, A), (N, N, F)):
            for o in ((x, y, z) for x in xs for y in ys for z in zs):
                cover[o] = cover.get(o, 0) + 1
        want = {(x, y, z) for x in box for y in box for z in box
                if max(abs(x), abs(y), abs(z)) > 1}
        assert set(cover) == want and set(cover.values()) == {1}
