"""GPU parity of the expansion engine and the explicit layer (through the C ABI).

Checker: the CPU oracle (float64 restatement, pinned to the reference by
tests/test_oracle_golden.py) and the reference's own golden vectors.
Tolerances: integer outputs bit-exact; float outputs rel-L2 <= 1e-5 against
the float64 reference on identical float32 inputs (BASELINE north_star).
"""

import numpy as np
import pytest
import torch

from conftest import golden
from oracle.fc2t2_oracle import Oracle, naive_grads, naive_sum, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def eng4(cuda):
    from paper_2111_00110_b200 import Engine, KernelModel
    return Engine(KernelModel("gaussian", 200.0, 4), 4, lsq=True, check_admissibility=False)


@pytest.fixture(scope="module")
def ora4():
    return Oracle(200.0, 4, 4)


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


# ------------------------------------------------------------ integer parity ---

@pytest.mark.parametrize("level", range(2, 8))
def test_find_box_bit_exact(cuda, level):
    from paper_2111_00110_b200.expansion import find_box
    g = golden("find_box")
    got = find_box(level, torch.from_numpy(g["pts"]).cuda())
    assert np.array_equal(got.cpu().numpy(), g[f"box_l{level}"])


@pytest.mark.parametrize("level", [2, 5, 6, 7])
def test_find_box_float32_edges(cuda, level):
    """The float32-only box_axis (csrc/common.cuh) at the inputs where it could
    part from the float64 floor((x + 1) res / 2) of expansion.py:85-93: x in
    [-2^-54, 0) (where float64 x + 1 rounds to 1), denormals, +-0, every
    plane and one float32 ulp either side, -1 and the largest x < 1."""
    from oracle.fc2t2_oracle import find_box as oracle_box
    from paper_2111_00110_b200.expansion import find_box
    res = 2 ** (level + 1)
    planes = (np.arange(res + 1) / (res / 2) - 1).astype(np.float32)
    v = np.concatenate([
        np.array([0.0, -0.0, -2.0**-54, -2.0**-55, -2.0**-53, -2.0**-52, 2.0**-54, -1e-45, 1e-45,
                  -1e-38, -1e-30, -1e-20, -1e-17, -1e-16, -1.0, np.nextafter(1.0, 0.0)], np.float32),
        planes, np.nextafter(planes, np.float32(2)), np.nextafter(planes, np.float32(-2))])
    v = v[np.abs(v) < 1]
    p = np.stack([v, v[::-1], np.roll(v, 7)], 1).astype(np.float32)
    got = find_box(level, torch.from_numpy(p).cuda()).cpu().numpy()
    assert np.array_equal(got, oracle_box(level, p.astype(np.float64)))


def _cell_key(p: np.ndarray, level: int) -> np.ndarray:
    from oracle.fc2t2_oracle import find_box
    res = 2 ** (level + 1)
    b = find_box(level, p.astype(np.float64))
    return (b[:, 0] * res + b[:, 1]) * res + b[:, 2]


@pytest.mark.parametrize("level,rho,C,n,heavy", [(4, 4, 1, 50_000, 0), (4, 4, 2, 50_000, 9_000),
                                                 (5, 4, 1, 200_000, 0), (6, 6, 1, 120_000, 3_000),
                                                 (3, 4, 3, 7, 0), (5, 4, 1, 0, 0)])
def test_brick_p2m_is_stable_and_matches_oracle(cuda, level, rho, C, n, heavy):
    """fc2t2_p2m_points (brick partition + per-brick P2M): equal to the float64
    oracle (expansion.py:186-198) to float32 rounding; bit-identical to itself
    run twice (deterministic) and to the same points pre-sorted STABLY by cell
    (the per-cell summation order is the index order, as np.add.at); heavy
    cells (> one 2048-record chunk of a brick) and level 6's 512-cell bricks."""
    from paper_2111_00110_b200 import Engine, KernelModel
    alpha = {3: 50.0, 4: 200.0, 5: 1000.0, 6: 4000.0}[level]
    eng = Engine(KernelModel("gaussian", alpha, rho), level, check_admissibility=False)
    rng = np.random.default_rng(level * 10 + C)
    p = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    if heavy:
        idx = rng.permutation(n)
        p[idx[:heavy]] = (p[idx[0]] * 0.999).astype(np.float32) + \
            rng.uniform(-1e-4, 1e-4, (heavy, 3)).astype(np.float32)
    w = rng.normal(size=(n, C)).astype(np.float32)
    pt, wt = torch.from_numpy(p).cuda(), torch.from_numpy(w).cuda()
    m1 = eng.p2m_device(pt, wt).storage.clone()
    m2 = eng.p2m_device(pt, wt).storage
    assert torch.equal(m1, m2)
    order = np.argsort(_cell_key(p, level), kind="stable")
    m3 = eng.p2m_device(torch.from_numpy(p[order]).cuda(), torch.from_numpy(w[order]).cuda()).storage
    assert torch.equal(m1, m3)
    ref = Oracle(alpha, rho, level, tables={"far": {}, "near": None}).p2m(p.astype(np.float64),
                                                                           w.astype(np.float64))
    got = m1.cpu().numpy().astype(np.float64)[..., :ref.shape[-1]]
    assert np.all(m1.cpu().numpy()[..., ref.shape[-1]:] == 0)
    if n:
        assert rel_l2(got, ref) < 1e-6
    else:
        assert np.all(got == 0)


@pytest.mark.parametrize("heavy", [0, 5000, 20_000])
def test_cell_sort_is_stable_counting_sort(eng4, heavy):
    """order == stable argsort by cell for every segment path of the sort:
    uniform cells (warp networks), a 5000-point cell (shared-memory block
    sort), a 20000-point cell (block runs + merge path) and a 300-point one."""
    rng = np.random.default_rng(0)
    p = rng.uniform(-1, 1, (50_000, 3)).astype(np.float32)
    if heavy:
        idx = rng.permutation(50_000)
        p[idx[:heavy]] = p[idx[0]]            # a heavy cell, scattered indices
        p[idx[heavy:heavy + 300]] = p[idx[heavy]]
    order, start = eng4.sort_points(torch.from_numpy(p).cuda())
    from oracle.fc2t2_oracle import find_box
    b = find_box(4, p.astype(np.float64))
    key = (b[:, 0] * 32 + b[:, 1]) * 32 + b[:, 2]
    ref = np.argsort(key, kind="stable")
    assert np.array_equal(order.cpu().numpy(), ref)
    pr = p[::-1].copy()        # reversed input: arrival order is mostly descending
    plain_r, _ = eng4.sort_points(torch.from_numpy(pr).cuda())
    assert np.array_equal(plain_r.cpu().numpy(), np.argsort(key[::-1], kind="stable"))
    counts = np.bincount(key, minlength=32 ** 3)
    assert np.array_equal(start.cpu().numpy(), np.concatenate([[0], np.cumsum(counts)]))


def test_key_sort_stable_with_no_cell_bucket(cuda):
    """fc2t2_key_sort (insertions): keys >= R (no cell) sort after every cell,
    everything stable; heavy keys exercise the block sort and merge paths."""
    from paper_2111_00110_b200 import _lib
    from paper_2111_00110_b200.expansion import _ptr, _stream
    lv = 3
    R = (1 << (lv + 1)) ** 3
    rng = np.random.default_rng(4)
    keys = rng.integers(0, R + 40, 60_000).astype(np.uint32)   # ~1 % no-cell
    keys[rng.permutation(60_000)[:9000]] = 17                  # > 8192 in one cell
    keys[keys >= R] = R + 7
    kd = torch.from_numpy(keys.astype(np.int64)).to(torch.int32).cuda()
    n = keys.size
    ws_b = int(_lib.lib().fc2t2_key_sort_workspace_size(lv, n))
    ws = torch.empty(ws_b, dtype=torch.uint8, device="cuda")
    order = torch.empty(n, dtype=torch.int32, device="cuda")
    start = torch.empty(R + 1, dtype=torch.int32, device="cuda")
    _lib.call("fc2t2_key_sort", lv, _ptr(kd), n, _ptr(order), _ptr(start), _ptr(ws), ws_b,
              _stream())
    ref = np.argsort(np.minimum(keys, R), kind="stable")
    assert np.array_equal(order.cpu().numpy(), ref)
    counts = np.bincount(keys[keys < R], minlength=R)
    assert np.array_equal(start.cpu().numpy(), np.concatenate([[0], np.cumsum(counts)]))


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "small"])
def test_device_interaction_lists_bit_exact(cuda, name):
    """The device lists are exactly the reference's active offsets, split by
    target parity the way expansion.py:246-249 restricts them."""
    from paper_2111_00110_b200 import Engine, KernelModel
    g = golden(f"tables_{name}")
    eng = Engine(KernelModel("gaussian", float(g["alpha"]), int(g["rho"])), int(g["levels"]),
                 check_admissibility=False)
    for level in range(2, int(g["levels"]) + 1):
        ent, starts = eng.interaction_list(level, 0)
        off = g[f"far{level}_offsets"][g[f"far{level}_active"]].astype(np.int32)
        if level == 2:
            assert np.array_equal(ent[:, :3], off)
            continue
        assert starts.shape[0] == 9
        for cls in range(8):
            par = [(cls >> 2) & 1, (cls >> 1) & 1, cls & 1]
            keep = np.ones(off.shape[0], bool)
            for a in range(3):
                keep &= ~((off[:, a] == -3) & (par[a] != 1))
                keep &= ~((off[:, a] == 3) & (par[a] != 0))
            assert np.array_equal(ent[starts[cls]:starts[cls + 1], :3], off[keep])
    ent, _ = eng.interaction_list(int(g["levels"]), 1)
    assert np.array_equal(ent[:, :3], g["near_offsets"][g["near_active"]].astype(np.int32))


# -------------------------------------------------------------- stage parity ---

def test_p2m_matches_oracle(eng4, ora4):
    from paper_2111_00110_b200 import SourceSet
    g = golden("expansion_l4")
    p, w = g["p"].astype(np.float64), g["w"].astype(np.float64)
    m = eng4.p2m(SourceSet(p, w))
    ref = ora4.p2m(p, w)
    assert rel_l2(_np(m.data), ref) < 1e-6
    # the golden moments of the reference itself (first 60 sources)
    m60 = _np(eng4.p2m(SourceSet(p[:60], w[:60])).data)
    c = g["p2m_cells"]
    assert rel_l2(m60[c[:, 0], c[:, 1], c[:, 2]], g["p2m_moments"]) < 1e-6
    assert np.count_nonzero(np.abs(m60).sum(axis=(3, 4))) == c.shape[0]


def test_m2m_l2l_m2l_match_oracle(eng4, ora4):
    rng = np.random.default_rng(5)
    m = eng4.zero_grid(4, 2, "M")
    mdata = rng.normal(size=tuple(m.data.shape)).astype(np.float32)
    m.data[:] = torch.from_numpy(mdata).cuda()
    md = mdata.astype(np.float64)
    coarse = eng4.m2m(m)
    assert rel_l2(_np(coarse.data), ora4.m2m(md, 4)) < 1e-6
    far = eng4.m2l_tables["far"][4]
    out = eng4.m2l(m, far)
    ref = ora4.m2l(md, ora4.tables["far"][4])
    assert rel_l2(_np(out.data), ref) < 1e-5
    near = eng4.m2l(m, eng4.m2l_tables["near"])
    assert rel_l2(_np(near.data), ora4.m2l(md, ora4.tables["near"])) < 1e-5
    c3 = eng4.zero_grid(3, 2, "M")
    c3.data[:] = torch.from_numpy(mdata[::2, ::2, ::2]).cuda()
    out3 = eng4.m2l(c3, eng4.m2l_tables["far"][3])
    assert rel_l2(_np(out3.data), ora4.m2l(md[::2, ::2, ::2], ora4.tables["far"][3])) < 1e-5
    c2 = eng4.zero_grid(2, 2, "M")
    c2.data[:] = torch.from_numpy(mdata[::4, ::4, ::4]).cuda()
    out2 = eng4.m2l(c2, eng4.m2l_tables["far"][2])
    assert rel_l2(_np(out2.data), ora4.m2l(md[::4, ::4, ::4], ora4.tables["far"][2])) < 1e-5
    lg = eng4.zero_grid(3, 2, "L")
    lg.data[:] = torch.from_numpy(mdata[::2, ::2, ::2]).cuda()
    fine = eng4.l2l(lg)
    assert rel_l2(_np(fine.data), ora4.l2l(md[::2, ::2, ::2], 3)) < 1e-6


def test_l2l_golden_exact_on_polynomials(eng4):
    from paper_2111_00110_b200 import Accessor
    g = golden("l2l_l3")
    coarse = eng4.zero_grid(3, 1, "L")
    coarse.data[:] = torch.from_numpy(g["coarse"]).cuda()
    fine = eng4.l2l(coarse)
    v = Accessor(fine, eng4.table).value(g["q"].astype(np.float64))
    assert rel_l2(v, g["fine_value"]) < 1e-6
    vc = Accessor(coarse, eng4.table).value(g["q"].astype(np.float64))
    assert rel_l2(vc, g["fine_value"]) < 1e-6


def test_expand_and_l2p_match_reference_golden(eng4):
    from paper_2111_00110_b200 import SourceSet
    g = golden("expansion_l4")
    p, w, q = (g[k].astype(np.float64) for k in ("p", "w", "q"))
    acc = eng4.expand(SourceSet(p, w))
    assert rel_l2(acc.value(q), g["value"]) < TOL
    assert rel_l2(acc.partials(q), g["partials"]) < TOL
    assert rel_l2(acc.partials2(q), g["partials2"]) < 1e-4  # second derivatives: 2 orders less


def test_expand_deterministic(eng4):
    from paper_2111_00110_b200 import SourceSet
    rng = np.random.default_rng(9)
    p = rng.uniform(-1, 1, (200_000, 3))
    w = rng.normal(size=(200_000, 1))
    s = SourceSet(p, w)
    a = eng4.expand(s).grid.storage.clone()
    b = eng4.expand(s).grid.storage
    assert torch.equal(a, b)


def test_domain_errors(eng4):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.expansion import DomainError
    with pytest.raises(DomainError):
        SourceSet(np.array([[0.0, 1.0, 0.0]]), np.array([1.0]))
    acc = eng4.expand(SourceSet(np.zeros((2, 3)), np.ones(2)))
    with pytest.raises(DomainError):
        acc.value(np.array([[1.0, 0.0, 0.0]]))
    # device tensors are checked by the kernel flag
    with pytest.raises(DomainError):
        acc.value(torch.tensor([[0.0, -1.0, 0.5]], device="cuda"))


def test_explicit_layer_domain_errors_and_recovery(eng4):
    """The explicit layer raises DomainError at return for device inputs
    (checked by early kernels, read without draining the stream); a valid
    call right after is unaffected (the trailing kernels' flag writes are
    cleared in stream order)."""
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.expansion import DomainError
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    rng = np.random.default_rng(4)
    p = torch.from_numpy(rng.uniform(-0.9, 0.9, (500, 3)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.normal(0, 1, (500, 1)).astype(np.float32)).cuda()
    q = torch.from_numpy(rng.uniform(-0.9, 0.9, (777, 3)).astype(np.float32)).cuda()
    ok = explicit_forward(eng4, SourceSet(p, w), q).values.clone()
    for bad_q in (1.0, float("nan"), -1.5):
        qb = q.clone()
        qb[700, 1] = bad_q
        with pytest.raises(DomainError):
            explicit_forward(eng4, SourceSet(p, w), qb)
        res = explicit_forward(eng4, SourceSet(p, w), q)
        assert torch.equal(res.values, ok)
        explicit_jvp(torch.ones(777, 1, device="cuda"), res)
    pb = p.clone()
    pb[3, 0] = -1.0
    with pytest.raises(DomainError):
        explicit_forward(eng4, SourceSet(pb, w), q)
    assert torch.equal(explicit_forward(eng4, SourceSet(p, w), q).values, ok)


def test_empty_sources(eng4):
    from paper_2111_00110_b200 import SourceSet
    acc = eng4.expand(SourceSet(np.zeros((0, 3)), np.zeros((0, 1))))
    assert float(acc.grid.storage.abs().max()) == 0.0
    assert acc.value(np.zeros((3, 3))).shape == (3, 1)


# ------------------------------------------------------------ explicit layer ---

def test_explicit_cfg1_matches_reference(eng4):
    """BASELINE config 1 (2D lifted to z=0.03125) vs the reference's outputs."""
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    g = golden("explicit_cfg1")
    p, w, q, yb = (g[k].astype(np.float64) for k in ("p", "w", "q", "y_bar"))
    res = explicit_forward(eng4, SourceSet(p, w), q)
    gr = explicit_jvp(yb, res)
    assert rel_l2(res.values, g["values"]) < TOL
    assert rel_l2(gr.w_bar, g["w_bar"]) < TOL
    assert rel_l2(gr.p_bar, g["p_bar"]) < TOL
    assert rel_l2(gr.q_bar, g["q_bar"]) < TOL
    # and the direct O(NM) sum with the reference's own bounds
    assert rel_l2(res.values, naive_sum(200.0, p, w, q)) <= 1e-2
    assert rel_l2(gr.w_bar, naive_sum(200.0, q, yb, p)) <= 1e-2
    assert rel_l2(gr.p_bar, np.einsum("nc,nca->na", w, naive_grads(200.0, q, yb, p))) <= 5e-2


def test_explicit_torch_io_and_counts(eng4):
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    rng = np.random.default_rng(1)
    p = torch.from_numpy(rng.uniform(-1, 1, (3000, 3)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.normal(size=(3000, 2)).astype(np.float32)).cuda()
    q = torch.from_numpy(rng.uniform(-1, 1, (5000, 3)).astype(np.float32)).cuda()
    before = eng4.expansion_count
    res = explicit_forward(eng4, SourceSet(p, w), q)
    assert isinstance(res.values, torch.Tensor) and res.values.shape == (5000, 2)
    assert eng4.expansion_count == before + 1
    yb = torch.randn(5000, 2, device="cuda")
    g = explicit_jvp(yb, res)
    assert eng4.expansion_count == before + 2
    assert g.w_bar.shape == (3000, 2) and g.p_bar.shape == (3000, 3) and g.q_bar.shape == (5000, 3)
    ora = Oracle(200.0, 4, 4)
    vals, wb, pb, qb = ora.explicit(_np(p), _np(w), _np(q), _np(yb))
    assert rel_l2(_np(res.values), vals) < TOL
    assert rel_l2(_np(g.w_bar), wb) < TOL
    assert rel_l2(_np(g.p_bar), pb) < TOL
    assert rel_l2(_np(g.q_bar), qb) < TOL


@pytest.mark.parametrize("m", [5001, 5])
def test_explicit_host_tensors_match_device(eng4, m):
    """Host (pinned / pageable) torch inputs take the chunked duplex-copy path
    (layers._explicit_*_host); every output must equal the device path bit for
    bit, for ragged chunk sizes."""
    import paper_2111_00110_b200.layers as layers
    from paper_2111_00110_b200 import SourceSet
    rng = np.random.default_rng(7)
    p = torch.from_numpy(rng.uniform(-1, 1, (3000, 3)).astype(np.float32))
    w = torch.from_numpy(rng.normal(size=(3000, 2)).astype(np.float32))
    q = torch.from_numpy(rng.uniform(-1, 1, (m, 3)).astype(np.float32))
    yb = torch.from_numpy(rng.normal(size=(m, 2)).astype(np.float32))
    rd = layers.explicit_forward(eng4, SourceSet(p.cuda(), w.cuda()), q.cuda())
    gd = layers.explicit_jvp(yb.cuda(), rd)
    src = SourceSet(p.pin_memory(), w.pin_memory()) if m > 100 else SourceSet(p, w)  # async / sync upload
    rh = layers.explicit_forward(eng4, src, q.pin_memory())
    gh = layers.explicit_jvp(yb, rh)          # pageable: staged through a pinned copy
    assert not rh.values.is_cuda and not gh.q_bar.is_cuda
    assert torch.equal(rh.values, rd.values.cpu())
    assert torch.equal(gh.q_bar, gd.q_bar.cpu())
    assert torch.equal(gh.w_bar, gd.w_bar.cpu())
    assert torch.equal(gh.p_bar, gd.p_bar.cpu())


def test_explicit_config2_full_size_properties(cuda):
    """Config 2 at full size (N=2^20, M=10^7, level 5): size-independent
    checks -- the adjoint (dot-product) identity <y, G w> = <w, G^T y> of the
    self-adjoint pipeline, linearity in w, and direct-sum accuracy on a sample."""
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    gen = torch.Generator(device="cuda").manual_seed(0)
    N, M = 1 << 20, 10_000_000
    p = torch.rand(N, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    w = torch.randn(N, 1, device="cuda", generator=gen) * 0.1
    q = torch.rand(M, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    yb = torch.randn(M, 1, device="cuda", generator=gen)
    res = explicit_forward(eng, SourceSet(p, w), q)
    g = explicit_jvp(yb, res)
    lhs = float((yb.double() * res.values.double()).sum())
    rhs = float((w.double() * g.w_bar.double()).sum())
    assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + abs(rhs))
    res2 = explicit_forward(eng, SourceSet(p, 2.0 * w), q)
    assert rel_l2(_np(res2.values), 2.0 * _np(res.values)) < 1e-6
    # direct sum on a sample of 512 queries (float64 on the device: checker only)
    idx = torch.arange(0, M, M // 512, device="cuda")[:512]
    qs, pd, wd = q[idx].double(), p.double(), w.double()
    exact = torch.zeros(qs.shape[0], 1, dtype=torch.float64, device="cuda")
    for lo in range(0, N, 1 << 16):
        d = qs[:, None, :] - pd[None, lo:lo + (1 << 16), :]
        exact += torch.exp(-1000.0 * (d * d).sum(-1)) @ wd[lo:lo + (1 << 16)]
    assert rel_l2(_np(res.values[idx]), _np(exact)) < 1e-2


def test_m2l_tensor_core_level5_matches_oracle(cuda):
    """The default level-5 cascade (separable finest far + near M2L, tcgen05
    fp16-split coarse levels) against the float64 oracle, and the level-5 far
    table through the dense tcgen05 kernel (Engine.m2l) against the oracle's
    per-table M2L."""
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    ora = Oracle(1000.0, 4, 5)
    rng = np.random.default_rng(21)
    p = rng.uniform(-1, 1, (20000, 3)).astype(np.float32).astype(np.float64)
    w = rng.normal(size=(20000, 1)).astype(np.float32).astype(np.float64)
    q = rng.uniform(-1, 1, (5000, 3)).astype(np.float32).astype(np.float64)
    acc = eng.expand(SourceSet(p, w))
    L = ora.expand(p, w)
    assert rel_l2(_np(acc.grid.data), L) < TOL
    assert rel_l2(acc.value(q), ora.evaluate(L, q)) < TOL
    # per-table tensor-core path vs the FFMA path on the same moments
    m = eng.p2m(SourceSet(p, w))
    far = eng.m2l_tables["far"][5]
    tc = _np(eng.m2l(m, far).data)
    assert rel_l2(tc, ora.m2l(_np(m.data), ora.tables["far"][5])) < TOL


@pytest.mark.parametrize("separable", [True, False])
def test_expand_slabs_assemble_full_cascade(cuda, separable):
    """fc2t2_expand_slab (one rank's x-slab of the sharded cascade, SURVEY
    8(e)): the finest cells of every slab equal the full cascade bit for bit
    (level 5, separable or dense tcgen05 finest level), so the multi-GPU
    all-gather reproduces the single-GPU grid exactly."""
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False,
                 separable=separable)
    assert eng.separable == separable
    gen = torch.Generator(device="cuda").manual_seed(3)
    p = torch.rand(200_000, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    w = torch.randn(200_000, 1, device="cuda", generator=gen)
    m = eng.p2m_device(p, w).storage
    full = eng.cascade_device(m)
    res = full.shape[0]
    for world in (2, 8):
        width = res // world
        parts = [eng.cascade_device(m, (r * width, (r + 1) * width))[r * width:(r + 1) * width]
                 for r in range(world)]
        assert torch.equal(torch.cat(parts), full)
    with pytest.raises(Exception):
        eng.cascade_device(m, (2, 16))        # not a multiple of 4


@pytest.mark.parametrize("rho,level,C,n", [(4, 4, 1, 4133), (4, 3, 3, 70), (6, 5, 1, 3001),
                                           (2, 3, 2, 33), (6, 3, 2, 1)])
def test_warp_cooperative_l2p_matches_per_thread_gather(cuda, rho, level, C, n):
    """Natural-order L2P uses the warp-cooperative row fetch (rows staged in
    shared memory by cp.async); an explicit order selects the per-thread
    gather.  With the identity order both evaluate the same arithmetic, so
    every mode (value, grad, Hessian, weighted grad), ragged tails and C > 1
    must agree bit for bit."""
    from paper_2111_00110_b200 import Engine, KernelModel, _lib
    from paper_2111_00110_b200.expansion import Accessor
    eng = Engine(KernelModel("gaussian", 300.0, rho), level, check_admissibility=False)
    gen = torch.Generator(device="cuda").manual_seed(11)
    L = eng._empty_grid(level, C, "L")
    L.storage.normal_(generator=gen)       # pad entries are never read by the contractions
    acc = Accessor(L, eng.table, eng.flops, flag=eng.flag)
    q = torch.rand(n, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    w = torch.randn(n, C, device="cuda", generator=gen)
    ident = torch.arange(n, dtype=torch.int32, device="cuda")
    for mode, keys in ((_lib.L2P_VALUE | _lib.L2P_WGRAD, ("value", "wgrad")),
                       (_lib.L2P_GRAD | _lib.L2P_HESS, ("grad", "hess")),
                       (_lib.L2P_VALUE | _lib.L2P_GRAD | _lib.L2P_HESS, ("value", "grad", "hess"))):
        nat = acc.eval_device(q, mode, wts=w)
        thr = acc.eval_device(q, mode, wts=w, order=ident)
        for k in keys:
            assert torch.isfinite(nat[k]).all()
            assert torch.equal(nat[k], thr[k]), (mode, k)


def test_graphed_explicit_replays_bit_identical(eng4):
    """CUDA-graph replay of the explicit layer step (graphs.GraphedExplicit):
    outputs equal the eager layer bit for bit, new inputs are picked up on
    replay, and an out-of-domain input raises DomainError after the replay."""
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.expansion import DomainError
    from paper_2111_00110_b200.graphs import GraphedExplicit
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    gen = torch.Generator(device="cuda").manual_seed(2)
    mk = lambda *s: torch.rand(*s, device="cuda", generator=gen) * 1.999998 - 0.999999  # noqa: E731
    p, q = mk(4096, 3), mk(4096, 3)
    w, yb = torch.randn(4096, 1, device="cuda", generator=gen), torch.randn(4096, 1, device="cuda", generator=gen)
    step = GraphedExplicit(eng4, p, w, q, yb)
    for it in range(2):
        if it:
            p, q = mk(4096, 3), mk(4096, 3)
        got = [t.clone() for t in step(p, w, q, yb)]
        r = explicit_forward(eng4, SourceSet(p, w), q)
        g = explicit_jvp(yb, r)
        for a, b in zip(got, (r.values, g.w_bar, g.p_bar, g.q_bar)):
            assert torch.equal(a, b)
    bad = q.clone()
    bad[7, 0] = 1.5
    with pytest.raises(DomainError):
        step(q=bad)
    step(q=q)   # the flag is re-zeroed inside the graph


@pytest.mark.parametrize("alpha,rho,level,C,lsq", [(1000.0, 4, 5, 1, True), (200.0, 4, 4, 2, True),
                                                   (200.0, 3, 4, 1, True), (1000.0, 4, 5, 1, False),
                                                   (1000.0, 5, 5, 1, True), (50.0, 2, 4, 3, True),
                                                   (200.0, 4, 5, 2, True)])
def test_separable_finest_m2l_matches_dense_and_oracle(cuda, alpha, rho, level, C, lsq):
    """The separable finest far + near M2L (csrc/m2l_sep.cu: per-axis
    triangular transforms around three 1-D convolutions) against the dense
    per-offset tables (tcgen05 path of the same engine configuration) and the
    float64 oracle cascade.  The orthonormal per-axis factors keep float32
    rounding at input level: rel-L2 of the finest L grid < 2e-6."""
    from paper_2111_00110_b200 import Engine, KernelModel
    from oracle.fc2t2_oracle import Oracle
    k = KernelModel("gaussian", alpha, rho)
    sep = Engine(k, level, lsq=lsq, check_admissibility=False, separable=True)
    dense = Engine(k, level, lsq=lsq, check_admissibility=False, separable=False)
    assert sep.separable and not dense.separable
    gen = torch.Generator(device="cuda").manual_seed(rho * 10 + level)
    n = 60_000
    p = torch.rand(n, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    w = torch.randn(n, C, device="cuda", generator=gen)
    m = sep.p2m_device(p, w).storage
    Ls = sep.cascade_device(m)
    Ld = dense.cascade_device(m)
    P = sep.P
    a, b = _np(Ls)[..., :P], _np(Ld)[..., :P]
    assert np.all(_np(Ls)[..., P:] == 0)
    assert rel_l2(a, b) < 2e-6
    ora = Oracle(alpha, rho, level, lsq=lsq)
    ref = ora.cascade(_np(m)[..., :P].astype(np.float64))
    assert rel_l2(a, ref) < 2e-6
    # per channel too (channels are independent convolutions)
    for c in range(C):
        assert rel_l2(a[..., c, :], ref[..., c, :]) < 2e-6


def test_query_gradient_recycling_is_bit_identical(eng4):
    """explicit_forward stores grad f(q) from its VALUE | GRAD L2P and
    explicit_jvp forms q_bar with fc2t2_weighted_grad: equal bit for bit to a
    second L2P pass with L2P_WGRAD (ref layers.py:183)."""
    from paper_2111_00110_b200 import SourceSet, _lib
    from paper_2111_00110_b200 import layers
    rng = np.random.default_rng(12)
    p = torch.from_numpy(rng.uniform(-1, 1, (3000, 3)).astype(np.float32)).cuda()
    w = torch.from_numpy(rng.normal(size=(3000, 2)).astype(np.float32)).cuda()
    q = torch.from_numpy(rng.uniform(-1, 1, (7001, 3)).astype(np.float32)).cuda()
    yb = torch.from_numpy(rng.normal(size=(7001, 2)).astype(np.float32)).cuda()
    r = layers.explicit_forward(eng4, SourceSet(p, w), q)
    g = layers.explicit_jvp(yb, r)
    second = r.accessor.eval_device(q, _lib.L2P_WGRAD, wts=yb)["wgrad"]
    assert torch.equal(g.q_bar, second)


@pytest.mark.parametrize("C", [1, 3])
def test_separable_post_with_fused_l2l_is_bit_identical(cuda, C):
    """The separable M2L's post transform with the finest L2L fused into it
    (run after the coarse chain) equals the separate accumulate-L2L launch bit
    for bit, for the full grid and for an x-slab."""
    from paper_2111_00110_b200 import Engine, KernelModel, _lib
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    assert eng.separable
    gen = torch.Generator(device="cuda").manual_seed(21)
    p = torch.rand(100_000, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    w = torch.randn(100_000, C, device="cuda", generator=gen)
    m = eng.p2m_device(p, w).storage
    lib = _lib.lib()
    out = {}
    for fuse in (1, 0):
        _lib.check(lib.fc2t2_engine_set_sep_fusion(eng.handle, fuse), "fusion")
        out[fuse] = (eng.cascade_device(m), eng.cascade_device(m, (16, 40))[16:40])
    _lib.check(lib.fc2t2_engine_set_sep_fusion(eng.handle, 1), "fusion")
    assert torch.equal(out[0][0], out[1][0])
    assert torch.equal(out[0][1], out[1][1])
    assert torch.equal(out[1][1], out[1][0][16:40])


def test_sharded_layer_single_rank_matches_layers(eng4):
    """The sharded explicit layer (parallel.py) with the device backend on one
    rank (no process group) equals layers.explicit_forward / explicit_jvp bit
    for bit: same early query sort, recycled q_bar and cascade."""
    from paper_2111_00110_b200 import SourceSet
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    from paper_2111_00110_b200.parallel import (DeviceBackend, explicit_forward_sharded,
                                                explicit_jvp_sharded)
    gen = torch.Generator(device="cuda").manual_seed(31)
    p = torch.rand(20_000, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    w = torch.randn(20_000, 1, device="cuda", generator=gen)
    q = torch.rand(50_000, 3, device="cuda", generator=gen) * 1.999998 - 0.999999
    yb = torch.randn(50_000, 1, device="cuda", generator=gen)
    be = DeviceBackend(eng4)
    rs = explicit_forward_sharded(be, p, w, q)
    wb, pb, qb = explicit_jvp_sharded(be, yb, rs)
    rl = explicit_forward(eng4, SourceSet(p, w), q)
    g = explicit_jvp(yb, rl)
    assert rs.q_grad is not None
    assert torch.equal(rs.values, rl.values)
    assert torch.equal(qb, g.q_bar) and torch.equal(wb, g.w_bar) and torch.equal(pb, g.p_bar)


# ------------------------------------------- separable far tables (coarse) ---

@pytest.mark.parametrize("alpha,levels,rho,level,C", [
    (1000.0, 5, 4, 4, 1),     # config 2: level 4 (32^3), 308 of 316 offsets active
    (1000.0, 5, 4, 3, 2),     # config 2: level 3 (16^3, 16-line tiles), 90 active
    (200.0, 4, 4, 3, 1),      # config 1: level 3, 308 active
    (60.0, 5, 3, 4, 1),       # wide kernel: every offset active
])
def test_separable_far_matches_dense_and_oracle(cuda, alpha, levels, rho, level, C):
    """A coarse level's far table through its per-axis factors (three disjoint
    separable pieces, csrc/m2l_sep.cu) against the dense tables of the same
    engine configuration and the float64 oracle (ref expansion.py:227-264)."""
    from paper_2111_00110_b200 import Engine, KernelModel
    k = KernelModel("gaussian", alpha, rho)
    eng = Engine(k, levels, check_admissibility=False)
    dense = Engine(k, levels, check_admissibility=False, separable=False)
    assert level in eng._sep_far and not dense._sep_far
    ora = Oracle(alpha, rho, levels)
    rng = np.random.default_rng(77 + level)
    m = eng.zero_grid(level, C, "M")
    # moment-like magnitudes: degree-n entries scale like (h/2)^n
    h = 2.0 / (1 << (level + 1))
    deg = eng.table.entries.sum(axis=1)
    mdata = (rng.normal(size=tuple(m.data.shape)) * (h / 2) ** deg).astype(np.float32)
    m.data[:] = torch.from_numpy(mdata).cuda()
    md = dense.zero_grid(level, C, "M")
    md.data[:] = m.data
    sep = _np(eng.m2l(m, eng.m2l_tables["far"][level]).data)
    den = _np(dense.m2l(md, dense.m2l_tables["far"][level]).data)
    ref = ora.m2l(mdata.astype(np.float64), ora.tables["far"][level])
    assert rel_l2(den, ref) < 1e-5
    assert rel_l2(sep, ref) < 2e-6
    # coefficient by coefficient (the degrees differ by orders of magnitude)
    for j in range(sep.shape[-1]):
        assert rel_l2(sep[..., j], ref[..., j]) < 1e-5, j
    # deterministic
    again = _np(eng.m2l(m, eng.m2l_tables["far"][level]).data)
    assert np.array_equal(sep, again)
