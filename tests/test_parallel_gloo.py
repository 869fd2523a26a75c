"""Multi-rank sharding of the explicit layer, world size 2 over gloo on CPU.

The sharding logic (paper_2111_00110_b200/parallel.py) runs with the CPU
oracle as its compute backend: two ranks each own half the sources and half
the queries, all-reduce the moment grids, and the concatenated per-rank results
must equal the single-process explicit layer.
"""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.fc2t2_oracle import Oracle
from paper_2111_00110_b200.parallel import (explicit_forward_sharded, explicit_jvp_sharded,
                                            shard_range, slab_range)


class OracleBackend:
    """The CPU oracle behind the sharding interface.  Everything a rank does
    not own is poisoned with NaN, so the test proves each phase reads only
    what the protocol delivered: the slab (M2M chain), the slab plus the
    3-plane halo (finest M2L), and the all-gathered coarse levels."""

    def __init__(self, ora):
        self.o = ora
        self.levels = ora.levels
        self.slabs = []

    def p2m_grid(self, p, w):
        return torch.from_numpy(self.o.p2m(p.numpy(), w.numpy()))

    def slab_split_ok(self, x0, x1):
        return True

    def cascade(self, m, x_range=None):
        L = torch.from_numpy(self.o.cascade(m.numpy()))
        if x_range is not None:
            L[:x_range[0]] = float("nan")
            L[x_range[1]:] = float("nan")
            self.slabs.append(tuple(x_range))
        return L

    def cascade_up(self, m, x_range):
        x0, x1 = x_range
        M = {self.levels: m.clone()}
        M[self.levels][:x0] = float("nan")
        M[self.levels][x1:] = float("nan")
        for lv in range(self.levels, 2, -1):
            M[lv - 1] = torch.from_numpy(self.o.m2m(M[lv].numpy(), lv))
        return M

    def coarse_views(self, M):
        return [(lv, M[lv]) for lv in range(2, self.levels)]

    def cascade_down(self, m, M, x_range):
        x0, x1 = x_range
        self.slabs.append(tuple(x_range))
        mf = m.clone()
        mf[:max(0, x0 - 3)] = float("nan")
        mf[x1 + 3:] = float("nan")
        for lv in range(2, self.levels):
            assert not torch.isnan(M[lv]).any()       # the coarse all-gathers completed
        o, t = self.o, self.o.tables
        L = o.m2l(M[2].numpy(), t["far"][2])
        for lv in range(3, self.levels):
            L = o.m2l(M[lv].numpy(), t["far"][lv]) + o.l2l(L, lv - 1)
        L = o.m2l(mf.numpy(), t["far"][self.levels]) + o.l2l(L, self.levels - 1) + \
            o.m2l(mf.numpy(), t["near"])
        L = torch.from_numpy(L)
        assert not torch.isnan(L[x0:x1]).any()
        L[:x0] = float("nan")
        L[x1:] = float("nan")
        return L

    def evaluate(self, L, pts, wts, value):
        Ln, x = L.numpy(), pts.numpy()
        v = torch.from_numpy(self.o.evaluate(Ln, x)) if value else None
        g = None
        if wts is not None:
            g = torch.from_numpy(np.einsum("nc,nca->na", wts.numpy(),
                                           self.o.evaluate(Ln, x, what="grad")))
        return v, g


def _data():
    rng = np.random.default_rng(5)
    p = rng.uniform(-0.9, 0.9, (300, 3))
    w = rng.normal(size=(300, 2))
    q = rng.uniform(-0.9, 0.9, (250, 3))
    yb = rng.normal(size=(250, 2))
    return p, w, q, yb


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p, w, q, yb = _data()
        a, b = shard_range(p.shape[0], rank, world)
        c, d = shard_range(q.shape[0], rank, world)
        be = OracleBackend(Oracle(50.0, 4, 3))
        t = torch.from_numpy
        res = explicit_forward_sharded(be, t(p[a:b]), t(w[a:b]), t(q[c:d]))
        wb, pb, qb = explicit_jvp_sharded(be, t(yb[c:d]), res)
        np.savez(os.path.join(out, f"rank{rank}.npz"), values=res.values.numpy(),
                 w_bar=wb.numpy(), p_bar=pb.numpy(), q_bar=qb.numpy(),
                 slabs=np.array(be.slabs))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for n in (0, 1, 7, 100):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_two_rank_explicit_layer_matches_single_process(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    p, w, q, yb = _data()
    ora = Oracle(50.0, 4, 3)
    values, w_bar, p_bar, q_bar = ora.explicit(p, w, q, yb)
    r = [np.load(tmp_path / f"rank{k}.npz") for k in range(2)]
    cat = lambda key: np.concatenate([x[key] for x in r])  # noqa: E731
    for got, ref in ((cat("values"), values), (cat("w_bar"), w_bar), (cat("p_bar"), p_bar),
                     (cat("q_bar"), q_bar)):
        assert np.allclose(got, ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())
    # each rank ran the down phase on its own x-slab of the level-3 (16^3)
    # grid, once per expansion
    assert [tuple(map(tuple, x["slabs"])) for x in r] == [((0, 8), (0, 8)), ((8, 16), (8, 16))]


def test_slab_range():
    assert [slab_range(128, r, 8) for r in range(8)] == [(16 * r, 16 * r + 16) for r in range(8)]
    assert slab_range(64, 1, 2) == (32, 64)
    assert slab_range(16, 0, 3) is None      # 4 units do not split over 3 ranks
    assert slab_range(16, 3, 4) == (12, 16)
