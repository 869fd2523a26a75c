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
    def __init__(self, ora):
        self.o = ora
        self.slabs = []

    def p2m_grid(self, p, w):
        return torch.from_numpy(self.o.p2m(p.numpy(), w.numpy()))

    def cascade_grid(self, m, x_range=None):
        L = torch.from_numpy(self.o.cascade(m.numpy()))
        if x_range is not None:
            # outside this rank's slab the grid is unspecified: poison it so
            # the test proves the all-gather assembles only owned slabs
            L[:x_range[0]] = float("nan")
            L[x_range[1]:] = float("nan")
            self.slabs.append(tuple(x_range))
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
    # each rank computed only its own x-slab of the level-3 (16^3) grid, twice
    assert [tuple(map(tuple, x["slabs"])) for x in r] == [((0, 8), (0, 8)), ((8, 16), (8, 16))]


def test_slab_range():
    assert [slab_range(128, r, 8) for r in range(8)] == [(16 * r, 16 * r + 16) for r in range(8)]
    assert slab_range(64, 1, 2) == (32, 64)
    assert slab_range(16, 0, 3) is None      # 4 units do not split over 3 ranks
    assert slab_range(16, 3, 4) == (12, 16)
