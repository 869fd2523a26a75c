"""The sharded device path (parallel.py) with two processes on one B200.

Two ranks share cuda:0 over a gloo group (collectives staged through the
host -- only one GPU is available; the NCCL code path differs only in the
collective calls).  No kernel of one rank waits on the other's: every
exchange is a host-side collective between launches.

Checks, per rank, against the single-process layers on the same inputs:
  * the sharded cascade (reduce-scatter, 3-plane halo, slab M2M chain,
    coarse all-gathers, slab M2L/L2L, finest all-gather) is BIT-identical to
    the one-GPU cascade when rank 0 holds all the moments (x + 0 = x);
  * explicit layer fwd + jvp on source / query shards: rel-L2 <= 1e-6 (the
    moment sums associate differently);
  * depth + normal and radiance layers on ray shards (sources sharded too);
  * an out-of-domain query on one rank raises DomainError on both.
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
        from paper_2111_00110_b200.expansion import DomainError
        from paper_2111_00110_b200.layers import (depth_forward, depth_surface_jvp,
                                                  explicit_forward, explicit_jvp,
                                                  volumetric_forward, volumetric_jvp)
        from paper_2111_00110_b200.parallel import (Comm, DeviceBackend, shard_range, sharded,
                                                    sharded_cascade)
        from paper_2111_00110_b200.ray import Camera, RayBundle, generate_rays
        dev = torch.device("cuda", 0)
        res = {}
        for name, alpha, rho, level in (("sep", 1000.0, 4, 5), ("dense", 4000.0, 6, 5)):
            eng = Engine(KernelModel("gaussian", alpha, rho), level, check_admissibility=False)
            gen = torch.Generator(device=dev).manual_seed(1)
            p = torch.rand(40_000, 3, device=dev, generator=gen) * 1.999998 - 0.999999
            w = torch.randn(40_000, 1, device=dev, generator=gen) * 0.1
            M = eng.p2m_device(p, w).storage
            full = eng.cascade_device(M.clone())
            mine = M.clone() if rank == 0 else torch.zeros_like(M)
            L = sharded_cascade(DeviceBackend(eng), mine, Comm())
            res[f"cascade_equal_{name}"] = bool(torch.equal(L, full))
            res[f"cascade_split_{name}"] = bool(DeviceBackend(eng).slab_split_ok(
                *[(0, 32), (32, 64)][rank]))
        # explicit layer on shards
        eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
        rng = np.random.default_rng(3)
        N, Mq = 30_000, 50_000
        p = rng.uniform(-1, 1, (N, 3)).astype(np.float32)
        w = rng.normal(0, 0.1, (N, 1)).astype(np.float32)
        q = rng.uniform(-1, 1, (Mq, 3)).astype(np.float32)
        yb = rng.normal(size=(Mq, 1)).astype(np.float32)
        a, b = shard_range(N, rank, world)
        c, d = shard_range(Mq, rank, world)
        T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
        with sharded(eng):
            r = explicit_forward(eng, SourceSet(T(p[a:b]), T(w[a:b])), T(q[c:d]))
            g = explicit_jvp(T(yb[c:d]), r)
        res["explicit"] = {k: v.cpu().numpy() for k, v in (
            ("values", r.values), ("w_bar", g.w_bar), ("p_bar", g.p_bar), ("q_bar", g.q_bar))}
        # depth + normal on ray shards (sources sharded too)
        cam = Camera(np.array([0.3, 0.8, 1.8]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 60.0,
                     64, 64)
        rays = generate_rays(cam)
        R = rays.count
        e, f = shard_range(R, rank, world)
        bundle = RayBundle(T(rays.origins[e:f]), T(rays.directions[e:f]))
        yl = rng.normal(size=R).astype(np.float32)
        yg = rng.normal(size=(R, 3)).astype(np.float32)
        with sharded(eng):
            rr = depth_forward(eng, SourceSet(T(p[a:b]), T(w[a:b])), bundle, bias=0.05)
            gd = depth_surface_jvp(T(yl[e:f]), T(yg[e:f]), rr)
        res["depth"] = {"lengths": rr.lengths.cpu().numpy(), "hit": rr.hit.cpu().numpy(),
                        "w_bar": gd.w_bar.cpu().numpy(), "p_bar": gd.p_bar.cpu().numpy()}
        # radiance on ray shards
        ws = np.abs(rng.normal(size=(N, 1))).astype(np.float32)
        wc = rng.uniform(0, 1, (N, 3)).astype(np.float32)
        yr = rng.normal(size=(R, 3)).astype(np.float32) * 1e-3
        with sharded(eng):
            rv = volumetric_forward(eng, T(p[a:b]), T(ws[a:b]), T(wc[a:b]), bundle, np.ones(3))
            gv = volumetric_jvp(T(yr[e:f]), rv)
        res["radiance"] = {"rgb": rv.rgb.cpu().numpy(), "w_bar": gv.w_bar.cpu().numpy(),
                           "p_bar": gv.p_bar.cpu().numpy()}
        # a bad query on rank 1 only: both ranks raise
        qq = T(q[c:d]).clone()
        if rank == 1:
            qq[3, 0] = 1.5
        raised = False
        try:
            with sharded(eng):
                explicit_forward(eng, SourceSet(T(p[a:b]), T(w[a:b])), qq)
        except DomainError:
            raised = True
        res["raised"] = raised
        np.save(os.path.join(out, f"rank{rank}.npy"), res, allow_pickle=True)
    finally:
        dist.destroy_process_group()


def test_two_rank_device_path_matches_single_process(tmp_path, cuda):
    import torch.multiprocessing as mp
    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import (depth_forward, depth_surface_jvp, explicit_forward,
                                              explicit_jvp, volumetric_forward, volumetric_jvp)
    from paper_2111_00110_b200.ray import Camera, RayBundle, generate_rays
    from oracle.fc2t2_oracle import rel_l2
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r = [np.load(tmp_path / f"rank{k}.npy", allow_pickle=True).item() for k in range(2)]
    for k in range(2):
        for name in ("sep", "dense"):
            assert r[k][f"cascade_split_{name}"]          # nothing replicated
            assert r[k][f"cascade_equal_{name}"], (k, name)
        assert r[k]["raised"]
    # single-process reference on the same inputs
    dev = torch.device("cuda", 0)
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    rng = np.random.default_rng(3)
    N, Mq = 30_000, 50_000
    p = rng.uniform(-1, 1, (N, 3)).astype(np.float32)
    w = rng.normal(0, 0.1, (N, 1)).astype(np.float32)
    q = rng.uniform(-1, 1, (Mq, 3)).astype(np.float32)
    yb = rng.normal(size=(Mq, 1)).astype(np.float32)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    rf = explicit_forward(eng, SourceSet(T(p), T(w)), T(q))
    g = explicit_jvp(T(yb), rf)
    ref = {"values": rf.values, "w_bar": g.w_bar, "p_bar": g.p_bar, "q_bar": g.q_bar}
    for k, v in ref.items():
        got = np.concatenate([r[0]["explicit"][k], r[1]["explicit"][k]])
        assert rel_l2(got, v.cpu().numpy()) < 1e-6, k
    cam = Camera(np.array([0.3, 0.8, 1.8]), np.zeros(3), np.array([0.0, 1.0, 0.0]), 60.0, 64, 64)
    rays = generate_rays(cam)
    R = rays.count
    bundle = RayBundle(T(rays.origins), T(rays.directions))
    yl = rng.normal(size=R).astype(np.float32)
    yg = rng.normal(size=(R, 3)).astype(np.float32)
    rr = depth_forward(eng, SourceSet(T(p), T(w)), bundle, bias=0.05)
    gd = depth_surface_jvp(T(yl), T(yg), rr)
    hit = np.concatenate([r[0]["depth"]["hit"], r[1]["depth"]["hit"]])
    assert np.array_equal(hit, rr.hit.cpu().numpy())
    lens = np.concatenate([r[0]["depth"]["lengths"], r[1]["depth"]["lengths"]])
    assert rel_l2(lens[hit], rr.lengths.cpu().numpy()[hit]) < 1e-6
    for k in ("w_bar", "p_bar"):
        got = np.concatenate([r[0]["depth"][k], r[1]["depth"][k]])
        assert rel_l2(got, getattr(gd, k).cpu().numpy()) < 1e-5, k
    ws = np.abs(rng.normal(size=(N, 1))).astype(np.float32)
    wc = rng.uniform(0, 1, (N, 3)).astype(np.float32)
    yr = rng.normal(size=(R, 3)).astype(np.float32) * 1e-3
    rv = volumetric_forward(eng, T(p), T(ws), T(wc), bundle, np.ones(3))
    gv = volumetric_jvp(T(yr), rv)
    got = np.concatenate([r[0]["radiance"]["rgb"], r[1]["radiance"]["rgb"]])
    assert rel_l2(got, rv.rgb.cpu().numpy()) < 1e-6
    for k in ("w_bar", "p_bar"):
        got = np.concatenate([r[0]["radiance"][k], r[1]["radiance"][k]])
        assert rel_l2(got, getattr(gv, k).cpu().numpy()) < 1e-5, k
