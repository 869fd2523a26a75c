"""How far is the atomic arrival order inside a cell from index order?
(fraction of cells already in order, adjacent inversions, max displacement)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel
CFG = bench.CFG
dev = torch.device("cuda")
eng = Engine(KernelModel("gaussian", CFG["alpha"], CFG["rho"]), CFG["levels"], check_admissibility=False)
_ = eng.handle
p, w, q, yb = (torch.from_numpy(a).to(dev) for a in bench.inputs(CFG["seed"], CFG["N"], CFG["M"]))
for name, pts in (("q", q), ("p", p)):
    st = eng.sort_points(pts, stable=True)
    bn = eng.sort_points(pts, stable=False)
    o_s, o_b, start = st[0].long(), bn[0].long(), st[1].long()
    n = o_s.numel()
    pos_s = torch.empty(n, dtype=torch.long, device=dev); pos_s[o_s] = torch.arange(n, device=dev)
    disp = (pos_s[o_b] - torch.arange(n, device=dev)).abs()
    same_cell = torch.ones(n - 1, dtype=torch.bool, device=dev)
    seg_id = torch.bucketize(torch.arange(n, device=dev), start[1:], right=True)
    same_cell = seg_id[1:] == seg_id[:-1]
    inv = (o_b[1:] < o_b[:-1]) & same_cell
    bad_seg = torch.zeros(start.numel(), dtype=torch.long, device=dev)
    bad_seg.index_add_(0, seg_id[1:][inv], torch.ones(int(inv.sum()), dtype=torch.long, device=dev))
    nonempty = (start[1:] - start[:-1]) > 1
    print(name, "n", n, "adjacent inversions frac", float(inv.sum()) / max(1, int(same_cell.sum())),
          "cells in order frac", float(((bad_seg[:-1] == 0) & nonempty).sum()) / max(1, int(nonempty.sum())),
          "max displacement", int(disp.max()), "mean displacement", float(disp.float().mean()), flush=True)
