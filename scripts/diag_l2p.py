"""L2P timing at config-5 scale (level 6, rho 6, 2^27 points): natural vs
cell-sorted order, value / wgrad modes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_00110_b200 import Engine, KernelModel, _lib
from paper_2111_00110_b200.expansion import Accessor
dev = torch.device("cuda")
lvl, rho = int(os.environ.get("LEVEL", 6)), int(os.environ.get("RHO", 6))
M = int(os.environ.get("M", 1 << 27))
eng = Engine(KernelModel("gaussian", 4000.0, rho), lvl, check_admissibility=False); _ = eng.handle
g = torch.Generator(device=dev).manual_seed(1)
q = torch.rand(M, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
y = torch.randn(M, 1, device=dev, generator=g)
L = eng._empty_grid(lvl, 1, "L")
L.storage.normal_()
acc = Accessor(L, eng.table, eng.flops, flag=eng.flag)
order, _ = eng.sort_points(q)
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n, 3)
for name, od in (("natural", None), ("sorted", order)):
    print("L2P", lvl, rho, M, name, "value", t(lambda: acc.eval_device(q, _lib.L2P_VALUE, order=od)),
          "wgrad", t(lambda: acc.eval_device(q, _lib.L2P_WGRAD, wts=y, order=od)), flush=True)
