"""L2P A/B at config-2 scale: M = 10^7 value+grad (mode 3) and N = 2^20
value+wgrad (mode 9), level 5, rho 4 (library chosen by FC2T2_LIB_OVERRIDE)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_00110_b200 import Engine, KernelModel, _lib
from paper_2111_00110_b200.expansion import Accessor
dev = torch.device("cuda")
eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False); _ = eng.handle
g = torch.Generator(device=dev).manual_seed(1)
L = eng._empty_grid(5, 1, "L"); L.storage.normal_(generator=g)
acc = Accessor(L, eng.table, eng.flops, flag=eng.flag)
q = torch.rand(10_000_000, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
p = torch.rand(1 << 20, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
w = torch.randn(1 << 20, 1, device=dev, generator=g)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def t(fn, n=10):
    fn(); torch.cuda.synchronize(); tot = 0.0
    for i in range(n):
        flush.fill_(i)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); tot += a.elapsed_time(b)
    return round(1000 * tot / n, 1)
r3 = acc.eval_device(q, 3)
print(os.environ.get("FC2T2_LIB_OVERRIDE", "default").split("/")[-1],
      "mode3_us", t(lambda: acc.eval_device(q, 3)), "mode9_us", t(lambda: acc.eval_device(p, 9, wts=w)),
      "checksum", float(r3["value"].double().sum()), float(r3["grad"].double().abs().sum()), flush=True)
