"""P2M A/B at config-2 scale: 10^7 queries and 2^20 sources, level 5, rho 4
(library chosen by FC2T2_LIB_OVERRIDE); moments checksum for equality."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_00110_b200 import Engine, KernelModel
dev = torch.device("cuda")
eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False); _ = eng.handle
g = torch.Generator(device=dev).manual_seed(1)
q = torch.rand(10_000_000, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
y = torch.randn(10_000_000, 1, device=dev, generator=g)
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
m = eng.p2m_device(q, y).storage
print(os.environ.get("FC2T2_LIB_OVERRIDE", "default").split("/")[-1],
      "q_us", t(lambda: eng.p2m_device(q, y)), "p_us", t(lambda: eng.p2m_device(p, w)),
      "checksum", float(m.double().sum()), float(m.double().abs().sum()), flush=True)
