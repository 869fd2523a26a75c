"""Repro: brick P2M at level 4 with 8M sources (bench training line)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(66)
for level, alpha in ((4, 200.0), (5, 1200.0), (6, 4000.0)):
    for n in (4096, 1 << 20, 8 << 20):
        eng = Engine(KernelModel("gaussian", alpha, 4), level, check_admissibility=False)
        p = torch.rand(n, 3, device=dev, generator=gen) * (2 * 0.99999994) - 0.99999994
        w = torch.randn(n, 1, device=dev, generator=gen)
        try:
            m = eng.p2m_device(p, w)
            torch.cuda.synchronize()
            print(level, n, "ok", float(m.storage.double().sum()), flush=True)
        except Exception as e:
            print(level, n, "FAIL", e, flush=True)
