"""Cell sort of 10^7 uniform points at level 5 (the config-2 query sort):
per-kernel times (library profiler) for ncu targeting."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_00110_b200 import Engine, KernelModel, _lib
dev = torch.device("cuda")
eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False); _ = eng.handle
g = torch.Generator(device=dev).manual_seed(1)
q = torch.rand(10_000_000, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
for _ in range(3):
    eng.sort_points(q)
torch.cuda.synchronize()
_lib.profile_enable(True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    eng.sort_points(q)
e1.record(); torch.cuda.synchronize()
prof = _lib.profile_read(); _lib.profile_enable(False)
print("SORT_MS", round(e0.elapsed_time(e1) / 10, 4), {k: (round(v[0] / 10, 4), v[1] // 10) for k, v in prof.items()})
