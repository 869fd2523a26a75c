"""Finest-level M2L timing at config-2 scale (level 5, rho 4) or config-5
scale: separable (m2l_sep.cu) vs dense, serialised cascade, per-kernel events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FC2T2_SERIAL_CASCADE", "1")
import torch
from paper_2111_00110_b200 import Engine, KernelModel, _lib
dev = torch.device("cuda")
lvl, rho, alpha = int(os.environ.get("LEVEL", 5)), int(os.environ.get("RHO", 4)), float(os.environ.get("ALPHA", 1000))
reps = int(os.environ.get("REPS", 5))
g = torch.Generator(device=dev).manual_seed(1)
p = torch.rand(1 << 20, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
w = torch.randn(1 << 20, 1, device=dev, generator=g) * 0.1
for sep in (True, False):
    eng = Engine(KernelModel("gaussian", alpha, rho), lvl, check_admissibility=False, separable=sep)
    m = eng.p2m_device(p, w).storage
    for _ in range(2):
        eng.cascade_device(m)
    torch.cuda.synchronize()
    lib = _lib.lib()
    st = {}
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        eng.cascade_device(m)
    b.record(); torch.cuda.synchronize()
    print(f"separable={sep}: cascade {a.elapsed_time(b)/reps:.3f} ms", flush=True)
    _lib.profile_enable(True)
    eng.cascade_device(m)
    torch.cuda.synchronize()
    print("  ", {k: round(v[0], 4) for k, v in _lib.profile_read().items()}, flush=True)
    _lib.profile_enable(False)
