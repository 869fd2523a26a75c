"""Per-launch time of the config-2 M2L kernels (library event profiler).
Run with FC2T2_TC_DIAG=0/1/2/3 (1: skip window gathers, 2: skip B loads) to
split the kernel's time between MMA issue and operand staging."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
from paper_2111_00110_b200.layers import explicit_forward
dev = torch.device("cuda")
level = int(os.environ.get("LEVEL", 5)); rho = int(os.environ.get("RHO", 4))
eng = Engine(KernelModel("gaussian", 1000.0, rho), level, check_admissibility=False); _ = eng.handle
g = torch.Generator(device=dev).manual_seed(1)
N, M = 1 << 20, 1 << 16
p = torch.rand(N, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
w = torch.randn(N, 1, device=dev, generator=g)
q = torch.rand(M, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
for _ in range(3):
    explicit_forward(eng, SourceSet(p, w), q)
torch.cuda.synchronize()
_lib.profile_enable(True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    explicit_forward(eng, SourceSet(p, w), q)
e1.record()
torch.cuda.synchronize()
print("FWD_MS", round(e0.elapsed_time(e1) / 10, 4))
prof = _lib.profile_read(); _lib.profile_enable(False)
print("DIAG", os.environ.get("FC2T2_TC_DIAG", "0"), {k: round(v[0] / v[1], 4) for k, v in prof.items() if "m2l" in k})
