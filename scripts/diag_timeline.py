"""Device timeline of one config-2 explicit step from the library's own
per-launch CUDA events (no profiler attached): begin/end of every launch on
its stream, relative to the step's first launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
CFG = bench.CFG
eng = Engine(KernelModel("gaussian", CFG["alpha"], CFG["rho"]), CFG["levels"], check_admissibility=False)
_ = eng.handle
p, w, q, yb = (torch.from_numpy(a).cuda() for a in bench.inputs(CFG["seed"], CFG["N"], CFG["M"]))
def step():
    res = explicit_forward(eng, SourceSet(p, w), q)
    return explicit_jvp(yb, res)
for _ in range(5):
    step()
torch.cuda.synchronize()
for rep in range(2):
    _lib.profile_enable(True)
    step(); step()
    torch.cuda.synchronize()
    tl = _lib.profile_timeline()
    _lib.profile_enable(False)
n = len(tl) // 2
t00 = tl[n][1]
for name, a, b in tl[n:]:
    print(f"{(a - t00) * 1e3:9.1f} {(b - t00) * 1e3:9.1f} {(b - a) * 1e3:8.1f}  {name}")
print(f"step span {(max(b for _, _, b in tl[n:]) - t00) * 1e3:.1f} us")
