"""Timeline of one device-resident explicit step (config 2, the headline)
via torch.profiler: every CUDA kernel / memset / memcpy interval, gaps
between them on each stream, and host syncs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
CFG = bench.CFG
eng = Engine(KernelModel("gaussian", CFG["alpha"], CFG["rho"]), CFG["levels"], check_admissibility=False)
_ = eng.handle
p, w, q, yb = (torch.from_numpy(a).cuda() for a in bench.inputs(CFG["seed"], CFG["N"], CFG["M"]))
def step():
    res = explicit_forward(eng, SourceSet(p, w), q)
    g = explicit_jvp(yb, res)
    return res.values, g.w_bar
for _ in range(5):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
rows = sorted(((e.time_range.start - t0) / 1000, (e.time_range.end - t0) / 1000, e.name[:70]) for e in ev)
busy_end = 0.0
gap_total = 0.0
for a, b, n in rows:
    gap = a - busy_end
    if gap > 0.003:
        gap_total += gap
    print(f"{a:8.3f} {b:8.3f} {b - a:7.3f} gap {max(gap, 0):6.3f}  {n}")
    busy_end = max(busy_end, b)
print(f"span {busy_end:.3f} ms, idle gaps {gap_total:.3f} ms")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and
       e.name in ("cudaStreamSynchronize", "cudaEventSynchronize", "cudaDeviceSynchronize",
                  "aten::item", "aten::_local_scalar_dense", "cudaMemcpyAsync")]
for e in cpu:
    print("CPU", e.name, f"{(e.time_range.start - t0)/1000:.3f} {(e.time_range.end - t0)/1000:.3f}")
