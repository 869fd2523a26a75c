"""Timeline of one host-tensor explicit step (config 2) via torch.profiler:
memcpy HtoD / DtoH and kernel intervals, to see where PCIe idles."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
CFG = bench.CFG
eng = Engine(KernelModel("gaussian", CFG["alpha"], CFG["rho"]), CFG["levels"], check_admissibility=False)
_ = eng.handle
p, w, q, yb = bench.inputs(CFG["seed"], CFG["N"], CFG["M"])
hp, hw, hq, hy = (torch.from_numpy(a).pin_memory() for a in (p, w, q, yb))
def step():
    res = explicit_forward(eng, SourceSet(hp, hw), hq)
    g = explicit_jvp(hy, res)
    return res.values, g.w_bar
for _ in range(3):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
rows = sorted(((e.time_range.start - t0) / 1000, (e.time_range.end - t0) / 1000, e.name[:60]) for e in ev)
for a, b, n in rows:
    if b - a > 0.02 or "Memcpy" in n or "memcpy" in n:
        print(f"{a:8.3f} {b:8.3f} {b - a:7.3f}  {n}")
# CPU side: the python calls
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU and e.name in ("cudaStreamSynchronize", "cudaEventSynchronize", "cudaDeviceSynchronize")]
for e in cpu:
    print("CPU", e.name, f"{(e.time_range.start - t0)/1000:.3f} {(e.time_range.end - t0)/1000:.3f}")

print("---- CPU ops")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
for e in sorted(cpu, key=lambda e: e.time_range.start):
    a = (e.time_range.start - t0) / 1000
    b = (e.time_range.end - t0) / 1000
    if -0.2 < a < 0.7 or 3.1 < a < 3.6:
        if b - a > 0.004:
            print(f"CPUOP {a:8.3f} {b:8.3f} {b-a:7.3f} {e.name[:70]}")
