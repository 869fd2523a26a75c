"""Config-3 step repeated: per-step host time, then a torch.profiler pass
listing the slowest CPU-side ops (finding host stalls)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import profile, ProfilerActivity
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
from paper_2111_00110_b200.layers import depth_forward, depth_surface_jvp
from paper_2111_00110_b200.ray import Camera, RayBundle, generate_rays
dev = torch.device("cuda")
rng = np.random.default_rng(33)
lo = np.nextafter(-1.0, 0.0)
N3 = 1 << 18
p = rng.uniform(lo, 1, (N3, 3)).astype(np.float32)
w = rng.normal(0.0, 0.1, (N3, 1)).astype(np.float32)
cam = Camera(2.0 * bench.seeded_direction(rng), np.zeros(3), np.array([0.0, 1.0, 0.0]), 60.0, 512, 512)
b3 = generate_rays(cam)
R3 = b3.count
yl = torch.from_numpy(rng.standard_normal(R3).astype(np.float32)).to(dev)
yg = torch.from_numpy(rng.standard_normal((R3, 3)).astype(np.float32)).to(dev)
b3 = RayBundle(torch.from_numpy(b3.origins).to(dev), torch.from_numpy(b3.directions).to(dev))
e5 = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
src3 = SourceSet(torch.from_numpy(p).to(dev), torch.from_numpy(w).to(dev))
def step3():
    res = depth_forward(e5, src3, b3, bias=0.05)
    return depth_surface_jvp(yl, yg, res), res
ts = []
for i in range(30):
    torch.cuda.synchronize(); t0 = time.perf_counter(); step3(); torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
print("STEP ms", [round(t, 2) for t in ts])
from paper_2111_00110_b200 import _lib
_lib.profile_enable(True)
for _ in range(10):
    step3()
torch.cuda.synchronize()
prof = _lib.profile_read(); _lib.profile_enable(False)
print("CFG3", {k: (round(v[0] / 10, 4), v[1] // 10) for k, v in sorted(prof.items(), key=lambda x: -x[1][0])})
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step3()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
