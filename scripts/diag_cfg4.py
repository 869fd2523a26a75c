"""Config-4 radiance step (8 poses x 400^2 rays, N = 2^20, level 5) for
profiling: per-kernel times via the library profiler."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel, _lib
from paper_2111_00110_b200.layers import volumetric_forward, volumetric_jvp
from paper_2111_00110_b200.ray import Camera, RayBundle, generate_rays
dev = torch.device("cuda")
rng = np.random.default_rng(44)
lo = np.nextafter(-1.0, 0.0)
N4 = 1 << 20
p = torch.from_numpy(rng.uniform(lo, 1, (N4, 3)).astype(np.float32)).to(dev)
ws = torch.from_numpy(np.abs(rng.standard_normal((N4, 1))).astype(np.float32)).to(dev)
wc = torch.from_numpy(rng.uniform(0, 1, (N4, 3)).astype(np.float32)).to(dev)
poses = int(os.environ.get("POSES", 8))
org, dirs = [], []
for _ in range(poses):
    bb = generate_rays(Camera(2.5 * bench.seeded_direction(rng), np.zeros(3), np.array([0.0, 1.0, 0.0]), 50.0, 400, 400))
    org.append(bb.origins); dirs.append(bb.directions)
b4 = RayBundle(torch.from_numpy(np.concatenate(org)).to(dev), torch.from_numpy(np.concatenate(dirs)).to(dev))
target = torch.from_numpy(rng.uniform(0, 1, (b4.count, 3)).astype(np.float32)).to(dev)
e5 = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
def step():
    res = volumetric_forward(e5, p, ws, wc, b4, np.ones(3))
    ybar = 2.0 * (res.rgb - target) / float(res.rgb.numel())
    return volumetric_jvp(ybar, res)
for _ in range(int(os.environ.get("WARM", 2))):
    step()
torch.cuda.synchronize()
_lib.profile_enable(True)
step(); torch.cuda.synchronize()
prof = _lib.profile_read(); _lib.profile_enable(False)
print("CFG4", {k: (round(v[0], 3), v[1]) for k, v in sorted(prof.items(), key=lambda x: -x[1][0])})
