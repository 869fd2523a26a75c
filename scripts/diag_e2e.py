"""Timeline of one end-to-end explicit-layer step with host tensors."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp

eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False); _ = eng.handle
p, w, q, yb = bench.inputs(3, 1 << 20, 10_000_000)
hp, hw, hq, hy = (torch.from_numpy(a).pin_memory() for a in (p, w, q, yb))
for _ in range(3):
    r = explicit_forward(eng, SourceSet(hp, hw), hq); g = explicit_jvp(hy, r)
torch.cuda.synchronize()
T = []
def mark(name): torch.cuda.synchronize(); T.append((name, time.perf_counter()))
for it in range(3):
    T.clear(); mark("start")
    s = SourceSet(hp, hw); mark("sourceset")
    r = explicit_forward(eng, s, hq); mark("forward")
    g = explicit_jvp(hy, r); mark("jvp")
    print(" | ".join(f"{b[0]} {1e3*(b[1]-a[1]):.2f}ms" for a, b in zip(T, T[1:])))
torch.cuda.synchronize(); a = time.perf_counter()
for _ in range(5):
    r = explicit_forward(eng, SourceSet(hp, hw), hq); g = explicit_jvp(hy, r)
torch.cuda.synchronize(); print("free-running step", (time.perf_counter() - a) / 5 * 1e3, "ms")
