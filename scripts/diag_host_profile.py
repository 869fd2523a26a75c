"""cProfile of the host side of the headline step (device inputs): where the
Python/ctypes time goes between kernel launches."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
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
# host time of the forward call alone while the GPU is idle at entry
ts = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = explicit_forward(eng, SourceSet(p, w), q)
    t1 = time.perf_counter()
    explicit_jvp(yb, res)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    ts.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (time.perf_counter() - t0)))
import numpy as np
print("host fwd / jvp / total ms (median):", np.median(np.array(ts), axis=0).round(3))
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
