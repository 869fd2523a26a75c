"""Uninstrumented times of the parts of a config-2 step, each in its own
loop (CUDA events around 30 back-to-back calls, L2 not flushed)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
CFG = bench.CFG
dev = torch.device("cuda")
eng = Engine(KernelModel("gaussian", CFG["alpha"], CFG["rho"]), CFG["levels"], check_admissibility=False)
_ = eng.handle
p, w, q, yb = (torch.from_numpy(a).to(dev) for a in bench.inputs(CFG["seed"], CFG["N"], CFG["M"]))

def timeit(fn, k=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k * 1e3

m_small = eng.p2m_device(p, w)
m_big = eng.p2m_device(q, yb)
acc = eng.accessor_from_moments(m_small.storage.clone())
print(f"p2m 2^20            {timeit(lambda: eng.p2m_device(p, w)):8.1f} us")
print(f"p2m 10^7            {timeit(lambda: eng.p2m_device(q, yb)):8.1f} us")
ms = m_small.storage.clone()
print(f"cascade             {timeit(lambda: eng.cascade_device(ms)):8.1f} us")
print(f"l2p 10^7 value+grad {timeit(lambda: acc.eval_device(q, _lib.L2P_VALUE | _lib.L2P_GRAD)):8.1f} us")
print(f"l2p 2^20 value+wgrad{timeit(lambda: acc.eval_device(p, _lib.L2P_VALUE | _lib.L2P_WGRAD, wts=w)):8.1f} us")
print(f"forward             {timeit(lambda: explicit_forward(eng, SourceSet(p, w), q)):8.1f} us")
res = explicit_forward(eng, SourceSet(p, w), q)
print(f"backward            {timeit(lambda: explicit_jvp(yb, res)):8.1f} us")
print(f"step                {timeit(lambda: explicit_jvp(yb, explicit_forward(eng, SourceSet(p, w), q))):8.1f} us")
os.environ["X"] = "1"
