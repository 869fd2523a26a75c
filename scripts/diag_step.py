"""One config-2 explicit fwd+bwd step between cudaProfilerStart/Stop (after
two warm-up steps), for `ncu --profile-from-start off` captures:
launch list / per-stage DRAM traffic of exactly one bench step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
CFG = bench.CFG
dev = torch.device("cuda")
eng = Engine(KernelModel("gaussian", CFG["alpha"], CFG["rho"]), CFG["levels"], check_admissibility=False)
_ = eng.handle
p, w, q, yb = (torch.from_numpy(a).to(dev) for a in bench.inputs(CFG["seed"], CFG["N"], CFG["M"]))
step = lambda: explicit_jvp(yb, explicit_forward(eng, SourceSet(p, w), q))  # noqa: E731
for _ in range(2):
    step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("step done")
