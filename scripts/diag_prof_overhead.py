"""Config-2 step with and without the library's per-launch profiling events
(bench.timed_steps): the cost of the stage instrumentation itself."""
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
step = lambda: explicit_jvp(yb, explicit_forward(eng, SourceSet(p, w), q))
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream()
for rep in range(3):
    ms0, _ = bench.timed_steps(step, 30, 5, flush, stream, None)
    st = {}
    ms1, _ = bench.timed_steps(step, 30, 5, flush, stream, st)
    print(f"plain {ms0 / 30:.4f} ms/step   with stage events {ms1 / 30:.4f} ms/step")
