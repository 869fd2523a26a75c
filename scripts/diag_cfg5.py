"""Config-5 step: device time under the bench's timed_steps with/without
result retention and the per-kernel profiler (finding host stalls)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
dev = torch.device("cuda")
stream = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
e6 = Engine(KernelModel("gaussian", 4000.0, 6), 6, check_admissibility=False); _ = e6.handle
g = torch.Generator(device=dev).manual_seed(5)
N, M = 1 << 24, 1 << 27
p = torch.rand(N, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
w = torch.randn(N, 1, device=dev, generator=g) * 0.1
q = torch.rand(M, 3, device=dev, generator=g) * 1.9999998 - 0.9999999
y = torch.randn(M, 1, device=dev, generator=g)
fn = lambda: explicit_jvp(y, explicit_forward(e6, SourceSet(p, w), q))
for label, st in (("plain", None), ("profiled", {}), ("plain", None), ("profiled", {})):
    t0 = time.perf_counter()
    ms, out = bench.timed_steps(fn, 2, 1, flush, stream, st)
    del out
    print(f"{label}: {ms/2:.1f} ms/step  wall {1e3*(time.perf_counter()-t0):.0f} ms "
          f"stage-sum {sum(st.values()) if st else 0:.1f}", flush=True)
