"""Repro of the bench's secondary -> training sequence with FC2T2_DEBUG_ERRORS=1."""
import os, sys
os.environ["FC2T2_DEBUG_ERRORS"] = "1"
sys.path.insert(0, ".")
import torch
import bench
dev = torch.device("cuda", 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
stream = torch.cuda.current_stream()
if "--skip-secondary" not in sys.argv:
    out = bench.secondary(dev, flush, stream, 4)
    print({k: v.get("ms_per_step") for k, v in out.items()}, flush=True)
out = bench.training_lines(dev, flush, stream, 4)
print({k: v.get("ms_per_step") for k, v in out.items()}, flush=True)
