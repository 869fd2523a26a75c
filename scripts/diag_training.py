"""bench.training_lines alone (quick check of the training bench lines)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = bench.training_lines(dev, flush, torch.cuda.current_stream(), int(sys.argv[1]) if len(sys.argv) > 1 else 20)
for k, v in out.items():
    print(k, json.dumps({a: b for a, b in v.items() if a != "workload"}))
