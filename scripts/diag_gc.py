"""Run bench.secondary() with gc callbacks logging collections > 5 ms, to
explain rare ~100 ms host stalls in single timed steps."""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
t = {}
def cb(phase, info):
    if phase == "start":
        t["s"] = time.perf_counter()
    else:
        d = 1e3 * (time.perf_counter() - t["s"])
        if d > 5:
            print(f"GC gen{info['generation']} {d:.1f} ms collected={info['collected']}", flush=True)
gc.callbacks.append(cb)
dev = torch.device("cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for rep in range(2):
    out = bench.secondary(dev, flush, torch.cuda.current_stream(), 20)
    print({k: (round(v["ms_per_step"], 2), v.get("stages_ms_per_step", {}).get("_step_ms_max")) for k, v in out.items()}, flush=True)
