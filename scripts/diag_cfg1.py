"""Config-1 step kernel breakdown (serial cascade for clean event timings)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
rng = np.random.default_rng(11)
n = 4096
lo = np.nextafter(-1.0, 0.0)
mk = lambda: torch.from_numpy(np.concatenate([rng.uniform(lo, 1, (n, 2)), np.full((n, 1), 0.03125)], 1).astype(np.float32)).cuda()
P, Q = mk(), mk()
W, YB = (torch.from_numpy(rng.standard_normal((n, 1)).astype(np.float32)).cuda() for _ in range(2))
e1 = Engine(KernelModel("gaussian", 200.0, 4), 4, check_admissibility=False)
step = lambda: explicit_jvp(YB, explicit_forward(e1, SourceSet(P, W), Q))
for _ in range(3): step()
torch.cuda.synchronize()
_lib.profile_enable(True)
for _ in range(10): step()
torch.cuda.synchronize()
prof = _lib.profile_read(); _lib.profile_enable(False)
tot = sum(v[0] for v in prof.values()) / 10
print("CFG1 total kernel ms/step", round(tot, 4), {k: (round(v[0] / 10, 4), v[1] // 10) for k, v in sorted(prof.items(), key=lambda x: -x[1][0])})
