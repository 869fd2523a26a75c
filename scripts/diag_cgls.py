"""CGLS vs the reference golden, per iteration count (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
from conftest import golden
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
from paper_2111_00110_b200.trainer import cgls_sdf
g = golden("training")
eng = Engine(KernelModel("gaussian", 12.0, 4), 3, check_admissibility=False)
for it in range(1, 5):
    out = cgls_sdf(eng, g["cgls_p"], g["cgls_q"], g["cgls_d"], it)
    w = out["w"].cpu().numpy()[:, 0]
    ref = g["cgls_w"][it - 1]
    print(it, "w rel", np.linalg.norm(w - ref) / np.linalg.norm(ref), "bias", out["bias"],
          g["cgls_bias"][it - 1], "mae", out["mae"][-1], g["cgls_mae"][it - 1])
# forward product check: A w for the golden w
acc = eng.expand_device(torch.from_numpy(g["cgls_p"]).float().cuda(),
                        torch.from_numpy(g["cgls_w"][0]).float().cuda().reshape(-1, 1))
