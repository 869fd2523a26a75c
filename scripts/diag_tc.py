"""Diagnostic: rel-L2 of the tcgen05 and FFMA M2L paths against the oracle."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.fc2t2_oracle import Oracle, rel_l2  # noqa: E402
from paper_2111_00110_b200 import Engine, KernelModel, SourceSet  # noqa: E402


def np_(t):
    return t.detach().cpu().numpy().astype(np.float64)


def run(level, alpha, data):
    eng = Engine(KernelModel("gaussian", alpha, 4), level, check_admissibility=False)
    ora = Oracle(alpha, 4, level)
    rng = np.random.default_rng(5)
    if data == "random":
        m = eng.zero_grid(level, 1, "M")
        md = rng.normal(size=tuple(m.data.shape)).astype(np.float32)
        m.data[:] = torch.from_numpy(md).cuda()
        md = md.astype(np.float64)
    else:
        p = rng.uniform(-1, 1, (200000, 3)).astype(np.float32).astype(np.float64)
        w = rng.normal(size=(200000, 1)).astype(np.float32).astype(np.float64)
        m = eng.p2m(SourceSet(p, w))
        md = np_(m.data)
    for tab_name in ("far", "near"):
        tab = eng.m2l_tables["far"][level] if tab_name == "far" else eng.m2l_tables["near"]
        ref = ora.m2l(md, ora.tables["far"][level] if tab_name == "far" else ora.tables["near"])
        out = {}
        for impl in ("tc", "ffma"):
            os.environ["FC2T2_M2L_FFMA"] = "1" if impl == "ffma" else "0"
            out[impl] = np_(eng.m2l(m, tab).data)
        os.environ["FC2T2_M2L_FFMA"] = "0"
        print(f"L{level} a={alpha} {data:6s} {tab_name:4s}: tc {rel_l2(out['tc'], ref):.2e}  "
              f"ffma {rel_l2(out['ffma'], ref):.2e}", flush=True)


if __name__ == "__main__":
    for lv, a in ((4, 200.0), (5, 1000.0)):
        for d in ("random", "points"):
            run(lv, a, d)
