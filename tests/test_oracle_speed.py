"""The oracle is the CPU baseline of bench.py (--impl reference and the
cpu_baseline key): it must be as fast as the reference it restates, or the
reported GPU/CPU ratios are inflated.  Times the oracle against the imported
reference on the same 2^14-source level-5 sample (P2M, one cascade, L2P value
and gradient at 2^16 queries) and asserts the oracle is within 1.3x.

Needs /root/reference (the build container); skipped elsewhere.
"""

import os
import sys
import time

import numpy as np
import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_oracle_is_speed_faithful_to_reference():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    try:
        from fc2t2.expansion import Engine, SourceSet
        from fc2t2.kernel import KernelModel
    finally:
        sys.path.remove(REF)
    from oracle.fc2t2_oracle import Oracle

    rng = np.random.default_rng(0)
    p = rng.uniform(-1, 1, (1 << 14, 3))
    w = rng.normal(size=(1 << 14, 1))
    q = rng.uniform(-1, 1, (1 << 16, 3))
    eng = Engine(KernelModel("gaussian", 1000.0, 4), 5, lsq=True, check_admissibility=False)
    tabs = {"far": {}, "near": None}
    for lvl, t in list(eng.m2l_tables["far"].items()) + [(None, eng.m2l_tables["near"])]:
        d = {"level": t.level, "near": bool(t.nearfield), "offsets": t.offsets, "hole": t.hole,
             "active": t.active, "coeffs": t.coeffs}
        if lvl is None:
            tabs["near"] = d
        else:
            tabs["far"][lvl] = d
    ora = Oracle(1000.0, 4, 5, tables=tabs)

    def ref_run():
        acc = eng.expand(SourceSet(p, w))
        return acc.value(q), acc.partials(q), acc.grid.data

    def ora_run():
        L = ora.expand(p, w)
        return ora.evaluate(L, q), ora.evaluate(L, q, what="grad"), L

    t0 = time.perf_counter()
    rv, rg, rL = ref_run()
    t1 = time.perf_counter()
    ov, og, oL = ora_run()
    t2 = time.perf_counter()
    t_ref, t_ora = t1 - t0, t2 - t1
    print(f"reference {t_ref:.2f} s, oracle {t_ora:.2f} s")
    # the same numbers (float64, same association per GEMM)
    assert np.abs(oL - rL).max() <= 1e-12 * np.abs(rL).max()
    assert np.allclose(ov, rv, rtol=1e-12, atol=1e-14)
    assert t_ora <= 1.3 * t_ref, (t_ora, t_ref)
