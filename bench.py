"""FC2T2 B200 benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
the 3D explicit layer, forward + backward w.r.t. w and p (and q), with
N = 2^20 sources ~ U(-1,1)^3, w ~ N(0, 0.1^2), M = 10^7 queries ~ U(-1,1)^3,
upstream gradient ~ N(0,1); level 5 (64^3 finest grid), rho 4 (P=35),
Gaussian alpha = 1000 (reference default kernel, DEFAULT_ALPHA[5]).

  value  (N+M) / device time of explicit_forward + explicit_jvp, inputs resident
         in HBM, CUDA events per step on the launching stream, L2 flushed
         between steps (outside the events); the median step (the
         mean and the slowest step are reported beside it).  The K timed steps
         run without the library's per-launch events; the same K steps run a
         second time with them on for the per-kernel times (the two event
         records around every launch cost ~9 % of a step).
  e2e    the same metric through the public API with pinned HOST torch tensors:
         H2D of p, w, q, y_bar and D2H of values, w_bar, p_bar, q_bar inside
         the timed region.
  roofline_stages  per stage: algorithmic bytes (inputs once, outputs once)
         and, for the separable M2L, executed FFMA flops; time from the
         library's per-launch CUDA events; frac = max(bytes / HBM peak,
         flops / FFMA peak) / time (peaks measured: MEASURED_PEAKS.json,
         profiles/r2_peaks.json).
  roofline  the dominant KERNEL: the launch label with the largest serialised
         time in the committed ncu capture (profiles/traffic.json), with its
         measured DRAM traffic; roofline_dominant_stage: the same for the
         multi-kernel stage groups; roofline_kernels: every launch label.
  cpu_baseline / --impl reference  the oracle port (float64 NumPy restatement
         of the reference, speed-faithful, all host threads for BLAS) on a
         1/32 slice of the step.

Multi-GPU (torchrun) and --config 5: BASELINE config 5 as strong scaling --
the global N = 2^24, M = 2^27, rho = 6, level 6 problem split over the ranks;
every expansion runs the sharded cascade (parallel.py: reduce-scatter into
x-slabs, 3-plane halos, slab cascade at every level, all-gathers); timing is
the max over ranks of the device time.

Secondary lines (rank 0, single GPU): configs 1, 3, 4 and one-GPU config 5
(explicit 2D-lifted, root-implicit depth+normal, radiance, rho 6) with their
own metrics (points/s, rays/s), and the fitting loops (training lines).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "FC²T² fwd+bwd points/sec (N+M) in 3D; rays/sec for root/integral layers"
UNIT = "points/s"
CFG = dict(N=1 << 20, M=10_000_000, levels=5, rho=4, alpha=1000.0, seed=2)
WORKLOAD = ("cfg2 explicit layer fwd+bwd (w, p, q adjoints): N=2^20 sources, M=10^7 queries "
            "uniform in [-1,1]^3, w~N(0,0.1^2), y_bar~N(0,1), level 5 (64^3), rho=4 (P=35), "
            "gaussian alpha=1000")

CFG5 = dict(N=1 << 24, M=1 << 27, levels=6, rho=6, alpha=4000.0, seed=5)
WORKLOAD5 = ("cfg5 explicit layer fwd+bwd (w, p, q adjoints), strong scaling: N=2^24 sources, "
             "M=2^27 queries uniform in [-1,1]^3 split evenly over the ranks, w~N(0,0.1^2), "
             "y_bar~N(0,1), level 6 (128^3), rho=6 (P=84), gaussian alpha=4000")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--small", action="store_true", help="reduced sizes for a quick check")
    ap.add_argument("--no-secondary", action="store_true", help="skip configs 1, 3, 4")
    ap.add_argument("--config", type=int, choices=[2, 5], default=None,
                    help="2: the headline (default at one GPU); 5: the multi-GPU scaling "
                         "config (default under torchrun), strong scaling over the ranks")
    return ap.parse_args()


def inputs(seed: int, N: int, M: int):
    rng = np.random.default_rng(seed)
    lo, hi = np.nextafter(-1.0, 0.0), 1.0
    p = rng.uniform(lo, hi, (N, 3)).astype(np.float32)
    w = (0.1 * rng.standard_normal((N, 1))).astype(np.float32)
    q = rng.uniform(lo, hi, (M, 3)).astype(np.float32)
    yb = rng.standard_normal((M, 1)).astype(np.float32)
    one = np.nextafter(np.float32(1), np.float32(0))
    np.clip(p, -one, one, out=p)
    np.clip(q, -one, one, out=q)
    return p, w, q, yb


# ------------------------------------------------------------- clocks ---

class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.out = ""

    def summary(self) -> dict:
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ------------------------------------------------------------- CPU arm ---

def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


SAMPLE_SLICES = 32   # one CPU step = 1/32 of the full config-2 step's work


def cpu_sample(steps: int, warmup: int, N: int, M: int, seed: int, cfg: dict | None = None,
               slices: int | None = None) -> dict:
    """The reference pipeline restated by the oracle (speed-faithful: power-table
    monomials, one contiguous GEMM per offset -- tests/test_oracle_speed.py
    holds it within 1.3x of the imported reference), timed on a BOUNDED SLICE
    of the full config-2 step.

    The full step's work is a list of units -- P2M of p and of q, L2P value +
    gradient at q and at p (per point), and for each of its two cascades every
    (level, active offset) M2L GEMM, every (level, child) M2M and L2L shift
    (expansion.py:200-264) -- dealt round-robin into SAMPLE_SLICES balanced
    slices.  Step s runs slice s mod SAMPLE_SLICES on real-sized grids (level 5,
    64^3) and (N + M) / SAMPLE_SLICES points; value = that slice's points per
    second, i.e. (N + M) / (SAMPLE_SLICES * t_slice).  No extrapolation beyond
    the uniform 1/32 share of the same work."""
    threads = len(os.sched_getaffinity(0))
    for var in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(var, str(threads))
    from itertools import product

    from oracle.fc2t2_oracle import COARSEST, Oracle, res_of, width_of
    cfg = cfg or CFG
    ora = Oracle(cfg["alpha"], cfg["rho"], cfg["levels"])
    S = slices or SAMPLE_SLICES
    L = cfg["levels"]
    rng = np.random.default_rng(seed + 7)
    # grids of the real sizes (values do not change the arithmetic)
    Mg = {l: rng.standard_normal((res_of(l),) * 3 + (1, ora.P)) for l in range(COARSEST, L + 1)}
    units = []
    for _cascade in range(2):
        for l in range(L, COARSEST, -1):
            units += [("m2m", l, c) for c in product((0, 1), repeat=3)]
        for l in range(COARSEST, L + 1):
            t = ora.tables["far"][l]
            units += [("m2l", l, i) for i in np.flatnonzero(t["active"])]
            if l > COARSEST:
                units += [("l2l", l - 1, c) for c in product((0, 1), repeat=3)]
        units += [("near", L, i) for i in np.flatnonzero(ora.tables["near"]["active"])]
    slices = [units[k::S] for k in range(S)]
    n_s, m_s = N // S, M // S
    shift_cache = {}

    def shift(kind, l, c):
        key = (kind, l, c)
        if key not in shift_cache:
            wf = width_of(l if kind == "m2m" else l + 1)
            shift_cache[key] = ora.shift((np.array(c) - 0.5) * wf, kind == "m2m").T.copy()
        return shift_cache[key]

    def run_unit(u):
        kind, l, x = u
        if kind == "m2m":
            f = Mg[l]
            _ = f[x[0]::2, x[1]::2, x[2]::2] @ shift(kind, l, x)
        elif kind == "l2l":
            _ = Mg[l] @ shift(kind, l, x)
        else:
            tab = ora.tables["near"] if kind == "near" else ora.tables["far"][l]
            one = dict(tab)
            one["active"] = np.zeros_like(tab["active"])
            one["active"][x] = True
            ora.m2l(Mg[l], one)

    times = []
    for it in range(warmup + steps):
        k = it % S
        p, w, q, yb = inputs(seed + 1 + it, n_s, m_s)
        p, w, q, yb = (a.astype(np.float64) for a in (p, w, q, yb))
        t0 = time.perf_counter()
        ora.p2m(p, w)                                   # forward P2M
        Lf = Mg[L]
        ora.evaluate(Lf, q)                             # values
        np.einsum("mc,mca->ma", yb, ora.evaluate(Lf, q, what="grad"))   # q_bar
        ora.p2m(q, yb)                                  # backward P2M
        ora.evaluate(Lf, p)                             # w_bar
        np.einsum("nc,nca->na", w, ora.evaluate(Lf, p, what="grad"))    # p_bar
        for u in slices[k]:
            run_unit(u)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    t = float(np.mean(times))
    return {"value": (n_s + m_s) / t, "unit": UNIT, "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": (f"oracle (float64 NumPy restatement of the reference, speed-faithful) on "
                       f"1/{S} of the full step per timed step: {n_s} sources + {m_s} "
                       f"queries through P2M and L2P value+grad, plus a round-robin 1/{S} of "
                       f"the two level-{L} cascades' M2L offsets and M2M/L2L child shifts on "
                       f"full-size grids; mean of {steps} steps"),
            "slices": S,
            "seconds_per_step": t, "seconds_per_full_step": S * t}


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    five = world > 1 or args.config == 5
    cfg, wl = (CFG5, WORKLOAD5) if five else (CFG, WORKLOAD)
    N, M = cfg["N"], cfg["M"]
    cb = cpu_sample(args.steps, args.warmup, N, M, cfg["seed"], cfg, 256 if five else None)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * cb["seconds_per_step"],
            "ms_per_full_step": 1000.0 * cb["seconds_per_full_step"],
            "higher_is_better": True, "scaling": "strong" if five else "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": wl, "N": N, "M": M,
                                            "parallelism": "cpu",
                                            "sample_fraction": 1.0 / cb["slices"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                "cpu_model")},
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- GPU arm ---

def seeded_direction(rng):
    """Unit vector, rejecting near-vertical ones (SURVEY 8(d) camera rule)."""
    while True:
        u = rng.normal(size=3)
        u /= np.linalg.norm(u)
        if abs(u[1]) <= 0.99:
            return u


# Stages of a config-2 step (library launch labels); two expansions per step:
# the forward of (p, w) and the backward of (q, y_bar).
STAGE_GROUPS = {
    "l2p": ["l2p"],
    "domain_check": ["domain_check"],
    "p2m": ["brick_hist", "brick_scan", "brick_scatter", "brick_p2m"],
    "m2l_finest": ["m2l_sep_pre", "m2l_sep_z", "m2l_sep_y", "m2l_sep_x", "m2l_sep_post",
                   "m2l_sep_post_l2l"],
    "m2l_coarse": ["m2l_sepfar_pre", "m2l_sepfar_z", "m2l_sepfar_y", "m2l_sepfar_x",
                   "m2l_sepfar_post", "m2l_absmax", "m2l_split", "m2l_tc_L4", "m2l_L3", "m2l_L2",
                   "m2l_reduce"],
    "l2l": ["l2l"],
    "m2m": ["m2m"],
    "wgrad_recycle": ["wgrad_recycle"],
}


def sep_ffma_per_cell(rho: int) -> int:
    """FFMAs the separable finest M2L executes per cell and expansion
    (csrc/m2l_sep.cu): the pre transform (lower-triangular per axis), the z,
    y and x passes (6 taps per output position, index sets truncated to total
    degree <= rho) and the post transform (upper-triangular per axis)."""
    R1 = rho + 1
    ex = [(a, b, c) for t in range(R1) for a in range(t + 1) for b in range(t - a + 1)
          for c in [t - a - b]]
    pre = sum(e[k] + 1 for e in ex for k in range(3))
    post = sum(rho - sum(e) + 1 for e in ex for _ in range(3))
    z = sum((R1 - a - b) * R1 * 6 for a in range(R1) for b in range(R1 - a))
    y = sum((R1 - a) * (R1 - c) * 6 for a in range(R1) for c in range(R1))
    x = sum(R1 * (R1 - b - c) * 6 for b in range(R1) for c in range(R1 - b))
    return pre + z + y + x + post


def stage_rooflines(eng, prof, steps, N, M, hbm_peak, ffma_peak):
    """Per stage: ALGORITHMIC bytes per step (what the operation must move:
    inputs read once, outputs written once -- not the kernels' own
    intermediates), executed FP32 FLOPs where the stage is compute heavy,
    time per step from the library's per-launch CUDA events on each launch's
    stream, and the fraction of the binding roofline: t_min / t, t_min =
    max(bytes / HBM peak, flops / FFMA peak).  The finest M2L runs on a side
    stream beside the coarse levels, so both spans include SM sharing."""
    P, PP, L = eng.P, eng.PP, eng.levels
    R = (2 ** (L + 1)) ** 3
    grid = 4 * PP * R
    sep_flops = 2 * 2 * sep_ffma_per_cell(eng.rho) * R   # two expansions, 2 flop per FFMA
    model = {
        "l2p": (M * (12 + 4 + 12) + grid + N * (12 + 4 + 4 + 12) + grid, 0,
                "q: 12 B in + 4 B value + 12 B grad; p: 12 B + 4 B w + 4 B w_bar + 12 B p_bar; "
                "+ one finest L grid read per launch (the 144 B row gathers are L2 traffic)"),
        "p2m": ((N + M) * (12 + 4) + 2 * grid, 0,
                "12 B point + 4 B weight in per point + the finest M grid written, per expansion"),
        "m2l_finest": (2 * (2 * grid + grid // 8), sep_flops,
                       "per expansion: finest M read + L written + the level above's L read "
                       "(fused L2L); flops = executed FFMAs of the separable form x 2"),
        "m2l_coarse": (2 * sum(2 * 4 * PP * (2 ** (l + 1)) ** 3 for l in range(2, L)), 0,
                       "per expansion and coarse level: M read + L written"),
        "l2l": (2 * sum(4 * PP * ((2 ** (l + 1)) ** 3 * 2 + (2 ** l) ** 3)
                        for l in range(3, L)), 0, "fine read+write + coarse read per level"),
        "m2m": (2 * sum(4 * PP * ((2 ** (l + 1)) ** 3 + (2 ** l) ** 3) for l in range(3, L + 1)),
                0, "fine read + coarse write per level"),
        "wgrad_recycle": (M * (12 + 4 + 12), 0, "12 B grad + 4 B y_bar in, 12 B q_bar out"),
        "domain_check": (M * 12, 0, "12 B per query read"),
    }
    out = {}
    for st, names in STAGE_GROUPS.items():
        hit = [n for n in names if n in prof]
        if not hit:
            continue
        ms = sum(prof[n][0] for n in hit) / steps
        launches = sum(prof[n][1] for n in hit) / steps
        b, fl, how = model[st]
        t = ms / 1000.0
        t_hbm, t_fl = b / (hbm_peak * 1e9), (fl / (ffma_peak * 1e12) if fl else 0.0)
        bound = "fp32_ffma" if t_fl > t_hbm else "hbm"
        e = {"kernels": hit, "ms_per_step": round(ms, 4), "launches_per_step": launches,
             "bytes_per_step": b, "achieved_gbps": round(b / t / 1e9, 1),
             "hbm_frac": round(t_hbm / t, 4), "bound": bound,
             "frac": round(max(t_hbm, t_fl) / t, 4), "model": how}
        if fl:
            e.update(flops_per_step=fl, achieved_tflops=round(fl / t / 1e12, 2),
                     ffma_frac=round(t_fl / t, 4))
        out[st] = e
    if "l2p" in out:
        # the cell-row gathers are L2 traffic: 5 sectors (160 B) per point and channel
        sect = (M + N) * 160
        o = out["l2p"]
        o["l2_sector_bytes_per_step"] = sect
        o["l2_tbps"] = round(sect / (o["ms_per_step"] / 1000.0) / 1e12, 2)
        o["l2_note"] = ("each point gathers its 144-byte cell row = 5 L2 sectors; the 37.7 MB "
                        "level-5 grid is L2 resident, so the binding resource is the L2 slice "
                        "throughput (~6300 B/clk chip-wide, B300_MICROARCH.md)")
    return out


def kernel_rooflines(eng, prof, steps, N, M, hbm_peak, ffma_peak):
    """The same accounting per library launch label (one kernel each): the
    bytes that kernel must read and write once, its executed FFMA flops where
    it is a separable pass, against the live event time per step."""
    P, PP, L, R1 = eng.P, eng.PP, eng.levels, eng.rho + 1
    R = (2 ** (L + 1)) ** 3
    grid = 4 * PP * R
    T = R1 * (R1 + 1) // 2 * R1
    zf = sum((R1 - a - b) * R1 * 6 for a in range(R1) for b in range(R1 - a))
    yf = sum((R1 - a) * (R1 - c) * 6 for a in range(R1) for c in range(R1))
    xf = sum(R1 * (R1 - b - c) * 6 for b in range(R1) for c in range(R1 - b))
    model = {
        "l2p": (M * (12 + 4 + 12) + grid + N * (12 + 4 + 4 + 12) + grid, 0,
                "per point 12 B in + value/grad (+ w_bar, p_bar) out, + the finest L grid once "
                "per launch; the 144 B row gathers are L2 traffic"),
        "brick_hist": ((N + M) * 12, 0, "12 B per point read"),
        "brick_scatter": ((N + M) * (16 + 16), 0, "12 B point + 4 B weight read, 16 B record written"),
        "brick_p2m": ((N + M) * 16 + 2 * grid, 0, "16 B record read per point + the finest M grid written"),
        "wgrad_recycle": (M * (12 + 4 + 12), 0, "12 B grad + 4 B y_bar in, 12 B q_bar out"),
        "domain_check": (M * 12, 0, "12 B per query read"),
        "m2l_sep_pre": (2 * (grid + 4 * P * R), 0, "M rows read, M' written, per expansion"),
        "m2l_sep_z": (2 * 4 * (P + T) * R, 2 * 2 * zf * R, "M' read, Z written; executed FFMAs x 2"),
        "m2l_sep_y": (2 * 4 * (T + T) * R, 2 * 2 * yf * R, "Z read, Y written; executed FFMAs x 2"),
        "m2l_sep_x": (2 * 4 * (T + P) * R, 2 * 2 * xf * R, "Y read, X written; executed FFMAs x 2"),
        "m2l_sep_post_l2l": (2 * (4 * P * R + grid + grid // 8), 0,
                             "X read, L rows written, the level above's L read"),
    }
    out = {}
    for lab, (b, fl, how) in model.items():
        if lab not in prof:
            continue
        t = prof[lab][0] / steps / 1000.0
        t_hbm, t_fl = b / (hbm_peak * 1e9), (fl / (ffma_peak * 1e12) if fl else 0.0)
        e = {"kernels": [lab], "ms_per_step": round(t * 1000.0, 4),
             "launches_per_step": prof[lab][1] / steps, "bytes_per_step": b,
             "achieved_gbps": round(b / t / 1e9, 1), "hbm_frac": round(t_hbm / t, 4),
             "bound": "fp32_ffma" if t_fl > t_hbm else "hbm",
             "frac": round(max(t_hbm, t_fl) / t, 4), "model": how}
        if fl:
            e.update(flops_per_step=fl, achieved_tflops=round(fl / t / 1e12, 2),
                     ffma_frac=round(t_fl / t, 4))
        out[lab] = e
    if "l2p" in out:
        o = out["l2p"]
        o["l2_sector_bytes_per_step"] = (M + N) * 160
        o["l2_tbps"] = round((M + N) * 160 / (o["ms_per_step"] / 1000.0) / 1e12, 2)
        o["l2_frac_of_lts_cap"] = round(o["l2_tbps"] / (6300 * 1.965e9 / 1e12), 3)
        o["l2_note"] = ("each point gathers its 144-byte cell row = 5 L2 sectors from the "
                        "L2-resident 37.7 MB grid: the kernel is bound by the L2 slice throughput "
                        "(~6300 B/clk chip-wide = 12.4 TB/s at 1.965 GHz, B300_MICROARCH.md), "
                        "not by HBM")
    return out


def _peaks():
    """(HBM GB/s, FP32 FFMA TFLOP/s): the measured peaks, else the fallbacks."""
    try:
        hbm = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 7672.0))
    except Exception:
        hbm = 7672.0
    return hbm, ffma_peak_tflops()[0]


def ffma_peak_tflops():
    """The FP32 FFMA peak measured on this pool's B200s by scripts/ubench/peaks.py
    (profiles/r2_peaks.json), else the nominal 148 SMs x 128 FMA/clk x 2 x
    1.965 GHz."""
    try:
        v = json.loads((ROOT / "profiles" / "r2_peaks.json").read_text())["ffma_tflops"]
        return float(v), "measured FFMA peak (profiles/r2_peaks.json, scripts/ubench/peaks.cu)"
    except Exception:
        return 74.45, "nominal 148 SM x 128 FMA/clk x 1.965 GHz"


def measured_traffic(kernels):
    """DRAM bytes per step of these kernels from the committed ncu --set full
    capture (profiles/traffic.json, written by scripts/ncu_traffic.py), or None."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic.json").read_text())
    except Exception:
        return None
    tot, ms, hit = 0.0, 0.0, False
    for k in kernels:
        if k in t.get("bytes_per_step", {}):
            tot += t["bytes_per_step"][k]
            ms += t.get("serial_ms_per_step", {}).get(k, 0.0)
            hit = True
    return {"bytes_per_step": tot, "serial_ms_per_step": ms or None,
            "source": t.get("source")} if hit else None


def timed_steps(fn, steps: int, warmup: int, flush, stream, stages: dict | None = None):
    """(median step in ms x `steps`, last result): per-step CUDA events on the
    launching stream, L2 flush between steps outside the events.  With
    ``stages`` a SECOND pass of the same `steps` steps runs with the library's
    per-launch CUDA events on (two event records around every kernel launch,
    ~9 % of a config-2 step) and stores the per-kernel profile (ms per step);
    the returned time is the first, uninstrumented pass."""
    import torch

    from paper_2111_00110_b200 import _lib
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()   # like timeit: no interpreter GC pause inside a timed step

    def one_pass():
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        res, host = None, 0.0
        for i in range(steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            h0 = time.perf_counter()
            res = fn()
            host += time.perf_counter() - h0
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        return sorted(a.elapsed_time(b) for a, b in ev), res, host

    per, out, host = one_pass()
    if stages is not None:
        _lib.profile_enable(True)
        per_i, _, _ = one_pass()
        stages.update({k: round(v[0] / steps, 4) for k, v in _lib.profile_read().items()})
        _lib.profile_enable(False)
        stages["_host_call_ms"] = round(1e3 * host / steps, 4)
        stages["_note"] = ("CUDA-event spans per kernel name on the launching stream, from a "
                           "second pass of the same steps with the per-launch events on (the "
                           "step time reported is the first pass, without them); the finest M2L "
                           "and the coarse levels run on their own streams, so spans include "
                           "waiting for SMs -- the serialised ncu launch list has the kernels' "
                           "own times")
        stages["_step_ms_instrumented"] = round(sum(per_i) / steps, 4)
        stages["_step_ms_median"] = round(float(np.median(per)), 4)
        stages["_step_ms_mean"] = round(sum(per) / steps, 4)
        stages["_step_ms_max"] = round(per[-1], 4)
    gc.enable()
    # the MEDIAN step times `steps` (median of >= 20 runs): one
    # host hiccup in a 20-step region moves the mean by several per cent
    return float(np.median(per)) * steps, out


def secondary(dev, flush, stream, steps: int) -> dict:
    """Configs 1, 3, 4 on one GPU (their own metrics, secondary to the headline)."""
    import torch

    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import (depth_forward, depth_surface_jvp,
                                              explicit_forward, explicit_jvp,
                                              volumetric_forward, volumetric_jvp)
    from paper_2111_00110_b200.ray import Camera, RayBundle, generate_rays, traverse
    out = {}
    hbm_peak, ffma_peak = _peaks()

    def ray_roofline(ms, nbytes, flops, how):
        """SURVEY 8(d), ray kernels: both bounds -- per-ray I/O plus the
        per-box coefficient gather (an HBM upper bound: the grid is mostly L2
        resident) and the paper's per-box FLOP counts against the measured
        FP32 FFMA peak; the higher fraction binds."""
        t = ms / 1e3
        fh, ff = nbytes / (hbm_peak * 1e9) / t, flops / (ffma_peak * 1e12) / t
        return {"ms_per_step": round(ms, 4), "bytes_per_step": int(nbytes),
                "flops_per_step": int(flops), "hbm_frac": round(fh, 4), "fp32_frac": round(ff, 4),
                "bound": "hbm" if fh >= ff else "fp32", "frac": round(max(fh, ff), 4),
                "model": how}
    # config 1: 2D explicit layer lifted to z = 0.03125, level 4
    rng = np.random.default_rng(11)
    n = 4096
    lo = np.nextafter(-1.0, 0.0)
    p = np.concatenate([rng.uniform(lo, 1, (n, 2)), np.full((n, 1), 0.03125)], 1).astype(np.float32)
    q = np.concatenate([rng.uniform(lo, 1, (n, 2)), np.full((n, 1), 0.03125)], 1).astype(np.float32)
    w = rng.standard_normal((n, 1)).astype(np.float32)
    yb = rng.standard_normal((n, 1)).astype(np.float32)
    P, Q, W, YB = (torch.from_numpy(a).to(dev) for a in (p, q, w, yb))
    e1 = Engine(KernelModel("gaussian", 200.0, 4), 4, check_admissibility=False)
    ms, _ = timed_steps(lambda: explicit_jvp(YB, explicit_forward(e1, SourceSet(P, W), Q)),
                        steps, 3, flush, stream)
    out["cfg1_explicit_2d"] = {"metric": "points/s (N+M)", "value": 2 * n / (ms / steps / 1e3),
                               "ms_per_step": ms / steps,
                               "workload": "N=M=4096, 2D lifted to z=0.03125, level 4, alpha 200"}
    # the same step replayed as one CUDA graph (graphs.GraphedExplicit): the
    # config is launch-bound, ~45 kernels for 8192 points
    from paper_2111_00110_b200.graphs import GraphedExplicit
    g1 = GraphedExplicit(e1, P, W, Q, YB)
    ms, _ = timed_steps(lambda: g1(P, W, Q, YB), steps, 3, flush, stream)
    out["cfg1_explicit_2d_graphed"] = {
        "metric": "points/s (N+M)", "value": 2 * n / (ms / steps / 1e3), "ms_per_step": ms / steps,
        "workload": "config 1 as a CUDA-graph replay (inputs copied in, domain flag read per step)"}
    del g1
    # one fit-sdf training epoch (cli.py:129-145) at config-2
    # size on the device: explicit layer fwd, MAE loss + tangent, JVP, Adam step
    from paper_2111_00110_b200.trainer import Optimizer, TrainConfig, fit_sdf_epoch
    rng_f = np.random.default_rng(22)
    e5f = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    Nf, Mf = 1 << 20, 10_000_000
    pf = torch.from_numpy(rng_f.uniform(-1 + 1e-6, 1 - 1e-6, (Nf, 3)).astype(np.float32)).to(dev)
    wf = torch.from_numpy(rng_f.uniform(-1e-2, 1e-2, (Nf, 1)).astype(np.float32)).to(dev)
    qf = torch.from_numpy(rng_f.uniform(lo, 1, (Mf, 3)).astype(np.float32)).to(dev)
    tf = torch.from_numpy(rng_f.normal(0, 0.1, (Mf, 1)).astype(np.float32)).to(dev)
    optf = Optimizer(TrainConfig(optimizer="adam", learning_rate=1e-3, l1_weight=1e-6))
    state = {"src": SourceSet(pf, wf), "bias": 0.0, "epoch": 0}

    def epoch_f():
        st = state
        st["src"], st["bias"], loss, _ = fit_sdf_epoch(e5f, st["src"], st["bias"], qf, tf, optf,
                                                       st["epoch"])
        st["epoch"] += 1
        return loss
    ms, _ = timed_steps(epoch_f, steps, 3, flush, stream)
    out["fit_sdf_epoch"] = {
        "metric": "epochs/s", "value": 1e3 / (ms / steps), "ms_per_step": ms / steps,
        "points_per_s": (Nf + Mf) / (ms / steps / 1e3),
        "workload": "fit-sdf epoch (cli.py:129-145): N=2^20 sources, batch M=10^7 samples, "
                    "level 5, Adam lr 1e-3, MAE, L1 1e-6; loss read back every epoch"}
    del pf, wf, qf, tf, state, optf, e5f
    # config 3: root-implicit depth + normal, 512x512 rays, level 5, bias +0.05
    rng = np.random.default_rng(33)
    N3 = 1 << 18
    p = rng.uniform(lo, 1, (N3, 3)).astype(np.float32)
    w = rng.normal(0.0, 0.1, (N3, 1)).astype(np.float32)
    cam = Camera(2.0 * seeded_direction(rng), np.zeros(3), np.array([0.0, 1.0, 0.0]), 60.0,
                 512, 512)
    b3 = generate_rays(cam)
    R3 = b3.count
    yl = torch.from_numpy(rng.standard_normal(R3).astype(np.float32)).to(dev)
    yg = torch.from_numpy(rng.standard_normal((R3, 3)).astype(np.float32)).to(dev)
    b3 = RayBundle(torch.from_numpy(b3.origins).to(dev), torch.from_numpy(b3.directions).to(dev))
    e5 = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    src3 = SourceSet(torch.from_numpy(p).to(dev), torch.from_numpy(w).to(dev))

    def step3():
        res = depth_forward(e5, src3, b3, bias=0.05)
        return depth_surface_jvp(yl, yg, res), res
    st3 = {}
    ms, (g3, r3) = timed_steps(step3, steps, 3, flush, stream, st3)
    # every line: value from the median step (as the headline); the mean is
    # kept beside it in the stage dict
    med3 = st3.get("_step_ms_median", ms / steps)
    # boxes the walker visits: every box entered before the first root (all of
    # a missing ray's), from the traversal and the hit lengths
    tr3 = traverse(b3, 5)
    len3 = torch.as_tensor(r3.lengths, device=dev).double()
    hit3 = torch.as_tensor(r3.hit, device=dev).bool()
    rid3 = tr3.ray_id.long()
    vis3 = int(((tr3.t0 < len3[rid3]) | ~hit3[rid3]).sum().item())
    nh3 = int(hit3.sum().item())
    P4, PP4, cells5 = 35, 36, 64 ** 3
    rl3 = {"visited_boxes": vis3, "total_boxes": int(tr3.t0.shape[0]), "hits": nh3}
    if "depth_walk" in st3:
        rl3["depth_walk"] = ray_roofline(
            st3["depth_walk"], R3 * (48 + 4 + 12 + 12 + 4) + vis3 * 4 * P4, vis3 * (668 + 136),
            "48 B ray in, length + point + gradient + denominator out, 140 B cell row per "
            "visited box; line2poly 668 + Ferrari 136 FLOP per visited box (PAPER.md:609, :624); "
            "the root finder itself runs in float64")
    if "insert" in st3:
        rl3["insert"] = ray_roofline(
            st3["insert"], 4 * nh3 * (4 + 4 * PP4) + 4 * PP4 * cells5, 4 * nh3 * P4,
            "depth + 3 normal-adjoint items per hit: 4 B key + one 144 B payload row each, and "
            "the finest M grid written; one add per coefficient")
    del tr3
    out["cfg3_root_depth_normal"] = {
        "roofline_kernels": rl3,
        "metric": "rays/s", "value": R3 / (ms / steps / 1e3), "ms_per_step": ms / steps,
        "median_ms_per_step": med3,
        "hit_fraction": float(r3.hit.float().mean().item()), "stages_ms_per_step": st3,
        "workload": "N=2^18, 512x512 rays, radius 2, fov 60, level 5, bias +0.05, depth+normal "
                    "adjoints in one fused insertion"}
    # config 4: radiance, 8 poses of 400x400 rays, N = 2^20, 3 colours
    rng = np.random.default_rng(44)
    N4 = 1 << 20
    p = torch.from_numpy(rng.uniform(lo, 1, (N4, 3)).astype(np.float32)).to(dev)
    ws = torch.from_numpy(np.abs(rng.standard_normal((N4, 1))).astype(np.float32)).to(dev)
    wc = torch.from_numpy(rng.uniform(0, 1, (N4, 3)).astype(np.float32)).to(dev)
    org, dirs = [], []
    for _ in range(8):
        bb = generate_rays(Camera(2.5 * seeded_direction(rng), np.zeros(3),
                                  np.array([0.0, 1.0, 0.0]), 50.0, 400, 400))
        org.append(bb.origins)
        dirs.append(bb.directions)
    b4 = RayBundle(torch.from_numpy(np.concatenate(org)).to(dev),
                   torch.from_numpy(np.concatenate(dirs)).to(dev))
    R4 = b4.count
    target = torch.from_numpy(rng.uniform(0, 1, (R4, 3)).astype(np.float32)).to(dev)
    bg = np.ones(3)

    def step4():
        res = volumetric_forward(e5, p, ws, wc, b4, bg)
        ybar = 2.0 * (res.rgb - target) / float(res.rgb.numel())   # MSE tangent (trainer.py:96-97)
        return volumetric_jvp(ybar, res)
    st4 = {}
    ms, _ = timed_steps(step4, max(2, steps // 4), 1, flush, stream, st4)
    k = max(2, steps // 4)
    med4 = st4.get("_step_ms_median", ms / k)
    res4 = volumetric_forward(e5, p, ws, wc, b4, bg)
    alive4 = int(torch.as_tensor(res4.alive).sum().item())
    del res4
    C4 = 4
    rl4 = {"alive_segments": alive4}
    if "vol_forward" in st4:
        rl4["vol_forward"] = ray_roofline(
            st4["vol_forward"], R4 * (48 + 12) + alive4 * 4 * C4 * P4, alive4 * 1563,
            "48 B ray in, 12 B rgb out, 560 B of cell rows (sigma + 3 colours) per alive box; "
            "1563 FLOP per box (PAPER.md:1118)")
    if "vol_payload" in st4:
        rl4["vol_payload"] = ray_roofline(
            st4["vol_payload"], R4 * (48 + 12) + alive4 * (4 * C4 * P4 + 112 + 4), alive4 * 2452,
            "ray + rgb tangent in, 560 B of cell rows per alive box, one 112 B segment record "
            "+ 4 B key out; 2452 FLOP per box (PAPER.md:1119)")
    if "insert" in st4:
        rl4["insert"] = ray_roofline(
            st4["insert"], alive4 * (112 + 4 + 4) + 4 * C4 * PP4 * cells5, alive4 * 1489,
            "112 B record + key + order per alive box, the 4-channel finest M grid written; "
            "1489 FLOP per box (PAPER.md:1120)")
    out["cfg4_radiance"] = {"metric": "rays/s", "value": R4 / (ms / k / 1e3), "ms_per_step": ms / k,
                            "roofline_kernels": rl4,
                            "median_ms_per_step": med4,
                            "stages_ms_per_step": st4,
                            "workload": "N=2^20 (|N(0,1)| density, U(0,1) RGB), 8 poses x 400x400, "
                                        "radius 2.5, fov 50, level 5, MSE vs U(0,1) target"}
    # config 5 on one GPU: rho = 6 (P = 84), level 6 (128^3), N = 2^24, M = 2^27
    del P, Q, W, YB, p, ws, wc, b4, target, src3, b3
    torch.cuda.empty_cache()
    e6 = Engine(KernelModel("gaussian", 4000.0, 6), 6, check_admissibility=False)
    _ = e6.handle
    gen = torch.Generator(device=dev).manual_seed(55)
    N5, M5 = 1 << 24, 1 << 27
    lo32 = -0.99999994
    p5 = torch.rand(N5, 3, device=dev, generator=gen) * (2 * 0.99999994) + lo32
    w5 = torch.randn(N5, 1, device=dev, generator=gen) * 0.1
    q5 = torch.rand(M5, 3, device=dev, generator=gen) * (2 * 0.99999994) + lo32
    y5 = torch.randn(M5, 1, device=dev, generator=gen)
    st5 = {}
    ms, _ = timed_steps(lambda: explicit_jvp(y5, explicit_forward(e6, SourceSet(p5, w5), q5)),
                        2, 1, flush, stream, st5)
    out["cfg5_explicit_rho6_1gpu"] = {
        "metric": "points/s (N+M)", "value": (N5 + M5) / (ms / 2 / 1e3), "ms_per_step": ms / 2,
        "stages_ms_per_step": st5,
        "workload": "N=2^24, M=2^27, level 6 (128^3), rho 6 (P=84), alpha 4000, one GPU "
                    "(the multi-GPU runs shard this with the grid all-reduce)"}
    return out


def training_lines(dev, flush, stream, steps: int) -> dict:
    """the reference CLI's fitting loops on the device, on the
    paper's own per-epoch workloads where it quotes one (PAPER.md:537-548
    SDF epochs, :820 inverse rendering; RTX 2080 Ti numbers in BASELINE.md)."""
    import torch

    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet
    from paper_2111_00110_b200.layers import depth_forward
    from paper_2111_00110_b200.ray import Camera, RayBundle, generate_rays
    from paper_2111_00110_b200.trainer import (Optimizer, TrainConfig, cgls_sdf,
                                               fit_depth_epoch, fit_radiance_epoch,
                                               fit_sdf_epoch)
    out = {}
    gen = torch.Generator(device=dev).manual_seed(66)
    lo32 = -0.99999994

    def upts(n):
        return torch.rand(n, 3, device=dev, generator=gen) * (2 * 0.99999994) + lo32
    # SDF epochs (fit-sdf loop, cli.py:129-145) at the paper's size: N = 8M
    # sources, M = 10M samples per epoch, levels 4 / 5 / 6, Adam, MAE, L1
    Ns, Ms = 8 << 20, 10_000_000
    qs, ts = upts(Ms), torch.randn(Ms, 1, device=dev, generator=gen) * 0.1
    for level, alpha, paper_ms in ((4, 200.0, 130.0), (5, 1200.0, 225.0), (6, 4000.0, 1200.0)):
        eng = Engine(KernelModel("gaussian", alpha, 4), level, check_admissibility=False)
        opt = Optimizer(TrainConfig(optimizer="adam", learning_rate=1e-3, l1_weight=1e-6))
        st = {"src": SourceSet(upts(Ns), (torch.rand(Ns, 1, device=dev, generator=gen) - 0.5)
                               * 0.02), "bias": 0.0, "epoch": 0}

        def epoch_f(st=st, eng=eng, opt=opt):
            st["src"], st["bias"], loss, _ = fit_sdf_epoch(eng, st["src"], st["bias"], qs, ts,
                                                           opt, st["epoch"])
            st["epoch"] += 1
            return loss
        k = max(3, steps // 2)
        ms, _ = timed_steps(epoch_f, k, 3, flush, stream)
        out[f"sdf_epoch_paper_L{level}"] = {
            "metric": "ms/epoch", "ms_per_step": ms / k, "value": ms / k,
            "paper_ms_rtx2080ti": paper_ms, "paper_over_ours": paper_ms / (ms / k),
            "workload": f"fit-sdf epoch: N=8M sources, M=10M samples, level {level}, "
                        f"alpha {alpha:g}, rho 4, Adam, MAE, L1; loss read back each epoch"}
        del st, eng, opt
    # CGLS solve (cli.py:173-224) at config-2 size: 4 iterations
    e5 = Engine(KernelModel("gaussian", 1000.0, 4), 5, check_admissibility=False)
    pc, qc = upts(1 << 20), upts(10_000_000)
    dc = torch.randn(10_000_000, device=dev, generator=gen) * 0.1
    k = max(3, steps // 4)
    ms, _ = timed_steps(lambda: cgls_sdf(e5, pc, qc, dc, 4), k, 3, flush, stream)
    out["cgls_sdf_4it"] = {
        "metric": "ms/solve", "ms_per_step": ms / k, "value": ms / k,
        "workload": "CGLS on (w, bias), N=2^20 sources, M=10^7 samples, level 5, alpha 1000: "
                    "4 iterations + setup (2 sorts, 1 adjoint, 1 final forward) = 11 products"}
    del pc, qc, dc
    # fit-depth epoch (cli.py:288-306) at the paper's inverse-rendering image
    # size (420 x 560, level 5); N = 2^18 sources as config 3
    rng = np.random.default_rng(67)
    N3 = 1 << 18
    src = SourceSet(torch.from_numpy(rng.uniform(-0.9, 0.9, (N3, 3)).astype(np.float32)).to(dev),
                    torch.from_numpy(rng.normal(0, 0.1, (N3, 1)).astype(np.float32)).to(dev))
    cam = Camera(2.0 * seeded_direction(rng), np.zeros(3), np.array([0.0, 1.0, 0.0]), 60.0,
                 560, 420)
    bb = generate_rays(cam)
    bundle = RayBundle(torch.from_numpy(bb.origins).to(dev), torch.from_numpy(bb.directions).to(dev))
    r0 = depth_forward(e5, src, bundle, bias=0.05)
    tgt = torch.where(r0.dev["hit"].bool(), r0.lengths, torch.full_like(r0.lengths, float("nan")))
    tgt = (tgt + 0.01 * torch.randn(tgt.shape, device=dev, dtype=tgt.dtype, generator=gen)).float()
    optd = Optimizer(TrainConfig(optimizer="adam", learning_rate=1e-4, l1_weight=1e-6))
    sd = {"src": src, "bias": 0.05, "epoch": 0}

    def depth_f():
        sd["src"], sd["bias"], loss, _ = fit_depth_epoch(e5, sd["src"], sd["bias"], bundle, tgt,
                                                         optd, sd["epoch"])
        sd["epoch"] += 1
        return loss
    k = max(3, steps // 2)
    st_d = {}
    ms, _ = timed_steps(depth_f, k, 3, flush, stream, st_d)
    out["fit_depth_epoch_420x560"] = {
        "metric": "ms/epoch", "ms_per_step": ms / k, "value": ms / k, "stages_ms_per_step": st_d,
        "paper_ms_rtx2080ti": 600.0,
        "paper_note": "the paper's ~600 ms epoch fits surface gradients (normals) at this image "
                      "size; this line fits depths (same root walk, same one-insertion backward)",
        "workload": "fit-depth epoch: 420x560 rays, N=2^18, level 5, alpha 1000, Adam, MAE, "
                    "miss penalty 0.1"}
    del src, bundle, r0, tgt, sd, optd
    # fit-radiance epoch (cli.py:363-382) at config 4: N = 2^20, minibatches of
    # 2^17 rays drawn on the device from the 8 x 400 x 400 pool
    rng = np.random.default_rng(44)
    N4 = 1 << 20
    p4 = torch.from_numpy(rng.uniform(-0.99, 0.99, (N4, 3)).astype(np.float32)).to(dev)
    ws4 = torch.from_numpy(np.abs(rng.standard_normal((N4, 1))).astype(np.float32)).to(dev)
    wc4 = torch.from_numpy(rng.uniform(0, 1, (N4, 3)).astype(np.float32)).to(dev)
    org, dirs = [], []
    for _ in range(8):
        b = generate_rays(Camera(2.5 * seeded_direction(rng), np.zeros(3),
                                 np.array([0.0, 1.0, 0.0]), 50.0, 400, 400))
        org.append(b.origins)
        dirs.append(b.directions)
    pool_o = torch.from_numpy(np.concatenate(org)).to(dev)
    pool_d = torch.from_numpy(np.concatenate(dirs)).to(dev)
    pool_t = torch.rand(pool_o.shape[0], 3, device=dev, generator=gen)
    optr = Optimizer(TrainConfig(optimizer="adam", learning_rate=1e-3, l1_weight=1e-6,
                                 loss="mse"))
    sr = {"p": p4, "ws": ws4, "wc": wc4, "epoch": 0}
    B = 1 << 17

    def rad_f():
        idx = torch.randperm(pool_o.shape[0], device=dev, generator=gen)[:B]
        mb = RayBundle(pool_o[idx], pool_d[idx])
        sr["p"], sr["ws"], sr["wc"], loss = fit_radiance_epoch(
            e5, sr["p"], sr["ws"], sr["wc"], mb, pool_t[idx], np.ones(3), optr, sr["epoch"])
        sr["epoch"] += 1
        return loss
    k = max(3, steps // 4)
    st_r = {}
    ms, _ = timed_steps(rad_f, k, 3, flush, stream, st_r)
    out["fit_radiance_epoch"] = {
        "metric": "ms/epoch", "ms_per_step": ms / k, "value": ms / k, "stages_ms_per_step": st_r,
        "workload": "fit-radiance epoch: N=2^20, 2^17-ray minibatch from 8 x 400x400 poses, "
                    "level 5, alpha 1000, Adam, MSE, L1"}
    return out


def run_ours(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
    from paper_2111_00110_b200.expansion import m2l_pairs
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    from paper_2111_00110_b200.parallel import (DeviceBackend, explicit_forward_sharded,
                                                explicit_jvp_sharded)

    local = _local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    N, M = (CFG["N"], CFG["M"]) if not args.small else (1 << 16, 1 << 20)

    t0 = time.perf_counter()
    eng = Engine(KernelModel("gaussian", CFG["alpha"], CFG["rho"]), CFG["levels"],
                 check_admissibility=False)
    _ = eng.handle
    t_tables = time.perf_counter() - t0

    # this rank's shard of the global problem (weak scaling: shard = config-2 size)
    p, w, q, yb = inputs(CFG["seed"] + 1000 * rank, N, M)
    P = torch.from_numpy(p).to(dev)
    W = torch.from_numpy(w).to(dev)
    Q = torch.from_numpy(q).to(dev)
    YB = torch.from_numpy(yb).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    backend = DeviceBackend(eng)

    def step_dev():
        if world > 1:
            res = explicit_forward_sharded(backend, P, W, Q)
            return explicit_jvp_sharded(backend, YB, res)
        res = explicit_forward(eng, SourceSet(P, W), Q)
        return explicit_jvp(YB, res)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step_dev()
    barrier()

    # ---- value: device-resident inputs, per-step events, L2 flush between steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    gc.collect()
    gc.disable()   # like timeit: no interpreter GC pause inside the timed region
    with Clocks(local) as clk:
        barrier()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            step_dev()
            ev[i][1].record(stream)
        barrier()
    launches = (_lib.launch_count() - launches0) // args.steps
    # the median of the K per-step times (the mean is kept beside
    # it): one host hiccup in a 20-step region moves the mean by several per cent
    per_step = [a.elapsed_time(b) for a, b in ev]
    ms_mean = float(sum(per_step)) / args.steps
    ms = float(np.median(per_step)) * args.steps
    # ---- the same K steps once more with the library's per-launch CUDA events
    # on, for the per-kernel times behind the rooflines: two event records
    # around every launch cost ~9 % of a step, so `value` is the pass above
    # and the instrumented pass is reported beside it
    ev_i = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(args.steps)]
    _lib.profile_enable(True)
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        ev_i[i][0].record(stream)
        step_dev()
        ev_i[i][1].record(stream)
    barrier()
    gc.enable()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    ms_instr = float(np.median([a.elapsed_time(b) for a, b in ev_i]))
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * (N + M) / (ms_step / 1000.0)

    # the same step replayed as one CUDA graph (graphs.GraphedExplicit; fresh
    # inputs copied in every step): the launch/host overhead of the eager path
    graphed = None
    if world == 1:
        from paper_2111_00110_b200.graphs import GraphedExplicit
        gstep = GraphedExplicit(eng, P, W, Q, YB)
        for _ in range(args.warmup):
            gstep(P, W, Q, YB)
        torch.cuda.synchronize()
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        gc.collect()
        gc.disable()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            gev[i][0].record(stream)
            gstep(P, W, Q, YB)
            gev[i][1].record(stream)
        torch.cuda.synchronize()
        gc.enable()
        gms = sum(a.elapsed_time(b) for a, b in gev) / args.steps
        graphed = {"value": (N + M) / (gms / 1000.0), "ms_per_step": gms,
                   "note": "GraphedExplicit replay, inputs copied in per step"}
        del gstep

    # ---- e2e: pinned host torch tensors through the public API
    hp, hw, hq, hy = (torch.from_numpy(a).pin_memory() for a in (p, w, q, yb))
    h2d = sum(a.numel() * 4 for a in (hp, hw, hq, hy))

    def step_host():
        if world > 1:
            res = explicit_forward_sharded(backend, hp.to(dev, non_blocking=True),
                                           hw.to(dev, non_blocking=True),
                                           hq.to(dev, non_blocking=True))
            wb, pb, qb = explicit_jvp_sharded(backend, hy.to(dev, non_blocking=True), res)
            outs = [t.to("cpu", non_blocking=True) for t in (res.values, wb, pb, qb)]
            torch.cuda.synchronize()
            return outs
        res = explicit_forward(eng, SourceSet(hp, hw), hq)
        g = explicit_jvp(hy, res)
        return res.values, g.w_bar, g.p_bar, g.q_bar

    outs = step_host()
    d2h = sum(o.numel() * 4 for o in outs)
    del outs  # release the pinned result buffers so the caching host allocator reuses them
    for _ in range(max(0, args.warmup - 1)):
        step_host()
    barrier()
    gc.collect()
    gc.disable()
    # every host step ends with its results readable on the host (the API
    # call synchronises its downloads), so the host clock per step is the end
    # to end time; median of the K steps as for `value`, the mean beside it
    e2e_per = []
    for _ in range(args.steps):
        te0 = time.perf_counter()
        step_host()
        torch.cuda.synchronize()
        e2e_per.append(1000.0 * (time.perf_counter() - te0))
    barrier()
    e2e_ms = float(np.median(e2e_per))
    e2e_mean = float(np.mean(e2e_per))
    gc.enable()
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e = world * (N + M) / (e2e_ms / 1000.0)

    if rank != 0:
        return

    # ---- rooflines: every stage against the bound SURVEY 8(d) gives it
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 7672.0))
    hbm_src = ("measured HBM copy bandwidth (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks
               else "fallback (B200_PROFILING.md)")
    ffma_peak, ffma_src = ffma_peak_tflops()
    rl_stages = stage_rooflines(eng, prof, args.steps, N, M, hbm_peak, ffma_peak)
    # dominant stage: the largest SERIALISED time (the committed ncu launch
    # capture, profiles/traffic.json) -- live event spans of the concurrent
    # cascade streams include waiting for SMs; live time when no capture
    for st, e in rl_stages.items():
        tr = measured_traffic(e["kernels"])
        e["ncu_serial_ms_per_step"] = tr["serial_ms_per_step"] if tr else None
    ser = {k: e["ncu_serial_ms_per_step"] for k, e in rl_stages.items() if e["ncu_serial_ms_per_step"]}
    dom = max(ser, key=ser.get) if ser else max(rl_stages, key=lambda k: rl_stages[k]["ms_per_step"])
    d = rl_stages[dom]
    traffic = measured_traffic(d["kernels"])
    if d["bound"] == "hbm":
        rl_core = {"bound": "hbm", "achieved": d["achieved_gbps"], "peak": hbm_peak,
                   "unit": "GB/s", "peak_source": hbm_src}
    else:
        rl_core = {"bound": "fp32_ffma", "achieved": d["achieved_tflops"], "peak": ffma_peak,
                   "unit": "TFLOP/s", "peak_source": ffma_src,
                   "hbm_frac": d["hbm_frac"], "hbm_peak_gbs": hbm_peak}
    ser_ms = d.get("ncu_serial_ms_per_step")
    roofline_stage = {"kernel": dom, **rl_core, "frac": d["frac"],
                "frac_at_ncu_serial_time": (round(d["frac"] * d["ms_per_step"] / ser_ms, 4)
                                            if ser_ms else None),
                "traffic": (traffic["bytes_per_step"] if traffic else None),
                "traffic_source": (traffic["source"] if traffic else None),
                "ncu_serial_ms_per_step": (traffic["serial_ms_per_step"] if traffic else None),
                "bytes_per_step": d["bytes_per_step"],
                "launch_ms": d["ms_per_step"] / max(d["launches_per_step"], 1),
                "launches_per_step": d["launches_per_step"], "bytes_model": d["model"]}
    if "l2_sector_bytes_per_step" in d:
        roofline_stage["l2_sector_bytes_per_step"] = d["l2_sector_bytes_per_step"]
        roofline_stage["l2_tbps"] = d["l2_tbps"]
        roofline_stage["l2_note"] = d["l2_note"]
    # `roofline`: the dominant KERNEL -- the launch label with the largest
    # serialised time per step in the committed ncu capture (live time when
    # there is none); `roofline_dominant_stage` keeps the multi-kernel stage
    rl_kernels = kernel_rooflines(eng, prof, args.steps, N, M, hbm_peak, ffma_peak)
    for lab, e in rl_kernels.items():
        tr = measured_traffic([lab])
        e["ncu_serial_ms_per_step"] = tr["serial_ms_per_step"] if tr else None
        e["traffic"] = tr["bytes_per_step"] if tr else None
        e["traffic_source"] = tr["source"] if tr else None
    kser = {k: e["ncu_serial_ms_per_step"] for k, e in rl_kernels.items()
            if e["ncu_serial_ms_per_step"]}
    kdom = (max(kser, key=kser.get) if kser
            else max(rl_kernels, key=lambda k: rl_kernels[k]["ms_per_step"]))
    kd = rl_kernels[kdom]
    roofline = {"kernel": kdom,
                "bound": "hbm" if kd["bound"] == "hbm" else "fp32_ffma",
                "achieved": kd["achieved_gbps"] if kd["bound"] == "hbm" else kd["achieved_tflops"],
                "peak": hbm_peak if kd["bound"] == "hbm" else ffma_peak,
                "unit": "GB/s" if kd["bound"] == "hbm" else "TFLOP/s",
                "peak_source": hbm_src if kd["bound"] == "hbm" else ffma_src,
                "frac": kd["frac"],
                "frac_at_ncu_serial_time": (round(kd["frac"] * kd["ms_per_step"]
                                                  / kd["ncu_serial_ms_per_step"], 4)
                                            if kd["ncu_serial_ms_per_step"] else None),
                "traffic": kd["traffic"], "traffic_source": kd["traffic_source"],
                "ncu_serial_ms_per_step": kd["ncu_serial_ms_per_step"],
                "bytes_per_step": kd["bytes_per_step"],
                "launch_ms": kd["ms_per_step"] / max(kd["launches_per_step"], 1),
                "launches_per_step": kd["launches_per_step"], "bytes_model": kd["model"],
                "share_of_step": round(kd["ms_per_step"] / ms_instr, 4),
                "timing": ("per-launch CUDA events on the launching stream over a second pass "
                           f"of the same {args.steps} steps ({ms_instr:.4f} ms per step with the "
                           "events on; `value` is the pass without them)")}
    for k in ("l2_sector_bytes_per_step", "l2_tbps", "l2_frac_of_lts_cap", "l2_note"):
        if k in kd:
            roofline[k] = kd[k]
    # the finest-level M2L against the reference's own FLOP count (8(a) a8):
    # a speed ratio only -- the separable form executes ~1/60 of these FLOPs
    m2l_keys = [k for k in prof if k.startswith("m2l_sep_") or k == f"m2l_tc_L{CFG['levels']}"]
    m2l_ms = sum(prof[k][0] for k in m2l_keys) / args.steps
    pairs = m2l_pairs(eng.m2l_tables["far"][CFG["levels"]]) + m2l_pairs(eng.m2l_tables["near"])
    flops_exp = pairs * 1 * eng.P * eng.P * 2
    m2l_line = {"kernels": sorted(m2l_keys), "ms_per_step": m2l_ms,
                "reference_flops_per_expansion": flops_exp,
                "reference_equivalent_tflops": 2 * flops_exp / (m2l_ms / 1000.0) / 1e12,
                "executed_flops_per_expansion": 2 * sep_ffma_per_cell(eng.rho) * (
                    2 ** (CFG["levels"] + 1)) ** 3 if eng.separable else None,
                "algorithm": ("separable: per-axis transforms + three 1-D convolutions "
                              "(FFMA -- see roofline_stages.m2l_finest)"
                              if eng.separable else
                              "dense tcgen05 kind::f16 two-term split")}
    stages = {k: round(v[0] / args.steps, 4) for k, v in sorted(prof.items())}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "step_statistic": "median of the K steps",
        "ms_per_step_mean": ms_mean, "ms_per_step_max": float(max(per_step)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "N": N, "M": M, "levels": CFG["levels"],
                   "rho": CFG["rho"], "alpha": CFG["alpha"],
                   "l2": "inputs 176 MB > 126 MB L2, and a 256 MB L2 flush between steps",
                   "parallelism": f"dp{world}" + (" (grid all-reduce, NCCL)" if world > 1 else "")},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "ms_per_step_mean": e2e_mean},
        "gpu_launches": int(launches),
        "roofline": roofline,
        "roofline_dominant_stage": roofline_stage,
        "roofline_kernels": rl_kernels,
        "roofline_stages": rl_stages,
        "m2l_finest_vs_reference_flops": m2l_line,
        "stages_ms_per_step": stages,
        "ms_per_step_instrumented": ms_instr,
        "graphed": graphed,
        "table_fit_s": t_tables,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_secondary and not args.small:
        line["secondary"] = secondary(dev, flush, stream, args.steps)
        line["training"] = training_lines(dev, flush, stream, args.steps)
    if not args.no_cpu_baseline and not args.small and world == 1:
        cb = cpu_sample(4, 1, N, M, CFG["seed"])
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                   "cpu_model")}
    print(json.dumps(line), flush=True)


def run_scaling(args, rank: int, world: int) -> None:
    """BASELINE config 5 as strong scaling: the global problem (N = 2^24
    sources, M = 2^27 queries) is split over the ranks; every expansion runs
    the sharded cascade (parallel.py: reduce-scatter into x-slabs, 3-plane
    halos, slab M2M / M2L / L2L at every level, all-gathers).  value =
    (N + M) / max over ranks of the device time per step."""
    import torch
    import torch.distributed as dist

    from paper_2111_00110_b200 import Engine, KernelModel, SourceSet, _lib
    from paper_2111_00110_b200.layers import explicit_forward, explicit_jvp
    from paper_2111_00110_b200.parallel import DeviceBackend, shard_range, sharded, slab_range

    local = _local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    C5 = dict(CFG5)
    if args.small:
        C5.update(N=1 << 18, M=1 << 21)
    N, M = C5["N"], C5["M"]
    eng = Engine(KernelModel("gaussian", C5["alpha"], C5["rho"]), C5["levels"],
                 check_admissibility=False)
    _ = eng.handle
    a, b = shard_range(N, rank, world)
    c, d = shard_range(M, rank, world)
    gen = torch.Generator(device=dev).manual_seed(C5["seed"] * 1000 + rank)
    one = 0.99999994
    P = torch.rand(b - a, 3, device=dev, generator=gen) * (2 * one) - one
    W = torch.randn(b - a, 1, device=dev, generator=gen) * 0.1
    Q = torch.rand(d - c, 3, device=dev, generator=gen) * (2 * one) - one
    YB = torch.randn(d - c, 1, device=dev, generator=gen)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    res = 2 ** (C5["levels"] + 1)
    sl = slab_range(res, rank, world)
    split = world == 1 or (sl is not None and DeviceBackend(eng).slab_split_ok(*sl))

    def step(p, w, q, yb):
        with sharded(eng):
            r = explicit_forward(eng, SourceSet(p, w), q)
            return explicit_jvp(yb, r), r

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(P, W, Q, YB)
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    gc.collect()
    gc.disable()
    with Clocks(local) as clk:
        barrier()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(stream)
            step(P, W, Q, YB)
            ev[i][1].record(stream)
        barrier()
    gc.enable()
    launches = (_lib.launch_count() - launches0) // args.steps
    per = [a_.elapsed_time(b_) for a_, b_ in ev]
    ms = float(np.median(per)) * args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    # e2e: this rank's shard in pinned host memory through the public API
    hp, hw, hq, hy = (t.cpu().pin_memory() for t in (P, W, Q, YB))
    del P, W, Q, YB
    torch.cuda.empty_cache()

    def step_host():
        g, r = step(hp.to(dev, non_blocking=True), hw.to(dev, non_blocking=True),
                    hq.to(dev, non_blocking=True), hy.to(dev, non_blocking=True))
        outs = [x.to("cpu", non_blocking=True) for x in (r.values, g.w_bar, g.p_bar, g.q_bar)]
        torch.cuda.synchronize()
        return outs
    outs = step_host()
    h2d = sum(x.numel() * 4 for x in (hp, hw, hq, hy))
    d2h = sum(o.numel() * 4 for o in outs)
    del outs
    barrier()
    k = max(2, args.steps // 4)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    te0 = time.perf_counter()
    e0.record(stream)
    for _ in range(k):
        step_host()
    e1.record(stream)
    barrier()
    e2e_ms = max(e0.elapsed_time(e1), 1000.0 * (time.perf_counter() - te0)) / k
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": (N + M) / (ms_step / 1000.0), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "step_statistic": "median of the K steps (max over ranks)",
        "ms_per_step_mean_rank0": float(np.mean(per)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD5, "N": N, "M": M, "levels": C5["levels"],
                   "rho": C5["rho"], "alpha": C5["alpha"],
                   "l2": "inputs 2.4 GB > 126 MB L2, and a 256 MB L2 flush between steps",
                   "parallelism": (f"dp{world}: reduce-scatter + 3-plane halo + slab cascade "
                                   f"at every level + all-gathers "
                                   f"({dist.get_backend().upper() if world > 1 else 'single GPU'})"),
                   "slab_cascade_no_replication": bool(split)},
        "e2e": {"value": (N + M) / (e2e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "note": "rank 0's shard bytes; every rank moves its own shard"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def _local_device() -> int:
    """This rank's GPU: LOCAL_RANK, or LOCAL_RANK modulo the visible GPUs when
    more ranks than GPUs run (functional check of the sharded path only)."""
    import torch
    local = int(os.environ.get("LOCAL_RANK", 0))
    n = torch.cuda.device_count()
    return local % n if n else local


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if args.impl == "ours":
            import torch
            torch.cuda.set_device(_local_device())
            # one process per GPU over NCCL (NVLink); with fewer GPUs than ranks
            # (a functional check on one GPU) gloo stages through the host
            dist.init_process_group("nccl" if torch.cuda.device_count() >= world else "gloo")
        else:
            dist.init_process_group("gloo")
    try:
        if args.impl == "reference":
            run_reference(args, rank)
        elif world > 1 or args.config == 5:
            run_scaling(args, rank, world)
        else:
            run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
