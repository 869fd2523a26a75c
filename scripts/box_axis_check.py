"""CPU sweep: the float32 box_axis / box_offset (csrc/common.cuh) against the
float64 forms (reference expansion.py:85-93) on random, extreme and one-ulp
boundary inputs at res = 4..512.  Emulates the float32 steps with numpy."""
import numpy as np
rng = np.random.default_rng(0)
def ref_axis(x, res):
    s = x.astype(np.float64) + 1.0
    with np.errstate(invalid="ignore"):
        b = np.floor(s * (0.5 * res))
        b = np.where(np.isnan(b), 0, b)
    return np.clip(b, 0, res - 1).astype(np.int64)
def f_axis(x, res):
    h = np.float32(res // 2)
    xs = np.where(x >= np.float32(-2.0**-54), np.maximum(x, np.float32(0)), x).astype(np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        y = xs * h
    y = np.fmax(y, -h)  # fmaxf semantics: NaN -> other
    y = np.minimum(y, h - 1)
    # __fadd_rd(y, 1.5*2^23): exact floor(y) + magic
    t = np.floor(y.astype(np.float64)).astype(np.int64)
    return t + res // 2
def ref_off(x, b, res):
    c = -1.0 + (b.astype(np.float64) + 0.5) * (2.0 / res)
    return (x.astype(np.float64) - c).astype(np.float32)
def f_off(x, b, res):
    c = (2 * b + 1 - res).astype(np.float32) * np.float32(1.0 / res)
    return (x - c).astype(np.float32)
bad = 0
for res in [4, 8, 16, 32, 64, 128, 256, 512]:
    parts = [rng.uniform(-1, 1, 2_000_000).astype(np.float32),
             (rng.standard_normal(200000) * 10.0 ** rng.integers(-45, 39, 200000)).astype(np.float32),
             np.array([0.0, -0.0, 1.0, -1.0, np.inf, -np.inf, np.nan, 2.0**-54, -2.0**-54, -2.0**-55,
                       -2.0**-53, -1e-45, 1e-45, -1e-30, 3e38, -3e38], np.float32)]
    planes = (np.arange(res + 1) / (res / 2) - 1).astype(np.float32)
    parts += [planes, np.nextafter(planes, np.float32(2)), np.nextafter(planes, np.float32(-2))]
    x = np.concatenate(parts)
    a, b = ref_axis(x, res), f_axis(x, res)
    m = a != b
    bad += m.sum()
    if m.any(): print(res, x[m][:10], a[m][:10], b[m][:10])
    fin = np.isfinite(x)
    o1, o2 = ref_off(x[fin], a[fin], res), f_off(x[fin], a[fin], res)
    mm = (o1.view(np.int32) != o2.view(np.int32))
    bad += mm.sum()
    if mm.any(): print("off", res, x[fin][mm][:5], o1[mm][:5], o2[mm][:5])
print("mismatches", bad)
