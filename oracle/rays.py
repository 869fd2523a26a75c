"""CPU oracle for the ray layers -- TEST INFRASTRUCTURE ONLY.

Float64 NumPy restatement of the reference's cameras, traversal, line
restriction, closed-form roots and the root-implicit / integral-implicit
layers (reference ray.py, poly1d.py, layers.py:55-544).  Same import rules as
fc2t2_oracle.py: tests / smoke / bench cpu leg only.  Pinned against the
reference by tests/test_oracle_golden.py (golden vectors from
tests/golden/make_golden.py).
"""

from __future__ import annotations

import math

import numpy as np

from .fc2t2_oracle import Oracle, box_centers, find_box, monos, res_of

MIN_SEGMENT = 1e-12          # ray.py:23
LEADING_EPS = 1e-12          # poly1d.py:19
EXP_CUTOFF = 4.5             # poly1d.py:22
EXP_FIT_RANGE = 5.0          # poly1d.py:23
IFT_DENOM_RTOL = 1e-8        # layers.py:39
ROOT_BOUNDARY_EPS = 1e-10    # layers.py:40


# ---------------------------------------------------------------- cameras ---

def camera_rays(position, look_at, up, fov_deg, width, height):
    """Pinhole rays through pixel centres, row-major (ray.py:42-48, :63-77)."""
    pos = np.asarray(position, dtype=np.float64)
    fwd = np.asarray(look_at, dtype=np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    tan = np.tan(np.radians(fov_deg) / 2.0)
    aspect = width / height
    xs = (np.arange(width) + 0.5) / width * 2.0 - 1.0
    ys = (np.arange(height) + 0.5) / height * 2.0 - 1.0
    gy, gx = np.meshgrid(ys, xs, indexing="ij")
    dirs = (fwd[None, :] + gx.reshape(-1, 1) * (tan * aspect) * right[None, :]
            + gy.reshape(-1, 1) * tan * down[None, :])
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return np.broadcast_to(pos, dirs.shape).copy(), dirs


# -------------------------------------------------------------- traversal ---

def span(o, d):
    """Slab test (ray.py:101-120)."""
    with np.errstate(divide="ignore", invalid="ignore"):
        lo = (-1.0 - o) / d
        hi = (1.0 - o) / d
    near = np.where(np.isnan(lo), -np.inf, np.minimum(lo, hi))
    far = np.where(np.isnan(hi), np.inf, np.maximum(lo, hi))
    par = d == 0.0
    inside = np.abs(o) < 1.0
    near = np.where(par, np.where(inside, -np.inf, np.inf), near)
    far = np.where(par, np.where(inside, np.inf, -np.inf), far)
    return np.maximum(near.max(axis=1), 0.0), far.min(axis=1)


def traverse(o, d, level):
    """Per-box segments (ray.py:123-157): dict ray_id, t0, t1, box, offsets."""
    res = res_of(level)
    R = o.shape[0]
    t_in, t_out = span(o, d)
    hit = t_in < t_out
    planes = -1.0 + (2.0 / res) * np.arange(res + 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        ts = (planes[None, None, :] - o[:, :, None]) / d[:, :, None]
    ts = ts.reshape(R, -1)
    ts = np.where(np.isfinite(ts), ts, np.inf)
    ts = np.where((ts > t_in[:, None]) & (ts < t_out[:, None]), ts, t_out[:, None])
    ts.sort(axis=1)
    b = np.concatenate([t_in[:, None], ts, t_out[:, None]], axis=1)
    st, en = b[:, :-1], b[:, 1:]
    keep = (en - st > MIN_SEGMENT) & hit[:, None]
    ray = np.broadcast_to(np.arange(R)[:, None], keep.shape)[keep]
    t0, t1 = st[keep], en[keep]
    mid = o[ray] + 0.5 * (t0 + t1)[:, None] * d[ray]
    mid = np.clip(mid, -1.0 + 1e-15, 1.0 - 1e-15)
    box = find_box(level, mid)
    offs = np.concatenate([[0], np.cumsum(np.bincount(ray, minlength=R))])
    return {"ray_id": ray, "t0": t0, "t1": t1, "box": box, "offsets": offs,
            "t_enter": np.where(hit, t_in, np.nan)}


def seg_geometry(trav, o, d, level):
    """(d, r, s) per segment (ray.py:249-258)."""
    oo, rr = o[trav["ray_id"]], d[trav["ray_id"]]
    base = oo + trav["t0"][:, None] * rr
    return base - box_centers(level, trav["box"]), rr, trav["t1"] - trav["t0"]


# ----------------------------------------------------------- 1D polynomials ---

def peval(c, x):
    """Ascending Horner (poly1d.py:30-37); rows when c is 2-D (layers.py:70-75)."""
    c = np.asarray(c, dtype=np.float64)
    if c.ndim == 1:
        y = np.zeros_like(np.asarray(x, dtype=np.float64))
        for v in c[::-1]:
            y = y * x + v
        return y
    y = np.zeros(c.shape[0])
    for v in c.T[::-1]:
        y = y * x + v
    return y


def pmul(a, b):
    """Row-wise products (layers.py:55-60)."""
    out = np.zeros((a.shape[0], a.shape[1] + b.shape[1] - 1))
    for i in range(a.shape[1]):
        out[:, i:i + b.shape[1]] += a[:, i:i + 1] * b
    return out


def pint(a):
    """Row-wise antiderivative, zero constant (layers.py:63-66)."""
    out = np.zeros((a.shape[0], a.shape[1] + 1))
    out[:, 1:] = a / np.arange(1, a.shape[1] + 1)[None, :]
    return out


def pcompose(outer, g):
    """Rows of outer(g(x)), Horner in g (layers.py:77-83)."""
    out = np.full((g.shape[0], 1), outer[-1])
    for c in outer[-2::-1]:
        out = pmul(out, g)
        out[:, 0] += c
    return out


def exp_fit():
    """Degree-4 fit of exp(-x) on [0, 5] with value 1 at 0 (poly1d.py:224-242)."""
    k = np.arange(64)
    x = 2.5 + 2.5 * np.cos((2 * k + 1) * np.pi / 128)
    V = x[:, None] ** np.arange(1, 5)[None, :]
    tail, *_ = np.linalg.lstsq(V, np.exp(-x) - 1.0, rcond=None)
    return np.concatenate([[1.0], tail])


def mexp(x):
    """Fitted exp(-x), 0 beyond the fit range (poly1d.py:251-255)."""
    x = np.asarray(x, dtype=np.float64)
    return np.where(x > EXP_FIT_RANGE, 0.0, peval(exp_fit(), x))


# ----------------------------------------------------------------- roots ---

def _quad(a2, a1, a0):
    disc = a1 * a1 - 4.0 * a2 * a0
    if disc < 0.0:
        return []
    if disc == 0.0:
        return [-a1 / (2.0 * a2)]
    sq = math.sqrt(disc)
    q = -0.5 * (a1 + math.copysign(sq, a1))
    return [q / a2, a0 / q if q != 0.0 else -a1 / (2.0 * a2)]


def _cubic(a3, a2, a1, a0):
    b, c, d = a2 / a3, a1 / a3, a0 / a3
    sh = b / 3.0
    p = c - b * b / 3.0
    q = 2.0 * b ** 3 / 27.0 - b * c / 3.0 + d
    disc = (q / 2.0) ** 2 + (p / 3.0) ** 3
    if disc > 0.0:
        s = math.sqrt(disc)
        u = math.copysign(abs(-q / 2.0 + s) ** (1.0 / 3.0), -q / 2.0 + s)
        v = math.copysign(abs(-q / 2.0 - s) ** (1.0 / 3.0), -q / 2.0 - s)
        r = [u + v]
    elif disc == 0.0:
        if q == 0.0:
            r = [0.0]
        else:
            u = math.copysign(abs(q / 2.0) ** (1.0 / 3.0), q / 2.0)
            r = [-2.0 * u, u]
    else:
        m = 2.0 * math.sqrt(-p / 3.0)
        th = math.acos(max(-1.0, min(1.0, 3.0 * q / (p * m)))) / 3.0
        r = [m * math.cos(th - 2.0 * math.pi * k / 3.0) for k in range(3)]
    return [x - sh for x in r]


def _quartic(a4, a3, a2, a1, a0):
    b, c, d, e = a3 / a4, a2 / a4, a1 / a4, a0 / a4
    sh = b / 4.0
    p = c - 3.0 * b * b / 8.0
    q = d - b * c / 2.0 + b ** 3 / 8.0
    r = e - b * d / 4.0 + b * b * c / 16.0 - 3.0 * b ** 4 / 256.0
    ys = []
    if abs(q) < LEADING_EPS * max(1.0, abs(p), abs(r)):
        for z in _quad(1.0, p, r):
            if z > 0.0:
                ys += [math.sqrt(z), -math.sqrt(z)]
            elif z == 0.0:
                ys.append(0.0)
        return [y - sh for y in ys]
    z = max(_cubic(1.0, -p, -4.0 * r, 4.0 * p * r - q * q))
    s = math.sqrt(max(z - p, 0.0))
    if s == 0.0:
        for z2 in _quad(1.0, 0.0, r):
            if z2 > 0:
                ys += [math.sqrt(z2), -math.sqrt(z2)]
            elif z2 == 0:
                ys.append(0.0)
    else:
        t = q / (2.0 * s)
        ys += _quad(1.0, s, z / 2.0 - t) + _quad(1.0, -s, z / 2.0 + t)
    return [y - sh for y in ys]


def quartic_roots(coeffs, tol=1e-9):
    """Real roots of a degree <= 4 polynomial (poly1d.py:185-218)."""
    c = np.zeros(5)
    c[:len(coeffs)] = coeffs
    scale = np.max(np.abs(c))
    if scale == 0.0:
        raise ValueError("zero polynomial")
    deg = 4
    while deg > 0 and abs(c[deg]) < LEADING_EPS * scale:
        deg -= 1
    if deg == 0:
        return np.empty(0)
    raw = {1: lambda: ([] if c[1] == 0.0 else [-c[0] / c[1]]),
           2: lambda: _quad(c[2], c[1], c[0]),
           3: lambda: _cubic(c[3], c[2], c[1], c[0]),
           4: lambda: _quartic(c[4], c[3], c[2], c[1], c[0])}[deg]()
    cc = c[:deg + 1]
    dc = cc[1:] * np.arange(1, deg + 1)
    pol = []
    for x in raw:
        fx, dfx = float(peval(cc, x)), float(peval(dc, x))
        if dfx != 0.0 and math.isfinite(dfx):
            st = fx / dfx
            if math.isfinite(st):
                x = x - st
        pol.append(x)
    out = []
    for x in sorted(pol):
        if not out or abs(x - out[-1]) > tol * max(1.0, abs(x)):
            out.append(x)
    return np.array(out)


# ------------------------------------------------------------- line2poly ---

def line2poly(coeffs, dd, rr, rho):
    """Exact restriction to x = d + t r (ray.py:184-210, Chebyshev values @ inverse Vandermonde)."""
    from .fc2t2_oracle import mi_entries
    ent = mi_entries(rho)
    u = np.cos(np.pi * np.arange(rho + 1) / rho)
    vinv = np.linalg.inv(u[:, None] ** np.arange(rho + 1)[None, :])
    S, C = coeffs.shape[0], coeffs.shape[1]
    out = np.empty((S, C, rho + 1))
    for lo in range(0, S, 65536):
        hi = min(lo + 65536, S)
        pts = dd[lo:hi, None, :] + u[None, :, None] * rr[lo:hi, None, :]
        mono = monos(ent, pts.reshape(-1, 3)).reshape(hi - lo, rho + 1, -1)
        out[lo:hi] = np.einsum("scp,sgp->scg", coeffs[lo:hi], mono) @ vinv.T
    return out


def line2taylor_h(dd, rr, s, h, rho):
    """Segment moments with polynomial weight h (ray.py:221-246), Gauss-Legendre exact."""
    from .fc2t2_oracle import mi_entries
    ent = mi_entries(rho)
    S, H = h.shape
    G = (rho + H - 1) // 2 + 1
    x, gw = np.polynomial.legendre.leggauss(G)
    out = np.empty((S, ent.shape[0]))
    for lo in range(0, S, 65536):
        hi = min(lo + 65536, S)
        half = 0.5 * s[lo:hi]
        t = half[:, None] * (x[None, :] + 1.0)
        hv = np.zeros_like(t)
        for mu in range(H - 1, -1, -1):
            hv = hv * t + h[lo:hi, mu:mu + 1]
        pts = dd[lo:hi, None, :] + t[..., None] * rr[lo:hi, None, :]
        mono = monos(ent, pts.reshape(-1, 3)).reshape(hi - lo, G, -1)
        out[lo:hi] = np.einsum("sgp,sg->sp", mono, hv * (half[:, None] * gw[None, :]))
    return out


# ------------------------------------------------------------------ layers ---

class RayOracle:
    """Root-implicit and integral-implicit layers (layers.py:193-544) on an Oracle."""

    def __init__(self, ora: Oracle):
        self.o = ora

    def _segments(self, L, o, d):
        tr = traverse(o, d, self.o.levels)
        dd, rr, s = seg_geometry(tr, o, d, self.o.levels)
        co = L[tr["box"][:, 0], tr["box"][:, 1], tr["box"][:, 2]]
        return tr, dd, rr, s, line2poly(co, dd, rr, self.o.rho)

    def first_root(self, polys, tr, bias, R):
        """layers.py:208-241."""
        a = polys[:, 0, :].copy()
        a[:, 0] += bias
        s = tr["t1"] - tr["t0"]
        smp = np.stack([peval(a, s * f) for f in (0.0, 0.25, 0.5, 0.75, 1.0)], axis=1)
        cand = smp.min(axis=1) <= 0.0
        lengths = np.full(R, np.nan)
        hit = np.zeros(R, bool)
        entry = np.zeros(R, bool)
        has = np.diff(tr["offsets"]) > 0
        entry[has] = a[tr["offsets"][:-1][has], 0] > 0.0
        for i in np.flatnonzero(cand):
            ray = tr["ray_id"][i]
            if hit[ray] or not entry[ray]:
                continue
            rt = quartic_roots(a[i]) if np.any(a[i]) else np.empty(0)
            rt = rt[(rt >= -ROOT_BOUNDARY_EPS) & (rt <= s[i] + ROOT_BOUNDARY_EPS)]
            if rt.size:
                lengths[ray] = tr["t0"][i] + float(np.clip(rt.min(), 0.0, s[i]))
                hit[ray] = True
        return lengths, hit

    def depth_forward(self, p, w, o, d, bias):
        """layers.py:244-272: dict of lengths, hit, points, grads, denom, L, trav."""
        L = self.o.expand(p, w)
        tr, dd, rr, s, polys = self._segments(L, o, d)
        lengths, hit = self.first_root(polys, tr, bias, o.shape[0])
        pts = np.zeros((o.shape[0], 3))
        grads = np.zeros((o.shape[0], 3))
        den = np.zeros(o.shape[0])
        if hit.any():
            pts[hit] = o[hit] + lengths[hit][:, None] * d[hit]
            grads[hit] = self.o.evaluate(L, pts[hit], what="grad")[:, 0, :]
            den[hit] = np.einsum("ra,ra->r", d[hit], grads[hit])
        return {"lengths": lengths, "hit": hit, "points": pts, "grads": grads, "denom": den,
                "L": L, "trav": tr}

    def _back(self, B, p, w):
        w = np.asarray(w, dtype=np.float64).reshape(p.shape[0], -1)
        return self.o.evaluate(B, p), np.einsum("nc,nca->na", w, self.o.evaluate(B, p, what="grad"))

    def depth_jvp(self, yb, fw, p, w):
        """layers.py:275-303."""
        h = fw["hit"]
        g = fw["grads"][h]
        den = fw["denom"][h]
        bad = np.abs(den) < IFT_DENOM_RTOL * np.maximum(np.linalg.norm(g, axis=1), 1e-300)
        u = np.where(bad, 0.0, -np.asarray(yb).reshape(-1)[h] / np.where(bad, 1.0, den))
        B = self.o.expand(fw["points"][h], u[:, None])
        return self._back(B, p, w)

    def surface_jvp(self, yb, fw, p, w, d):
        """layers.py:313-356 (monopole + dipole payload, one expansion)."""
        h = fw["hit"]
        pts = fw["points"][h]
        rd = d[h]
        h2 = self.o.evaluate(fw["L"], pts, what="hess")[:, 0, :]
        H = np.empty((pts.shape[0], 3, 3))
        H[:, 0, 0], H[:, 1, 1], H[:, 2, 2] = h2[:, 0], h2[:, 1], h2[:, 2]
        H[:, 0, 1] = H[:, 1, 0] = h2[:, 3]
        H[:, 0, 2] = H[:, 2, 0] = h2[:, 4]
        H[:, 1, 2] = H[:, 2, 1] = h2[:, 5]
        num = np.einsum("ria,ra->ri", H, rd)
        den = fw["denom"][h]
        bad = np.abs(den) < IFT_DENOM_RTOL * np.maximum(np.linalg.norm(fw["grads"][h], axis=1), 1e-300)
        kap = np.where(bad[:, None], 0.0, num / np.where(bad, 1.0, den)[:, None])
        ybh = np.asarray(yb)[h]
        mu = -np.einsum("ri,ri->r", ybh, kap)
        lev = self.o.levels
        box = find_box(lev, pts)
        mono = monos(self.o.e, pts - box_centers(lev, box))
        pay = mu[:, None] * mono
        for j, n in enumerate(self.o.e):
            for a in range(3):
                if n[a] >= 1:
                    lowr = tuple(int(n[k]) - (k == a) for k in range(3))
                    pay[:, j] += ybh[:, a] * mono[:, self.o.lookup[lowr]]
        B = self.o.cascade(self.o.insert(box, pay[:, None, :]))
        return self._back(B, p, w)

    def line_integral(self, p, w, o, d):
        """layers.py:371-386."""
        L = self.o.expand(p, w)
        tr, dd, rr, s, polys = self._segments(L, o, d)
        R, C = o.shape[0], polys.shape[1]
        vals = np.zeros((R, C))
        for c in range(C):
            vals[:, c] = np.bincount(tr["ray_id"], weights=peval(pint(polys[:, c, :]), s),
                                     minlength=R)
        return vals, tr

    def line_integral_jvp(self, yb, tr, p, w, o, d):
        """layers.py:389-402."""
        dd, rr, s = seg_geometry(tr, o, d, self.o.levels)
        mom = line2taylor_h(dd, rr, s, np.ones((s.shape[0], 1)), self.o.rho)
        yb = np.asarray(yb).reshape(o.shape[0], -1)
        B = self.o.cascade(self.o.insert(tr["box"], yb[tr["ray_id"]][:, :, None] * mom[:, None, :]))
        return self._back(B, p, w)

    def volumetric(self, p, w_sigma, w_color, o, d, bg):
        """layers.py:427-480; returns rgb and the caches of the JVP."""
        w_sigma = np.asarray(w_sigma, dtype=np.float64).reshape(-1, 1)
        w_color = np.asarray(w_color, dtype=np.float64)
        C = w_color.shape[1]
        L = self.o.expand(p, np.concatenate([np.maximum(w_sigma, 0.0), w_color], axis=1))
        tr, dd, rr, s, polys = self._segments(L, o, d)
        R = o.shape[0]
        sigma = polys[:, 0, :]
        sa = pint(sigma)
        send = peval(sa, s)
        ce = np.cumsum(send) - send
        depth0 = ce - ce[tr["offsets"][:-1][tr["ray_id"]]]
        alive = depth0 <= EXP_CUTOFF
        dfin = np.bincount(tr["ray_id"], weights=np.where(alive, send, 0.0), minlength=R)
        sig_a, col_a = sigma[alive], polys[alive][:, 1:, :]
        saa = sa[alive].copy()
        saa[:, 0] += depth0[alive]
        trans = pcompose(exp_fit(), saa)
        ray_a, s_a = tr["ray_id"][alive], s[alive]
        rgb = np.zeros((R, C))
        anti = np.zeros((alive.sum(), C, trans.shape[1] + 2 * self.o.rho + 1))
        for c in range(C):
            a = pint(pmul(pmul(col_a[:, c, :], sig_a), trans))
            anti[:, c, :] = a
            rgb[:, c] = np.bincount(ray_a, weights=peval(a, s_a), minlength=R)
        rgb += mexp(dfin)[:, None] * np.asarray(bg, dtype=np.float64)[None, :]
        return rgb, {"trav": tr, "alive": alive, "sigma": sig_a, "color": col_a, "trans": trans,
                     "depth0": depth0, "anti": anti, "dfin": dfin, "w_sigma": w_sigma,
                     "w_color": w_color, "bg": np.asarray(bg, dtype=np.float64)}

    def volumetric_jvp(self, yb, cache, p, o, d):
        """layers.py:483-544."""
        tr, alive = cache["trav"], cache["alive"]
        C = cache["w_color"].shape[1]
        dd, rr, s = seg_geometry(tr, o, d, self.o.levels)
        da, ra, sa_ = dd[alive], rr[alive], s[alive]
        ray_a = tr["ray_id"][alive]
        yb = np.asarray(yb, dtype=np.float64)
        ya = yb[ray_a]
        fit = exp_fit()
        dm = fit[1:] * np.arange(1, 5)
        sig_anti = pint(cache["sigma"])
        sig_anti[:, 0] += cache["depth0"][alive]
        tprime = pcompose(dm, sig_anti)
        tp_inf = np.where(cache["dfin"] > EXP_FIT_RANGE, 0.0, peval(dm, cache["dfin"]))
        dim = cache["anti"].shape[2]
        hs = np.zeros((alive.sum(), dim))
        R = o.shape[0]
        for c in range(C):
            tc = pmul(cache["trans"], cache["color"][:, c, :])
            hs[:, :tc.shape[1]] += ya[:, c:c + 1] * tc
            ap = pint(pmul(pmul(cache["color"][:, c, :], cache["sigma"]), tprime))
            cp = peval(ap, sa_)
            tot = np.bincount(ray_a, weights=cp, minlength=R)
            ce = np.cumsum(cp) - cp
            first = np.concatenate([[True], ray_a[1:] != ray_a[:-1]]) if ray_a.size else np.zeros(0, bool)
            run = np.cumsum(first) - 1
            before = ce - ce[np.flatnonzero(first)][run] if ray_a.size else ce
            hs[:, :ap.shape[1]] -= ya[:, c:c + 1] * ap
            hs[:, 0] += ya[:, c] * (tot[ray_a] - before + tp_inf[ray_a] * cache["bg"][c])
        ins = np.empty((alive.sum(), 1 + C, self.o.P))
        ins[:, 0, :] = line2taylor_h(da, ra, sa_, hs, self.o.rho)
        tsig = pmul(cache["trans"], cache["sigma"])
        for c in range(C):
            ins[:, 1 + c, :] = line2taylor_h(da, ra, sa_, ya[:, c:c + 1] * tsig, self.o.rho)
        B = self.o.cascade(self.o.insert(tr["box"][alive], ins))
        val = self.o.evaluate(B, p)
        grad = self.o.evaluate(B, p, what="grad")
        ws = cache["w_sigma"][:, 0]
        wsb = (ws > 0.0).astype(np.float64) * val[:, 0]
        p_bar = (np.maximum(cache["w_sigma"], 0.0) * grad[:, 0, :]
                 + np.einsum("nc,nca->na", cache["w_color"], grad[:, 1:, :]))
        return np.concatenate([wsb[:, None], val[:, 1:]], axis=1), p_bar
