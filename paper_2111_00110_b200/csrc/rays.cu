// Ray kernels of the root-implicit and integral-implicit layers.
//
// One thread walks one ray through the finest grid (reference ray.py:101-157):
// float64 slab test, the 3(res+1) plane crossings merged in order (every
// per-axis sequence is monotone, so a 3-way merge equals np.sort), segments
// shorter than 1e-12 dropped, box = find_box of the clipped midpoint -- the
// same float64 operations in the same order as the reference, so the box
// lists are bit-exact.  Per segment the cell polynomial is restricted to the
// ray (line2poly, reference ray.py:184-210) by the exact per-axis binomial
// expansion instead of Chebyshev interpolation (both are exact; SURVEY 8(a)
// note 6) and consumed on the fly: no per-segment arrays unless a backward
// insertion needs them.
#include <math_constants.h>

#include "common.cuh"
#include "kernels.cuh"
#include "raywalk.cuh"

namespace fc2t2 {

namespace {

using namespace ray;

__global__ void traverse_count_kernel(const double* __restrict__ org,
                                      const double* __restrict__ dir, int64_t R, int res,
                                      uint32_t* __restrict__ counts) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    counts[r] = (uint32_t)walk_ray(o, d, res, [](double, double, int, int, int) { return true; });
  }
}

__global__ void traverse_fill_kernel(const double* __restrict__ org, const double* __restrict__ dir,
                                     int64_t R, int res, const uint32_t* __restrict__ offsets,
                                     int32_t* __restrict__ ray_id, double* __restrict__ t0,
                                     double* __restrict__ t1, int32_t* __restrict__ box) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    int64_t i = offsets[r];
    walk_ray(o, d, res, [&](double a, double b, int x, int y, int z) {
      ray_id[i] = (int32_t)r;
      t0[i] = a;
      t1[i] = b;
      box[3 * i] = x;
      box[3 * i + 1] = y;
      box[3 * i + 2] = z;
      ++i;
      return true;
    });
  }
}

// --------------------------------------------------------------- roots ---
// Closed-form real roots for degree <= 4 + one Newton polish, sorted and
// de-duplicated (reference poly1d.py:99-218), float64.
__device__ __forceinline__ int roots_quadratic(double a2, double a1, double a0, double* r) {
  const double disc = a1 * a1 - 4.0 * a2 * a0;
  if (disc < 0.0) return 0;
  if (disc == 0.0) {
    r[0] = -a1 / (2.0 * a2);
    return 1;
  }
  const double sq = sqrt(disc);
  const double q = -0.5 * (a1 + copysign(sq, a1));
  r[0] = q / a2;
  r[1] = q != 0.0 ? a0 / q : -a1 / (2.0 * a2);
  return 2;
}

__device__ __forceinline__ int roots_cubic(double a3, double a2, double a1, double a0, double* r) {
  const double b = a2 / a3, c = a1 / a3, d = a0 / a3;
  const double sh = b / 3.0;
  const double p = c - b * b / 3.0;
  const double q = 2.0 * b * b * b / 27.0 - b * c / 3.0 + d;
  const double disc = (q / 2.0) * (q / 2.0) + (p / 3.0) * (p / 3.0) * (p / 3.0);
  int n;
  if (disc > 0.0) {
    const double s = sqrt(disc);
    const double u = copysign(pow(fabs(-q / 2.0 + s), 1.0 / 3.0), -q / 2.0 + s);
    const double v = copysign(pow(fabs(-q / 2.0 - s), 1.0 / 3.0), -q / 2.0 - s);
    r[0] = u + v;
    n = 1;
  } else if (disc == 0.0) {
    if (q == 0.0) {
      r[0] = 0.0;
      n = 1;
    } else {
      const double u = copysign(pow(fabs(q / 2.0), 1.0 / 3.0), q / 2.0);
      r[0] = -2.0 * u;
      r[1] = u;
      n = 2;
    }
  } else {
    const double m = 2.0 * sqrt(-p / 3.0);
    const double th = acos(fmax(-1.0, fmin(1.0, 3.0 * q / (p * m)))) / 3.0;
    for (int k = 0; k < 3; ++k) r[k] = m * cos(th - 2.0 * CUDART_PI * k / 3.0);
    n = 3;
  }
  for (int i = 0; i < n; ++i) r[i] -= sh;
  return n;
}

__device__ __forceinline__ int roots_quartic(double a4, double a3, double a2, double a1, double a0,
                                             double* r) {
  const double b = a3 / a4, c = a2 / a4, d = a1 / a4, e = a0 / a4;
  const double sh = b / 4.0;
  const double p = c - 3.0 * b * b / 8.0;
  const double q = d - b * c / 2.0 + b * b * b / 8.0;
  const double rr = e - b * d / 4.0 + b * b * c / 16.0 - 3.0 * b * b * b * b / 256.0;
  int n = 0;
  if (fabs(q) < LEADING_EPS * fmax(1.0, fmax(fabs(p), fabs(rr)))) {
    double z[2];
    const int nz = roots_quadratic(1.0, p, rr, z);
    for (int i = 0; i < nz; ++i) {
      if (z[i] > 0.0) {
        r[n++] = sqrt(z[i]);
        r[n++] = -sqrt(z[i]);
      } else if (z[i] == 0.0) {
        r[n++] = 0.0;
      }
    }
  } else {
    double zc[3];
    const int nc = roots_cubic(1.0, -p, -4.0 * rr, 4.0 * p * rr - q * q, zc);
    double z = zc[0];
    for (int i = 1; i < nc; ++i) z = fmax(z, zc[i]);
    const double s = sqrt(fmax(z - p, 0.0));
    if (s == 0.0) {
      double z2[2];
      const int nz = roots_quadratic(1.0, 0.0, rr, z2);
      for (int i = 0; i < nz; ++i) {
        if (z2[i] > 0.0) {
          r[n++] = sqrt(z2[i]);
          r[n++] = -sqrt(z2[i]);
        } else if (z2[i] == 0.0) {
          r[n++] = 0.0;
        }
      }
    } else {
      const double t = q / (2.0 * s);
      n += roots_quadratic(1.0, s, z / 2.0 - t, r + n);
      n += roots_quadratic(1.0, -s, z / 2.0 + t, r + n);
    }
  }
  for (int i = 0; i < n; ++i) r[i] -= sh;
  return n;
}

// all real roots of c[0] + c[1] x + ... + c[4] x^4, ascending; returns count
__device__ int quartic_roots(const double c[5], double* out) {
  double scale = 0.0;
  for (int i = 0; i < 5; ++i) scale = fmax(scale, fabs(c[i]));
  if (scale == 0.0) return 0;
  int deg = 4;
  while (deg > 0 && fabs(c[deg]) < LEADING_EPS * scale) --deg;
  double raw[4];
  int n = 0;
  if (deg == 0) return 0;
  if (deg == 1) {
    if (c[1] != 0.0) raw[n++] = -c[0] / c[1];
  } else if (deg == 2) {
    n = roots_quadratic(c[2], c[1], c[0], raw);
  } else if (deg == 3) {
    n = roots_cubic(c[3], c[2], c[1], c[0], raw);
  } else {
    n = roots_quartic(c[4], c[3], c[2], c[1], c[0], raw);
  }
  // one Newton step per root (poly1d.py:88-96)
  for (int i = 0; i < n; ++i) {
    double x = raw[i], fx = 0.0, dfx = 0.0;
    for (int k = deg; k >= 0; --k) fx = fx * x + c[k];
    for (int k = deg; k >= 1; --k) dfx = dfx * x + k * c[k];
    if (dfx != 0.0 && isfinite(dfx)) {
      const double st = fx / dfx;
      if (isfinite(st)) x = x - st;
    }
    raw[i] = x;
  }
  for (int i = 1; i < n; ++i)  // insertion sort
    for (int j = i; j > 0 && raw[j] < raw[j - 1]; --j) {
      const double t = raw[j];
      raw[j] = raw[j - 1];
      raw[j - 1] = t;
    }
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (m == 0 || fabs(raw[i] - out[m - 1]) > 1e-9 * fmax(1.0, fabs(raw[i]))) out[m++] = raw[i];
  return m;
}

__device__ __forceinline__ double horner(const double* c, int n, double x) {
  double y = 0.0;
  for (int k = n - 1; k >= 0; --k) y = y * x + c[k];
  return y;
}

// ----------------------------------------------------------- depth walk ---
// depth_forward (layers.py:244-272) fused with _first_root_per_ray (:208-241),
// the hit point, and the field gradient / Hessian at the hit (L2P, :261-267).
template <int RHO>
__global__ void __launch_bounds__(128)
depth_walk_kernel(const float* __restrict__ L, int res, const double* __restrict__ org,
                  const double* __restrict__ dir, int64_t R, double bias,
                  double* __restrict__ lengths, uint8_t* __restrict__ hit,
                  double* __restrict__ points, float* __restrict__ grads,
                  float* __restrict__ hess, float* __restrict__ denom) {
  constexpr MI<RHO> mi{};
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    const float dirf[3] = {(float)d[0], (float)d[1], (float)d[2]};
    bool found = false, first = true, entry_ok = false;
    double len = CUDART_NAN;
    walk_ray(o, d, res, [&](double t0, double t1, int b0, int b1, int b2) {
      float base[3];
      seg_base(o, d, t0, b0, b1, b2, res, base);
      const float* row = L + (((int64_t)b0 * res + b1) * res + b2) * PP;  // channel 0
      float pf[RHO + 1];
      line_poly<RHO>(row, base, dirf, pf);
      double a[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      for (int j = 0; j <= RHO && j < 5; ++j) a[j] = (double)pf[j];
      a[0] += bias;
      if (first) {
        first = false;
        entry_ok = a[0] > 0.0;  // dead-pixel rule (layers.py:225-228)
        if (!entry_ok) return false;
      }
      const double s = t1 - t0;
      double mn = CUDART_INF;
      const double fr[5] = {0.0, 0.25, 0.5, 0.75, 1.0};
      for (int k = 0; k < 5; ++k) mn = fmin(mn, horner(a, RHO + 1, s * fr[k]));
      if (!(mn <= 0.0)) return true;  // 5-sample candidate screen (:212-219)
      bool any = false;
      for (int j = 0; j <= RHO; ++j) any |= a[j] != 0.0;
      if (!any) return true;
      double rt[4];
      const int nr = quartic_roots(a, rt);
      for (int k = 0; k < nr; ++k)
        if (rt[k] >= -ROOT_BOUNDARY_EPS && rt[k] <= s + ROOT_BOUNDARY_EPS) {
          len = t0 + fmin(fmax(rt[k], 0.0), s);  // smallest in-range root
          found = true;
          return false;
        }
      return true;
    });
    lengths[r] = found ? len : CUDART_NAN;
    hit[r] = found ? 1 : 0;
    double pt[3] = {0.0, 0.0, 0.0};
    float g[3] = {0.f, 0.f, 0.f}, h[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, den = 0.f;
    if (found) {
      int b[3];
      float off[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        pt[k] = __dadd_rn(o[k], __dmul_rn(len, d[k]));
        b[k] = box_axis(pt[k], res);
        off[k] = (float)(pt[k] - (-1.0 + ((double)b[k] + 0.5) * (2.0 / (double)res)));
      }
      const float* row = L + (((int64_t)b[0] * res + b[1]) * res + b[2]) * PP;
      float a[PP];
#pragma unroll
      for (int k = 0; k < PP; k += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(row + k));
        a[k] = v.x; a[k + 1] = v.y; a[k + 2] = v.z; a[k + 3] = v.w;
      }
      float mono[P];
      monomials<RHO>(off[0], off[1], off[2], mono);
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        float acc = 0.f;
#pragma unroll
        for (int j = 0; j < P; ++j)
          if (mi.up[s][j] >= 0) acc = fmaf(a[mi.up[s][j]], mono[j], acc);
        if (s < 3) g[s] = acc; else h[s - 3] = acc;
      }
      den = dirf[0] * g[0] + dirf[1] * g[1] + dirf[2] * g[2];
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      points[3 * r + k] = pt[k];
      grads[3 * r + k] = g[k];
    }
    if (hess)
#pragma unroll
      for (int k = 0; k < 6; ++k) hess[6 * r + k] = h[k];
    denom[r] = den;
  }
}

// --------------------------------------------------- root JVP payloads ---
// Per hit ray: cell key and moment payload (layers.py:275-356).  depth:
// u = -y_len / <r, grad f> (0 where the IFT denominator is invalid) times the
// point moments; surface gradient: mu = -sum_i y_i kappa_i with
// kappa_i = <H_i, r> / <grad f, r>, plus the dipoles y_a * mono[n - e_a].
// Both share one insertion when both tangents are given.  Misses get the
// out-of-grid key res^3 (sorted last, inserted nowhere).
template <int RHO>
__global__ void __launch_bounds__(128)
root_payload_kernel(int res, const double* __restrict__ dir, int64_t R,
                    const uint8_t* __restrict__ hit, const double* __restrict__ points,
                    const float* __restrict__ grads, const float* __restrict__ hess,
                    const float* __restrict__ denom, const float* __restrict__ y_len,
                    const float* __restrict__ y_grad, uint32_t* __restrict__ keys,
                    float* __restrict__ payload, int32_t* __restrict__ n_clamped) {
  constexpr MI<RHO> mi{};
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  int clamped = 0;
  const uint32_t none = (uint32_t)res * res * res;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    float out[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) out[j] = 0.f;
    uint32_t key = none;
    if (hit[r]) {
      const float g0 = grads[3 * r], g1 = grads[3 * r + 1], g2 = grads[3 * r + 2];
      const float den = denom[r];
      const float gn = sqrtf(g0 * g0 + g1 * g1 + g2 * g2);
      const bool bad = fabsf(den) < (float)IFT_DENOM_RTOL * fmaxf(gn, 1e-30f);
      clamped += bad ? 1 : 0;
      float wmono = 0.f, ya[3] = {0.f, 0.f, 0.f};
      if (y_len && !bad) wmono += -y_len[r] / den;
      if (y_grad) {
        ya[0] = y_grad[3 * r];
        ya[1] = y_grad[3 * r + 1];
        ya[2] = y_grad[3 * r + 2];
        if (!bad) {
          const float rx = (float)dir[3 * r], ry = (float)dir[3 * r + 1], rz = (float)dir[3 * r + 2];
          const float* H = hess + 6 * r;  // xx yy zz xy xz yz
          const float k0 = (H[0] * rx + H[3] * ry + H[4] * rz) / den;
          const float k1 = (H[3] * rx + H[1] * ry + H[5] * rz) / den;
          const float k2 = (H[4] * rx + H[5] * ry + H[2] * rz) / den;
          wmono += -(ya[0] * k0 + ya[1] * k1 + ya[2] * k2);
        }
      }
      int b[3];
      float off[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double x = points[3 * r + k];
        b[k] = box_axis(x, res);
        off[k] = (float)(x - (-1.0 + ((double)b[k] + 0.5) * (2.0 / (double)res)));
      }
      key = ((uint32_t)b[0] * res + b[1]) * res + b[2];
      float mono[P];
      monomials<RHO>(off[0], off[1], off[2], mono);
#pragma unroll
      for (int j = 0; j < P; ++j) {
        float v = wmono * mono[j];
        // dipole_a[n] = mono[n - e_a]  (layers.py:127-141)
        const int j0 = MI<RHO>::index(mi.e0[j] - 1, mi.e1[j], mi.e2[j]);
        const int j1 = MI<RHO>::index(mi.e0[j], mi.e1[j] - 1, mi.e2[j]);
        const int j2 = MI<RHO>::index(mi.e0[j], mi.e1[j], mi.e2[j] - 1);
        if (j0 >= 0) v = fmaf(ya[0], mono[j0], v);
        if (j1 >= 0) v = fmaf(ya[1], mono[j1], v);
        if (j2 >= 0) v = fmaf(ya[2], mono[j2], v);
        out[j] = v;
      }
    }
    keys[r] = key;
#pragma unroll
    for (int k = 0; k < PP; k += 4)
      *reinterpret_cast<float4*>(payload + r * PP + k) =
          make_float4(out[k], out[k + 1], out[k + 2], out[k + 3]);
  }
  if (n_clamped) {
    clamped = __reduce_add_sync(0xffffffffu, clamped);
    if ((threadIdx.x & 31) == 0 && clamped) atomicAdd(n_clamped, clamped);
  }
}

// ------------------------------------------------------ line integral ---
// forward: sum over segments of int_0^s poly_c (layers.py:371-386)
template <int RHO>
__global__ void __launch_bounds__(128)
line_integral_kernel(const float* __restrict__ L, int res, int C, const double* __restrict__ org,
                     const double* __restrict__ dir, int64_t R, float* __restrict__ values) {
  constexpr int PP = MI<RHO>::PP;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    const float dirf[3] = {(float)d[0], (float)d[1], (float)d[2]};
    for (int c = 0; c < C; ++c) {
      double acc = 0.0;
      walk_ray(o, d, res, [&](double t0, double t1, int b0, int b1, int b2) {
        float base[3];
        seg_base(o, d, t0, b0, b1, b2, res, base);
        const float* row = L + ((((int64_t)b0 * res + b1) * res + b2) * C + c) * PP;
        float pf[RHO + 1];
        line_poly<RHO>(row, base, dirf, pf);
        const double s = t1 - t0;
        double v = 0.0;  // antiderivative at s (Horner)
        for (int j = RHO; j >= 0; --j) v = (v + (double)pf[j] / (double)(j + 1)) * s;
        acc += v;
        return true;
      });
      values[r * C + c] = (float)acc;
    }
  }
}

// backward payload per segment: y_c * line2taylor(d, r, s) (ray.py:213-246),
// Gauss-Legendre with G = floor(rho / 2) + 1 nodes (exact for h = 1)
template <int RHO>
__global__ void __launch_bounds__(128)
line_payload_kernel(int res, int C, const double* __restrict__ org,
                    const double* __restrict__ dir, int64_t R, const uint32_t* __restrict__ offsets,
                    const float* __restrict__ y, const double* __restrict__ gl_x,
                    const double* __restrict__ gl_w, int G, uint32_t* __restrict__ keys,
                    float* __restrict__ payload) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    int64_t i = offsets[r];
    walk_ray(o, d, res, [&](double t0, double t1, int b0, int b1, int b2) {
      float base[3];
      seg_base(o, d, t0, b0, b1, b2, res, base);
      const double s = t1 - t0, half = 0.5 * s;
      float mom[P];
#pragma unroll
      for (int j = 0; j < P; ++j) mom[j] = 0.f;
      for (int gq = 0; gq < G; ++gq) {
        const double t = half * (gl_x[gq] + 1.0);
        const float wt = (float)(half * gl_w[gq]);
        float mono[P];
        monomials<RHO>(base[0] + (float)t * (float)d[0], base[1] + (float)t * (float)d[1],
                       base[2] + (float)t * (float)d[2], mono);
#pragma unroll
        for (int j = 0; j < P; ++j) mom[j] = fmaf(wt, mono[j], mom[j]);
      }
      keys[i] = ((uint32_t)b0 * res + b1) * res + b2;
      for (int c = 0; c < C; ++c) {
        const float yc = y[r * C + c];
        float* dst = payload + (i * C + c) * PP;
#pragma unroll
        for (int k = 0; k < PP; k += 4)
          *reinterpret_cast<float4*>(dst + k) =
              make_float4(k < P ? yc * mom[k] : 0.f, k + 1 < P ? yc * mom[k + 1] : 0.f,
                          k + 2 < P ? yc * mom[k + 2] : 0.f, k + 3 < P ? yc * mom[k + 3] : 0.f);
      }
      ++i;
      return true;
    });
  }
}

// ----------------------------------------------------------- insertion ---
// Sum per-item payload rows into their cells in sorted (deterministic) order
// (reference _insert_moments, layers.py:144-153).
// Light cells (<= INS_LIGHT items): one thread per (cell, channel) sums the
// rows in sorted order.  Heavier cells (surface cells collecting hundreds of
// root payloads, or the segment moments of the radiance backward) are summed
// by one warp each in a second kernel (a warp per (cell, channel), light ones
// skipped): PP/4 lanes read one row (coalesced), WR = 32 /
// (PP/4) rows in flight; lane (r, q) accumulates float4 q of rows r, r+WR, ...
// and the WR partial sums are added in fixed order.  The summation order
// depends only on the cell's item count -> deterministic.
constexpr int INS_LIGHT = 8;

template <int PP>
__global__ void __launch_bounds__(128)
insert_sorted_kernel(const float* __restrict__ payload, int C, int64_t R,
                     const int32_t* __restrict__ order, const int32_t* __restrict__ cell_start,
                     float* __restrict__ M) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < R * C;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / C;
    const int c = (int)(g - cell * C);
    const int beg = cell_start[cell], end = cell_start[cell + 1];
    if (end - beg > INS_LIGHT) continue;   // insert_heavy_kernel
    float acc[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) acc[j] = 0.f;
    for (int k = beg; k < end; ++k) {
      const float* src = payload + ((int64_t)order[k] * C + c) * PP;
#pragma unroll
      for (int j = 0; j < PP; j += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(src + j));
        acc[j] += v.x; acc[j + 1] += v.y; acc[j + 2] += v.z; acc[j + 3] += v.w;
      }
    }
#pragma unroll
    for (int j = 0; j < PP; j += 4)
      *reinterpret_cast<float4*>(M + g * PP + j) =
          make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
}

template <int PP>
__global__ void __launch_bounds__(256)
insert_heavy_kernel(const float* __restrict__ payload, int C, int64_t R,
                    const int32_t* __restrict__ order, const int32_t* __restrict__ cell_start,
                    float* __restrict__ M) {
  constexpr int Q = PP / 4;                  // float4 per row
  constexpr int WR = 32 / Q > 0 ? 32 / Q : 1;  // rows in flight per warp
  const int lane = threadIdx.x & 31;
  const int r = lane / Q, q = lane - r * Q;
  const bool active = r < WR && q < Q;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t g = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); g < R * C;
       g += warps) {
    const int64_t cell = g / C;
    const int c = (int)(g - cell * C);
    const int beg = cell_start[cell], end = cell_start[cell + 1];
    if (end - beg <= INS_LIGHT) continue;
    float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
    if (active)
      for (int k = beg + r; k < end; k += WR) {
        const float4 v =
            __ldg(reinterpret_cast<const float4*>(payload + ((int64_t)order[k] * C + c) * PP) + q);
        a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
      }
    // fixed-order sum of the WR row partials into lanes 0..Q-1
    for (int rr = 1; rr < WR; ++rr) {
      const float bx = __shfl_sync(0xffffffffu, a.x, rr * Q + q);
      const float by = __shfl_sync(0xffffffffu, a.y, rr * Q + q);
      const float bz = __shfl_sync(0xffffffffu, a.z, rr * Q + q);
      const float bw = __shfl_sync(0xffffffffu, a.w, rr * Q + q);
      if (r == 0) { a.x += bx; a.y += by; a.z += bz; a.w += bw; }
    }
    if (r == 0 && q < Q) reinterpret_cast<float4*>(M + g * PP)[q] = a;
  }
}

}  // namespace

// ---------------------------------------------------------------- host ---

cudaError_t traverse_count(int level, const double* org, const double* dir, int64_t R,
                           uint32_t* counts, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  FC2T2_LAUNCH("traverse", s,
               traverse_count_kernel<<<grid_blocks(R, 128, 148 * 32), 128, 0, s>>>(
                   org, dir, R, 1 << (level + 1), counts));
  return cudaGetLastError();
}

cudaError_t traverse_fill(int level, const double* org, const double* dir, int64_t R,
                          const uint32_t* offsets, int32_t* ray_id, double* t0, double* t1,
                          int32_t* box, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  FC2T2_LAUNCH("traverse", s,
               traverse_fill_kernel<<<grid_blocks(R, 128, 148 * 32), 128, 0, s>>>(
                   org, dir, R, 1 << (level + 1), offsets, ray_id, t0, t1, box));
  return cudaGetLastError();
}

cudaError_t depth_walk(int rho, int level, const float* L, const double* org, const double* dir,
                       int64_t R, double bias, double* lengths, uint8_t* hit, double* points,
                       float* grads, float* hess, float* denom, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  if (rho > 4) return cudaErrorNotSupported;  // quartic line polynomials (multiindex.py:17)
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("depth_walk", s,
      depth_walk_kernel<RHO><<<grid_blocks(R, 128, 148 * 32), 128, 0, s>>>(
          L, 1 << (level + 1), org, dir, R, bias, lengths, hit, points, grads, hess, denom)));
  return cudaGetLastError();
}

cudaError_t root_payload(int rho, int level, const double* dir, int64_t R, const uint8_t* hit,
                         const double* points, const float* grads, const float* hess,
                         const float* denom, const float* y_len, const float* y_grad,
                         uint32_t* keys, float* payload, int32_t* n_clamped, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("root_payload", s,
      root_payload_kernel<RHO><<<grid_blocks(R, 128, 148 * 32), 128, 0, s>>>(
          1 << (level + 1), dir, R, hit, points, grads, hess, denom, y_len, y_grad, keys,
          payload, n_clamped)));
  return cudaGetLastError();
}

cudaError_t line_integral(int rho, int level, int C, const float* L, const double* org,
                          const double* dir, int64_t R, float* values, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("line_integral", s,
      line_integral_kernel<RHO><<<grid_blocks(R, 128, 148 * 32), 128, 0, s>>>(
          L, 1 << (level + 1), C, org, dir, R, values)));
  return cudaGetLastError();
}

cudaError_t line_payload(int rho, int level, int C, const double* org, const double* dir,
                         int64_t R, const uint32_t* offsets, const float* y, const double* gl_x,
                         const double* gl_w, int G, uint32_t* keys, float* payload,
                         cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("line_payload", s,
      line_payload_kernel<RHO><<<grid_blocks(R, 128, 148 * 32), 128, 0, s>>>(
          1 << (level + 1), C, org, dir, R, offsets, y, gl_x, gl_w, G, keys, payload)));
  return cudaGetLastError();
}

cudaError_t insert_sorted(int rho, int level, int C, const float* payload, const int32_t* order,
                          const int32_t* cell_start, float* M, cudaStream_t s) {
  const int64_t res = (int64_t)1 << (level + 1);
  const int64_t R = res * res * res;
  const int PP = pad4(index_count(rho));
  switch (PP) {
#define FC2T2_INS(V)                                                                         \
  case V:                                                                                    \
    FC2T2_LAUNCH("insert", s, insert_sorted_kernel<V><<<grid_blocks(R * C, 128, 148 * 64),  \
                                                        128, 0, s>>>(payload, C, R, order,   \
                                                                     cell_start, M));        \
    FC2T2_LAUNCH("insert", s, insert_heavy_kernel<V><<<grid_blocks(R * C * 32, 256, 148 * 32), \
                                  256, 0, s>>>(payload, C, R, order, cell_start, M));        \
    break;
    FC2T2_INS(4)
    FC2T2_INS(12)
    FC2T2_INS(20)
    FC2T2_INS(36)
    FC2T2_INS(56)
    FC2T2_INS(84)
#undef FC2T2_INS
    default:
      return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

}  // namespace fc2t2
