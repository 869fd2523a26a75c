// Shared device code of the ray kernels: float64 traversal walker (reference
// ray.py:101-157) and the exact line restriction of a cell polynomial
// (ray.py:184-210).  Included by rays.cu and volume.cu.
#pragma once
#include <math_constants.h>

#include "common.cuh"

namespace fc2t2 {
namespace ray {

constexpr double MIN_SEGMENT = 1e-12;        // ray.py:23
constexpr double LEADING_EPS = 1e-12;        // poly1d.py:19
constexpr double ROOT_BOUNDARY_EPS = 1e-10;  // layers.py:40
constexpr double IFT_DENOM_RTOL = 1e-8;      // layers.py:39

// ------------------------------------------------------------ traversal ---

__device__ __forceinline__ void domain_span(const double o[3], const double d[3], double& t_in,
                                            double& t_out) {
  double near = -CUDART_INF, far = CUDART_INF;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double n, f;
    if (d[a] == 0.0) {
      const bool inside = fabs(o[a]) < 1.0;
      n = inside ? -CUDART_INF : CUDART_INF;
      f = inside ? CUDART_INF : -CUDART_INF;
    } else {
      const double lo = __ddiv_rn(__dadd_rn(-1.0, -o[a]), d[a]);
      const double hi = __ddiv_rn(__dadd_rn(1.0, -o[a]), d[a]);
      n = fmin(lo, hi);
      f = fmax(lo, hi);
    }
    near = fmax(near, n);
    far = fmin(far, f);
  }
  t_in = fmax(near, 0.0);
  t_out = far;
}

// Walk the ray's segments in order; seg(t0, t1, b0, b1, b2) returns false to stop.
template <class F>
__device__ __forceinline__ int walk_ray(const double o[3], const double d[3], int res, F&& seg) {
  double t_in, t_out;
  domain_span(o, d, t_in, t_out);
  if (!(t_in < t_out)) return 0;
  const double width = 2.0 / (double)res;
  int k[3], step[3];
  double nxt[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (d[a] == 0.0) {
      nxt[a] = CUDART_INF;
      k[a] = 0;
      step[a] = 0;
      continue;
    }
    step[a] = d[a] > 0.0 ? 1 : -1;
    k[a] = d[a] > 0.0 ? 0 : res;
    // first plane strictly after t_in
    for (;;) {
      if (k[a] < 0 || k[a] > res) { nxt[a] = CUDART_INF; break; }
      const double pl = __dadd_rn(-1.0, __dmul_rn(width, (double)k[a]));
      const double t = __ddiv_rn(__dadd_rn(pl, -o[a]), d[a]);
      if (t > t_in) { nxt[a] = t; break; }
      k[a] += step[a];
    }
  }
  const double lo_clip = -1.0 + 1e-15, hi_clip = 1.0 - 1e-15;
  double prev = t_in;
  int count = 0;
  for (;;) {
    int am = 0;
    double t = nxt[0];
    if (nxt[1] < t) { t = nxt[1]; am = 1; }
    if (nxt[2] < t) { t = nxt[2]; am = 2; }
    const bool last = !(t < t_out);
    const double end = last ? t_out : t;
    if (__dadd_rn(end, -prev) > MIN_SEGMENT) {
      const double tm = __dmul_rn(0.5, __dadd_rn(prev, end));
      int b[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        double m = __dadd_rn(o[a], __dmul_rn(tm, d[a]));
        m = fmin(fmax(m, lo_clip), hi_clip);
        b[a] = box_axis(m, res);
      }
      ++count;
      if (!seg(prev, end, b[0], b[1], b[2])) return count;
    }
    if (last) break;
    prev = end;
    k[am] += step[am];
    if (k[am] < 0 || k[am] > res) {
      nxt[am] = CUDART_INF;
    } else {
      const double pl = __dadd_rn(-1.0, __dmul_rn(width, (double)k[am]));
      nxt[am] = __ddiv_rn(__dadd_rn(pl, -o[am]), d[am]);
    }
  }
  return count;
}

__device__ __forceinline__ void load_ray(const double* __restrict__ org,
                                         const double* __restrict__ dir, int64_t r, double o[3],
                                         double d[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    o[a] = org[3 * r + a];
    d[a] = dir[3 * r + a];
  }
}

// segment base offset from its box centre, d = (o + t0 r) - centre (ray.py:249-258)
__device__ __forceinline__ void seg_base(const double o[3], const double d[3], double t0, int b0,
                                         int b1, int b2, int res, float base[3]) {
  const int b[3] = {b0, b1, b2};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double x = __dadd_rn(o[a], __dmul_rn(t0, d[a]));
    const double c = -1.0 + ((double)b[a] + 0.5) * (2.0 / (double)res);
    base[a] = (float)(x - c);
  }
}

// ------------------------------------------------------------ line2poly ---
// f(centre + base + t r) as ascending coefficients in t: per axis
// U[k](t) = (base + t r)^k / k!, then sum_n L[n] Ux[n0] Uy[n1] Uz[n2].
template <int RHO>
__device__ __forceinline__ void axis_polys(float b, float r, float (&U)[RHO + 1][RHO + 1]) {
#pragma unroll
  for (int k = 0; k <= RHO; ++k)
#pragma unroll
    for (int j = 0; j <= RHO; ++j) U[k][j] = 0.f;
  U[0][0] = 1.f;
#pragma unroll
  for (int k = 1; k <= RHO; ++k) {
    const float inv = 1.f / (float)k;
#pragma unroll
    for (int j = 0; j <= k; ++j) {
      float v = j < k ? U[k - 1][j] * b : 0.f;
      if (j > 0) v = fmaf(U[k - 1][j - 1], r, v);
      U[k][j] = v * inv;
    }
  }
}

template <int RHO>
__device__ __forceinline__ void line_poly(const float* __restrict__ row, const float base[3],
                                          const float dir[3], float (&out)[RHO + 1]) {
  constexpr MI<RHO> mi{};
  float Ux[RHO + 1][RHO + 1], Uy[RHO + 1][RHO + 1], Uz[RHO + 1][RHO + 1];
  axis_polys<RHO>(base[0], dir[0], Ux);
  axis_polys<RHO>(base[1], dir[1], Uy);
  axis_polys<RHO>(base[2], dir[2], Uz);
  float a[MI<RHO>::PP];
#pragma unroll
  for (int k = 0; k < MI<RHO>::PP; k += 4) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(row + k));
    a[k] = v.x; a[k + 1] = v.y; a[k + 2] = v.z; a[k + 3] = v.w;
  }
#pragma unroll
  for (int j = 0; j <= RHO; ++j) out[j] = 0.f;
#pragma unroll
  for (int n0 = 0; n0 <= RHO; ++n0) {
    float Y[RHO + 1];
#pragma unroll
    for (int j = 0; j <= RHO; ++j) Y[j] = 0.f;
#pragma unroll
    for (int n1 = 0; n0 + n1 <= RHO; ++n1) {
      float Z[RHO + 1];
#pragma unroll
      for (int j = 0; j <= RHO; ++j) Z[j] = 0.f;
#pragma unroll
      for (int n2 = 0; n0 + n1 + n2 <= RHO; ++n2) {
        const float c = a[MI<RHO>::index(n0, n1, n2)];
#pragma unroll
        for (int j = 0; j <= n2; ++j) Z[j] = fmaf(c, Uz[n2][j], Z[j]);
      }
      // Y += Uy[n1] * Z   (deg Z <= RHO - n0 - n1)
#pragma unroll
      for (int i = 0; i <= n1; ++i)
#pragma unroll
        for (int j = 0; i + j <= RHO - n0; ++j) Y[i + j] = fmaf(Uy[n1][i], Z[j], Y[i + j]);
    }
#pragma unroll
    for (int i = 0; i <= n0; ++i)
#pragma unroll
      for (int j = 0; i + j <= RHO; ++j) out[i + j] = fmaf(Ux[n0][i], Y[j], out[i + j]);
  }
  (void)mi;
}

}  // namespace ray
}  // namespace fc2t2
