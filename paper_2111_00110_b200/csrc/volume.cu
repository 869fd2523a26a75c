// Integral-implicit radiance layer (reference layers.py:405-544) on the device.
//
// Forward, one thread per ray walking its segments in order:
//   sigma, colour polynomials = line2poly of the 1+CC channels (raywalk.cuh),
//   S(x) = int sigma, depth0 = per-ray exclusive prefix of S(s) (float64),
//   alive = depth0 <= 4.5, rgb_c += int_0^s c sigma E(S + depth0) dx,
//   rgb_c += E(depth_final) bg_c.
// The integrand is a polynomial of degree 4(rho+1) + 2 rho (28 at rho = 4),
// so a 15-node Gauss-Legendre rule (exact to degree 29) integrates it exactly
// -- the same value the
// reference gets from its explicit polynomial algebra, without the degree-29
// coefficient arrays (the register footprint is what bounded the first
// version of these kernels).
// Backward (volumetric_jvp): pass A recomputes the per-ray totals of
// int_0^s E'(S + depth0) sigma c; pass B builds per alive segment the weights
// h_sigma(u) and y_c T(u) sigma(u) at the 15 Gauss nodes and inserts their
// closed-form segment moments (line2taylor_h, exact at this degree).  The one
// nested integral, int_0^u c sigma T', is polynomial algebra in float32 with
// E' Taylor-shifted to depth0 in float64 first.
#include "common.cuh"
#include "kernels.cuh"
#include "raywalk.cuh"

namespace fc2t2 {

namespace {

using namespace ray;

constexpr double EXP_CUTOFF = 4.5;     // poly1d.py:22
constexpr double EXP_FIT_RANGE = 5.0;  // poly1d.py:23
constexpr int GN = 15;                 // Gauss-Legendre nodes, exact to degree 29 >= 28

__constant__ double GL_X[GN] = {
    -0.9879925180204854, -0.9372733924007058, -0.8482065834104272, -0.7244177313601701,
    -0.5709721726085388, -0.3941513470775634, -0.20119409399743451, 0.0, 0.20119409399743451,
    0.3941513470775634, 0.5709721726085388, 0.7244177313601701, 0.8482065834104272,
    0.9372733924007058, 0.9879925180204854};
__constant__ double GL_W[GN] = {
    0.030753241996117203, 0.0703660474881084, 0.10715922046717141, 0.13957067792615444,
    0.16626920581699398, 0.1861610000155622, 0.1984314853271116, 0.2025782419255613,
    0.1984314853271116, 0.1861610000155622, 0.16626920581699398, 0.13957067792615444,
    0.10715922046717141, 0.0703660474881084, 0.030753241996117203};

template <int N>
__device__ __forceinline__ float hornerf(const float (&a)[N], float x) {
  float y = 0.f;
#pragma unroll
  for (int k = N - 1; k >= 0; --k) y = fmaf(y, x, a[k]);
  return y;
}

template <int NA, int NB>
__device__ __forceinline__ void pmulf(const float (&a)[NA], const float (&b)[NB],
                                      float (&o)[NA + NB - 1]) {
#pragma unroll
  for (int k = 0; k < NA + NB - 1; ++k) o[k] = 0.f;
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) o[i + j] = fmaf(a[i], b[j], o[i + j]);
}

__device__ __forceinline__ double efit_eval(const double* e, double y) {
  return (((e[4] * y + e[3]) * y + e[2]) * y + e[1]) * y + e[0];
}

__device__ __forceinline__ double efit_deriv(const double* e, double y) {
  return ((4.0 * e[4] * y + 3.0 * e[3]) * y + 2.0 * e[2]) * y + e[1];
}

// segment: sigma line polynomial, its antiderivative coefficients and S(s)
template <int RHO>
__device__ __forceinline__ double segment_sigma(const float* row, const float base[3],
                                                const float dirf[3], double s,
                                                float (&sg)[RHO + 1], float (&S)[RHO + 2]) {
  line_poly<RHO>(row, base, dirf, sg);
  S[0] = 0.f;
#pragma unroll
  for (int k = 0; k <= RHO; ++k) S[k + 1] = sg[k] / (float)(k + 1);
  double v = 0.0;  // S(s) in float64 (feeds the optical-depth prefix)
#pragma unroll
  for (int k = RHO; k >= 0; --k) v = (v + (double)sg[k] / (double)(k + 1)) * s;
  return v;
}

// ------------------------------------------------------------- forward ---
template <int RHO, int CC>
__global__ void __launch_bounds__(128)
vol_forward_kernel(const float* __restrict__ L, int res, const double* __restrict__ org,
                   const double* __restrict__ dir, int64_t R, const double* __restrict__ efit,
                   const double* __restrict__ bg, float* __restrict__ rgb,
                   double* __restrict__ depth_final, const uint32_t* __restrict__ seg_offsets,
                   uint8_t* __restrict__ seg_alive, uint32_t* __restrict__ n_alive,
                   double* __restrict__ totals) {
  // With n_alive / totals the walk also produces the backward's pass-A
  // quantities (same node arithmetic as vol_totals_kernel, bit-identical), so
  // volumetric_jvp can skip that pass.
  constexpr int PP = MI<RHO>::PP, NCH = 1 + CC;
  double e[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) e[k] = efit[k];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    const float dirf[3] = {(float)d[0], (float)d[1], (float)d[2]};
    double depth = 0.0, dfin = 0.0, acc[CC], tot[CC];
#pragma unroll
    for (int c = 0; c < CC; ++c) acc[c] = tot[c] = 0.0;
    uint32_t na = 0;
    int64_t j = seg_offsets ? (int64_t)seg_offsets[r] : 0;
    walk_ray(o, d, res, [&](double t0, double t1, int b0, int b1, int b2) {
      float base[3];
      seg_base(o, d, t0, b0, b1, b2, res, base);
      const float* row = L + (((int64_t)b0 * res + b1) * res + b2) * NCH * PP;
      const double s = t1 - t0;
      float sg[RHO + 1], S[RHO + 2];
      const double send = segment_sigma<RHO>(row, base, dirf, s, sg, S);
      const bool alive = depth <= EXP_CUTOFF;
      if (alive) {
        float col[CC][RHO + 1];
#pragma unroll
        for (int c = 0; c < CC; ++c) line_poly<RHO>(row + (1 + c) * PP, base, dirf, col[c]);
        const double half = 0.5 * s;
#pragma unroll 1
        for (int g = 0; g < GN; ++g) {
          const double x = half * (GL_X[g] + 1.0);
          const float xf = (float)x;
          const double y = (double)hornerf(S, xf) + depth;
          const double T = efit_eval(e, y);
          const double sgx = (double)hornerf(sg, xf);
          const double wts = half * GL_W[g] * T * sgx;
          if (totals) {
            const double wtp = half * GL_W[g] * efit_deriv(e, y) * sgx;
#pragma unroll
            for (int c = 0; c < CC; ++c) {
              const double cx = (double)hornerf(col[c], xf);
              acc[c] += wts * cx;
              tot[c] += wtp * cx;
            }
          } else {
#pragma unroll
            for (int c = 0; c < CC; ++c) acc[c] += wts * (double)hornerf(col[c], xf);
          }
        }
        dfin += send;
        ++na;
      }
      if (seg_alive) seg_alive[j++] = alive ? 1 : 0;
      depth += send;
      return true;
    });
    const double te = dfin > EXP_FIT_RANGE ? 0.0 : efit_eval(e, dfin);
#pragma unroll
    for (int c = 0; c < CC; ++c) rgb[r * CC + c] = (float)(acc[c] + te * bg[c]);
    depth_final[r] = dfin;
    if (totals) {
      n_alive[r] = na;
#pragma unroll
      for (int c = 0; c < CC; ++c) totals[r * CC + c] = tot[c];
    }
  }
}

// ------------------------------------------------- backward pass A ---
// per ray: number of alive segments and totals of int_0^s c sigma E'(S + depth0)
template <int RHO, int CC>
__global__ void __launch_bounds__(128)
vol_totals_kernel(const float* __restrict__ L, int res, const double* __restrict__ org,
                  const double* __restrict__ dir, int64_t R, const double* __restrict__ efit,
                  uint32_t* __restrict__ n_alive, double* __restrict__ totals,
                  double* __restrict__ depth_final) {
  constexpr int PP = MI<RHO>::PP, NCH = 1 + CC;
  double e[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) e[k] = efit[k];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    const float dirf[3] = {(float)d[0], (float)d[1], (float)d[2]};
    double depth = 0.0, dfin = 0.0, tot[CC];
#pragma unroll
    for (int c = 0; c < CC; ++c) tot[c] = 0.0;
    uint32_t na = 0;
    walk_ray(o, d, res, [&](double t0, double t1, int b0, int b1, int b2) {
      float base[3];
      seg_base(o, d, t0, b0, b1, b2, res, base);
      const float* row = L + (((int64_t)b0 * res + b1) * res + b2) * NCH * PP;
      const double s = t1 - t0;
      float sg[RHO + 1], S[RHO + 2];
      const double send = segment_sigma<RHO>(row, base, dirf, s, sg, S);
      if (depth <= EXP_CUTOFF) {
        float col[CC][RHO + 1];
#pragma unroll
        for (int c = 0; c < CC; ++c) line_poly<RHO>(row + (1 + c) * PP, base, dirf, col[c]);
        const double half = 0.5 * s;
#pragma unroll 1
        for (int g = 0; g < GN; ++g) {
          const double x = half * (GL_X[g] + 1.0);
          const float xf = (float)x;
          const double Tp = efit_deriv(e, (double)hornerf(S, xf) + depth);
          const double wts = half * GL_W[g] * Tp * (double)hornerf(sg, xf);
#pragma unroll
          for (int c = 0; c < CC; ++c) tot[c] += wts * (double)hornerf(col[c], xf);
        }
        dfin += send;
        ++na;
      }
      depth += send;
      return true;
    });
    n_alive[r] = na;
#pragma unroll
    for (int c = 0; c < CC; ++c) totals[r * CC + c] = tot[c];
    depth_final[r] = dfin;
  }
}

// ------------------------------------------------- backward pass B ---
// Per alive segment (layers.py:513-534):
//   h_sigma(u) = sum_c y_c [ T(u) c(u) - int_0^u c sigma T' + total_c - before_c + tp_inf bg_c ]
//   payload[0]   = sum_g W_g h_sigma(u_g) mono(d + u_g r)
//   payload[1+c] = sum_g W_g y_c T(u_g) sigma(u_g) mono(d + u_g r)
// T(u) = E(S(u) + depth0), T' = E'(S(u) + depth0).  int_0^u c sigma T' is a
// degree-(3(rho+1) + 2 rho + 1) polynomial built in float32 from
// E'_shift(y) = E'(y + depth0) (shift in float64) composed with S.
// Moments of NCH node-weighted point sets on one segment line p(x) = base +
// x dir: pay[ch][n] = sum_g wn[ch][g] mono_n(p(x_g)).  Each monomial is a
// polynomial in x, mono_n(p(x)) = inv_fact[n] prod_a (base_a + x dir_a)^{n_a}
// = sum_i c_{n,i} x^i (|n| <= RHO), so pay[ch][n] = sum_i c_{n,i} mu[ch][i] with
// the power moments mu[ch][i] = sum_g wn[ch][g] x_g^i.  A segment is therefore
// fully described by the record {base, dir, mu} (VOL_REC floats): the
// backward's walker writes records (not NCH x PP payload rows), and the
// per-cell insertion expands them while it sums (vol_insert_kernel).
template <int RHO, int NCH, int GNODES>
__device__ __forceinline__ void segment_power_moments(const float (&xs)[GNODES], const float* wn,
                                                      float (&mu)[NCH][RHO + 1]) {
#pragma unroll
  for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
    for (int i = 0; i <= RHO; ++i) mu[ch][i] = 0.f;
#pragma unroll 1
  for (int g = 0; g < GNODES; ++g) {
    const float x = xs[g];
    float w[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) w[ch] = wn[ch * GNODES + g];
#pragma unroll
    for (int i = 0; i <= RHO; ++i) {
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) mu[ch][i] += w[ch];
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) w[ch] *= x;
    }
  }
}

// acc[ch][n - N0] += pay[ch][n] for n in [N0, N1) and every channel: the
// segment's rows restricted to one slice of the coefficient index
template <int RHO, int NCH, int N0, int N1>
__device__ __forceinline__ void add_segment_rows(const float base[3], const float dirf[3],
                                                 const float (&mu)[NCH][RHO + 1],
                                                 float (&acc)[NCH][N1 - N0]) {
  constexpr MI<RHO> mi{};
  constexpr int P = MI<RHO>::P;
  // per-axis binomial polynomials Q[a][k][i] = coefficient of x^i in (b + x d)^k
  float Q[3][RHO + 1][RHO + 1];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    Q[a][0][0] = 1.f;
#pragma unroll
    for (int k = 1; k <= RHO; ++k)
#pragma unroll
      for (int i = 0; i <= k; ++i)
        Q[a][k][i] = (i < k ? Q[a][k - 1][i] * base[a] : 0.f) +
                     (i > 0 ? Q[a][k - 1][i - 1] * dirf[a] : 0.f);
  }
#pragma unroll
  for (int n = N0; n < N1 && n < P; ++n) {
    const int n0 = mi.e0[n], n1 = mi.e1[n], n2 = mi.e2[n];
    float c01[RHO + 1], c[RHO + 1];
#pragma unroll
    for (int i = 0; i <= RHO; ++i) c01[i] = c[i] = 0.f;
#pragma unroll
    for (int i = 0; i <= RHO; ++i)
#pragma unroll
      for (int j = 0; j <= RHO; ++j)
        if (i <= n0 && j <= n1) c01[i + j] = fmaf(Q[0][n0][i], Q[1][n1][j], c01[i + j]);
#pragma unroll
    for (int i = 0; i <= RHO; ++i)
#pragma unroll
      for (int j = 0; j <= RHO; ++j)
        if (i <= n0 + n1 && j <= n2 && i + j <= RHO) c[i + j] = fmaf(c01[i], Q[2][n2][j], c[i + j]);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
      float v = 0.f;
#pragma unroll
      for (int i = 0; i <= RHO; ++i)
        if (i <= n0 + n1 + n2) v = fmaf(c[i], mu[ch][i], v);
      acc[ch][n - N0] = __fadd_rn(acc[ch][n - N0], __fmul_rn(v, mi.inv_fact[n]));
    }
  }
}

// record floats: base 3 + dir 3 + NCH x (RHO + 1) power moments, 16-byte rows
__host__ __device__ constexpr int vol_rec_floats(int rho, int nch) {
  return (6 + nch * (rho + 1) + 3) / 4 * 4;
}

constexpr int VOL_THREADS = 128;

template <int RHO, int CC>
__global__ void __launch_bounds__(VOL_THREADS, 3)
vol_payload_kernel(const float* __restrict__ L, int res, const double* __restrict__ org,
                   const double* __restrict__ dir, int64_t R, const double* __restrict__ efit,
                   const double* __restrict__ bg, const float* __restrict__ ybar,
                   const uint32_t* __restrict__ alive_offsets, const double* __restrict__ totals,
                   const double* __restrict__ depth_final, uint32_t* __restrict__ keys,
                   float* __restrict__ payload) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP, NCH = 1 + CC;
  constexpr int NS = RHO + 2, NS2 = 2 * NS - 1, NS3 = NS2 + NS - 1;  // S, S^2, S^3
  constexpr int NCS = 2 * RHO + 1;                                   // c * sigma
  constexpr int NQ = NCS + NS3 - 1;                                  // c sigma T'
  __shared__ float wn_s[VOL_THREADS][NCH * GN + 1];                  // node weights
  // T at the nodes, once per segment, when it fits the 48 KB static limit
  constexpr bool TN = (NCH * GN + 1 + GN) * 4 * VOL_THREADS <= 48 * 1024;
  __shared__ float tn_s[TN ? GN : 1][VOL_THREADS];
  float* wn = wn_s[threadIdx.x];
  double e[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) e[k] = efit[k];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    const float dirf[3] = {(float)d[0], (float)d[1], (float)d[2]};
    const double dfin = depth_final[r];
    const double tp_inf = dfin > EXP_FIT_RANGE ? 0.0 : efit_deriv(e, dfin);  // layers.py:510-511
    double yb[CC], before[CC];
#pragma unroll
    for (int c = 0; c < CC; ++c) {
      yb[c] = (double)ybar[r * CC + c];
      before[c] = 0.0;
    }
    int64_t item = alive_offsets[r];
    double depth = 0.0;
    walk_ray(o, d, res, [&](double t0, double t1, int b0, int b1, int b2) {
      float base[3];
      seg_base(o, d, t0, b0, b1, b2, res, base);
      const float* row = L + (((int64_t)b0 * res + b1) * res + b2) * NCH * PP;
      const double s = t1 - t0;
      float sg[RHO + 1], S[NS];
      const double send = segment_sigma<RHO>(row, base, dirf, s, sg, S);
      if (depth <= EXP_CUTOFF) {
        // T'(x) = a0 + a1 S + a2 S^2 + a3 S^3 with a = E' shifted to depth0 (float64)
        const float a0 = (float)efit_deriv(e, depth);
        const float a1 = (float)((12.0 * e[4] * depth + 6.0 * e[3]) * depth + 2.0 * e[2]);
        const float a2 = (float)(12.0 * e[4] * depth + 3.0 * e[3]);
        const float a3 = (float)(4.0 * e[4]);
        float S2[NS2], S3[NS3], Tp[NS3];
        pmulf(S, S, S2);
        pmulf(S2, S, S3);
#pragma unroll
        for (int k = 0; k < NS3; ++k) {
          float v = a3 * S3[k];
          if (k < NS2) v = fmaf(a2, S2[k], v);
          if (k < NS) v = fmaf(a1, S[k], v);
          if (k == 0) v += a0;
          Tp[k] = v;
        }
        const double half = 0.5 * s;
        // T(x_g) = E(S(x_g) + depth0) once per node (shared by every channel
        // and by the weight loop below)
        if constexpr (TN) {
#pragma unroll 1
          for (int g = 0; g < GN; ++g)
            tn_s[g][threadIdx.x] =
                (float)efit_eval(e, (double)hornerf(S, (float)(half * (GL_X[g] + 1.0))) + depth);
        }
        auto t_at = [&](int g, float xf) -> double {
          if constexpr (TN) return (double)tn_s[g][threadIdx.x];
          else return efit_eval(e, (double)hornerf(S, xf) + depth);
        };
        // node weights: channel 0 accumulates h_sigma, colours y_c T sigma
        float hs_const = 0.f;
#pragma unroll
        for (int g = 0; g < GN; ++g) wn[g] = 0.f;
#pragma unroll 1
        for (int c = 0; c < CC; ++c) {
          float col[RHO + 1], cs[NCS], q[NQ];
          line_poly<RHO>(row + (1 + c) * PP, base, dirf, col);
          pmulf(col, sg, cs);
          pmulf(cs, Tp, q);
          const double k_c = totals[r * CC + c] - before[c] + tp_inf * bg[c];
          hs_const += (float)(yb[c] * k_c);
          // int_0^u q, evaluated at the nodes and at s
          double cp = 0.0;
#pragma unroll 1
          for (int g = 0; g <= GN; ++g) {
            const double x = g < GN ? half * (GL_X[g] + 1.0) : s;
            const float xf = (float)x;
            float aq = 0.f;
#pragma unroll
            for (int k = NQ - 1; k >= 0; --k) aq = (aq + q[k] / (float)(k + 1)) * xf;
            if (g == GN) {
              cp = (double)aq;
              break;
            }
            const double T = t_at(g, xf);
            wn[g] += (float)(yb[c] * (T * (double)hornerf(col, xf) - (double)aq));
          }
          before[c] += cp;
        }
#pragma unroll 1
        for (int g = 0; g < GN; ++g) {
          const double x = half * (GL_X[g] + 1.0);
          const float xf = (float)x;
          const double W = half * GL_W[g];
          const double T = t_at(g, xf);
          wn[g] = (float)(W * ((double)wn[g] + (double)hs_const));
          const double ts = W * T * (double)hornerf(sg, xf);
#pragma unroll
          for (int c = 0; c < CC; ++c) wn[(1 + c) * GN + g] = (float)(yb[c] * ts);
        }
        keys[item] = ((uint32_t)b0 * res + b1) * res + b2;
        float xs[GN];
#pragma unroll
        for (int g = 0; g < GN; ++g) xs[g] = (float)(half * (GL_X[g] + 1.0));
        float mu[NCH][RHO + 1];
        segment_power_moments<RHO, NCH, GN>(xs, wn, mu);
        constexpr int RV = vol_rec_floats(RHO, NCH);
        float rv[RV];
        rv[0] = base[0]; rv[1] = base[1]; rv[2] = base[2];
        rv[3] = dirf[0]; rv[4] = dirf[1]; rv[5] = dirf[2];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int i = 0; i <= RHO; ++i) rv[6 + ch * (RHO + 1) + i] = mu[ch][i];
#pragma unroll
        for (int k = 6 + NCH * (RHO + 1); k < RV; ++k) rv[k] = 0.f;
        float4* dst = reinterpret_cast<float4*>(payload + item * RV);
#pragma unroll
        for (int k = 0; k < RV / 4; ++k)
          dst[k] = make_float4(rv[4 * k], rv[4 * k + 1], rv[4 * k + 2], rv[4 * k + 3]);
        ++item;
      }
      depth += send;
      return true;
    });
  }
}

// Per (cell, channel), in the key sort's order: the segment records of the
// cell expanded to payload rows and summed (the same float32 row values the
// row-materialising version wrote and summed, without the NCH x PP rows in HBM)
// Per (cell, channel), in the key sort's order: the cell's segment records
// expanded to payload rows and summed -- the same float32 row values the
// row-materialising version wrote and summed, without the NCH x PP rows in
// HBM.  (Measured alternatives: three threads per cell splitting the
// coefficient index, 3.6 ms vs 2.4 ms at config 4 -- 168 registers.)
template <int RHO, int NCH>
__global__ void __launch_bounds__(128)
vol_insert_kernel(const float* __restrict__ rec, int64_t R3, const int32_t* __restrict__ order,
                  const int32_t* __restrict__ cell_start, float* __restrict__ M) {
  constexpr int PP = MI<RHO>::PP, RV = vol_rec_floats(RHO, NCH);
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < R3 * NCH;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / NCH;
    const int ch = (int)(g - cell * NCH);
    const int beg = cell_start[cell], end = cell_start[cell + 1];
    float acc[1][PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) acc[0][j] = 0.f;
    for (int k = beg; k < end; ++k) {
      const float* r = rec + (int64_t)order[k] * RV;
      const float4 a = __ldg(reinterpret_cast<const float4*>(r));
      const float2 b = __ldg(reinterpret_cast<const float2*>(r + 4));
      const float base[3] = {a.x, a.y, a.z}, dirf[3] = {a.w, b.x, b.y};
      float mu[1][RHO + 1];
#pragma unroll
      for (int i = 0; i <= RHO; ++i) mu[0][i] = __ldg(r + 6 + ch * (RHO + 1) + i);
      add_segment_rows<RHO, 1, 0, PP>(base, dirf, mu, acc);
    }
#pragma unroll
    for (int j = 0; j < PP; j += 4)
      *reinterpret_cast<float4*>(M + g * PP + j) =
          make_float4(acc[0][j], acc[0][j + 1], acc[0][j + 2], acc[0][j + 3]);
  }
}

#define FC2T2_VOL_DISPATCH(CCV, ...)                       \
  switch (CCV) {                                           \
    case 1: { constexpr int CC = 1; __VA_ARGS__; } break;  \
    case 2: { constexpr int CC = 2; __VA_ARGS__; } break;  \
    case 3: { constexpr int CC = 3; __VA_ARGS__; } break;  \
    case 4: { constexpr int CC = 4; __VA_ARGS__; } break;  \
    default: return cudaErrorNotSupported;                 \
  }

}  // namespace

int vol_gauss_nodes(int rho) { return GN; }

int vol_record_floats(int CC) { return vol_rec_floats(4, 1 + CC); }

cudaError_t vol_insert(int rho, int level, int CC, const float* rec, const int32_t* order,
                       const int32_t* cell_start, float* M, cudaStream_t s) {
  if (rho != 4) return cudaErrorNotSupported;
  constexpr int RHO = 4;
  const int64_t res = (int64_t)1 << (level + 1), R3 = res * res * res;
  FC2T2_VOL_DISPATCH(CC, FC2T2_LAUNCH("insert", s,
      vol_insert_kernel<RHO, 1 + CC><<<grid_blocks(R3 * (1 + CC), 128, 148 * 64), 128, 0, s>>>(
          rec, R3, order, cell_start, M)));
  return cudaGetLastError();
}

cudaError_t vol_forward(int rho, int level, int CC, const float* L, const double* org,
                        const double* dir, int64_t R, const double* efit, const double* bg,
                        float* rgb, double* depth_final, const uint32_t* seg_offsets,
                        uint8_t* seg_alive, cudaStream_t s, uint32_t* n_alive, double* totals) {
  if (R <= 0) return cudaSuccess;
  if (rho != 4) return cudaErrorNotSupported;
  constexpr int RHO = 4;
  const int blocks = grid_blocks(R, 128, 148 * 32);
  FC2T2_VOL_DISPATCH(CC, FC2T2_LAUNCH("vol_forward", s,
      vol_forward_kernel<RHO, CC><<<blocks, 128, 0, s>>>(L, 1 << (level + 1), org, dir, R, efit,
                                                         bg, rgb, depth_final, seg_offsets,
                                                         seg_alive, n_alive, totals)));
  return cudaGetLastError();
}

cudaError_t vol_totals(int rho, int level, int CC, const float* L, const double* org,
                       const double* dir, int64_t R, const double* efit, uint32_t* n_alive,
                       double* totals, double* depth_final, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  if (rho != 4) return cudaErrorNotSupported;
  constexpr int RHO = 4;
  const int blocks = grid_blocks(R, 128, 148 * 32);
  FC2T2_VOL_DISPATCH(CC, FC2T2_LAUNCH("vol_totals", s,
      vol_totals_kernel<RHO, CC><<<blocks, 128, 0, s>>>(L, 1 << (level + 1), org, dir, R, efit,
                                                        n_alive, totals, depth_final)));
  return cudaGetLastError();
}

cudaError_t vol_payload(int rho, int level, int CC, const float* L, const double* org,
                        const double* dir, int64_t R, const double* efit, const double* bg,
                        const float* ybar, const uint32_t* alive_offsets, const double* totals,
                        const double* depth_final, const double* gl_x, const double* gl_w,
                        uint32_t* keys, float* payload, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  if (rho != 4) return cudaErrorNotSupported;
  constexpr int RHO = 4;
  (void)gl_x;
  (void)gl_w;
  const int blocks = grid_blocks(R, VOL_THREADS, 148 * 32);
  FC2T2_VOL_DISPATCH(CC, FC2T2_LAUNCH("vol_payload", s,
      vol_payload_kernel<RHO, CC><<<blocks, VOL_THREADS, 0, s>>>(
          L, 1 << (level + 1), org, dir, R, efit, bg, ybar, alive_offsets, totals, depth_final,
          keys, payload)));
  return cudaGetLastError();
}

}  // namespace fc2t2
