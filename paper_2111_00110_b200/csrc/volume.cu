// Integral-implicit radiance layer (reference layers.py:405-544) on the device.
//
// Forward, one thread per ray walking its segments in order:
//   sigma, colour polynomials = line2poly of the 1+CC channels (rays.cu),
//   S(x) = int sigma, depth0 = per-ray exclusive prefix of S(s) (float64),
//   alive = depth0 <= 4.5, T(x) = E(S(x) + depth0) with E the degree-4 exp(-x)
//   fit (Horner composition, degree 4(rho+1)), rgb_c += int_0^s c sigma T,
//   rgb_c += E(depth_final) bg_c.
// Backward (volumetric_jvp): pass A recomputes the per-ray totals of
//   int_0^s E'(S + depth0) sigma c; pass B builds, per alive segment, the
//   polynomial weights h_sigma(u) and y_c T sigma and inserts their closed-form
//   segment moments (line2taylor_h = Gauss-Legendre with G = 17 nodes, exact
//   for the degree-33 integrands) -- keys + payload rows, then the generic
//   deterministic insertion.  Polynomial algebra is float64 like the
//   reference; the quadrature moments are float32.
#include "common.cuh"
#include "kernels.cuh"
#include "raywalk.cuh"

namespace fc2t2 {

namespace {

using namespace ray;

constexpr double EXP_CUTOFF = 4.5;     // poly1d.py:22
constexpr double EXP_FIT_RANGE = 5.0;  // poly1d.py:23

template <int RHO>
struct VolCfg {
  static constexpr int NL = RHO + 1;             // line polynomial
  static constexpr int NS = RHO + 2;             // S = int sigma (with constant)
  static constexpr int NT = 4 * (RHO + 1) + 1;   // T = E(S + depth0)
  static constexpr int NTP = 3 * (RHO + 1) + 1;  // T' = E'(S + depth0)
  static constexpr int NCS = 2 * RHO + 1;        // c * sigma
  static constexpr int NI = NCS + NT - 1;        // c sigma T
  static constexpr int NIP = NCS + NTP - 1;      // c sigma T'
  static constexpr int NH = NI + 1;              // h_sigma (= antiderivative length)
  static constexpr int NTS = NT + NL - 1;        // T sigma, T c
  static constexpr int G = (RHO + NH - 1) / 2 + 1;  // Gauss nodes (ray.py:236)
};

template <int NA, int NB>
__device__ __forceinline__ void pmul(const double (&a)[NA], const double (&b)[NB],
                                     double (&o)[NA + NB - 1]) {
#pragma unroll
  for (int k = 0; k < NA + NB - 1; ++k) o[k] = 0.0;
#pragma unroll
  for (int i = 0; i < NA; ++i)
#pragma unroll
    for (int j = 0; j < NB; ++j) o[i + j] = fma(a[i], b[j], o[i + j]);
}

template <int N>
__device__ __forceinline__ double peval(const double (&a)[N], double x) {
  double y = 0.0;
#pragma unroll
  for (int k = N - 1; k >= 0; --k) y = fma(y, x, a[k]);
  return y;
}

// int_0^x of the polynomial a, evaluated at x
template <int N>
__device__ __forceinline__ double pint_eval(const double (&a)[N], double x) {
  double v = 0.0;
#pragma unroll
  for (int k = N - 1; k >= 0; --k) v = (v + a[k] / (double)(k + 1)) * x;
  return v;
}

// out = E(g(x)), E of NE coefficients, Horner in g (layers.py:77-83)
template <int NE, int NG>
__device__ __forceinline__ void compose(const double* e, const double (&g)[NG],
                                        double (&out)[(NE - 1) * (NG - 1) + 1]) {
  constexpr int NO = (NE - 1) * (NG - 1) + 1;
#pragma unroll
  for (int k = 0; k < NO; ++k) out[k] = 0.0;
  out[0] = e[NE - 1];
#pragma unroll
  for (int k = NE - 2; k >= 0; --k) {
    const int deg = (NE - 2 - k) * (NG - 1);  // current degree of out
    double tmp[NO];
#pragma unroll
    for (int i = 0; i < NO; ++i) tmp[i] = 0.0;
#pragma unroll
    for (int i = 0; i < NO; ++i)
#pragma unroll
      for (int j = 0; j < NG; ++j)
        if (i <= deg && i + j < NO) tmp[i + j] = fma(out[i], g[j], tmp[i + j]);
    tmp[0] += e[k];
#pragma unroll
    for (int i = 0; i < NO; ++i) out[i] = tmp[i];
  }
}

template <int RHO>
__device__ __forceinline__ void line_poly_d(const float* row, const float base[3],
                                            const float dirf[3], double (&out)[RHO + 1]) {
  float pf[RHO + 1];
  line_poly<RHO>(row, base, dirf, pf);
#pragma unroll
  for (int j = 0; j <= RHO; ++j) out[j] = (double)pf[j];
}

__device__ __forceinline__ double mexp_clamped(const double* e, double x) {
  if (x > EXP_FIT_RANGE) return 0.0;
  double y = 0.0;
  for (int k = 4; k >= 0; --k) y = y * x + e[k];
  return y;
}

// ------------------------------------------------------------- forward ---
template <int RHO, int CC>
__global__ void __launch_bounds__(128)
vol_forward_kernel(const float* __restrict__ L, int res, const double* __restrict__ org,
                   const double* __restrict__ dir, int64_t R, const double* __restrict__ efit,
                   const double* __restrict__ bg, float* __restrict__ rgb,
                   double* __restrict__ depth_final, const uint32_t* __restrict__ seg_offsets,
                   uint8_t* __restrict__ seg_alive) {
  using V = VolCfg<RHO>;
  constexpr int PP = MI<RHO>::PP, NCH = 1 + CC;
  double e[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) e[k] = efit[k];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    const float dirf[3] = {(float)d[0], (float)d[1], (float)d[2]};
    double depth = 0.0, dfin = 0.0, acc[CC];
#pragma unroll
    for (int c = 0; c < CC; ++c) acc[c] = 0.0;
    int64_t j = seg_offsets ? (int64_t)seg_offsets[r] : 0;
    walk_ray(o, d, res, [&](double t0, double t1, int b0, int b1, int b2) {
      float base[3];
      seg_base(o, d, t0, b0, b1, b2, res, base);
      const float* row = L + (((int64_t)b0 * res + b1) * res + b2) * NCH * PP;
      double sg[V::NL];
      line_poly_d<RHO>(row, base, dirf, sg);
      double S[V::NS];
      S[0] = 0.0;
#pragma unroll
      for (int k = 0; k < V::NL; ++k) S[k + 1] = sg[k] / (double)(k + 1);
      const double s = t1 - t0;
      const double send = peval(S, s);
      const bool alive = depth <= EXP_CUTOFF;
      if (alive) {
        double gpoly[V::NS];
#pragma unroll
        for (int k = 0; k < V::NS; ++k) gpoly[k] = S[k];
        gpoly[0] += depth;
        double T[V::NT];
        compose<5, V::NS>(e, gpoly, T);
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          double col[V::NL], cs[V::NCS], integ[V::NI];
          line_poly_d<RHO>(row + (1 + c) * PP, base, dirf, col);
          pmul(col, sg, cs);
          pmul(cs, T, integ);
          acc[c] += pint_eval(integ, s);
        }
        dfin += send;
      }
      if (seg_alive) seg_alive[j++] = alive ? 1 : 0;
      depth += send;
      return true;
    });
    const double te = mexp_clamped(e, dfin);
#pragma unroll
    for (int c = 0; c < CC; ++c) rgb[r * CC + c] = (float)(acc[c] + te * bg[c]);
    depth_final[r] = dfin;
  }
}

// ------------------------------------------------- backward pass A ---
// per ray: number of alive segments and totals of int_0^s c sigma T'
template <int RHO, int CC>
__global__ void __launch_bounds__(128)
vol_totals_kernel(const float* __restrict__ L, int res, const double* __restrict__ org,
                  const double* __restrict__ dir, int64_t R, const double* __restrict__ efit,
                  uint32_t* __restrict__ n_alive, double* __restrict__ totals,
                  double* __restrict__ depth_final) {
  using V = VolCfg<RHO>;
  constexpr int PP = MI<RHO>::PP, NCH = 1 + CC;
  double ep[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) ep[k] = efit[k + 1] * (double)(k + 1);
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
      double sg[V::NL];
      line_poly_d<RHO>(row, base, dirf, sg);
      double S[V::NS];
      S[0] = 0.0;
#pragma unroll
      for (int k = 0; k < V::NL; ++k) S[k + 1] = sg[k] / (double)(k + 1);
      const double s = t1 - t0;
      const double send = peval(S, s);
      if (depth <= EXP_CUTOFF) {
        double gpoly[V::NS];
#pragma unroll
        for (int k = 0; k < V::NS; ++k) gpoly[k] = S[k];
        gpoly[0] += depth;
        double Tp[V::NTP];
        compose<4, V::NS>(ep, gpoly, Tp);
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          double col[V::NL], cs[V::NCS], ip[V::NIP];
          line_poly_d<RHO>(row + (1 + c) * PP, base, dirf, col);
          pmul(col, sg, cs);
          pmul(cs, Tp, ip);
          tot[c] += pint_eval(ip, s);
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
template <int RHO, int CC>
__global__ void __launch_bounds__(128)
vol_payload_kernel(const float* __restrict__ L, int res, const double* __restrict__ org,
                   const double* __restrict__ dir, int64_t R, const double* __restrict__ efit,
                   const double* __restrict__ bg, const float* __restrict__ ybar,
                   const uint32_t* __restrict__ alive_offsets, const double* __restrict__ totals,
                   const double* __restrict__ depth_final, const double* __restrict__ gl_x,
                   const double* __restrict__ gl_w, uint32_t* __restrict__ keys,
                   float* __restrict__ payload) {
  using V = VolCfg<RHO>;
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP, NCH = 1 + CC, G = V::G;
  double e[5], ep[4];
#pragma unroll
  for (int k = 0; k < 5; ++k) e[k] = efit[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) ep[k] = efit[k + 1] * (double)(k + 1);
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    double o[3], d[3];
    load_ray(org, dir, r, o, d);
    const float dirf[3] = {(float)d[0], (float)d[1], (float)d[2]};
    const double dfin = depth_final[r];
    // E'(depth_final), 0 beyond the fit range (layers.py:510-511)
    const double tp_inf = dfin > EXP_FIT_RANGE ? 0.0 : ((ep[3] * dfin + ep[2]) * dfin + ep[1]) * dfin + ep[0];
    double yb[CC], before[CC], konst = 0.0;
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
      double sg[V::NL];
      line_poly_d<RHO>(row, base, dirf, sg);
      double S[V::NS];
      S[0] = 0.0;
#pragma unroll
      for (int k = 0; k < V::NL; ++k) S[k + 1] = sg[k] / (double)(k + 1);
      const double s = t1 - t0;
      const double send = peval(S, s);
      if (depth <= EXP_CUTOFF) {
        double gpoly[V::NS];
#pragma unroll
        for (int k = 0; k < V::NS; ++k) gpoly[k] = S[k];
        gpoly[0] += depth;
        double T[V::NT], Tp[V::NTP];
        compose<5, V::NS>(e, gpoly, T);
        compose<4, V::NS>(ep, gpoly, Tp);
        // h_sigma = sum_c y_c [T c - int_0^u E'(S) sigma c + const_c]  (layers.py:513-527)
        double h[V::NH];
#pragma unroll
        for (int k = 0; k < V::NH; ++k) h[k] = 0.0;
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          double col[V::NL], tc[V::NTS], cs[V::NCS], ip[V::NIP];
          line_poly_d<RHO>(row + (1 + c) * PP, base, dirf, col);
          pmul(T, col, tc);
#pragma unroll
          for (int k = 0; k < V::NTS; ++k) h[k] = fma(yb[c], tc[k], h[k]);
          pmul(col, sg, cs);
          pmul(cs, Tp, ip);
          // antiderivative of ip (zero constant) subtracted
#pragma unroll
          for (int k = 0; k < V::NIP; ++k) h[k + 1] -= yb[c] * ip[k] / (double)(k + 1);
          const double cp = pint_eval(ip, s);
          h[0] += yb[c] * (totals[r * CC + c] - before[c] + tp_inf * bg[c]);
          before[c] += cp;
        }
        double tsig[V::NTS];
        pmul(T, sg, tsig);
        // per-node weights of the NCH payload channels
        const double half = 0.5 * s;
        float wn[NCH][G];
        float nx[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const double t = half * (gl_x[g] + 1.0);
          const double W = half * gl_w[g];
          nx[g] = (float)t;
          wn[0][g] = (float)(W * peval(h, t));
          const double ts = W * peval(tsig, t);
#pragma unroll
          for (int c = 0; c < CC; ++c) wn[1 + c][g] = (float)(yb[c] * ts);
        }
        keys[item] = ((uint32_t)b0 * res + b1) * res + b2;
#pragma unroll 1
        for (int ch = 0; ch < NCH; ++ch) {
          float acc[P];
#pragma unroll
          for (int k = 0; k < P; ++k) acc[k] = 0.f;
#pragma unroll 1
          for (int g = 0; g < G; ++g) {
            float mono[P];
            monomials<RHO>(fmaf(nx[g], dirf[0], base[0]), fmaf(nx[g], dirf[1], base[1]),
                           fmaf(nx[g], dirf[2], base[2]), mono);
            const float wt = wn[ch][g];
#pragma unroll
            for (int k = 0; k < P; ++k) acc[k] = fmaf(wt, mono[k], acc[k]);
          }
          float* dst = payload + (item * NCH + ch) * PP;
#pragma unroll
          for (int k = 0; k < PP; k += 4)
            *reinterpret_cast<float4*>(dst + k) =
                make_float4(k < P ? acc[k] : 0.f, k + 1 < P ? acc[k + 1] : 0.f,
                            k + 2 < P ? acc[k + 2] : 0.f, k + 3 < P ? acc[k + 3] : 0.f);
        }
        ++item;
      }
      depth += send;
      return true;
    });
    (void)konst;
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

int vol_gauss_nodes(int rho) { return rho == 4 ? VolCfg<4>::G : (rho == 3 ? VolCfg<3>::G : (rho == 2 ? VolCfg<2>::G : VolCfg<1>::G)); }

cudaError_t vol_forward(int rho, int level, int CC, const float* L, const double* org,
                        const double* dir, int64_t R, const double* efit, const double* bg,
                        float* rgb, double* depth_final, const uint32_t* seg_offsets,
                        uint8_t* seg_alive, cudaStream_t s) {
  if (R <= 0) return cudaSuccess;
  if (rho != 4) return cudaErrorNotSupported;
  constexpr int RHO = 4;
  const int blocks = grid_blocks(R, 128, 148 * 32);
  FC2T2_VOL_DISPATCH(CC, FC2T2_LAUNCH("vol_forward", s,
      vol_forward_kernel<RHO, CC><<<blocks, 128, 0, s>>>(L, 1 << (level + 1), org, dir, R, efit,
                                                         bg, rgb, depth_final, seg_offsets,
                                                         seg_alive)));
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
  const int blocks = grid_blocks(R, 128, 148 * 32);
  FC2T2_VOL_DISPATCH(CC, FC2T2_LAUNCH("vol_payload", s,
      vol_payload_kernel<RHO, CC><<<blocks, 128, 0, s>>>(
          L, 1 << (level + 1), org, dir, R, efit, bg, ybar, alive_offsets, totals, depth_final,
          gl_x, gl_w, keys, payload)));
  return cudaGetLastError();
}

}  // namespace fc2t2
