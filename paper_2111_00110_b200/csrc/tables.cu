// On-device fitting of the M2L translation tables.
//
// The reference fits every active offset's table on the host in float64
// (kernel.py:180-204): A(o) = pinv(V) Psi(o) pinv(V)^T over a G^3 Chebyshev
// tensor grid per box, stored transposed as coeffs[o] = A^T [k_local][n_moment],
// with the fit residual max |V A V^T - Psi| (kernel.py:202).  Psi(o) is the
// Kronecker product of three per-axis G x G node-pair kernels
//     e_a[p][q] = exp(-alpha (o_a w + x_p - x_q)^2),
// so the two-sided product is applied one axis at a time (3 G-point passes
// per row of pinv(V)) instead of forming the G^3 x G^3 pair matrix.
//
// One CTA per offset, float64 throughout (the tables feed a float64 host
// copy and the fp32 / split-fp16 device tables).  pinv(V) and V (G^3 x P)
// are computed once per level on the host (one small SVD) and read here
// through L2.  Shared memory per CTA: the P x G^3 row block (the contracted
// rows, later A V^T) plus A itself: 70 KB at rho = 4, 201 KB at rho = 6.
#include <cmath>

#include "../../include/fc2t2_b200.h"
#include "common.cuh"

namespace fc2t2 {
namespace {

constexpr int FIT_THREADS = 256;
constexpr int FIT_WARPS = FIT_THREADS / 32;
constexpr int G = 6;                 // Chebyshev nodes per axis (reference default)
constexpr int G3 = G * G * G;

__device__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// pv: (P, G^3) row-major = pinv(V) reshaped (P, gx, gy, gz); v: (G^3, P);
// x1: G node coordinates (already scaled by width / 2); offsets: (K, 3).
__global__ void __launch_bounds__(FIT_THREADS) fit_tables_kernel(
    int P, const double* __restrict__ pv, const double* __restrict__ v,
    const double* __restrict__ x1, double alpha, double width, const int32_t* __restrict__ offsets,
    double* __restrict__ coeffs, double* __restrict__ resid) {
  extern __shared__ double sm[];
  double* W = sm;                          // P x G3: contracted rows, then A V^T
  double* A = W + (size_t)P * G3;          // P x P: A[n][k]
  double* tmp = A + (size_t)P * P;         // FIT_WARPS x G3 per-warp scratch
  __shared__ double e[3][G][G];
  __shared__ double red[FIT_WARPS];
  const int o = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid < 3 * G * G) {
    const int a = tid / (G * G), p = (tid / G) % G, q = tid % G;
    const double d = offsets[3 * o + a] * width + x1[p] - x1[q];
    e[a][p][q] = exp(-alpha * d * d);
  }
  __syncthreads();

  // rows k of pinv(V): w[k,a,b,c] = sum_xyz ex[a,x] ey[b,y] ez[c,z] pv[k,x,y,z]
  double* t = tmp + warp * G3;
  for (int k = warp; k < P; k += FIT_WARPS) {
    const double* src = pv + (size_t)k * G3;
    double* row = W + (size_t)k * G3;
    for (int i = lane; i < G3; i += 32) {           // z pass: t[x,y,c]
      const int x = i / (G * G), y = (i / G) % G, c = i % G;
      const double* s = src + (x * G + y) * G;
      double acc = 0.0;
#pragma unroll
      for (int z = 0; z < G; ++z) acc = fma(e[2][c][z], __ldg(s + z), acc);
      t[i] = acc;
    }
    __syncwarp();
    for (int i = lane; i < G3; i += 32) {           // y pass: row[x,b,c]
      const int x = i / (G * G), b = (i / G) % G, c = i % G;
      double acc = 0.0;
#pragma unroll
      for (int y = 0; y < G; ++y) acc = fma(e[1][b][y], t[(x * G + y) * G + c], acc);
      row[i] = acc;
    }
    __syncwarp();
    for (int i = lane; i < G3; i += 32) {           // x pass: t[a,b,c]
      const int a = i / (G * G), bc = i % (G * G);
      double acc = 0.0;
#pragma unroll
      for (int x = 0; x < G; ++x) acc = fma(e[0][a][x], row[x * G * G + bc], acc);
      t[i] = acc;
    }
    __syncwarp();
    for (int i = lane; i < G3; i += 32) row[i] = t[i];
    __syncwarp();
  }
  __syncthreads();

  // A[n][k] = sum_i pv[n,i] w[k,i]; stored transposed: coeffs[o][k][n]
  double* out = coeffs + (size_t)o * P * P;
  for (int q = tid; q < P * P; q += FIT_THREADS) {
    const int n = q / P, k = q % P;
    const double* pn = pv + (size_t)n * G3;
    const double* wk = W + (size_t)k * G3;
    double acc = 0.0;
    for (int i = 0; i < G3; ++i) acc = fma(__ldg(pn + i), wk[i], acc);
    A[n * P + k] = acc;
    out[k * P + n] = acc;
  }
  __syncthreads();

  // residual max |V A V^T - Psi|: B[n][j] = sum_k A[n][k] V[j][k] (into W)
  for (int q = tid; q < P * G3; q += FIT_THREADS) {
    const int n = q / G3, j = q % G3;
    const double* vj = v + (size_t)j * P;
    double acc = 0.0;
    for (int k = 0; k < P; ++k) acc = fma(A[n * P + k], __ldg(vj + k), acc);
    W[q] = acc;
  }
  __syncthreads();
  double worst = 0.0;
  for (int q = tid; q < G3 * G3; q += FIT_THREADS) {
    const int i = q / G3, j = q % G3;
    const double* vi = v + (size_t)i * P;
    double acc = 0.0;
    for (int n = 0; n < P; ++n) acc = fma(__ldg(vi + n), W[(size_t)n * G3 + j], acc);
    const double psi = e[0][i / (G * G)][j / (G * G)] * e[1][(i / G) % G][(j / G) % G] *
                       e[2][i % G][j % G];
    worst = fmax(worst, fabs(acc - psi));
  }
  worst = warp_max(worst);
  if (lane == 0) red[warp] = worst;
  __syncthreads();
  if (tid == 0) {
    double m = red[0];
    for (int w = 1; w < FIT_WARPS; ++w) m = fmax(m, red[w]);
    resid[o] = m;
  }
}

size_t fit_smem(int P) { return ((size_t)P * G3 + (size_t)P * P + FIT_WARPS * G3) * sizeof(double); }

}  // namespace
}  // namespace fc2t2

extern "C" size_t fc2t2_fit_tables_smem(int rho) {
  const int P = (rho + 1) * (rho + 2) * (rho + 3) / 6;
  return fc2t2::fit_smem(P);
}

extern "C" int fc2t2_fit_tables(int rho, int nodes, const double* d_pinv, const double* d_v,
                                const double* d_nodes, double alpha, double width,
                                const int32_t* d_offsets, int64_t count, double* d_coeffs,
                                double* d_resid, void* stream) {
  using namespace fc2t2;
  if (rho < 1 || rho > 6) return FC2T2_EORDER;
  if (nodes != G || count < 0 || !(alpha > 0.0) || !(width > 0.0)) return FC2T2_EVALUE;
  if (count == 0) return FC2T2_OK;
  const int P = (rho + 1) * (rho + 2) * (rho + 3) / 6;
  const size_t smem = fit_smem(P);
  static unsigned long long attr = 0;   // devices configured, for the largest rho
  if (attr_needed(attr)) {
    if (cudaFuncSetAttribute(fit_tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)fit_smem(84)) != cudaSuccess)
      return FC2T2_ECUDA;
  }
  cudaStream_t s = (cudaStream_t)stream;
  FC2T2_LAUNCH("fit_tables", s,
               fit_tables_kernel<<<(unsigned)count, FIT_THREADS, smem, s>>>(
                   P, d_pinv, d_v, d_nodes, alpha, width, d_offsets, d_coeffs, d_resid));
  return cudaGetLastError() == cudaSuccess ? FC2T2_OK : FC2T2_ECUDA;
}
