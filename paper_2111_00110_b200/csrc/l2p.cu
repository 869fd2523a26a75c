// L2P: evaluate the finest local expansions at free points.
//
// Reference: Accessor._local/value/partials/partials2 (expansion.py:335-373):
// bit-exact box lookup, in-box offset d, then per channel the contractions
// value = sum_n A_n d^n / n!, the gradient (coefficient shift n -> n + e_a,
// reference _shift_indices :309-329) and the Hessian (xx yy zz xy xz yz).
// L2P_WGRAD fuses the adjoint contraction sum_c wts_c grad f_c used by the
// explicit layer's q_bar and p_bar (reference layers.py:183, :186-187).
//
// Row fetch (warp-cooperative): a thread-per-point gather makes every float4
// load instruction of a warp touch 32 different cell rows.  Here the warp
// copies its 32 points' rows into shared memory with consecutive lanes on
// consecutive 16-byte pieces of the same row (~2.5 rows per instruction),
// then each thread reads its own row back (row stride PP words: the 8 lanes
// of a 128-bit shared access hit distinct bank quads for PP = 4, 12, 20, 36,
// 84).
//
// Contraction (nested, no monomial table): with X_a = dx^a/a!, Y_b, Z_c,
//   T[a][b]  = sum_c Z_c A[a,b,c]          S[a]  = sum_b Y_b T[a][b]
//   value    = sum_a X_a S[a]
//   d/dx     = sum_{a>=1} X_{a-1} S[a]      d/dy = sum_a X_a sum_{b>=1} Y_{b-1} T[a][b]
//   d/dz     = sum_a X_a sum_b Y_b sum_{c>=1} Z_{c-1} A[a,b,c]
// (and the second derivatives alike): 55 + 30 + 15 FMAs for value + gradient
// at rho = 4 instead of a 35-entry monomial table (105 multiplies) and four
// 35-term dot products -- half the registers, twice the resident warps.
// With a cell-sorted `order`, thread t evaluates point order[t] (outputs
// stay indexed by point).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.cuh"

#include <cstring>

namespace fc2t2 {

namespace {

__device__ __forceinline__ void l2p_cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// sum_c Z[c - s] A[a, b, c] over c >= s (s = 0, 1, 2: the z shift)
template <int RHO, int S>
__device__ __forceinline__ float zsum(const float (&A)[MI<RHO>::PP], const float (&Z)[RHO + 1],
                                      int a, int b) {
  float t = 0.f;
#pragma unroll
  for (int c = S; c <= RHO - a - b; ++c) t = fmaf(Z[c - S], A[MI<RHO>::index(a, b, c)], t);
  return t;
}

// One point, one channel: value / gradient / Hessian of its cell row A.
template <int RHO, int MODE>
__device__ __forceinline__ void l2p_nested(const float (&A)[MI<RHO>::PP], const float (&X)[RHO + 1],
                                           const float (&Y)[RHO + 1], const float (&Z)[RHO + 1],
                                           float& v, float (&g)[3], float (&h)[6]) {
  constexpr bool G = (MODE & (L2P_GRAD | L2P_WGRAD)) != 0, H = (MODE & L2P_HESS) != 0;
  float S[RHO + 1], Sy[RHO + 1], Sz[RHO + 1], Syy[RHO + 1], Szz[RHO + 1], Syz[RHO + 1];
#pragma unroll
  for (int a = 0; a <= RHO; ++a) {
    float s = 0.f, sy = 0.f, sz = 0.f, syy = 0.f, szz = 0.f, syz = 0.f;
#pragma unroll
    for (int b = 0; b <= RHO - a; ++b) {
      const float t = zsum<RHO, 0>(A, Z, a, b);
      s = fmaf(Y[b], t, s);
      if constexpr (G || H) {
        if (b >= 1) sy = fmaf(Y[b - 1], t, sy);
        const float tz = zsum<RHO, 1>(A, Z, a, b);
        sz = fmaf(Y[b], tz, sz);
        if constexpr (H) {
          if (b >= 2) syy = fmaf(Y[b - 2], t, syy);
          if (b >= 1) syz = fmaf(Y[b - 1], tz, syz);
          szz = fmaf(Y[b], zsum<RHO, 2>(A, Z, a, b), szz);
        }
      }
    }
    S[a] = s; Sy[a] = sy; Sz[a] = sz; Syy[a] = syy; Szz[a] = szz; Syz[a] = syz;
  }
  v = 0.f;
#pragma unroll
  for (int a = 0; a <= RHO; ++a) v = fmaf(X[a], S[a], v);
  if constexpr (G || H) {
    g[0] = g[1] = g[2] = 0.f;
#pragma unroll
    for (int a = 0; a <= RHO; ++a) {
      if (a >= 1) g[0] = fmaf(X[a - 1], S[a], g[0]);
      g[1] = fmaf(X[a], Sy[a], g[1]);
      g[2] = fmaf(X[a], Sz[a], g[2]);
    }
  }
  if constexpr (H) {
#pragma unroll
    for (int d = 0; d < 6; ++d) h[d] = 0.f;
#pragma unroll
    for (int a = 0; a <= RHO; ++a) {
      if (a >= 2) h[0] = fmaf(X[a - 2], S[a], h[0]);     // xx
      h[1] = fmaf(X[a], Syy[a], h[1]);                     // yy
      h[2] = fmaf(X[a], Szz[a], h[2]);                     // zz
      if (a >= 1) h[3] = fmaf(X[a - 1], Sy[a], h[3]);     // xy
      if (a >= 1) h[4] = fmaf(X[a - 1], Sz[a], h[4]);     // xz
      h[5] = fmaf(X[a], Syz[a], h[5]);                     // yz
    }
  }
}

template <int RHO>
__device__ __forceinline__ void axis_table(float d, float (&T)[RHO + 1]) {
  T[0] = 1.f;
#pragma unroll
  for (int k = 1; k <= RHO; ++k) T[k] = T[k - 1] * d * (1.f / (float)k);
}

template <int RHO, int MODE>
constexpr int l2p_min_blocks() {
#ifdef FC2T2_L2P_MINB
  return (RHO <= 4 && !(MODE & L2P_HESS)) ? FC2T2_L2P_MINB : 2;
#else
  // 4 with the TMA row fetch (10^7-point value + grad: 190 us at 4 blocks,
  // 212 at 3, 256 at 2; the cp.async fetch was L1/TEX bound and slower at 4)
  return (RHO <= 4 && !(MODE & L2P_HESS)) ? 4 : 2;
#endif
}

template <int RHO, int MODE>
__global__ void __launch_bounds__(256, (l2p_min_blocks<RHO, MODE>()))
l2p_kernel(const float* __restrict__ L, const float* __restrict__ q, int64_t n, int C, int res,
           const int32_t* __restrict__ order, const float* __restrict__ wts,
           float* __restrict__ value, float* __restrict__ grad, float* __restrict__ hess,
           float* __restrict__ wgrad, int32_t* __restrict__ flag) {
  constexpr int PP = MI<RHO>::PP, F4 = PP / 4;
  extern __shared__ __align__(16) float l2p_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* rows = l2p_smem + warp * 32 * PP;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  int bad = 0;
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32; base < n;
       base += warps_total * 32) {
    const int64_t t = base + lane;
    const bool valid = t < n;
    const int64_t i = valid ? (order ? (int64_t)order[t] : t) : 0;
    float x = 0.f, y = 0.f, z = 0.f;
    if (valid) { x = q[3 * i]; y = q[3 * i + 1]; z = q[3 * i + 2]; }
    bad |= valid && outside_domain(x, y, z);
    const int b0 = box_axis(x, res), b1 = box_axis(y, res), b2 = box_axis(z, res);
    float X[RHO + 1], Y[RHO + 1], Z[RHO + 1];
    axis_table<RHO>(box_offset(x, b0, res), X);
    axis_table<RHO>(box_offset(y, b1, res), Y);
    axis_table<RHO>(box_offset(z, b2, res), Z);
    const int64_t rowoff = ((((int64_t)b0 * res + b1) * res + b2) * C) * PP;
    float wg0 = 0.f, wg1 = 0.f, wg2 = 0.f;
    for (int c = 0; c < C; ++c) {
      // the tangent weight is read before the copy wait so its latency
      // overlaps the row fetch
      const float wv = ((MODE & L2P_WGRAD) && valid) ? wts[i * C + c] : 0.f;
#pragma unroll
      for (int k = 0; k < F4; ++k) {
        const int j = k * 32 + lane;
        const int pt = j / F4, f = j - pt * F4;
        const int64_t src = __shfl_sync(0xffffffffu, rowoff, pt);
        l2p_cp_async16(rows + pt * PP + 4 * f, L + src + c * PP + 4 * f);
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
      float A[PP];
#pragma unroll
      for (int k = 0; k < PP; k += 4) {
        const float4 v4 = *reinterpret_cast<const float4*>(rows + lane * PP + k);
        A[k] = v4.x; A[k + 1] = v4.y; A[k + 2] = v4.z; A[k + 3] = v4.w;
      }
      __syncwarp();
      float v, g[3], h[6];
      l2p_nested<RHO, MODE>(A, X, Y, Z, v, g, h);
      if (valid) {
        if constexpr (MODE & L2P_VALUE) value[i * C + c] = v;
        if constexpr (MODE & L2P_GRAD) {
          grad[(i * C + c) * 3 + 0] = g[0];
          grad[(i * C + c) * 3 + 1] = g[1];
          grad[(i * C + c) * 3 + 2] = g[2];
        }
        if constexpr (MODE & L2P_HESS) {
#pragma unroll
          for (int d = 0; d < 6; ++d) hess[(i * C + c) * 6 + d] = h[d];
        }
        if constexpr (MODE & L2P_WGRAD) {
          wg0 = fmaf(wv, g[0], wg0);
          wg1 = fmaf(wv, g[1], wg1);
          wg2 = fmaf(wv, g[2], wg2);
        }
      }
    }
    if constexpr (MODE & L2P_WGRAD) {
      if (valid) {
        wgrad[3 * i + 0] = wg0;
        wgrad[3 * i + 1] = wg1;
        wgrad[3 * i + 2] = wg2;
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

// Row fetch by TMA gather4 (FC2T2_L2P_TMA): lanes 0..7 of a warp each load
// four of its 32 points' rows (a 2-D tensor map over the grid as
// [cells * C, PP] floats) straight into shared memory -- the L1/TEX pipe
// then only serves the read-back.
struct L2PMap {
  CUtensorMap m;
};

template <int RHO, int MODE>
__global__ void __launch_bounds__(256, (l2p_min_blocks<RHO, MODE>()))
l2p_tma_kernel(const __grid_constant__ L2PMap map, const float* __restrict__ q, int64_t n, int C,
               int res, const int32_t* __restrict__ order, const float* __restrict__ wts,
               float* __restrict__ value, float* __restrict__ grad, float* __restrict__ hess,
               float* __restrict__ wgrad, int32_t* __restrict__ flag) {
  constexpr int PP = MI<RHO>::PP;
  constexpr int GS = (4 * PP * 4 + 127) / 128 * 32;   // floats per 128-byte aligned group of 4 rows
  extern __shared__ __align__(128) float l2p_tma_smem_raw[];
  __shared__ __align__(8) uint64_t bars[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* sm0 = reinterpret_cast<float*>(
      reinterpret_cast<unsigned char*>(l2p_tma_smem_raw) +
      ((128 - ((unsigned)__cvta_generic_to_shared(l2p_tma_smem_raw) & 127)) & 127));
  float* rows = sm0 + warp * 8 * GS;   // group k = points 4k..4k+3 at k * GS
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[warp]);
  const uint32_t dst = (uint32_t)__cvta_generic_to_shared(rows);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  uint32_t phase = 0;
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  int bad = 0;
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + warp) * 32; base < n;
       base += warps_total * 32) {
    const int64_t t = base + lane;
    const bool valid = t < n;
    const int64_t i = valid ? (order ? (int64_t)order[t] : t) : 0;
    float x = 0.f, y = 0.f, z = 0.f;
    if (valid) { x = q[3 * i]; y = q[3 * i + 1]; z = q[3 * i + 2]; }
    bad |= valid && outside_domain(x, y, z);
    const int b0 = box_axis(x, res), b1 = box_axis(y, res), b2 = box_axis(z, res);
    float X[RHO + 1], Y[RHO + 1], Z[RHO + 1];
    axis_table<RHO>(box_offset(x, b0, res), X);
    axis_table<RHO>(box_offset(y, b1, res), Y);
    axis_table<RHO>(box_offset(z, b2, res), Z);
    const int cellrow = ((b0 * res + b1) * res + b2) * C;
    float wg0 = 0.f, wg1 = 0.f, wg2 = 0.f;
    for (int c = 0; c < C; ++c) {
      const float wv = ((MODE & L2P_WGRAD) && valid) ? wts[i * C + c] : 0.f;
      const int r = cellrow + c;
      const int r0 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4);
      const int r1 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4 + 1);
      const int r2 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4 + 2);
      const int r3 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4 + 3);
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar),
                     "r"(32 * PP * 4));
      __syncwarp();
      if (lane < 8) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
            "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst + lane * GS * 4),
            "l"(reinterpret_cast<uint64_t>(&map.m)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
            "r"(bar)
            : "memory");
      }
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "L2PW_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra L2PW_%=;\n\t}\n" ::"r"(bar),
          "r"(phase)
          : "memory");
      phase ^= 1u;
      float A[PP];
#pragma unroll
      for (int k = 0; k < PP; k += 4) {
        const float4 v4 =
            *reinterpret_cast<const float4*>(rows + (lane >> 2) * GS + (lane & 3) * PP + k);
        A[k] = v4.x; A[k + 1] = v4.y; A[k + 2] = v4.z; A[k + 3] = v4.w;
      }
      __syncwarp();
      float v, g[3], h[6];
      l2p_nested<RHO, MODE>(A, X, Y, Z, v, g, h);
      if (valid) {
        if constexpr (MODE & L2P_VALUE) value[i * C + c] = v;
        if constexpr (MODE & L2P_GRAD) {
          grad[(i * C + c) * 3 + 0] = g[0];
          grad[(i * C + c) * 3 + 1] = g[1];
          grad[(i * C + c) * 3 + 2] = g[2];
        }
        if constexpr (MODE & L2P_HESS) {
#pragma unroll
          for (int d = 0; d < 6; ++d) hess[(i * C + c) * 6 + d] = h[d];
        }
        if constexpr (MODE & L2P_WGRAD) {
          wg0 = fmaf(wv, g[0], wg0);
          wg1 = fmaf(wv, g[1], wg1);
          wg2 = fmaf(wv, g[2], wg2);
        }
      }
    }
    if constexpr (MODE & L2P_WGRAD) {
      if (valid) {
        wgrad[3 * i + 0] = wg0;
        wgrad[3 * i + 1] = wg1;
        wgrad[3 * i + 2] = wg2;
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

template <int RHO>
constexpr int l2p_tma_smem() {
  return 8 * 8 * ((4 * MI<RHO>::PP * 4 + 127) / 128 * 128) + 128;
}

// 2-D tensor map [rows = cells * C, PP floats] over the grid; false on failure
template <int RHO>
bool l2p_map(L2PMap& out, const float* L, int res, int C) {
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tensor_map_encoder());
  if (!enc) return false;
  constexpr int PP = MI<RHO>::PP;
  const cuuint64_t rows = (cuuint64_t)res * res * res * C;
  cuuint64_t dims[2] = {(cuuint64_t)PP, rows};
  cuuint64_t strides[1] = {(cuuint64_t)PP * 4};
  cuuint32_t box[2] = {(cuuint32_t)PP, 1}, es[2] = {1, 1};
  std::memset(&out, 0, sizeof(out));
  return enc(&out.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(L), dims, strides, box,
             es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int RHO, int M>
cudaError_t l2p_launch(int blocks, int C, int res, const float* L, const float* q, int64_t n,
                       const int32_t* order, const float* wts, float* value, float* grad,
                       float* hess, float* wgrad, int32_t* flag, cudaStream_t s) {
  constexpr int smem = 8 * 32 * MI<RHO>::PP * (int)sizeof(float);
  static unsigned long long configured = 0;
  if (smem > 48 * 1024 && attr_needed(configured)) {
    const cudaError_t e = cudaFuncSetAttribute(l2p_kernel<RHO, M>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
#ifndef FC2T2_L2P_NO_TMA
  {
    L2PMap map;
    if ((int64_t)res * res * res * C < (int64_t)INT32_MAX && l2p_map<RHO>(map, L, res, C)) {
      constexpr int tsm = l2p_tma_smem<RHO>();
      static unsigned long long cfg2 = 0;
      if (tsm > 48 * 1024 && attr_needed(cfg2)) {
        const cudaError_t e = cudaFuncSetAttribute(
            l2p_tma_kernel<RHO, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, tsm);
        if (e != cudaSuccess) return e;
      }
      FC2T2_LAUNCH("l2p", s, l2p_tma_kernel<RHO, M><<<blocks, 256, tsm, s>>>(
          map, q, n, C, res, order, wts, value, grad, hess, wgrad, flag));
      return cudaGetLastError();
    }
  }
#endif
  FC2T2_LAUNCH("l2p", s, l2p_kernel<RHO, M><<<blocks, 256, smem, s>>>(
      L, q, n, C, res, order, wts, value, grad, hess, wgrad, flag));
  return cudaGetLastError();
}

template <int RHO>
cudaError_t l2p_rho(int level, int C, const float* L, const float* q, int64_t n, int mode,
                    const int32_t* order, const float* wts, float* value, float* grad,
                    float* hess, float* wgrad, int32_t* flag, cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int blocks = grid_blocks(n, 256, 148 * 16);
#define FC2T2_L2P_CASE(M)                                                                 \
  case M:                                                                                 \
    return l2p_launch<RHO, M>(blocks, C, res, L, q, n, order, wts, value, grad, hess,    \
                              wgrad, flag, s);
  switch (mode) {
    FC2T2_L2P_CASE(1)
    FC2T2_L2P_CASE(2)
    FC2T2_L2P_CASE(3)
    FC2T2_L2P_CASE(4)
    FC2T2_L2P_CASE(6)
    FC2T2_L2P_CASE(7)
    FC2T2_L2P_CASE(8)
    FC2T2_L2P_CASE(9)
    default:
      return cudaErrorInvalidValue;
  }
#undef FC2T2_L2P_CASE
}

// out[i] = sum_c w[i, c] grad[i, c, :], the same fmaf sequence as L2P_WGRAD
__global__ void __launch_bounds__(256)
weighted_grad_kernel(const float* __restrict__ grad, const float* __restrict__ w, int64_t n,
                     int C, float* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float wg0 = 0.f, wg1 = 0.f, wg2 = 0.f;
    for (int c = 0; c < C; ++c) {
      const float wv = w[i * C + c];
      const float* g = grad + (i * C + c) * 3;
      wg0 = fmaf(wv, g[0], wg0);
      wg1 = fmaf(wv, g[1], wg1);
      wg2 = fmaf(wv, g[2], wg2);
    }
    out[3 * i + 0] = wg0;
    out[3 * i + 1] = wg1;
    out[3 * i + 2] = wg2;
  }
}

}  // namespace

cudaError_t weighted_grad(const float* grad, const float* w, int64_t n, int C, float* out,
                          cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  FC2T2_LAUNCH("wgrad_recycle", s,
               weighted_grad_kernel<<<grid_blocks(n, 256, 148 * 16), 256, 0, s>>>(grad, w, n, C, out));
  return cudaGetLastError();
}

cudaError_t l2p(int rho, int level, int C, const float* L, const float* q, int64_t n, int mode,
                const int32_t* order, const float* wts, float* value, float* grad, float* hess,
                float* wgrad, int32_t* flag, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  FC2T2_DISPATCH_RHO(rho, return l2p_rho<RHO>(level, C, L, q, n, mode, order, wts, value, grad,
                                              hess, wgrad, flag, s));
  return cudaSuccess;
}

}  // namespace fc2t2
