// L2P: evaluate the finest local expansions at free points.
//
// Reference: Accessor._local/value/partials/partials2 (expansion.py:335-373).
// One thread per point: bit-exact box lookup, in-box offset, monomials, then
// per channel a 16-byte-vectorised read of the cell's coefficient row and
// contractions for the value, the gradient (coefficient shift n -> n + e_a,
// reference _shift_indices :309-329) and the Hessian (xx yy zz xy xz yz).
// L2P_WGRAD fuses the adjoint contraction sum_c wts_c grad f_c used by the
// explicit layer's q_bar and p_bar (reference layers.py:183, :186-187).
//
// With a cell-sorted `order` (the stable sort P2M needs anyway), thread t
// evaluates point order[t]: neighbouring threads share cell rows, which then
// come from L1 instead of one 144-byte L2 gather per point.  With
// L2P_PRESORTED the inputs (q, wts) are already permuted into that order
// (fc2t2_cell_sort_ex / fc2t2_permute_rows), so they are read coalesced and
// only the outputs are scattered to order[t].
#include "../csrc/common.cuh"
#include "../csrc/kernels.cuh"

#include <cstdlib>

namespace fc2t2 {

namespace {

// Contractions of one point's cell row `a` (PP floats of channel c).
template <int RHO, int MODE>
__device__ __forceinline__ void l2p_contract(const float (&a)[MI<RHO>::PP], const float (&mono)[MI<RHO>::P],
                                             int64_t i, int c, int C, float wv,
                                             float* __restrict__ value,
                                             float* __restrict__ grad, float* __restrict__ hess,
                                             float& wg0, float& wg1, float& wg2) {
  constexpr MI<RHO> mi{};
  constexpr int P = MI<RHO>::P;
  if constexpr (MODE & L2P_VALUE) {
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < P; ++j) s = fmaf(a[j], mono[j], s);
    value[i * C + c] = s;
  }
  if constexpr ((MODE & L2P_GRAD) || (MODE & L2P_WGRAD)) {
    float g[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (mi.up[d][j] >= 0) s = fmaf(a[mi.up[d][j]], mono[j], s);
      g[d] = s;
    }
    if constexpr (MODE & L2P_GRAD) {
      grad[(i * C + c) * 3 + 0] = g[0];
      grad[(i * C + c) * 3 + 1] = g[1];
      grad[(i * C + c) * 3 + 2] = g[2];
    }
    if constexpr (MODE & L2P_WGRAD) {
      wg0 = fmaf(wv, g[0], wg0);
      wg1 = fmaf(wv, g[1], wg1);
      wg2 = fmaf(wv, g[2], wg2);
    }
  }
  if constexpr (MODE & L2P_HESS) {
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < P; ++j)
        if (mi.up[3 + d][j] >= 0) s = fmaf(a[mi.up[3 + d][j]], mono[j], s);
      hess[(i * C + c) * 6 + d] = s;
    }
  }
}

__device__ __forceinline__ void l2p_cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// Warp-cooperative row fetch.  A thread-per-point gather makes every float4
// load instruction of a warp touch 32 different cell rows (32 L1 tag lookups
// / wavefronts per instruction, PP/4 instructions per point).  Here the warp
// copies its 32 points' rows into shared memory with consecutive lanes on
// consecutive 16-byte pieces of the same row (about 2.5 rows = 4-6 lines per
// instruction, same PP/4 instructions per lane), then each thread reads its
// own row back from shared memory (row stride PP words: the 8 lanes of a
// 128-bit shared access hit distinct bank quads for PP = 4, 12, 20, 36, 84).
template <int RHO, int MODE>
__global__ void __launch_bounds__(256)
l2p_warp_kernel(const float* __restrict__ L, const float* __restrict__ q, int64_t n, int C, int res,
                const int32_t* __restrict__ order, bool presorted, const float* __restrict__ wts,
                float* __restrict__ value, float* __restrict__ grad, float* __restrict__ hess,
                float* __restrict__ wgrad, int32_t* __restrict__ flag) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP, F4 = PP / 4;
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
    const int64_t in = presorted ? (valid ? t : 0) : i;
    float x = 0.f, y = 0.f, z = 0.f;
    if (valid) { x = q[3 * in]; y = q[3 * in + 1]; z = q[3 * in + 2]; }
    bad |= valid && outside_domain(x, y, z);
    const int b0 = box_axis(x, res), b1 = box_axis(y, res), b2 = box_axis(z, res);
    float mono[P];
    monomials<RHO>(box_offset(x, b0, res), box_offset(y, b1, res), box_offset(z, b2, res), mono);
    const int64_t rowoff = ((((int64_t)b0 * res + b1) * res + b2) * C) * PP;
    float wg0 = 0.f, wg1 = 0.f, wg2 = 0.f;
    for (int c = 0; c < C; ++c) {
      // the tangent weight is read before the copy barrier so its latency
      // overlaps the row fetch
      const float wv = ((MODE & L2P_WGRAD) && valid) ? wts[in * C + c] : 0.f;
#pragma unroll
      for (int k = 0; k < F4; ++k) {
        const int j = k * 32 + lane;
        const int pt = j / F4, f = j - pt * F4;
        const int64_t src = __shfl_sync(0xffffffffu, rowoff, pt);
        l2p_cp_async16(rows + pt * PP + 4 * f, L + src + c * PP + 4 * f);
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
      float a[PP];
#pragma unroll
      for (int k = 0; k < PP; k += 4) {
        const float4 v = *reinterpret_cast<const float4*>(rows + lane * PP + k);
        a[k] = v.x; a[k + 1] = v.y; a[k + 2] = v.z; a[k + 3] = v.w;
      }
      __syncwarp();
      if (valid) l2p_contract<RHO, MODE>(a, mono, i, c, C, wv, value, grad, hess, wg0, wg1, wg2);
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

template <int RHO, int MODE>
__global__ void __launch_bounds__(256)
l2p_kernel(const float* __restrict__ L, const float* __restrict__ q, int64_t n, int C, int res,
           const int32_t* __restrict__ order, bool presorted, const float* __restrict__ wts,
           float* __restrict__ value, float* __restrict__ grad, float* __restrict__ hess,
           float* __restrict__ wgrad, int32_t* __restrict__ flag) {
  constexpr MI<RHO> mi{};
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  int bad = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    // outputs at point i; inputs at i, or at t when they are pre-permuted
    const int64_t i = order ? (int64_t)order[t] : t;
    const int64_t in = presorted ? t : i;
    const float x = q[3 * in], y = q[3 * in + 1], z = q[3 * in + 2];
    bad |= outside_domain(x, y, z);
    const int b0 = box_axis(x, res), b1 = box_axis(y, res), b2 = box_axis(z, res);
    float mono[P];
    monomials<RHO>(box_offset(x, b0, res), box_offset(y, b1, res), box_offset(z, b2, res), mono);
    const float* row = L + ((((int64_t)b0 * res + b1) * res + b2) * C) * PP;
    float wg0 = 0.f, wg1 = 0.f, wg2 = 0.f;
    for (int c = 0; c < C; ++c) {
      float a[PP];
#pragma unroll
      for (int k = 0; k < PP; k += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(row + c * PP + k));
        a[k] = v.x; a[k + 1] = v.y; a[k + 2] = v.z; a[k + 3] = v.w;
      }
      const float wv = (MODE & L2P_WGRAD) ? wts[in * C + c] : 0.f;
      l2p_contract<RHO, MODE>(a, mono, i, c, C, wv, value, grad, hess, wg0, wg1, wg2);
    }
    if constexpr (MODE & L2P_WGRAD) {
      wgrad[3 * i + 0] = wg0;
      wgrad[3 * i + 1] = wg1;
      wgrad[3 * i + 2] = wg2;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

bool l2p_thread_per_point() {
  static const bool v = [] {
    const char* e = std::getenv("FC2T2_L2P_THREAD");
    return e && e[0] == '1';
  }();
  return v;
}

template <int RHO, int M>
cudaError_t l2p_launch(int blocks, int C, int res, const float* L, const float* q, int64_t n,
                       const int32_t* order, bool presorted, const float* wts, float* value,
                       float* grad, float* hess, float* wgrad, int32_t* flag, cudaStream_t s) {
  // a cell-coherent order makes neighbouring threads share rows (L1
  // broadcast), which the per-thread gather exploits and the cooperative copy
  // would duplicate
  if (order || l2p_thread_per_point()) {
    FC2T2_LAUNCH("l2p", s, l2p_kernel<RHO, M><<<blocks, 256, 0, s>>>(
        L, q, n, C, res, order, presorted, wts, value, grad, hess, wgrad, flag));
    return cudaGetLastError();
  }
  constexpr int smem = 8 * 32 * MI<RHO>::PP * (int)sizeof(float);
  static unsigned long long configured = 0;
  if (smem > 48 * 1024 && attr_needed(configured))
    cudaFuncSetAttribute(l2p_warp_kernel<RHO, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  FC2T2_LAUNCH("l2p", s, l2p_warp_kernel<RHO, M><<<blocks, 256, smem, s>>>(
      L, q, n, C, res, order, presorted, wts, value, grad, hess, wgrad, flag));
  return cudaGetLastError();
}

template <int RHO>
cudaError_t l2p_rho(int level, int C, const float* L, const float* q, int64_t n, int mode,
                    const int32_t* order, const float* wts, float* value, float* grad,
                    float* hess, float* wgrad, int32_t* flag, cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int blocks = grid_blocks(n, 256, 148 * 16);
  const bool presorted = (mode & 16) != 0;
  mode &= ~16;
#define FC2T2_L2P_CASE(M)                                                              \
  case M:                                                                              \
    return l2p_launch<RHO, M>(blocks, C, res, L, q, n, order, presorted, wts, value,  \
                              grad, hess, wgrad, flag, s);
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
