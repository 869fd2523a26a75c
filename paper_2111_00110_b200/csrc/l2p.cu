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
#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

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
          const float wv = wts[in * C + c];
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
    if constexpr (MODE & L2P_WGRAD) {
      wgrad[3 * i + 0] = wg0;
      wgrad[3 * i + 1] = wg1;
      wgrad[3 * i + 2] = wg2;
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

template <int RHO>
cudaError_t l2p_rho(int level, int C, const float* L, const float* q, int64_t n, int mode,
                    const int32_t* order, const float* wts, float* value, float* grad,
                    float* hess, float* wgrad, int32_t* flag, cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int blocks = grid_blocks(n, 256, 148 * 16);
  const bool presorted = (mode & L2P_PRESORTED) != 0;
  mode &= ~L2P_PRESORTED;
#define FC2T2_L2P_CASE(M)                                                               \
  case M:                                                                               \
    FC2T2_LAUNCH("l2p", s, l2p_kernel<RHO, M><<<blocks, 256, 0, s>>>(                   \
        L, q, n, C, res, order, presorted, wts, value, grad, hess, wgrad, flag));                  \
    break;
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
  return cudaGetLastError();
}

}  // namespace

cudaError_t l2p(int rho, int level, int C, const float* L, const float* q, int64_t n, int mode,
                const int32_t* order, const float* wts, float* value, float* grad, float* hess,
                float* wgrad, int32_t* flag, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  FC2T2_DISPATCH_RHO(rho, return l2p_rho<RHO>(level, C, L, q, n, mode, order, wts, value, grad,
                                              hess, wgrad, flag, s));
  return cudaSuccess;
}

}  // namespace fc2t2
