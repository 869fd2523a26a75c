// Training glue on the device: losses with their output
// tangents and the SGD / Adam parameter step of the reference trainer
// (reference trainer.py:70-152), fused so a training epoch stays on the GPU
// around the layers.
//
// Losses (trainer.py:70-105): diff = pred + bias - target over valid entries
// (mask optional, broadcast over columns); MAE value sum|diff|/count, tangent
// sign(diff)/count; MSE value sum diff^2/count, tangent 2 diff/count.  Sums
// are float64 block partials reduced in block order (deterministic).
//
// Step (trainer.py:122-152): grad (+ l1 * sign(w), trainer.py:108-112);
// Adam m += (1-b1)(g-m), v += (1-b2)(g^2-v), d = (m/c1)/(sqrt(v/c2)+eps),
// c_i = 1 - b_i^t; SGD d = g; x -= lr d; positions clipped to
// [-1 + 1e-6, 1 - 1e-6].  A device flag set by the non-finite check makes
// the step a no-op (the reference raises before updating).
#include <cmath>
#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

constexpr int TR_THREADS = 256;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  __syncthreads();
  return t;  // valid in thread 0
}

// pass 1: per block (count of valid entries, sum |diff| or diff^2)
__global__ void __launch_bounds__(TR_THREADS)
loss_partial_kernel(const float* __restrict__ pred, const float* __restrict__ target,
                    const uint8_t* __restrict__ mask, int64_t n, int cols, float bias, int mse,
                    double* __restrict__ part) {
  __shared__ double sh[TR_THREADS / 32];
  double cnt = 0.0, acc = 0.0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n * cols;
       g += (int64_t)gridDim.x * blockDim.x) {
    if (mask && !mask[g / cols]) continue;
    const double d = (double)pred[g] + (double)bias - (double)target[g];
    cnt += 1.0;
    acc += mse ? d * d : fabs(d);
  }
  cnt = block_sum(cnt, sh);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = cnt;
    part[2 * blockIdx.x + 1] = acc;
  }
}

// pass 2 (one block): out[0] = count, out[1] = loss (0 for an empty set)
__global__ void __launch_bounds__(TR_THREADS)
loss_finish_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  __shared__ double sh[TR_THREADS / 32];
  double cnt = 0.0, acc = 0.0;
  // fixed assignment of partials to threads -> deterministic
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
    cnt += part[2 * i];
    acc += part[2 * i + 1];
  }
  cnt = block_sum(cnt, sh);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    out[0] = cnt;
    out[1] = cnt > 0.0 ? acc / cnt : 0.0;
  }
}

// pass 3: tangent + per-block tangent sums
__global__ void __launch_bounds__(TR_THREADS)
tangent_kernel(const float* __restrict__ pred, const float* __restrict__ target,
               const uint8_t* __restrict__ mask, int64_t n, int cols, float bias, int mse,
               const double* __restrict__ stats, float* __restrict__ tangent,
               double* __restrict__ part) {
  __shared__ double sh[TR_THREADS / 32];
  const double cnt = stats[0];
  double acc = 0.0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n * cols;
       g += (int64_t)gridDim.x * blockDim.x) {
    float t = 0.f;
    if (cnt > 0.0 && !(mask && !mask[g / cols])) {
      const double d = (double)pred[g] + (double)bias - (double)target[g];
      const double v = mse ? 2.0 * d / cnt : (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) / cnt;
      t = (float)v;
    }
    tangent[g] = t;
    acc += (double)t;
  }
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(TR_THREADS)
tangent_finish_kernel(const double* __restrict__ part, int nparts, double* __restrict__ out) {
  __shared__ double sh[TR_THREADS / 32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += part[i];
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) out[2] = acc;
}

__global__ void nonfinite_kernel(const float* __restrict__ x, int64_t n,
                                 int32_t* __restrict__ flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(x[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

__global__ void opt_step_kernel(float* __restrict__ x, const float* __restrict__ g,
                                float* __restrict__ m, float* __restrict__ v, int64_t n, int adam,
                                float lr, float c1, float c2, float l1, int clip,
                                const int32_t* __restrict__ flag) {
  if (flag && *flag) return;  // non-finite gradient: no update (reference raises)
  // 1 - beta as float constants: (1.f - 0.999f) would be off by 1.3e-5 relative
  constexpr float omb1 = 0.1f, omb2 = 0.001f, eps = 1e-8f;
  const float lo = -1.f + 1e-6f, hi = 1.f - 1e-6f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float xi = x[i];
    float gi = g[i];
    if (l1 != 0.f) gi += l1 * (xi > 0.f ? 1.f : (xi < 0.f ? -1.f : 0.f));
    float d = gi;
    if (adam) {
      const float mi = m[i] + omb1 * (gi - m[i]);
      const float vi = v[i] + omb2 * (gi * gi - v[i]);
      m[i] = mi;
      v[i] = vi;
      d = (mi / c1) / (sqrtf(vi / c2) + eps);
    }
    xi -= lr * d;
    if (clip) xi = fminf(fmaxf(xi, lo), hi);
    x[i] = xi;
  }
}

}  // namespace

size_t loss_workspace_bytes(int64_t n, int cols) {
  const int blocks = grid_blocks(n * cols, TR_THREADS, 148 * 8);
  return (size_t)blocks * 2 * sizeof(double) + 4 * sizeof(double);
}

cudaError_t loss_tangent(const float* pred, const float* target, const uint8_t* mask, int64_t n,
                         int cols, float bias, int mse, float* tangent, double* stats, void* ws,
                         cudaStream_t s) {
  const int blocks = grid_blocks(n * cols, TR_THREADS, 148 * 8);
  double* part = (double*)ws;
  FC2T2_LAUNCH("loss", s, loss_partial_kernel<<<blocks, TR_THREADS, 0, s>>>(
                              pred, target, mask, n, cols, bias, mse, part));
  FC2T2_LAUNCH("loss", s, loss_finish_kernel<<<1, TR_THREADS, 0, s>>>(part, blocks, stats));
  FC2T2_LAUNCH("loss", s, tangent_kernel<<<blocks, TR_THREADS, 0, s>>>(
                              pred, target, mask, n, cols, bias, mse, stats, tangent, part));
  FC2T2_LAUNCH("loss", s, tangent_finish_kernel<<<1, TR_THREADS, 0, s>>>(part, blocks, stats));
  return cudaGetLastError();
}

cudaError_t nonfinite(const float* x, int64_t n, int32_t* flag, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  FC2T2_LAUNCH("opt_check", s,
               nonfinite_kernel<<<grid_blocks(n, 256, 148 * 8), 256, 0, s>>>(x, n, flag));
  return cudaGetLastError();
}

cudaError_t opt_step(float* x, const float* g, float* m, float* v, int64_t n, int adam, float lr,
                     float c1, float c2, float l1, int clip, const int32_t* flag,
                     cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  FC2T2_LAUNCH("opt_step", s,
               opt_step_kernel<<<grid_blocks(n, 256, 148 * 8), 256, 0, s>>>(
                   x, g, m, v, n, adam, lr, c1, c2, l1, clip, flag));
  return cudaGetLastError();
}

}  // namespace fc2t2
