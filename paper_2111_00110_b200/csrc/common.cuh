// Shared device-side definitions for the FC2T2 B200 kernels.
//
// Layout contract:
//   * A coefficient grid at level l is row-major over cells
//     cell = (b0 * res + b1) * res + b2  (reference expansion.py:195), then
//     channel, then the graded-lex coefficient index padded to PP floats
//     (PP = P rounded up to 4, so every row is 16-byte aligned).  The pad
//     entries are always zero.
//   * Points are (n, 3) float32, weights (n, C) float32.
//
// MI<RHO> regenerates the graded-lex multi-index order of
// paper_2111_00110_b200/multiindex.py (reference multiindex.py:74-96) at
// compile time so every kernel loop over coefficients fully unrolls with
// constant exponents.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>

namespace fc2t2 {

constexpr int index_count(int rho) { return (rho + 1) * (rho + 2) * (rho + 3) / 6; }
constexpr int pad4(int p) { return (p + 3) & ~3; }

template <int RHO>
struct MI {
  static constexpr int P = index_count(RHO);
  static constexpr int PP = pad4(P);
  int e0[P], e1[P], e2[P];
  float inv_fact[P];
  double inv_fact_d[P];
  int up[9][P];    // ordinal of e_j + s for s in x,y,z,xx,yy,zz,xy,xz,yz, else -1
  constexpr MI() : e0(), e1(), e2(), inv_fact(), inv_fact_d(), up() {
    int k = 0;
    for (int t = 0; t <= RHO; ++t)
      for (int x = 0; x <= t; ++x)
        for (int y = 0; y <= t - x; ++y) {
          e0[k] = x; e1[k] = y; e2[k] = t - x - y;
          double f = 1.0;
          for (int i = 2; i <= x; ++i) f *= i;
          for (int i = 2; i <= y; ++i) f *= i;
          for (int i = 2; i <= t - x - y; ++i) f *= i;
          inv_fact_d[k] = 1.0 / f;
          inv_fact[k] = (float)(1.0 / f);
          ++k;
        }
    const int sh[9][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {2, 0, 0}, {0, 2, 0},
                          {0, 0, 2}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}};
    for (int s = 0; s < 9; ++s)
      for (int j = 0; j < P; ++j) up[s][j] = index(e0[j] + sh[s][0], e1[j] + sh[s][1], e2[j] + sh[s][2]);
  }
  // ordinal of (x, y, z); -1 if outside the table
  // closed form of the graded-lex ordinal: entries of lower total order,
  // then (within total t) those with a smaller first, then second, index
  static constexpr int index(int x, int y, int z) {
    if (x < 0 || y < 0 || z < 0 || x + y + z > RHO) return -1;
    const int t = x + y + z;
    return t * (t + 1) * (t + 2) / 6 + x * (t + 1) - x * (x - 1) / 2 + y;
  }
};

// Bit-exact point -> box index along one axis: floor((x + 1) * res / 2) in
// float64 round-to-nearest, clipped to [0, res-1] (reference
// expansion.py:85-93).  For float32 x the sum is the same double the
// reference computes from the float32-quantized input.
__device__ __forceinline__ int box_axis(double x, int res) {
  double s = __dadd_rn(x, 1.0);
  int b = (int)floor(__dmul_rn(s, 0.5 * (double)res));
  return b < 0 ? 0 : (b > res - 1 ? res - 1 : b);
}

// Offset of x from its box centre, one rounding: -1 + (b + 0.5) * width is
// exact in float64 and so is the difference; the result is rounded once.
__device__ __forceinline__ float box_offset(double x, int b, int res) {
  double c = -1.0 + ((double)b + 0.5) * (2.0 / (double)res);
  return (float)(x - c);
}

// The same two functions for float32 x in float32 arithmetic only (no
// float64 conversions on the hot kernels), bit-identical to the float64
// forms above for every float32 input, NaN and +-inf included
// (scripts/box_axis_check.py sweeps this on the CPU):
//  * (x + 1) * h, h = res / 2, has floor(x * h) + h as its exact floor; x * h
//    is exact (h a power of two).  The float64 sum x + 1 rounds to 1 only
//    for x in [-2^-54, 0), which the select maps to 0.  Clamping to
//    [-h, h - 1] before the floor is the clip (NaN -> -h -> box 0, as the
//    float64 cast gives 0); floor is a round-down add of 1.5 * 2^23.
//  * the centre (2b + 1 - res) / res is exact in float32 and x - c is rounded
//    once, which the float64 difference also is: it is exact in float64
//    unless |x| < 2^-37, where both round to -c.
__device__ __forceinline__ int box_axis(float x, int res) {
  const float h = (float)(res >> 1);
  const float xs = x >= -0x1p-54f ? fmaxf(x, 0.f) : x;
  const float y = fminf(fmaxf(xs * h, -h), h - 1.f);
  return __float_as_int(__fadd_rd(y, 12582912.f)) - 0x4B400000 + (res >> 1);
}

__device__ __forceinline__ float box_offset(float x, int b, int res) {
  const float c = (float)(2 * b + 1 - res) * (1.f / (float)res);
  return __fsub_rn(x, c);
}

// Per-axis power tables x^0..x^RHO.
template <int RHO, typename T>
__device__ __forceinline__ void powers(T x, T (&p)[RHO + 1]) {
  p[0] = T(1);
#pragma unroll
  for (int k = 1; k <= RHO; ++k) p[k] = p[k - 1] * x;
}

// mono[j] = d^n_j / n_j!  (reference expansion.py:96-113)
template <int RHO, typename T>
__device__ __forceinline__ void monomials(T dx, T dy, T dz, T (&mono)[index_count(RHO)]) {
  constexpr MI<RHO> mi{};
  T px[RHO + 1], py[RHO + 1], pz[RHO + 1];
  powers<RHO>(dx, px);
  powers<RHO>(dy, py);
  powers<RHO>(dz, pz);
#pragma unroll
  for (int j = 0; j < MI<RHO>::P; ++j) {
    if constexpr (sizeof(T) == 8)
      mono[j] = px[mi.e0[j]] * py[mi.e1[j]] * pz[mi.e2[j]] * mi.inv_fact_d[j];
    else
      mono[j] = px[mi.e0[j]] * py[mi.e1[j]] * pz[mi.e2[j]] * mi.inv_fact[j];
  }
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024,
// a multiple of 32); `total` = the block sum.  Contains __syncthreads.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* warp_tot,
                                                         uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive warp prefix
  }
  __syncthreads();
  total = warp_tot[(blockDim.x >> 5) - 1];
  uint32_t before = warp > 0 ? warp_tot[warp - 1] : 0u;
  __syncthreads();
  return before + x - v;
}

// Domain flag bits (read once per layer call by the host shim).
enum : int { FLAG_DOMAIN = 1 };

__device__ __forceinline__ bool outside_domain(float x, float y, float z) {
  // reference rejects max |x| >= 1 (expansion.py:45-46, :337-338); NaN fails too
  return !(fabsf(x) < 1.0f && fabsf(y) < 1.0f && fabsf(z) < 1.0f);
}

// Function attributes are per device: `mask` (one per kernel instantiation)
// records the devices already configured, so a launch path sets them once per
// device and issues nothing but launches afterwards (CUDA-graph capture).
inline bool attr_needed(unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask & bit) return false;
  mask |= bit;
  return true;
}

inline int grid_blocks(int64_t n, int threads, int cap = 148 * 32) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)(b > cap ? cap : b);
}

// Launch bookkeeping (abi.cu): every kernel launch bumps a counter (the
// bench's gpu_launches) and, when profiling is on, is bracketed by CUDA
// events on its own stream so bench.py can time individual kernels live.
void prof_begin(const char* name, cudaStream_t s);
void prof_end(cudaStream_t s);

}  // namespace fc2t2

#define FC2T2_LAUNCH(name, stream, ...)      \
  do {                                       \
    ::fc2t2::prof_begin(name, stream);       \
    __VA_ARGS__;                             \
    ::fc2t2::prof_end(stream);               \
  } while (0)

// Dispatch a templated launcher on rho in {1..6}.
#define FC2T2_DISPATCH_RHO(rho, ...)            \
  switch (rho) {                                \
    case 1: { constexpr int RHO = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int RHO = 2; __VA_ARGS__; } break; \
    case 3: { constexpr int RHO = 3; __VA_ARGS__; } break; \
    case 4: { constexpr int RHO = 4; __VA_ARGS__; } break; \
    case 5: { constexpr int RHO = 5; __VA_ARGS__; } break; \
    case 6: { constexpr int RHO = 6; __VA_ARGS__; } break; \
    default: return cudaErrorNotSupported;      \
  }
