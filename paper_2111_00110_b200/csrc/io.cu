// Device side of the data formats (reference dataio.py).
//
// FCPT point files and FCCK checkpoints store float64 rows; the device path
// wants float32 columns.  unpack_rows reads the interleaved rows
// (x, y, z, v1..vC) coalesced -- consecutive threads take consecutive
// doubles -- and scatters them to p (M, 3) and values (M, C) as float32,
// fusing the (-1, 1)^3 domain check of PointSampleSet (dataio.py:49-51):
// the first offending row index is kept with atomicMin so the error names
// the same point the reference names.  One HBM pass: 8 (3 + C) bytes read,
// 4 (3 + C) written per row.
#include <cstdint>

#include "../../include/fc2t2_b200.h"
#include "common.cuh"

namespace fc2t2 {
namespace {

__global__ void unpack_rows_kernel(const double* __restrict__ rows, int64_t m, int c,
                                   float* __restrict__ p, float* __restrict__ v,
                                   unsigned long long* __restrict__ first_bad) {
  const int width = 3 + c;
  const int64_t n = m * width;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / width;
    const int col = (int)(i - r * width);
    const double x = __ldcs(rows + i);
    if (col < 3) {
      p[r * 3 + col] = (float)x;
      // NaN fails "strictly inside" as well
      if (first_bad && !(fabs(x) < 1.0)) atomicMin(first_bad, (unsigned long long)r);
    } else {
      v[r * c + (col - 3)] = (float)x;
    }
  }
}

// Domain check only: every coordinate strictly inside (-1, 1) (NaN fails),
// over the flat (n * 3) float array with 16-byte loads; one flag write per
// offending block.  Used where a layer must raise DomainError at return but
// its own kernels would only see the points at the very end.
__global__ void domain_check_kernel(const float* __restrict__ x, int64_t nf, int32_t* flag) {
  bool bad = false;
  const int64_t n4 = nf >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldcs(x4 + i);
    bad |= !(fabsf(v.x) < 1.f) | !(fabsf(v.y) < 1.f) | !(fabsf(v.z) < 1.f) | !(fabsf(v.w) < 1.f);
  }
  if (blockIdx.x == 0 && threadIdx.x < (nf & 3)) bad |= !(fabsf(x[(n4 << 2) + threadIdx.x]) < 1.f);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, FLAG_DOMAIN);
}

}  // namespace
}  // namespace fc2t2

extern "C" int fc2t2_domain_check(const float* d_pts, int64_t n, int32_t* d_flag, void* stream) {
  if (n < 0 || (n > 0 && (!d_pts || !d_flag))) return FC2T2_EVALUE;
  if (n == 0) return FC2T2_OK;
  if (reinterpret_cast<uintptr_t>(d_pts) & 15) return FC2T2_EVALUE;   // 16-byte loads
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t nf = 3 * n;
  FC2T2_LAUNCH("domain_check", s,
               fc2t2::domain_check_kernel<<<fc2t2::grid_blocks((nf + 3) / 4, 256, 148 * 8), 256,
                                             0, s>>>(d_pts, nf, d_flag));
  return cudaGetLastError() == cudaSuccess ? FC2T2_OK : FC2T2_ECUDA;
}

extern "C" int fc2t2_unpack_rows(const double* d_rows, int64_t m, int c, float* d_p, float* d_v,
                                 uint64_t* d_first_bad, void* stream) {
  if (m < 0 || c < 0 || (m > 0 && (!d_rows || !d_p || (c > 0 && !d_v)))) return FC2T2_EVALUE;
  if (m == 0) return FC2T2_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t n = m * (3 + c);
  FC2T2_LAUNCH("unpack_rows", s,
               fc2t2::unpack_rows_kernel<<<fc2t2::grid_blocks(n, 256, 148 * 16), 256, 0, s>>>(
                   d_rows, m, c, d_p, d_v, (unsigned long long*)d_first_bad));
  return cudaGetLastError() == cudaSuccess ? FC2T2_OK : FC2T2_ECUDA;
}
