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

}  // namespace
}  // namespace fc2t2

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
