// Point -> cell keys and a stable sort by cell.
//
// Replaces the reference's find_box + np.add.at key (reference
// expansion.py:85-93, :195): P2M wants every cell's points contiguous and in
// ascending source index so that the per-cell sum is accumulated in the same
// order as np.add.at and is bit-reproducible run to run.  The output is the
// stable sort by cell id -- order = points sorted by (cell, index) -- plus
// every cell's [start, end) range, computed as a counting sort:
//   1. keys + arrival ranks: rank = atomicAdd(&count[cell], 1) (an arbitrary
//      order inside a cell), 2. exclusive scan of the counts = cell_start,
//   3. order[cell_start[cell] + rank] = i, 4. every cell's segment sorted by
//      index (cells hold tens of points: a warp bitonic network up to 1024,
//      a shared-memory block sort up to 8192, a block merge sort beyond).
// Step 4 makes the result independent of the atomics' interleaving, i.e.
// identical to a stable sort.  No float atomics anywhere: P2M is deterministic.
#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096

constexpr int WARP_SEG_MAX = 1024;    // warp bitonic network (up to 32 per lane)
constexpr int BLOCK_SEG_MAX = 8192;   // shared-memory bitonic sort
constexpr int SEG_BLOCK = 1024;

// ---------------------------------------------------------------- keys ---

__global__ void cell_keys_kernel(const float* __restrict__ pts, int64_t n, int res,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ ranks,
                                 uint32_t* __restrict__ counts, int32_t* __restrict__ flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    bad |= outside_domain(x, y, z);
    int b0 = box_axis(x, res), b1 = box_axis(y, res), b2 = box_axis(z, res);
    uint32_t key = ((uint32_t)b0 * res + b1) * res + b2;
    keys[i] = key;
    ranks[i] = atomicAdd(&counts[key], 1u);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

__global__ void find_box_kernel(const float* __restrict__ pts, int64_t n, int res,
                                int32_t* __restrict__ box, int32_t* __restrict__ flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    bad |= outside_domain(x, y, z);
    box[3 * i] = box_axis(x, res);
    box[3 * i + 1] = box_axis(y, res);
    box[3 * i + 2] = box_axis(z, res);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

}  // namespace

// ---------------------------------------------------------------- scan ---
// Exclusive scan of uint32, three phases (tile scan, scan of tile sums,
// add-back), recursion on the tile sums.

__global__ void scan_tiles_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                  int64_t n, uint32_t* __restrict__ tile_sums) {
  __shared__ uint32_t warp_tot[32];
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  uint32_t v[SCAN_ITEMS];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + k;
    v[k] = i < n ? in[i] : 0u;
    s += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(s, warp_tot, total);
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; ++k) {
    int64_t i = base + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
  if (threadIdx.x == 0 && tile_sums) tile_sums[blockIdx.x] = total;
}

__global__ void scan_add_kernel(uint32_t* __restrict__ out, int64_t n,
                                const uint32_t* __restrict__ tile_offsets) {
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  const uint32_t off = tile_offsets[blockIdx.x];
  for (int k = threadIdx.x; k < SCAN_TILE; k += blockDim.x) {
    int64_t i = base + k;
    if (i < n) out[i] += off;
  }
}

size_t scan_ws_words(int64_t n) {
  size_t w = 0;
  while (n > SCAN_TILE) {
    n = (n + SCAN_TILE - 1) / SCAN_TILE;
    w += (size_t)n;
  }
  return w;
}

cudaError_t exclusive_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* ws,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  uint32_t* sums = tiles > 1 ? ws : nullptr;
  FC2T2_LAUNCH("scan", s, scan_tiles_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(in, out, n, sums));
  if (tiles > 1) {
    cudaError_t e = exclusive_scan(sums, sums, tiles, ws + tiles, s);
    if (e != cudaSuccess) return e;
    FC2T2_LAUNCH("scan", s, scan_add_kernel<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(out, n, sums));
  }
  return cudaGetLastError();
}

namespace {

// ------------------------------------------------------- counting sort ---

// nocell_rank (key sorts only): stable ranks of the key-R items, an exclusive
// scan of their flags, so the no-cell bucket needs no segment sort
__global__ void place_kernel(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ranks,
                             int64_t n, int64_t R, const uint32_t* __restrict__ start,
                             const uint32_t* __restrict__ nocell_rank,
                             uint32_t* __restrict__ order) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys[i];
    const uint32_t r = (nocell_rank && (int64_t)k == R) ? nocell_rank[i] : ranks[i];
    const uint32_t slot = start[k] + r;
    order[slot] = (uint32_t)i;
  }
}

// keys >= R (no cell) go to bucket R, after every cell; flags[i] = 1 for them
__global__ void key_rank_kernel(const uint32_t* __restrict__ keys_in, int64_t n, int64_t R,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ ranks,
                                uint32_t* __restrict__ counts, uint32_t* __restrict__ flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys_in[i];
    const bool cell = (int64_t)k < R;
    keys[i] = cell ? k : (uint32_t)R;
    ranks[i] = cell ? atomicAdd(&counts[k], 1u) : 0u;
    flags[i] = cell ? 0u : 1u;
  }
}

// Bitonic sort of 32*K values held as v[j] = element j*32 + lane.
template <int K, class T>
__device__ __forceinline__ void warp_bitonic(T (&v)[K], int lane) {
  constexpr int N = 32 * K;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      if (jj >= 32) {
        const int js = jj >> 5;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const int q = j ^ js;
          if (q > j) {
            const bool up = (((j << 5) | lane) & k) == 0;
            const T a = v[j], b = v[q];
            if ((a > b) == up) {
              v[j] = b;
              v[q] = a;
            }
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const T o = __shfl_xor_sync(0xffffffffu, v[j], jj);
          const bool up = (((j << 5) | lane) & k) == 0;
          const bool lower = (lane & jj) == 0;
          v[j] = (lower == up) ? min(v[j], o) : max(v[j], o);
        }
      }
    }
  }
}

// Sorts one segment of `order` by index (32 * K >= size).
template <int K>
__device__ __forceinline__ void warp_sort_segment(uint32_t* order, int64_t b, int size, int lane) {
  uint32_t v[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int e = j * 32 + lane;
    v[j] = e < size ? order[b + e] : 0xffffffffu;
  }
  warp_bitonic<K, uint32_t>(v, lane);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int e = j * 32 + lane;
    if (e < size) order[b + e] = v[j];
  }
}

__device__ __forceinline__ void warp_sort_any(uint32_t* order, int64_t b, int size, int lane) {
  if (size <= 32) warp_sort_segment<1>(order, b, size, lane);
  else if (size <= 64) warp_sort_segment<2>(order, b, size, lane);
  else if (size <= 128) warp_sort_segment<4>(order, b, size, lane);
  else if (size <= 256) warp_sort_segment<8>(order, b, size, lane);
  else if (size <= 512) warp_sort_segment<16>(order, b, size, lane);
  else warp_sort_segment<32>(order, b, size, lane);
}

// segment c = [start[c], c < R ? start[c+1] : n); one warp per segment,
// segments above WARP_SEG_MAX go to the block worklist
__global__ void __launch_bounds__(256)
segment_sort_warp_kernel(uint32_t* __restrict__ order, const uint32_t* __restrict__ start,
                         int64_t nseg, int64_t R, int64_t n, uint32_t* __restrict__ work) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < nseg;
       c += warps) {
    const int64_t b = start[c];
    const int64_t e = c < R ? (int64_t)start[c + 1] : n;
    const int64_t size = e - b;
    if (size <= 1) continue;
    if (size > WARP_SEG_MAX) {
      if (lane == 0) work[1 + atomicAdd(work, 1u)] = (uint32_t)c;
      continue;
    }
    warp_sort_any(order, b, (int)size, lane);
  }
}

// shared-memory bitonic sort of one run (len <= BLOCK_SEG_MAX), in place
__device__ void block_sort_run(uint32_t* run, int len, uint32_t* sm) {
  int N = 1;
  while (N < len) N <<= 1;
  for (int i = threadIdx.x; i < N; i += blockDim.x) sm[i] = i < len ? run[i] : 0xffffffffu;
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1)
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int p = i ^ jj;
        if (p > i) {
          const bool up = (i & k) == 0;
          const uint32_t a = sm[i], b = sm[p];
          if ((a > b) == up) {
            sm[i] = b;
            sm[p] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < len; i += blockDim.x) run[i] = sm[i];
  __syncthreads();
}

__device__ __forceinline__ int64_t lmin(int64_t a, int64_t b) { return a < b ? a : b; }

// first index of the merge of sorted a[0,na) and b[0,nb) at diagonal d
__device__ __forceinline__ int64_t merge_path(const uint32_t* a, int64_t na, const uint32_t* b,
                                              int64_t nb, int64_t d) {
  int64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int64_t m = (lo + hi) >> 1;
    if (a[m] < b[d - 1 - m]) lo = m + 1;
    else hi = m;
  }
  return lo;  // elements taken from a
}

// segments from the worklist: one block each; runs of BLOCK_SEG_MAX sorted in
// shared memory, then merged pairwise through `tmp` (merge path per thread)
__global__ void __launch_bounds__(SEG_BLOCK)
segment_sort_block_kernel(uint32_t* __restrict__ order, uint32_t* __restrict__ tmp,
                          const uint32_t* __restrict__ start, int64_t R, int64_t n,
                          const uint32_t* __restrict__ work) {
  extern __shared__ uint32_t sm[];
  const uint32_t count = work[0];
  for (uint32_t w = blockIdx.x; w < count; w += gridDim.x) {
    const int64_t c = work[1 + w];
    const int64_t b = start[c];
    const int64_t e = c < R ? (int64_t)start[c + 1] : n;
    const int64_t size = e - b;
    for (int64_t r = 0; r < size; r += BLOCK_SEG_MAX)
      block_sort_run(order + b + r, (int)lmin(BLOCK_SEG_MAX, size - r), sm);
    uint32_t* src = order + b;
    uint32_t* dst = tmp + b;
    for (int64_t width = BLOCK_SEG_MAX; width < size; width <<= 1) {
      for (int64_t r0 = 0; r0 < size; r0 += 2 * width) {
        const int64_t na = lmin(width, size - r0);
        const int64_t nb = lmin(width, size - r0 - na);
        const uint32_t* A = src + r0;
        const uint32_t* B = A + na;
        const int64_t tot = na + nb;
        const int64_t per = (tot + blockDim.x - 1) / blockDim.x;
        const int64_t d0 = lmin(tot, per * threadIdx.x), d1 = lmin(tot, d0 + per);
        int64_t ia = merge_path(A, na, B, nb, d0), ib = d0 - ia;
        for (int64_t d = d0; d < d1; ++d) {
          const bool takeA = ib >= nb || (ia < na && A[ia] <= B[ib]);
          dst[r0 + d] = takeA ? A[ia++] : B[ib++];
        }
      }
      __syncthreads();
      uint32_t* t = src;
      src = dst;
      dst = t;
    }
    if (src != order + b)
      for (int64_t i = threadIdx.x; i < size; i += blockDim.x) order[b + i] = src[i];
    __syncthreads();
  }
}

struct SortWs {
  uint32_t *keys, *ranks, *tmp, *counts, *scan, *work;
};

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

SortWs carve(void* ws, int64_t n, int64_t R) {
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { char* q = p; p += align256(bytes); return (uint32_t*)q; };
  SortWs w;
  w.keys = take(4 * (size_t)n);
  w.ranks = take(4 * (size_t)n);
  w.tmp = take(4 * (size_t)n);    // key-sort flags
  w.counts = take(4 * (size_t)(R + 1));
  w.scan = take(4 * std::max(scan_ws_words(R + 1), scan_ws_words(n)) + 4);
  w.work = take(4 * (size_t)(R + 2));
  return w;
}

size_t ws_bytes(int64_t n, int64_t R) {
  return 3 * align256(4 * (size_t)n) + align256(4 * (size_t)(R + 1)) +
         align256(4 * std::max(scan_ws_words(R + 1), scan_ws_words(n)) + 4) +
         align256(4 * (size_t)(R + 2));
}

// keys/ranks/counts prepared: cell ranges, placement, per-cell index sort.
// nocell: key sorts, whose bucket R is ranked stably by a scan of w.tmp flags.
cudaError_t sort_ranked(SortWs& w, int64_t n, int64_t R, int32_t* order, int32_t* cell_start,
                        bool nocell, cudaStream_t s) {
  cudaError_t e = exclusive_scan(w.counts, (uint32_t*)cell_start, R + 1, w.scan, s);
  if (e != cudaSuccess || n == 0) return e != cudaSuccess ? e : cudaGetLastError();
  if (nocell) {
    e = exclusive_scan(w.tmp, w.tmp, n, w.scan, s);
    if (e != cudaSuccess) return e;
  }
  uint32_t* ord = (uint32_t*)order;
  FC2T2_LAUNCH("sort_place", s,
               place_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(
                   w.keys, w.ranks, n, R, (const uint32_t*)cell_start, nocell ? w.tmp : nullptr,
                   ord));
  e = cudaMemsetAsync(w.work, 0, 4, s);
  if (e != cudaSuccess) return e;
  const int64_t nseg = nocell ? R : R + 1;
  FC2T2_LAUNCH("sort_segments", s,
               segment_sort_warp_kernel<<<grid_blocks(nseg * 32, 256), 256, 0, s>>>(
                   ord, (const uint32_t*)cell_start, nseg, R, n, w.work));
  static unsigned long long attr = 0;   // devices configured
  if (attr_needed(attr)) {
    e = cudaFuncSetAttribute(segment_sort_block_kernel,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, BLOCK_SEG_MAX * 4);
    if (e != cudaSuccess) return e;
  }
  FC2T2_LAUNCH("sort_segments", s,
               segment_sort_block_kernel<<<148, SEG_BLOCK, BLOCK_SEG_MAX * 4, s>>>(
                   ord, w.ranks, (const uint32_t*)cell_start, R, n, w.work));
  return cudaGetLastError();
}

}  // namespace

size_t cell_sort_workspace(int level, int64_t n) {
  const int64_t R = (int64_t)1 << (3 * (level + 1));
  return ws_bytes(n, R);
}

cudaError_t cell_sort(int level, const float* pts, int64_t n, int32_t* order, int32_t* cell_start,
                      int32_t* flag, void* ws, size_t ws_bytes_, cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int64_t R = (int64_t)res * res * res;
  if (ws_bytes_ < cell_sort_workspace(level, n)) return cudaErrorInvalidValue;
  SortWs w = carve(ws, n, R);
  cudaError_t e = cudaMemsetAsync(w.counts, 0, 4 * (size_t)(R + 1), s);
  if (e != cudaSuccess) return e;
  if (n > 0)
    FC2T2_LAUNCH("cell_keys", s,
                 cell_keys_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(pts, n, res, w.keys, w.ranks,
                                                                      w.counts, flag));
  return sort_ranked(w, n, R, order, cell_start, false, s);
}

size_t key_sort_workspace(int level, int64_t n) { return cell_sort_workspace(level, n); }

cudaError_t key_sort(int level, const uint32_t* keys, int64_t n, int32_t* order,
                     int32_t* cell_start, void* ws, size_t ws_bytes_, cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int64_t R = (int64_t)res * res * res;
  if (ws_bytes_ < key_sort_workspace(level, n)) return cudaErrorInvalidValue;
  SortWs w = carve(ws, n, R);
  cudaError_t e = cudaMemsetAsync(w.counts, 0, 4 * (size_t)(R + 1), s);
  if (e != cudaSuccess) return e;
  if (n > 0)
    FC2T2_LAUNCH("keys_prep", s,
                 key_rank_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(keys, n, R, w.keys, w.ranks,
                                                                     w.counts, w.tmp));
  return sort_ranked(w, n, R, order, cell_start, true, s);
}

cudaError_t find_box(int level, const float* pts, int64_t n, int32_t* box, int32_t* flag,
                     cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  FC2T2_LAUNCH("find_box", s,
               find_box_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(pts, n, 1 << (level + 1), box,
                                                                   flag));
  return cudaGetLastError();
}

}  // namespace fc2t2
