// Point -> cell keys and a stable counting/radix sort by cell.
//
// Replaces the reference's find_box + np.add.at key (reference
// expansion.py:85-93, :195): P2M wants every cell's points contiguous and in
// ascending source index so that the per-cell sum is accumulated in the same
// order as np.add.at and is bit-reproducible run to run.  That is a *stable*
// sort by cell id, done here as an LSD radix sort of (cell, index) pairs with
// 6-8 bit digits (2-3 passes for 15-21 bit keys), plus a cell histogram whose
// exclusive scan gives every cell's [start, end) range.  No float atomics
// anywhere, so P2M is deterministic.
#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096

constexpr int RADIX_THREADS = 256;
constexpr int RADIX_ROUNDS = 16;
constexpr int RADIX_TILE = RADIX_THREADS * RADIX_ROUNDS;  // 4096 keys per block
constexpr int RADIX_WARPS = RADIX_THREADS / 32;
constexpr int RADIX_MAX_BITS = 9;  // 512 bins: 18-bit cell keys sort in 2 passes
constexpr int RADIX_MAX_BINS = 1 << RADIX_MAX_BITS;

// ---------------------------------------------------------------- keys ---

__global__ void cell_keys_kernel(const float* __restrict__ pts, int64_t n, int res,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                 uint32_t* __restrict__ counts, int32_t* __restrict__ flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    bad |= outside_domain(x, y, z);
    int b0 = box_axis(x, res), b1 = box_axis(y, res), b2 = box_axis(z, res);
    uint32_t key = ((uint32_t)b0 * res + b1) * res + b2;
    keys[i] = key;
    vals[i] = (uint32_t)i;
    atomicAdd(&counts[key], 1u);
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

// --------------------------------------------------------------- radix ---

__global__ void radix_hist_kernel(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                  int bits, int nblocks, uint32_t* __restrict__ hist) {
  __shared__ uint32_t h[RADIX_MAX_BINS];
  const int nbins = 1 << bits;
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RADIX_TILE;
  const uint32_t mask = (uint32_t)nbins - 1;
  for (int k = threadIdx.x; k < RADIX_TILE; k += blockDim.x) {
    int64_t i = base + k;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & mask], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbins; b += blockDim.x)
    hist[(int64_t)b * nblocks + blockIdx.x] = h[b];
}

// Stable scatter.  Warp w of a block owns keys [w*512, (w+1)*512) of the
// block's 4096-key tile and ranks them in index order with warp match_any
// against its own digit histogram (no block barriers inside the loop); one
// exclusive scan across the warps per digit then places every warp's run
// after the earlier warps' runs, so the scatter is stable.
constexpr int RADIX_ITEMS = RADIX_TILE / RADIX_THREADS;  // 16 keys per thread

__global__ void __launch_bounds__(RADIX_THREADS)
radix_scatter_kernel(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                     uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out,
                     int64_t n, int shift, int bits, int nblocks,
                     const uint32_t* __restrict__ offsets) {
  extern __shared__ uint32_t rsm[];
  const int nbins = 1 << bits;
  uint32_t* whist_base = rsm;                          // [RADIX_WARPS][nbins]
  uint32_t* dstart = rsm + RADIX_WARPS * nbins;        // [nbins]
  uint32_t* gstart = dstart + nbins;                   // [nbins]
  uint32_t* skey = gstart + nbins;                     // [RADIX_TILE]
  uint32_t* sval = skey + RADIX_TILE;                  // [RADIX_TILE]
  auto whist = [&](int w, uint32_t b) -> uint32_t& { return whist_base[w * nbins + b]; };
  const uint32_t mask = (uint32_t)nbins - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = threadIdx.x; b < RADIX_WARPS * nbins; b += blockDim.x) whist_base[b] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RADIX_TILE + (int64_t)warp * (32 * RADIX_ITEMS);
  const uint32_t lt_mask = (1u << lane) - 1u;
  uint32_t key[RADIX_ITEMS], val[RADIX_ITEMS], pos[RADIX_ITEMS];
#pragma unroll
  for (int r = 0; r < RADIX_ITEMS; ++r) {
    const int64_t i = base + r * 32 + lane;
    const bool valid = i < n;
    key[r] = valid ? keys_in[i] : 0xffffffffu;
    val[r] = valid ? vals_in[i] : 0u;
  }
#pragma unroll
  for (int r = 0; r < RADIX_ITEMS; ++r) {
    const bool valid = key[r] != 0xffffffffu;
    const uint32_t d = valid ? (key[r] >> shift) & mask : 0xffffffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (lane == leader && valid) {
      old = whist(warp, d);
      whist(warp, d) = old + __popc(peers);
    }
    old = __shfl_sync(0xffffffffu, old, leader);
    pos[r] = old + __popc(peers & lt_mask);
    __syncwarp();
  }
  __syncthreads();
  // block-local digit runs: per-warp prefix inside each digit, then an
  // exclusive scan over the digits (warp 0, 8 bins per lane)
  for (int b = threadIdx.x; b < nbins; b += blockDim.x) {
    uint32_t acc = 0;
#pragma unroll
    for (int w = 0; w < RADIX_WARPS; ++w) {
      const uint32_t c = whist(w, b);
      whist(w, b) = acc;
      acc += c;
    }
    dstart[b] = acc;  // digit total for now
    gstart[b] = offsets[(int64_t)b * nblocks + blockIdx.x];
  }
  __syncthreads();
  if (warp == 0) {
    constexpr int PER = RADIX_MAX_BINS / 32;
    uint32_t v[PER], sum = 0;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int b = lane * PER + k;
      v[k] = b < nbins ? dstart[b] : 0u;
      sum += v[k];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t run = x - sum;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int b = lane * PER + k;
      if (b < nbins) dstart[b] = run;
      run += v[k];
    }
  }
  __syncthreads();
  // stage the tile in digit order, then write every digit run contiguously
#pragma unroll
  for (int r = 0; r < RADIX_ITEMS; ++r) {
    if (key[r] == 0xffffffffu) continue;
    const uint32_t d = (key[r] >> shift) & mask;
    const uint32_t lp = dstart[d] + whist(warp, d) + pos[r];
    skey[lp] = key[r];
    sval[lp] = val[r];
  }
  __syncthreads();
  const int64_t tbase = (int64_t)blockIdx.x * RADIX_TILE;
  const int cnt = (int)((n - tbase) < RADIX_TILE ? (n - tbase) : RADIX_TILE);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const uint32_t k = skey[i];
    const uint32_t d = (k >> shift) & mask;
    const uint32_t gp = gstart[d] + (uint32_t)i - dstart[d];
    keys_out[gp] = k;
    vals_out[gp] = sval[i];
  }
}

struct SortWs {
  uint32_t *keys, *keys2, *vals, *vals2, *hist, *scan, *counts;
};

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

}  // namespace

size_t cell_sort_workspace(int level, int64_t n) {
  const int64_t R = (int64_t)1 << (3 * (level + 1));
  const int64_t nblocks = (n + RADIX_TILE - 1) / RADIX_TILE;
  const int64_t hist = RADIX_MAX_BINS * (nblocks > 0 ? nblocks : 1);
  size_t b = 0;
  b += 4 * align256(4 * (size_t)n);  // keys, keys2, vals, vals2
  b += align256(4 * (size_t)hist);
  b += align256(4 * std::max(scan_ws_words(hist), scan_ws_words(R + 1)) + 4);
  b += align256(4 * (size_t)(R + 1));  // counts
  return b;
}

namespace {

__global__ void keys_prep_kernel(const uint32_t* __restrict__ keys_in, int64_t n, int64_t R,
                                 uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                 uint32_t* __restrict__ counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = keys_in[i];
    keys[i] = k;
    vals[i] = (uint32_t)i;
    if ((int64_t)k < R) atomicAdd(&counts[k], 1u);  // keys >= R sort last, belong to no cell
  }
}

SortWs carve(void* ws, int64_t n, int64_t R) {
  const int64_t nblocks = std::max<int64_t>(1, (n + RADIX_TILE - 1) / RADIX_TILE);
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { char* q = p; p += align256(bytes); return (uint32_t*)q; };
  SortWs w;
  w.keys = take(4 * (size_t)n);
  w.keys2 = take(4 * (size_t)n);
  w.vals = take(4 * (size_t)n);
  w.vals2 = take(4 * (size_t)n);
  w.hist = take(4 * (size_t)(RADIX_MAX_BINS * nblocks));
  w.scan = take(4 * std::max(scan_ws_words(RADIX_MAX_BINS * nblocks), scan_ws_words(R + 1)) + 4);
  w.counts = take(4 * (size_t)(R + 1));
  return w;
}

// keys/vals/counts already prepared in w: cell ranges + LSD radix passes
cudaError_t sort_prepared(SortWs& w, int64_t n, int key_bits, int64_t R, int32_t* order,
                          int32_t* cell_start, cudaStream_t s) {
  const int64_t nblocks = std::max<int64_t>(1, (n + RADIX_TILE - 1) / RADIX_TILE);
  cudaError_t e = exclusive_scan(w.counts, (uint32_t*)cell_start, R + 1, w.scan, s);
  if (e != cudaSuccess || n == 0) return e != cudaSuccess ? e : cudaGetLastError();
  const int passes = (key_bits + RADIX_MAX_BITS - 1) / RADIX_MAX_BITS;
  const int digit = (key_bits + passes - 1) / passes;
  uint32_t *kin = w.keys, *vin = w.vals;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = ps * digit;
    const int bits = std::min(digit, key_bits - shift);
    const bool last = ps == passes - 1;
    uint32_t* kout = (kin == w.keys) ? w.keys2 : w.keys;
    uint32_t* vout = last ? (uint32_t*)order : ((vin == w.vals) ? w.vals2 : w.vals);
    FC2T2_LAUNCH("radix_hist", s,
                 radix_hist_kernel<<<(unsigned)nblocks, RADIX_THREADS, 0, s>>>(
                     kin, n, shift, bits, (int)nblocks, w.hist));
    e = exclusive_scan(w.hist, w.hist, (int64_t)(1 << bits) * nblocks, w.scan, s);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)(RADIX_WARPS * (1 << bits) + 2 * (1 << bits) + 2 * RADIX_TILE) * 4;
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(radix_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
      if (e != cudaSuccess) return e;
    }
    FC2T2_LAUNCH("radix_scatter", s,
                 radix_scatter_kernel<<<(unsigned)nblocks, RADIX_THREADS, smem, s>>>(
                     kin, vin, kout, vout, n, shift, bits, (int)nblocks, w.hist));
    kin = kout;
    vin = vout;
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t cell_sort(int level, const float* pts, int64_t n, int32_t* order, int32_t* cell_start,
                      int32_t* flag, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int64_t R = (int64_t)res * res * res;
  if (ws_bytes < cell_sort_workspace(level, n)) return cudaErrorInvalidValue;
  SortWs w = carve(ws, n, R);
  cudaError_t e = cudaMemsetAsync(w.counts, 0, 4 * (size_t)(R + 1), s);
  if (e != cudaSuccess) return e;
  if (n > 0)
    FC2T2_LAUNCH("cell_keys", s,
                 cell_keys_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(pts, n, res, w.keys, w.vals,
                                                                      w.counts, flag));
  return sort_prepared(w, n, 3 * (level + 1), R, order, cell_start, s);
}

size_t key_sort_workspace(int level, int64_t n) { return cell_sort_workspace(level, n); }

cudaError_t key_sort(int level, const uint32_t* keys, int64_t n, int32_t* order,
                     int32_t* cell_start, void* ws, size_t ws_bytes, cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int64_t R = (int64_t)res * res * res;
  if (ws_bytes < key_sort_workspace(level, n)) return cudaErrorInvalidValue;
  SortWs w = carve(ws, n, R);
  cudaError_t e = cudaMemsetAsync(w.counts, 0, 4 * (size_t)(R + 1), s);
  if (e != cudaSuccess) return e;
  if (n > 0)
    FC2T2_LAUNCH("keys_prep", s,
                 keys_prep_kernel<<<grid_blocks(n, 256), 256, 0, s>>>(keys, n, R, w.keys, w.vals,
                                                                      w.counts));
  // one extra key bit so the out-of-grid sentinel R sorts after every cell
  return sort_prepared(w, n, 3 * (level + 1) + 1, R, order, cell_start, s);
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
