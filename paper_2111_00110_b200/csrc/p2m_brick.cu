// P2M from unsorted points: a deterministic, stable partition of the points
// into bricks of cells, then one CTA per brick sums each cell's points in
// source index order (reference Engine.p2m, expansion.py:186-198: np.add.at
// over the cell key of :195 -- the per-cell summation order is the point
// order).
//
//   K1 brick_hist     CTA tiles of TILE consecutive points (2048 up to level
//                     5); per tile a shared-memory histogram over bricks ->
//                     cnt[tile][brick]
//   S  brick_scan     per brick, the exclusive prefix of cnt over the tiles
//                     (blocks of 32 bricks x 128 tiles read row-wise: segment
//                     sums, their scan, the in-segment fill); brick_start =
//                     exclusive scan of the brick totals (one CTA), folded
//                     into cnt by the fill: cnt[tile][brick] = the first
//                     record of the tile's run of the brick
//   K3 brick_scatter  a CTA bulk-copies its tile's points and weights into
//                     shared memory, finds every point's brick and a
//                     deterministic rank (per-warp counters, lane-order ranks
//                     among lanes sharing a brick), counting-sorts the tile
//                     by brick and writes the runs contiguously as records
//                     {x, y, z, w..}: a STABLE partition, coalesced stores
//                     (level 6, 4096 bricks: smem atomics + a fix-up sort of
//                     the short runs)
//   K4 brick_p2m      one CTA per brick, one thread per cell.  The brick's
//                     records stream through shared memory in chunks of 2048
//                     (one bulk copy each): cell keys and deterministic ranks
//                     as in K3, a counting sort (every cell's run is in record
//                     = index order), and each thread accumulates its cell's
//                     moment row in registers.
//
// No float atomics, and every summation order is the point order: moments are
// bit-reproducible run to run (the atomics only count).  Bytes per point: 12 (K1) + 12 + 4C (K3 in) +
// 2 x 4 RS (K3 out, K4 in), RS = record floats; plus the grid write.  No
// random gathers (the round-1 cell sort + gather P2M read every point through
// an index).
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

struct BrickGeom {
  int res, bz, bzs, nbx, nby, nbz, nb, cb;
};

// 8 x 8 x BZ cells per brick; BZ = 4 (256 cells) up to level 5, 8 (512 cells)
// at level 6.  Level >= 7 is not served by this path.
__host__ __device__ inline BrickGeom brick_geom(int level) {
  BrickGeom g;
  g.res = 1 << (level + 1);
  g.bz = level >= 6 ? 8 : 4;
  g.bzs = level >= 6 ? 3 : 2;   // log2(bz)
  g.nbx = g.res >= 8 ? g.res >> 3 : 1;
  g.nby = g.nbx;
  g.nbz = g.res >= g.bz ? g.res >> g.bzs : 1;
  g.nb = g.nbx * g.nby * g.nbz;
  g.cb = 64 * g.bz;
  return g;
}

__device__ __forceinline__ int point_brick(float x, float y, float z, const BrickGeom& g) {
  const int cx = box_axis(x, g.res), cy = box_axis(y, g.res), cz = box_axis(z, g.res);
  return ((cx >> 3) * g.nby + (cy >> 3)) * g.nbz + (cz >> g.bzs);
}

// In-place insertion sort of a short uint16 run (ascending): restores the
// index order inside a bucket filled in atomic-arrival order.  Runs longer
// than kShortRun (clustered points) are rebuilt by warp_compact_run instead.
constexpr int kShortRun = 32;
constexpr int kMaxLong = 256;   // >= tile / (kShortRun + 1) and chunk / (kShortRun + 1)
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// One warp writes, in index order, the positions k < n whose key >> shift ==
// want: 32 keys per step, matches compacted with a ballot (O(n / 32) steps).
__device__ __forceinline__ void warp_compact_run(uint16_t* out, const uint32_t* key, int n,
                                                 uint32_t want, int shift) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = lanemask_lt();
  uint32_t base = 0;
  for (int k0 = 0; k0 < n; k0 += 32) {
    const int k = k0 + lane;
    const bool hit = k < n && (key[k] >> shift) == want;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (hit) out[base + __popc(m & lt)] = (uint16_t)k;
    base += __popc(m);
  }
}

__device__ __forceinline__ void sort_run(uint16_t* a, int n) {
  for (int i = 1; i < n; ++i) {
    const uint16_t v = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > v) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = v;
  }
}

// ------------------------------------------------------------------- K1 ---
constexpr int K13_THREADS = 256;   // K1
constexpr int K3_THREADS = 1024;   // K3: one CTA per SM (smem), 32 warps

__global__ void __launch_bounds__(K13_THREADS)
brick_hist_kernel(const float* __restrict__ pts, int64_t n, int level, int tile,
                  uint32_t* __restrict__ cnt, int32_t* __restrict__ flag) {
  extern __shared__ uint32_t sh[];
  const BrickGeom g = brick_geom(level);
  for (int b = threadIdx.x; b < g.nb; b += blockDim.x) sh[b] = 0u;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * tile, hi = min(n, lo + tile);
  int bad = 0;
#pragma unroll 4
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const float x = __ldg(pts + 3 * i), y = __ldg(pts + 3 * i + 1), z = __ldg(pts + 3 * i + 2);
    bad |= outside_domain(x, y, z);
    atomicAdd(sh + point_brick(x, y, z, g), 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < g.nb; b += blockDim.x) cnt[(size_t)blockIdx.x * g.nb + b] = sh[b];
  if (__syncthreads_or(bad) && threadIdx.x == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

// ------------------------------------------------------------------- S ---
// cnt[t][b] <- exclusive prefix over tiles t; tot[b] = the column total.
// Blocks of 32 bricks x SEG_T tiles, read row-wise (128-byte coalesced rows):
//   S1 brick_segsum   per block and brick the segment sum -> part[seg][b]
//   S2 brick_segscan  per brick the exclusive scan of part over segments, tot
//   S3 brick_segfill  per block: warps' sums, their prefix, then each warp
//                     rewrites its SEG_T / 8 tiles with the running prefix
constexpr int SEG_T = 128;   // tiles per segment (8 warps x 16)

__global__ void __launch_bounds__(256)
brick_segsum_kernel(const uint32_t* __restrict__ cnt, int nt, int nb, uint32_t* __restrict__ part) {
  __shared__ uint32_t ws[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x * 32 + lane, seg = blockIdx.y;
  const int t0 = seg * SEG_T + w * (SEG_T / 8), t1 = min(nt, t0 + SEG_T / 8);
  uint32_t s = 0;
  if (b < nb)
#pragma unroll 8
    for (int t = t0; t < t1; ++t) s += cnt[(size_t)t * nb + b];
  ws[w][lane] = s;
  __syncthreads();
  if (w == 0 && b < nb) {
    uint32_t tot = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) tot += ws[q][lane];
    part[(size_t)seg * nb + b] = tot;
  }
}

__global__ void __launch_bounds__(256)
brick_segscan_kernel(uint32_t* __restrict__ part, int nseg, int nb, uint32_t* __restrict__ tot) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);   // a warp per brick
  if (b >= nb) return;
  uint32_t carry = 0;
  for (int g0 = 0; g0 < nseg; g0 += 32) {
    const int g = g0 + lane;
    const uint32_t v = g < nseg ? part[(size_t)g * nb + b] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (g < nseg) part[(size_t)g * nb + b] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) tot[b] = carry;
}

__global__ void __launch_bounds__(256)
brick_segfill_kernel(uint32_t* __restrict__ cnt, int nt, int nb, const uint32_t* __restrict__ part,
                     const uint32_t* __restrict__ bstart) {
  __shared__ uint32_t ws[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x * 32 + lane, seg = blockIdx.y;
  const int t0 = seg * SEG_T + w * (SEG_T / 8), t1 = min(nt, t0 + SEG_T / 8);
  uint32_t s = 0;
  if (b < nb)
#pragma unroll 8
    for (int t = t0; t < t1; ++t) s += cnt[(size_t)t * nb + b];
  ws[w][lane] = s;
  __syncthreads();
  if (b >= nb) return;
  uint32_t run = part[(size_t)seg * nb + b] + bstart[b];
  for (int q = 0; q < w; ++q) run += ws[q][lane];
  for (int t = t0; t < t1; ++t) {
    const uint32_t v = cnt[(size_t)t * nb + b];
    cnt[(size_t)t * nb + b] = run;
    run += v;
  }
}

// one CTA: brick_start = exclusive scan of the brick totals (nb + 1 entries)
__global__ void __launch_bounds__(1024)
brick_start_kernel(const uint32_t* __restrict__ tot, int nb, uint32_t* __restrict__ brick_start) {
  __shared__ uint32_t warp_tot[32];
  const int per = (nb + blockDim.x - 1) / blockDim.x;   // <= 4 (nb <= 4096)
  const int b0 = threadIdx.x * per;
  uint32_t mine = 0;
  for (int k = 0; k < per && b0 + k < nb; ++k) mine += tot[b0 + k];
  uint32_t total;
  uint32_t run = block_exclusive_scan(mine, warp_tot, total);
  for (int k = 0; k < per && b0 + k < nb; ++k) {
    brick_start[b0 + k] = run;
    run += tot[b0 + k];
  }
  if (threadIdx.x == blockDim.x - 1) brick_start[nb] = total;
}

// Small inputs (nt <= kSmallScanTiles): S1-S3 and the brick starts in one
// launch -- a CTA per 32 bricks scans all their tiles (32 warps x nt / 32 tiles),
// the brick totals meet at a grid barrier (at most 64 CTAs, all resident;
// the counters reset themselves; one slot per launch in flight), and every
// CTA derives its bricks' starts from the totals before it.  Same cnt / tot /
// brick_start contents as the four-kernel path.
constexpr int kSmallScanTiles = 2048;
constexpr int kSmallScanCtas = 64;   // two such launches in flight still leave SMs free
constexpr int kScanSlots = 32;
__device__ unsigned int g_scan_sync[kScanSlots][2];

__global__ void __launch_bounds__(1024)
brick_scan_small_kernel(uint32_t* __restrict__ cnt, int nt, int nb, uint32_t* __restrict__ tot,
                        uint32_t* __restrict__ brick_start, int slot) {
  __shared__ uint32_t ws[32][32];
  __shared__ uint32_t red[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = blockIdx.x * 32 + lane;
  const int per = (nt + 31) / 32;
  const int t0 = w * per, t1 = min(nt, t0 + per);
  uint32_t s = 0;
  if (b < nb)
#pragma unroll 16
    for (int t = t0; t < t1; ++t) s += cnt[(size_t)t * nb + b];
  ws[w][lane] = s;
  __syncthreads();
  if (w == 0 && b < nb) {
    uint32_t t = 0;
#pragma unroll
    for (int q = 0; q < 32; ++q) t += ws[q][lane];
    tot[b] = t;
  }
  // grid barrier: every CTA's totals are visible past it
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(&g_scan_sync[slot][0], 1u);
    while (*reinterpret_cast<volatile unsigned int*>(&g_scan_sync[slot][0]) < gridDim.x) {
    }
    __threadfence();
  }
  __syncthreads();
  // the totals of the bricks before this CTA's
  uint32_t part = 0;
  for (int i = threadIdx.x; i < (int)blockIdx.x * 32; i += blockDim.x) part += __ldcg(tot + i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[w] = part;
  __syncthreads();
  uint32_t base = 0;
#pragma unroll
  for (int q = 0; q < 32; ++q) base += red[q];
  const uint32_t mine = b < nb ? __ldcg(tot + b) : 0u;
  uint32_t x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const uint32_t start = base + x - mine;
  if (w == 0 && b < nb) {
    brick_start[b] = start;
    if (b == nb - 1) brick_start[nb] = start + mine;
  }
  if (b < nb) {
    uint32_t run = start;
    for (int q = 0; q < w; ++q) run += ws[q][lane];
    for (int t = t0; t < t1; ++t) {
      const uint32_t v = cnt[(size_t)t * nb + b];
      cnt[(size_t)t * nb + b] = run;
      run += v;
    }
  }
  // the last CTA out resets the slot
  if (threadIdx.x == 0 && atomicAdd(&g_scan_sync[slot][1], 1u) == gridDim.x - 1) {
    g_scan_sync[slot][0] = 0u;
    g_scan_sync[slot][1] = 0u;
    __threadfence();
  }
}

// ------------------------------------------------------------------- K3 ---
// records: RS floats per point (x, y, z, w_0..w_{C-1}, zero pad), RS % 4 == 0.
// Shared memory (K3Smem): the tile's raw points and weights (copied with
// 16-byte loads, one round trip), a key per point (brick << 13 | arrival rank),
// the tile's brick counts and starts, the global run starts and the sorting
// permutation (uint16).
struct K3Smem {
  size_t pts, wts, key, bcnt, lstart, gbase, perm, total;
};
__host__ __device__ inline K3Smem k3_smem(int tile, int C, int nb) {
  K3Smem m;
  size_t o = 0;
  auto take = [&](size_t b) { const size_t r = o; o += (b + 15) & ~(size_t)15; return r; };
  m.pts = take((size_t)tile * 12);
  m.wts = take((size_t)tile * C * 4);
  m.key = take((size_t)tile * 4);
  m.bcnt = take((size_t)nb * 4);
  m.lstart = take((size_t)nb * 4);
  m.gbase = take((size_t)nb * 4);
  m.perm = take((size_t)tile * 2);
  m.total = o;
  return m;
}

// copy nf floats global -> shared (16-byte loads when the source is aligned)
__device__ __forceinline__ void stage_floats(float* dst, const float* __restrict__ src, int nf) {
  if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const int n4 = nf >> 2;
    for (int j = threadIdx.x; j < n4; j += blockDim.x)
      reinterpret_cast<float4*>(dst)[j] = __ldg(reinterpret_cast<const float4*>(src) + j);
    for (int j = 4 * n4 + threadIdx.x; j < nf; j += blockDim.x) dst[j] = __ldg(src + j);
  } else {
    for (int j = threadIdx.x; j < nf; j += blockDim.x) dst[j] = __ldg(src + j);
  }
}

// A tile: bricks by smem atomics (arrival order), a tile-local counting sort,
// then every brick's run sorted back into index order (runs are short: the
// tile holds ~8 points per brick), then the runs written out contiguously.
__global__ void __launch_bounds__(K3_THREADS)
brick_scatter_kernel(const float* __restrict__ pts, const float* __restrict__ wts, int C, int RS,
                     int64_t n, int level, int tile, const uint32_t* __restrict__ cpre,
                     float* __restrict__ rec) {
  extern __shared__ __align__(16) unsigned char sm3[];
  const BrickGeom g = brick_geom(level);
  const K3Smem L = k3_smem(tile, C, g.nb);
  float* sp = reinterpret_cast<float*>(sm3 + L.pts);
  float* sw = reinterpret_cast<float*>(sm3 + L.wts);
  uint32_t* key = reinterpret_cast<uint32_t*>(sm3 + L.key);
  uint32_t* bcnt = reinterpret_cast<uint32_t*>(sm3 + L.bcnt);
  uint32_t* lstart = reinterpret_cast<uint32_t*>(sm3 + L.lstart);
  uint32_t* gbase = reinterpret_cast<uint32_t*>(sm3 + L.gbase);
  uint16_t* perm = reinterpret_cast<uint16_t*>(sm3 + L.perm);
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t nlong;
  __shared__ uint16_t longs[kMaxLong];
  const int64_t t0 = (int64_t)blockIdx.x * tile;
  const int tn = (int)min((int64_t)tile, n - t0);
  // 1. the tile's points and weights into shared memory
  stage_floats(sp, pts + 3 * t0, 3 * tn);
  stage_floats(sw, wts + (int64_t)C * t0, C * tn);
  for (int b = threadIdx.x; b < g.nb; b += blockDim.x) {
    bcnt[b] = 0u;
    gbase[b] = cpre[(size_t)blockIdx.x * g.nb + b];
  }
  __syncthreads();
  // 2. brick and arrival rank of every point
  for (int tp = threadIdx.x; tp < tn; tp += blockDim.x) {
    const int b = point_brick(sp[3 * tp], sp[3 * tp + 1], sp[3 * tp + 2], g);
    key[tp] = ((uint32_t)b << 13) | atomicAdd(&bcnt[b], 1u);
  }
  __syncthreads();
  // 3. tile-local brick starts
  const int bpt = (g.nb + blockDim.x - 1) / blockDim.x;   // bricks per thread (<= 16)
  uint32_t mine = 0;
  for (int k = 0; k < bpt; ++k) {
    const int b = threadIdx.x * bpt + k;
    if (b < g.nb) mine += bcnt[b];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(mine, warp_tot, total);
  for (int k = 0; k < bpt; ++k) {
    const int b = threadIdx.x * bpt + k;
    if (b >= g.nb) break;
    lstart[b] = run;
    run += bcnt[b];
  }
  __syncthreads();
  // 4. counting-sort placement (arrival order inside a brick) ...
  for (int tp = threadIdx.x; tp < tn; tp += blockDim.x) {
    const uint32_t k = key[tp];
    perm[lstart[k >> 13] + (k & 8191u)] = (uint16_t)tp;
  }
  __syncthreads();
  // ... and every brick's run back in index order (deterministic, stable):
  // short runs by one thread each, long runs (clustered points) by a warp
  if (threadIdx.x == 0) nlong = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < g.nb; b += blockDim.x) {
    const int cnt = (int)bcnt[b];
    if (cnt <= kShortRun) sort_run(perm + lstart[b], cnt);
    else longs[atomicAdd(&nlong, 1u)] = (uint16_t)b;
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x >> 5; i < nlong; i += blockDim.x >> 5)
    warp_compact_run(perm + lstart[longs[i]], key, tn, longs[i], 13);
  __syncthreads();
  // 5. brick runs out, coalesced
  if (RS == 4) {
    for (int s = threadIdx.x; s < tn; s += blockDim.x) {
      const int tp = perm[s];
      const int b = (int)(key[tp] >> 13);
      const size_t gs = (size_t)gbase[b] + (s - lstart[b]);
      reinterpret_cast<float4*>(rec)[gs] =
          make_float4(sp[3 * tp], sp[3 * tp + 1], sp[3 * tp + 2], sw[tp]);
    }
  } else {
    const int r4 = RS / 4;
    for (int e = threadIdx.x; e < tn * r4; e += blockDim.x) {
      const int s = e / r4, f = e - s * r4;
      const int tp = perm[s];
      const int b = (int)(key[tp] >> 13);
      const size_t gs = (size_t)gbase[b] + (s - lstart[b]);
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = 4 * f + j;
        v[j] = c < 3 ? sp[3 * tp + c] : (c < 3 + C ? sw[C * tp + c - 3] : 0.f);
      }
      reinterpret_cast<float4*>(rec)[gs * r4 + f] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

// K3r (levels <= 5, <= 1024 bricks): the same tile partition with
// deterministic ranks and no fix-up sort.  Warp w of the 512-thread CTA (two
// per SM, so one CTA's loads overlap the other's ranking) owns
// tile points [128 w, 128 w + 128) and ranks them 32 at a time against the
// warp's own 16-bit brick counters: a lane alone on its brick in the group
// (counter read before and after the group's atomicAdds differ by one) takes
// the old count; lanes sharing a brick (~40 % of the groups at 1024 bricks)
// add their lane-order rank among those peers (__match_any_sync over the
// clashing lanes only) -- deterministic whatever order the atomics ran in.
// Then slot = tile start of the brick + the counts of the brick in earlier
// warps + rank; the tile's points arrive by one bulk copy (TMA) while the
// counters are cleared, and cpre already holds every brick's global start
// for this tile (brick_segfill folds brick_start in).
constexpr int K3R_PER_WARP = 128;
constexpr int K3R_THREADS = 512;                              // 2 CTAs per SM
constexpr int K3R_NW = K3R_THREADS / 32;
constexpr int K3R_TILE = K3R_PER_WARP * K3R_NW;               // 2048

struct K3RSmem {
  size_t pts, wts, key, wc, delta, perm, total;
};
__host__ __device__ inline K3RSmem k3r_smem(int C, int nb) {
  K3RSmem m;
  size_t o = 0;
  auto take = [&](size_t b) { const size_t r = o; o += (b + 15) & ~(size_t)15; return r; };
  m.pts = take((size_t)K3R_TILE * 12);
  m.wts = take((size_t)K3R_TILE * C * 4);
  m.key = take((size_t)K3R_TILE * 4);
  m.wc = take((size_t)K3R_NW * nb * 2);    // packed 16-bit counters [NW][nb]
  m.delta = take((size_t)nb * 4);
  m.perm = take((size_t)K3R_TILE * 2);
  m.total = o;
  return m;
}

// bulk (TMA) copy of nbytes global -> shared on barrier bar when both ends
// are 16-byte aligned (the sub-16-byte tail by plain loads); false: caller
// stages with ordinary loads.  Issued by thread 0; the tail by threads 1..3.
__device__ __forceinline__ bool bulk_stage(void* dst, const void* src, uint32_t nbytes,
                                           uint32_t bar, uint32_t& expect) {
  if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) != 0)
    return false;
  const uint32_t body = nbytes & ~15u;
  if (threadIdx.x == 0 && body)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
        "[%3];\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(body), "r"(bar)
        : "memory");
  const uint32_t tail = (nbytes - body) >> 2;
  if (threadIdx.x >= 1 && threadIdx.x <= tail)
    reinterpret_cast<float*>(dst)[(body >> 2) + threadIdx.x - 1] =
        __ldg(reinterpret_cast<const float*>(src) + (body >> 2) + threadIdx.x - 1);
  expect += body;
  return true;
}

__global__ void __launch_bounds__(K3R_THREADS)
brick_scatter_rank_kernel(const float* __restrict__ pts, const float* __restrict__ wts, int C,
                          int RS, int64_t n, int level, const uint32_t* __restrict__ gstart,
                          float* __restrict__ rec) {
  extern __shared__ __align__(16) unsigned char sm3[];
  constexpr int NW = K3R_NW;
  const BrickGeom g = brick_geom(level);
  const K3RSmem L = k3r_smem(C, g.nb);
  float* sp = reinterpret_cast<float*>(sm3 + L.pts);
  float* sw = reinterpret_cast<float*>(sm3 + L.wts);
  uint32_t* key = reinterpret_cast<uint32_t*>(sm3 + L.key);
  uint32_t* wcw = reinterpret_cast<uint32_t*>(sm3 + L.wc);          // [NW][nb / 2] words
  uint16_t* wc = reinterpret_cast<uint16_t*>(sm3 + L.wc);           // [NW][nb]
  uint32_t* delta = reinterpret_cast<uint32_t*>(sm3 + L.delta);     // global - tile slot
  uint16_t* perm = reinterpret_cast<uint16_t*>(sm3 + L.perm);
  __shared__ uint32_t warp_tot[32];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t t0 = (int64_t)blockIdx.x * K3R_TILE;
  const int tn = (int)min((int64_t)K3R_TILE, n - t0);
  const int nbw = g.nb >> 1;   // counter words per warp (nb even, <= 1024)
  // 0. the tile's points and weights: one bulk copy each (TMA)
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  uint32_t expect = 0;
  if (!bulk_stage(sp, pts + 3 * t0, (uint32_t)(12 * tn), bar_s, expect))
    stage_floats(sp, pts + 3 * t0, 3 * tn);
  if (!bulk_stage(sw, wts + (int64_t)C * t0, (uint32_t)(4 * C * tn), bar_s, expect))
    stage_floats(sw, wts + (int64_t)C * t0, C * tn);
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s),
                 "r"(expect));
  // ... meanwhile: clear the counters
  for (int i = threadIdx.x; i < NW * nbw / 4; i += blockDim.x)
    reinterpret_cast<uint4*>(wcw)[i] = make_uint4(0u, 0u, 0u, 0u);
  __syncthreads();
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "K3W_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
      "@!p bra K3W_%=;\n\t}\n" ::"r"(bar_s)
      : "memory");
  // 1. ranks within the warp's points, in index order
  const unsigned lt = lanemask_lt();
  uint32_t* myw = wcw + (size_t)w * nbw;
#pragma unroll
  for (int grp = 0; grp < K3R_PER_WARP; grp += 32) {
    const int tp = w * K3R_PER_WARP + grp + lane;
    const bool ok = tp < tn;
    const int b = ok ? point_brick(sp[3 * tp], sp[3 * tp + 1], sp[3 * tp + 2], g) : 0;
    const uint32_t sh = (uint32_t)(b & 1) << 4;
    const uint32_t pre = (myw[b >> 1] >> sh) & 0xffffu;   // only this warp writes its row
    __syncwarp();
    if (ok) atomicAdd(myw + (b >> 1), 1u << sh);
    __syncwarp();
    // more than one lane on this brick: rank the group in lane order
    const bool clash = ok && ((myw[b >> 1] >> sh) & 0xffffu) != pre + 1;
    const unsigned cm = __ballot_sync(0xffffffffu, clash);
    uint32_t r = pre;
    if (clash) r += (uint32_t)__popc(__match_any_sync(cm, b) & lt);
    if (ok) key[tp] = ((uint32_t)b << 13) | r;
    __syncwarp();
  }
  __syncthreads();
  // 2. thread t owns counter word t (bricks 2t, 2t + 1): the exclusive
  //    prefix over the warps (packed: both halves stay < 2^11), the tile
  //    starts, then every warp's counter := tile slot of its first point
  uint32_t pre[NW], run = 0;
  const int t = threadIdx.x;
  if (t < nbw) {
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      pre[q] = run;
      run += wcw[q * nbw + t];
    }
  }
  const uint32_t c0 = run & 0xffffu, c1 = run >> 16;
  uint32_t total;
  const uint32_t st = block_exclusive_scan(c0 + c1, warp_tot, total);
  if (t < nbw) {
    const uint32_t base = st | ((st + c0) << 16);
#pragma unroll
    for (int q = 0; q < NW; ++q) wcw[q * nbw + t] = pre[q] + base;
    const uint32_t* gs = gstart + (size_t)blockIdx.x * g.nb + 2 * t;
    delta[2 * t] = __ldg(gs) - st;
    delta[2 * t + 1] = __ldg(gs + 1) - (st + c0);
  }
  __syncthreads();
  // 3. tile slot of every point
  for (int tp = threadIdx.x; tp < tn; tp += blockDim.x) {
    const uint32_t k = key[tp];
    perm[wc[(tp / K3R_PER_WARP) * g.nb + (k >> 13)] + (k & 8191u)] = (uint16_t)tp;
  }
  __syncthreads();
  // 4. brick runs out, coalesced: slot s -> record delta[brick] + s
  if (RS == 4) {
    for (int s = threadIdx.x; s < tn; s += blockDim.x) {
      const int tp = perm[s];
      const uint32_t gsl = delta[key[tp] >> 13] + (uint32_t)s;
      reinterpret_cast<float4*>(rec)[gsl] =
          make_float4(sp[3 * tp], sp[3 * tp + 1], sp[3 * tp + 2], sw[tp]);
    }
  } else {
    const int r4 = RS / 4;
    for (int e = threadIdx.x; e < tn * r4; e += blockDim.x) {
      const int s = e / r4, f = e - s * r4;
      const int tp = perm[s];
      const size_t gsl = delta[key[tp] >> 13] + (uint32_t)s;
      float v[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = 4 * f + j;
        v[j] = c < 3 ? sp[3 * tp + c] : (c < 3 + C ? sw[C * tp + c - 3] : 0.f);
      }
      reinterpret_cast<float4*>(rec)[gsl * r4 + f] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
}

// ------------------------------------------------------------------- K4 ---
// One CTA (CB threads) per brick; thread = cell of the brick, one channel at
// a time.  The brick's records stream through shared memory in chunks of
// K4_CHUNK.  Warp w ranks records [w K4_CHUNK / NW, ...) of the chunk, 32 at
// a time, against its own 16-bit cell counters (the K3r scheme: an atomicAdd
// per lane, lanes that share a cell in the group ranked in lane order by
// __match_any_sync) -- so every cell's run comes out in record (= index)
// order with no fix-up sort.  Per cell the exclusive prefix over the warps
// and the chunk's counting-sort starts, then each thread accumulates its
// cell's run in order.  Coefficient tables per axis carry the factorials
// (and the weight): px[k] = w dx^k / k!, so w d^n / n! = px[a] py[b] pz[c]
// (expansion.py:96-113).
#ifndef FC2T2_K4_CHUNK
#define FC2T2_K4_CHUNK 2048
#endif
#ifndef FC2T2_K4_MINB
#define FC2T2_K4_MINB 4
#endif
constexpr int K4_CHUNK = FC2T2_K4_CHUNK;

template <int RHO, int CB>
constexpr int k4_min_blocks() {
  return CB >= 512 ? 1 : (RHO >= 5 ? 2 : FC2T2_K4_MINB);   // rho >= 5: 56+ accumulators
}

// records per warp and the key layout: cell-in-brick << RB | rank in warp
template <int CB>
struct K4Keys {
  static constexpr int NW = CB / 32, PER_WARP = K4_CHUNK / NW;
  static constexpr int RB = CB >= 512 ? 7 : 8;
  static_assert(PER_WARP <= (1 << RB) && (CB - 1) < (1 << (16 - RB)), "16-bit keys");
  static_assert(PER_WARP % 32 == 0, "whole groups");
};

template <int CB>
constexpr size_t k4_smem() {
  // srec float4 + key uint16 + perm uint16 per record; per-warp packed 16-bit
  // cell counters; per cell its chunk start and count
  return (size_t)K4_CHUNK * (16 + 2 + 2) + (size_t)(CB / 32) * CB * 2 + (size_t)CB * 8;
}

template <int RHO, int CB>
__global__ void __launch_bounds__(CB, (k4_min_blocks<RHO, CB>()))
brick_p2m_kernel(const float* __restrict__ rec, int C, int RS, int level,
                 const uint32_t* __restrict__ brick_start, float* __restrict__ M) {
  constexpr int PP = MI<RHO>::PP;
  constexpr int BZ = CB / 64, BZS = BZ == 8 ? 3 : 2;
  using KK = K4Keys<CB>;
  constexpr int NW = KK::NW, PW = KK::PER_WARP, RB = KK::RB, CW = CB / 2;
  extern __shared__ __align__(16) unsigned char smem[];
  float4* srec = reinterpret_cast<float4*>(smem);                      // [K4_CHUNK]
  uint16_t* key = reinterpret_cast<uint16_t*>(srec + K4_CHUNK);        // [K4_CHUNK]
  uint16_t* perm = key + K4_CHUNK;                                     // [K4_CHUNK]
  uint32_t* wcw = reinterpret_cast<uint32_t*>(perm + K4_CHUNK);        // [NW][CB / 2]
  uint16_t* wc = reinterpret_cast<uint16_t*>(wcw);                     // [NW][CB]
  uint32_t* cst = wcw + NW * CW;                                       // [CB]
  uint32_t* ccnt = cst + CB;                                           // [CB]
  __shared__ uint32_t warp_tot[32];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(&bar);
  if (RS == 4 && threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  uint32_t phase = 0;

  const BrickGeom g = brick_geom(level);
  const int brick = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = lanemask_lt();
  const int bz = brick % g.nbz, by = (brick / g.nbz) % g.nby, bx = brick / (g.nbz * g.nby);
  // this thread's cell
  const int ccx = bx * 8 + (tid >> (3 + BZS)), ccy = by * 8 + ((tid >> BZS) & 7),
            ccz = bz * BZ + (tid & (BZ - 1));
  const int64_t cell = ((int64_t)ccx * g.res + ccy) * g.res + ccz;
  const uint32_t beg = brick_start[brick], end = brick_start[brick + 1];
  uint32_t* myw = wcw + warp * CW;

  for (int c = 0; c < C; ++c) {
    float acc[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) acc[j] = 0.f;
    for (uint32_t c0 = beg; c0 < end; c0 += K4_CHUNK) {
      const int nc = (int)umin((uint32_t)K4_CHUNK, end - c0);
      for (int i = tid; i < NW * CW; i += CB) wcw[i] = 0u;
      __syncthreads();   // also: the previous chunk's walk is done with srec / perm
      if (RS == 4) {
        // C = 1: the chunk's records are contiguous -- one bulk copy (TMA)
        if (threadIdx.x == 0) {
          // the previous chunk's generic-proxy stores to srec precede the copy
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s),
                       "r"((uint32_t)nc * 16u));
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
              "[%3];\n" ::"r"((uint32_t)__cvta_generic_to_shared(srec)),
              "l"(rec + (size_t)c0 * 4), "r"((uint32_t)nc * 16u), "r"(bar_s)
              : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "W4_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra W4_%=;\n\t}\n" ::"r"(bar_s),
            "r"(phase)
            : "memory");
        phase ^= 1u;
      } else {
        for (int k = tid; k < nc; k += CB) {
          const float* r = rec + (size_t)(c0 + k) * RS;
          srec[k] = make_float4(__ldg(r), __ldg(r + 1), __ldg(r + 2), __ldg(r + 3 + c));
        }
        __syncthreads();
      }
      // (x, y, z, w) -> (dx, dy, dz, w) in place; cell-in-brick key and the
      // deterministic rank within the warp's records
#pragma unroll 2
      for (int k0 = warp * PW; k0 < warp * PW + PW; k0 += 32) {
        const int k = k0 + lane;
        const bool ok = k < nc;
        uint32_t cib = 0;
        if (ok) {
          const float4 v = srec[k];
          const int cx = box_axis(v.x, g.res), cy = box_axis(v.y, g.res), cz = box_axis(v.z, g.res);
          srec[k] = make_float4(box_offset(v.x, cx, g.res), box_offset(v.y, cy, g.res),
                                box_offset(v.z, cz, g.res), v.w);
          cib = (uint32_t)((((cx & 7) << 3) | (cy & 7)) << BZS) | (cz & (BZ - 1));
        }
        const uint32_t sh = (cib & 1u) << 4;
        const uint32_t pre = (myw[cib >> 1] >> sh) & 0xffffu;
        __syncwarp();
        if (ok) atomicAdd(myw + (cib >> 1), 1u << sh);
        __syncwarp();
        const bool clash = ok && ((myw[cib >> 1] >> sh) & 0xffffu) != pre + 1;
        const unsigned cm = __ballot_sync(0xffffffffu, clash);
        uint32_t r = pre;
        if (clash) r += (uint32_t)__popc(__match_any_sync(cm, cib) & lt);
        if (ok) key[k] = (uint16_t)((cib << RB) | r);
        __syncwarp();
      }
      __syncthreads();
      // per cell: prefix over the warps (thread t < CB / 2 owns cells 2t,
      // 2t + 1; packed halves stay < 2^12), chunk starts, then every warp's
      // counter := chunk slot of its first record of the cell
      uint32_t pre[NW], run = 0;
      if (tid < CW) {
#pragma unroll
        for (int q = 0; q < NW; ++q) {
          pre[q] = run;
          run += wcw[q * CW + tid];
        }
      }
      const uint32_t n0 = run & 0xffffu, n1 = run >> 16;
      uint32_t total;
      const uint32_t st = block_exclusive_scan(n0 + n1, warp_tot, total);
      if (tid < CW) {
        const uint32_t base = st | ((st + n0) << 16);
#pragma unroll
        for (int q = 0; q < NW; ++q) wcw[q * CW + tid] = pre[q] + base;
        cst[2 * tid] = st;
        cst[2 * tid + 1] = st + n0;
        ccnt[2 * tid] = n0;
        ccnt[2 * tid + 1] = n1;
      }
      __syncthreads();
      for (int k = tid; k < nc; k += CB) {
        const uint32_t kk = key[k];
        perm[wc[(k / PW) * CB + (kk >> RB)] + (kk & ((1u << RB) - 1u))] = (uint16_t)k;
      }
      __syncthreads();
      // this cell's run, in index order
      const uint32_t mine = ccnt[tid];
      const uint16_t* mine_run = perm + cst[tid];
      for (uint32_t e = 0; e < mine; ++e) {
        const float4 v = srec[mine_run[e]];
        float px[RHO + 1], py[RHO + 1], pz[RHO + 1];
        px[0] = v.w;      // the weight rides on the x table
        py[0] = 1.f;
        pz[0] = 1.f;
#pragma unroll
        for (int q = 1; q <= RHO; ++q) {
          const float inv = 1.f / (float)q;
          px[q] = px[q - 1] * v.x * inv;
          py[q] = py[q - 1] * v.y * inv;
          pz[q] = pz[q - 1] * v.z * inv;
        }
#pragma unroll
        for (int a = 0; a <= RHO; ++a)
#pragma unroll
          for (int b = 0; b <= RHO - a; ++b) {
            const float wxy = px[a] * py[b];
#pragma unroll
            for (int cc = 0; cc <= RHO - a - b; ++cc)
              acc[MI<RHO>::index(a, b, cc)] = fmaf(wxy, pz[cc], acc[MI<RHO>::index(a, b, cc)]);
          }
      }
    }
    float* dst = M + ((size_t)cell * C + c) * PP;
#pragma unroll
    for (int j = 0; j < PP; j += 4)
      *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
}

struct BrickWs {
  uint32_t *cnt, *part, *tot, *bstart;
  float* rec;
};

size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

int rec_floats(int C) { return 4 * ((3 + C + 3) / 4); }

// points per K1/K3 tile: ~8 per brick (short runs for the in-order fix-up),
// between 256 and 6144, and at most 96 KB of raw points + weights in smem
bool rank_scatter(int level, int C) {
  const BrickGeom g = brick_geom(level);
  return g.nb <= 1024 && k3r_smem(C, g.nb).total <= 100 * 1024 && g.nb >= 64;
}

int brick_tile(int level, int C) {
  const BrickGeom g = brick_geom(level);
  if (rank_scatter(level, C)) return K3R_TILE;
  const int cap = std::min(6144, 98304 / ((3 + C) * 4) / K13_THREADS * K13_THREADS);
  const int want = (8 * g.nb + K13_THREADS - 1) / K13_THREADS * K13_THREADS;
  return std::max(K13_THREADS, std::min(cap, want));
}

int64_t brick_tiles(int64_t n, int level, int C) {
  const int t = brick_tile(level, C);
  return std::max<int64_t>(1, (n + t - 1) / t);
}

BrickWs brick_carve(void* ws, int level, int64_t n, int C) {
  const BrickGeom g = brick_geom(level);
  const int64_t nt = brick_tiles(n, level, C);
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { char* q = p; p += al256(bytes); return (void*)q; };
  BrickWs w;
  w.cnt = (uint32_t*)take((size_t)nt * g.nb * 4);
  w.part = (uint32_t*)take((size_t)((nt + SEG_T - 1) / SEG_T) * g.nb * 4);
  w.tot = (uint32_t*)take((size_t)g.nb * 4);
  w.bstart = (uint32_t*)take((size_t)(g.nb + 1) * 4);
  w.rec = (float*)take((size_t)std::max<int64_t>(n, 1) * rec_floats(C) * 4);
  return w;
}

// K4 launch; the shared-memory attribute is set once per device and per
// <RHO, CB> instantiation
template <int RHO, int CB>
cudaError_t launch_k4(const BrickWs& b, int C, int RS, int level, int nb, float* M,
                      cudaStream_t s) {
  constexpr size_t sm = k4_smem<CB>();
  static unsigned long long configured = 0;
  // static + dynamic shared memory above 48 KB needs the opt-in (the
  // kernel's static part is ~0.6 KB, so set it from 32 KB of dynamic)
  if (sm > 32 * 1024 && attr_needed(configured)) {
    cudaError_t e = cudaFuncSetAttribute(brick_p2m_kernel<RHO, CB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  FC2T2_LAUNCH("brick_p2m", s,
               brick_p2m_kernel<RHO, CB><<<(unsigned)nb, CB, sm, s>>>(b.rec, C, RS, level,
                                                                    b.bstart, M));
  return cudaSuccess;
}

}  // namespace

bool p2m_brick_supported(int level, int C) {
  return level >= 2 && level <= 6 && C >= 1 && C <= 8;
}

size_t p2m_brick_workspace(int level, int64_t n, int C) {
  const BrickGeom g = brick_geom(level);
  const int64_t nt = brick_tiles(n, level, C);
  return al256((size_t)nt * g.nb * 4) + al256((size_t)((nt + SEG_T - 1) / SEG_T) * g.nb * 4) +
         al256((size_t)g.nb * 4) + al256((size_t)(g.nb + 1) * 4) +
         al256((size_t)std::max<int64_t>(n, 1) * rec_floats(C) * 4);
}

cudaError_t p2m_brick(int rho, int level, int C, const float* pts, const float* w, int64_t n,
                      float* M, int32_t* flag, void* ws, size_t ws_bytes, cudaStream_t s,
                      int phase) {
  if (!p2m_brick_supported(level, C) || n < 0 || n > (int64_t)UINT32_MAX - 1)
    return cudaErrorNotSupported;
  if (ws_bytes < p2m_brick_workspace(level, n, C)) return cudaErrorInvalidValue;
  const BrickGeom g = brick_geom(level);
  BrickWs b = brick_carve(ws, level, n, C);
  const int tile = brick_tile(level, C);
  const int64_t nt = brick_tiles(n, level, C);
  if (nt > INT32_MAX / 2) return cudaErrorInvalidValue;
  const int RS = rec_floats(C);
  const bool rk = rank_scatter(level, C);
  const size_t sm3 = rk ? k3r_smem(C, g.nb).total : k3_smem(tile, C, g.nb).total;
  static unsigned long long attr = 0;
  if (attr_needed(attr)) {
    cudaError_t e = cudaFuncSetAttribute(brick_scatter_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(brick_scatter_rank_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
  }
  if (sm3 > 200 * 1024) return cudaErrorInvalidValue;
  if (phase & P2M_PREPARE) {
  FC2T2_LAUNCH("brick_hist", s,
               brick_hist_kernel<<<(unsigned)nt, K13_THREADS, g.nb * 4, s>>>(pts, n, level, tile,
                                                                            b.cnt, flag));
  const int nseg = (int)((nt + SEG_T - 1) / SEG_T);
  const dim3 sgrid((unsigned)((g.nb + 31) / 32), (unsigned)nseg);
  if (nt <= kSmallScanTiles && (g.nb + 31) / 32 <= kSmallScanCtas) {
    static std::atomic<unsigned> next_slot{0};
    const int slot = (int)(next_slot.fetch_add(1, std::memory_order_relaxed) % kScanSlots);
    FC2T2_LAUNCH("brick_scan", s,
                 brick_scan_small_kernel<<<(unsigned)((g.nb + 31) / 32), 1024, 0, s>>>(
                     b.cnt, (int)nt, g.nb, b.tot, b.bstart, slot));
  } else {
  FC2T2_LAUNCH("brick_scan", s,
               brick_segsum_kernel<<<sgrid, 256, 0, s>>>(b.cnt, (int)nt, g.nb, b.part));
  FC2T2_LAUNCH("brick_scan", s,
               brick_segscan_kernel<<<(g.nb + 7) / 8, 256, 0, s>>>(b.part, nseg, g.nb, b.tot));
  FC2T2_LAUNCH("brick_scan", s, brick_start_kernel<<<1, 1024, 0, s>>>(b.tot, g.nb, b.bstart));
  FC2T2_LAUNCH("brick_scan", s,
               brick_segfill_kernel<<<sgrid, 256, 0, s>>>(b.cnt, (int)nt, g.nb, b.part, b.bstart));
  }
  }
  if (!(phase & P2M_FINISH)) return cudaGetLastError();
  if (n > 0 && rk)
    FC2T2_LAUNCH("brick_scatter", s,
                 brick_scatter_rank_kernel<<<(unsigned)nt, K3R_THREADS, sm3, s>>>(
                     pts, w, C, RS, n, level, b.cnt, b.rec));
  else if (n > 0)
    FC2T2_LAUNCH("brick_scatter", s,
                 brick_scatter_kernel<<<(unsigned)nt, K3_THREADS, sm3, s>>>(
                     pts, w, C, RS, n, level, tile, b.cnt, b.rec));
  cudaError_t e = cudaSuccess;
  FC2T2_DISPATCH_RHO(rho, {
    if (g.cb == 512) e = launch_k4<RHO, 512>(b, C, RS, level, g.nb, M, s);
    else e = launch_k4<RHO, 256>(b, C, RS, level, g.nb, M, s);
  });
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace fc2t2
