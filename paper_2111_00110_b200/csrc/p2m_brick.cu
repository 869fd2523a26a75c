// P2M from unsorted points: a deterministic partition of the points into
// bricks of cells, then one CTA per brick sums each cell's points in source
// index order (reference Engine.p2m, expansion.py:186-198: np.add.at over
// the cell key of :195 -- the per-cell summation order is the point order).
//
//   K1 brick_hist     warp tiles of consecutive points; per tile a histogram
//                     over bricks (shared memory, counts only: order free)
//   S1-S3             per brick, the exclusive prefix over tiles (a column
//                     scan of the tile x brick count matrix) plus the brick
//                     start offsets  -> every (tile, brick) its first slot
//   K3 brick_scatter  every warp re-walks its tile 32 points at a time; lanes
//                     with equal bricks are ranked by __match_any_sync (lane
//                     order), the group leader advances the warp's own cursor:
//                     a STABLE partition -- inside a brick, points stay in
//                     index order -- written as records {x, y, z, w...}
//   K4 brick_p2m      one CTA per brick, one thread per cell; the brick's
//                     records stream through shared memory in chunks, a
//                     stable counting sort by cell (per-warp counters) lists
//                     each cell's points in index order, and every thread
//                     accumulates its cell's moment row in registers.
//
// No float atomics and no data-dependent ordering anywhere: moments are
// bit-reproducible run to run.  Bytes per point: 12 (K1) + 12 + 4C (K3 in)
// + 4 RS (K3 out, K4 in, RS = record floats) -- no random gathers (the
// previous cell sort + gather P2M read every point through an index).
#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

struct BrickGeom {
  int res, bz, nbx, nby, nbz, nb, cb;
};

// 8 x 8 x BZ cells per brick; BZ = 4 (256 cells) up to level 5, 8 (512 cells)
// at level 6.  Level >= 7 is not served by this path.
__host__ __device__ inline BrickGeom brick_geom(int level) {
  BrickGeom g;
  g.res = 1 << (level + 1);
  g.bz = level >= 6 ? 8 : 4;
  g.nbx = g.res / 8;
  g.nby = g.res / 8;
  g.nbz = g.res / g.bz;
  g.nb = g.nbx * g.nby * g.nbz;
  g.cb = 64 * g.bz;
  return g;
}

__device__ __forceinline__ void point_brick(float x, float y, float z, const BrickGeom& g,
                                            int& b, int& cx, int& cy, int& cz) {
  cx = box_axis(x, g.res);
  cy = box_axis(y, g.res);
  cz = box_axis(z, g.res);
  b = ((cx >> 3) * g.nby + (cy >> 3)) * g.nbz + cz / g.bz;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ------------------------------------------------------------------- K1 ---
__global__ void brick_hist_kernel(const float* __restrict__ pts, int64_t n, int level,
                                  int64_t tile, int ntiles, uint32_t* __restrict__ cnt,
                                  int32_t* __restrict__ flag) {
  extern __shared__ uint32_t sh[];
  const BrickGeom g = brick_geom(level);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * (blockDim.x >> 5) + w;
  if (t >= ntiles) return;
  uint32_t* h = sh + (size_t)w * g.nb;
  for (int b = lane; b < g.nb; b += 32) h[b] = 0u;
  __syncwarp();
  const int64_t lo = (int64_t)t * tile, hi = min(n, lo + tile);
  int bad = 0;
#pragma unroll 4
  for (int64_t i = lo + lane; i < hi; i += 32) {
    const float x = __ldg(pts + 3 * i), y = __ldg(pts + 3 * i + 1), z = __ldg(pts + 3 * i + 2);
    bad |= outside_domain(x, y, z);
    int b, cx, cy, cz;
    point_brick(x, y, z, g, b, cx, cy, cz);
    atomicAdd(h + b, 1u);
  }
  __syncwarp();
  uint32_t* row = cnt + (size_t)t * g.nb;
  for (int b = lane; b < g.nb; b += 32) row[b] = h[b];
  if (__any_sync(0xffffffffu, bad) && lane == 0 && flag) atomicOr(flag, FLAG_DOMAIN);
}

// ---------------------------------------------------------------- S1-S3 ---
constexpr int GT = 32;   // tiles per group of the column scan

// gsum[grp][b] = sum of cnt[t][b] over the group's tiles
__global__ void brick_colsum_kernel(const uint32_t* __restrict__ cnt, int ntiles, int nb,
                                    uint32_t* __restrict__ gsum) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int grp = blockIdx.y;
  if (b >= nb) return;
  const int t0 = grp * GT, t1 = min(ntiles, t0 + GT);
  uint32_t s = 0;
#pragma unroll 8
  for (int t = t0; t < t1; ++t) s += cnt[(size_t)t * nb + b];
  gsum[(size_t)grp * nb + b] = s;
}

// one CTA: brick totals, their exclusive scan (brick_start, nb + 1 entries)
// and gsum turned into each group's first slot per brick
__global__ void __launch_bounds__(1024)
brick_start_kernel(uint32_t* __restrict__ gsum, int ngrp, int nb,
                   uint32_t* __restrict__ brick_start) {
  __shared__ uint32_t warp_tot[32];
  const int per = (nb + blockDim.x - 1) / blockDim.x;   // <= 4 (nb <= 4096)
  const int b0 = threadIdx.x * per;
  uint32_t tot[4] = {0u, 0u, 0u, 0u};
  uint32_t mine = 0;
  for (int k = 0; k < per; ++k) {
    const int b = b0 + k;
    if (b >= nb) break;
    uint32_t s = 0;
    for (int grp = 0; grp < ngrp; ++grp) s += gsum[(size_t)grp * nb + b];
    tot[k] = s;
    mine += s;
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(mine, warp_tot, total);
  for (int k = 0; k < per; ++k) {
    const int b = b0 + k;
    if (b >= nb) break;
    brick_start[b] = run;
    uint32_t r = run;
    for (int grp = 0; grp < ngrp; ++grp) {
      const uint32_t v = gsum[(size_t)grp * nb + b];
      gsum[(size_t)grp * nb + b] = r;
      r += v;
    }
    run += tot[k];
  }
  if (threadIdx.x == blockDim.x - 1) brick_start[nb] = total;
}

// cnt[t][b] <- first slot of (tile t, brick b)
__global__ void brick_offsets_kernel(uint32_t* __restrict__ cnt, int ntiles, int nb,
                                     const uint32_t* __restrict__ gpre) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  const int grp = blockIdx.y;
  if (b >= nb) return;
  const int t0 = grp * GT, t1 = min(ntiles, t0 + GT);
  uint32_t run = gpre[(size_t)grp * nb + b];
#pragma unroll 8
  for (int t = t0; t < t1; ++t) {
    const uint32_t c = cnt[(size_t)t * nb + b];
    cnt[(size_t)t * nb + b] = run;
    run += c;
  }
}

// ------------------------------------------------------------------- K3 ---
// records: RS floats per point (dx, dy, dz, w_0..w_{C-1}, zero pad), RS % 4
// == 0, with d = the offset from the cell centre (box_offset: float64
// difference, one rounding -- the reference's expansion.py:190 in float32),
// and cib = the cell's index inside its brick (uint16).  Each lane handles
// U points per step (U independent loads in flight).
constexpr int K3_U = 4;

__global__ void __launch_bounds__(256)
brick_scatter_kernel(const float* __restrict__ pts, const float* __restrict__ wts, int C, int RS,
                     int64_t n, int level, int64_t tile, int ntiles,
                     const uint32_t* __restrict__ off, float* __restrict__ rec,
                     uint16_t* __restrict__ cibs) {
  extern __shared__ uint32_t sh[];
  const BrickGeom g = brick_geom(level);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = blockIdx.x * (blockDim.x >> 5) + w;
  if (t >= ntiles) return;
  uint32_t* cur = sh + (size_t)w * g.nb;
  const uint32_t* row = off + (size_t)t * g.nb;
  for (int b = lane; b < g.nb; b += 32) cur[b] = row[b];
  __syncwarp();
  const int64_t lo = (int64_t)t * tile, hi = min(n, lo + tile);
  const unsigned lt = lanemask_lt();
  for (int64_t base = lo; base < hi; base += 32 * K3_U) {
    float dx[K3_U], dy[K3_U], dz[K3_U], w0[K3_U];
    int bk[K3_U], cib[K3_U];
#pragma unroll
    for (int u = 0; u < K3_U; ++u) {
      const int64_t i = base + u * 32 + lane;
      bk[u] = g.nb + lane;            // unique key for idle lanes
      cib[u] = 0;
      dx[u] = dy[u] = dz[u] = w0[u] = 0.f;
      if (i < hi) {
        const float x = __ldg(pts + 3 * i), y = __ldg(pts + 3 * i + 1), z = __ldg(pts + 3 * i + 2);
        w0[u] = __ldg(wts + i * C);
        int cx, cy, cz;
        point_brick(x, y, z, g, bk[u], cx, cy, cz);
        cib[u] = ((cx & 7) * 8 + (cy & 7)) * g.bz + cz % g.bz;
        dx[u] = box_offset(x, cx, g.res);
        dy[u] = box_offset(y, cy, g.res);
        dz[u] = box_offset(z, cz, g.res);
      }
    }
#pragma unroll
    for (int u = 0; u < K3_U; ++u) {
      const int64_t i = base + u * 32 + lane;
      const bool ok = i < hi;
      const unsigned grp = __match_any_sync(0xffffffffu, bk[u]);
      const int leader = __ffs(grp) - 1;
      uint32_t slot = 0;
      if (ok && lane == leader) {
        slot = cur[bk[u]];
        cur[bk[u]] = slot + (uint32_t)__popc(grp);
      }
      slot = __shfl_sync(0xffffffffu, slot, leader) + (uint32_t)__popc(grp & lt);
      __syncwarp();
      if (ok) {
        float* r = rec + (size_t)slot * RS;
        cibs[slot] = (uint16_t)cib[u];
        if (RS == 4) {
          *reinterpret_cast<float4*>(r) = make_float4(dx[u], dy[u], dz[u], w0[u]);
        } else {
          r[0] = dx[u];
          r[1] = dy[u];
          r[2] = dz[u];
          r[3] = w0[u];
          for (int c = 1; c < C; ++c) r[3 + c] = __ldg(wts + i * C + c);
          for (int c = 3 + C; c < RS; ++c) r[c] = 0.f;
        }
      }
    }
  }
}

// ------------------------------------------------------------------- K4 ---
// One CTA (CB threads) per brick; thread = cell of the brick, one channel at
// a time.  Coefficient tables per axis carry the factorials (and the weight):
// px[k] = w dx^k / k!, so w d^n / n! = px[a] py[b] pz[c] (expansion.py:96-113).
constexpr int K4_CHUNK = 1024;   // records per shared-memory chunk

template <int RHO, int CB>
constexpr int k4_min_blocks() {
  return CB >= 512 ? 1 : (MI<RHO>::PP <= 36 ? 3 : 2);
}

template <int RHO, int CB>
__global__ void __launch_bounds__(CB, (k4_min_blocks<RHO, CB>()))
brick_p2m_kernel(const float* __restrict__ rec, const uint16_t* __restrict__ cibs, int C, int RS,
                 int level, const uint32_t* __restrict__ brick_start, float* __restrict__ M) {
  constexpr int PP = MI<RHO>::PP;
  constexpr int NW = CB / 32;
  constexpr int BZ = CB / 64;
  extern __shared__ __align__(16) unsigned char smem[];
  float4* srec = reinterpret_cast<float4*>(smem);                            // [K4_CHUNK]
  uint16_t* scell = reinterpret_cast<uint16_t*>(srec + K4_CHUNK);           // [K4_CHUNK]
  uint16_t* perm = scell + K4_CHUNK;                                         // [K4_CHUNK]
  uint32_t* wcnt = reinterpret_cast<uint32_t*>(perm + K4_CHUNK);             // [CB][NW]
  uint32_t* cstart = wcnt + CB * NW;                                         // [CB + 1]
  __shared__ uint32_t warp_tot[32];

  const BrickGeom g = brick_geom(level);
  const int brick = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int bz = brick % g.nbz, by = (brick / g.nbz) % g.nby, bx = brick / (g.nbz * g.nby);
  // this thread's cell
  const int ccx = bx * 8 + (tid / (8 * BZ)), ccy = by * 8 + ((tid / BZ) & 7),
            ccz = bz * BZ + (tid % BZ);
  const int64_t cell = ((int64_t)ccx * g.res + ccy) * g.res + ccz;
  const uint32_t beg = brick_start[brick], end = brick_start[brick + 1];
  const unsigned lt = lanemask_lt();

  for (int c = 0; c < C; ++c) {
    float acc[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) acc[j] = 0.f;
    for (uint32_t c0 = beg; c0 < end; c0 += K4_CHUNK) {
      const int nc = (int)umin((uint32_t)K4_CHUNK, end - c0);
      for (int k = tid; k < CB * NW; k += CB) wcnt[k] = 0u;
      // load the chunk (dx, dy, dz, w_c) and each record's cell in the brick
      for (int k = tid; k < nc; k += CB) {
        const float* r = rec + (size_t)(c0 + k) * RS;
        srec[k] = RS == 4 ? __ldg(reinterpret_cast<const float4*>(r))
                          : make_float4(__ldg(r), __ldg(r + 1), __ldg(r + 2), __ldg(r + 3 + c));
        scell[k] = __ldg(cibs + c0 + k);
      }
      __syncthreads();
      // stable counting sort by cell: warp `warp` owns items [r0, r1)
      const int per = (nc + NW - 1) / NW;
      const int r0 = min(nc, warp * per), r1 = min(nc, r0 + per);
      for (int k = r0 + lane; k < r1; k += 32) atomicAdd(&wcnt[(int)scell[k] * NW + warp], 1u);
      __syncthreads();
      // exclusive scan over (cell, warp), cell-major: thread = cell
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < NW; ++q) s += wcnt[tid * NW + q];
      uint32_t total;
      uint32_t run = block_exclusive_scan(s, warp_tot, total);
      cstart[tid] = run;
      if (tid == CB - 1) cstart[CB] = total;
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        const uint32_t v = wcnt[tid * NW + q];
        wcnt[tid * NW + q] = run;
        run += v;
      }
      __syncthreads();
      for (int k0 = r0; k0 < r1; k0 += 32) {
        const int k = k0 + lane;
        const int key = k < r1 ? (int)scell[k] : CB + lane;
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(grp) - 1;
        uint32_t slot = 0;
        if (k < r1 && lane == leader) {
          slot = wcnt[key * NW + warp];
          wcnt[key * NW + warp] = slot + (uint32_t)__popc(grp);
        }
        slot = __shfl_sync(0xffffffffu, slot, leader) + (uint32_t)__popc(grp & lt);
        if (k < r1) perm[slot] = (uint16_t)k;
        __syncwarp();
      }
      __syncthreads();
      // this cell's points of the chunk, in index order
      const int e1 = (int)cstart[tid + 1];
      for (int e = (int)cstart[tid]; e < e1; ++e) {
        const float4 v = srec[perm[e]];
        float px[RHO + 1], py[RHO + 1], pz[RHO + 1];
        px[0] = v.w;      // the weight rides on the x table
        py[0] = 1.f;
        pz[0] = 1.f;
#pragma unroll
        for (int k = 1; k <= RHO; ++k) {
          const float inv = 1.f / (float)k;
          px[k] = px[k - 1] * v.x * inv;
          py[k] = py[k - 1] * v.y * inv;
          pz[k] = pz[k - 1] * v.z * inv;
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
      __syncthreads();
    }
    float* dst = M + ((size_t)cell * C + c) * PP;
#pragma unroll
    for (int j = 0; j < PP; j += 4)
      *reinterpret_cast<float4*>(dst + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
  }
}

template <int CB>
size_t k4_smem() {
  return (size_t)K4_CHUNK * (16 + 2 + 2) + (size_t)CB * (CB / 32) * 4 + (size_t)(CB + 1) * 4;
}

struct BrickWs {
  uint32_t *cnt, *gsum, *bstart;
  float* rec;
  uint16_t* cib;
};

size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

int brick_tiles(int64_t n, int nb) {
  const int64_t maxt = nb > 1024 ? 148 * 12 : 148 * 16;
  int64_t t = (n + 1023) / 1024;
  if (t < 1) t = 1;
  return (int)std::min<int64_t>(t, maxt);
}

int rec_floats(int C) { return 4 * ((3 + C + 3) / 4); }

BrickWs brick_carve(void* ws, int level, int64_t n, int C) {
  const BrickGeom g = brick_geom(level);
  const int nt = brick_tiles(n, g.nb), ng = (nt + GT - 1) / GT;
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { char* q = p; p += al256(bytes); return (void*)q; };
  BrickWs w;
  w.cnt = (uint32_t*)take((size_t)nt * g.nb * 4);
  w.gsum = (uint32_t*)take((size_t)ng * g.nb * 4);
  w.bstart = (uint32_t*)take((size_t)(g.nb + 1) * 4);
  w.rec = (float*)take((size_t)std::max<int64_t>(n, 1) * rec_floats(C) * 4);
  w.cib = (uint16_t*)take((size_t)std::max<int64_t>(n, 1) * 2);
  return w;
}

}  // namespace

bool p2m_brick_supported(int level, int C) {
  return level >= 2 && level <= 6 && C >= 1 && C <= 8;
}

size_t p2m_brick_workspace(int level, int64_t n, int C) {
  const BrickGeom g = brick_geom(level);
  const int nt = brick_tiles(n, g.nb), ng = (nt + GT - 1) / GT;
  return al256((size_t)nt * g.nb * 4) + al256((size_t)ng * g.nb * 4) +
         al256((size_t)(g.nb + 1) * 4) + al256((size_t)std::max<int64_t>(n, 1) * rec_floats(C) * 4) +
         al256((size_t)std::max<int64_t>(n, 1) * 2);
}

cudaError_t p2m_brick(int rho, int level, int C, const float* pts, const float* w, int64_t n,
                      float* M, int32_t* flag, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (!p2m_brick_supported(level, C) || n < 0 || n > (int64_t)UINT32_MAX - 1)
    return cudaErrorNotSupported;
  if (ws_bytes < p2m_brick_workspace(level, n, C)) return cudaErrorInvalidValue;
  const BrickGeom g = brick_geom(level);
  BrickWs b = brick_carve(ws, level, n, C);
  const int nt = brick_tiles(n, g.nb), ng = (nt + GT - 1) / GT;
  const int64_t tile = ((std::max<int64_t>(n, 1) + nt - 1) / nt + 31) / 32 * 32;
  const int nw = g.nb > 1024 ? 4 : 8;
  const size_t sm13 = (size_t)nw * g.nb * 4;
  static unsigned long long attr = 0;
  if (attr_needed(attr)) {
    cudaError_t e = cudaFuncSetAttribute(brick_hist_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4096 * 4);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(brick_scatter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               4 * 4096 * 4);
    if (e != cudaSuccess) return e;
  }
  const unsigned blocks13 = (unsigned)((nt + nw - 1) / nw);
  FC2T2_LAUNCH("brick_hist", s,
               brick_hist_kernel<<<blocks13, 32 * nw, sm13, s>>>(pts, n, level, tile, nt, b.cnt,
                                                                 flag));
  const dim3 cgrid((unsigned)((g.nb + 255) / 256), (unsigned)ng);
  FC2T2_LAUNCH("brick_scan", s,
               brick_colsum_kernel<<<cgrid, 256, 0, s>>>(b.cnt, nt, g.nb, b.gsum));
  FC2T2_LAUNCH("brick_scan", s,
               brick_start_kernel<<<1, 1024, 0, s>>>(b.gsum, ng, g.nb, b.bstart));
  FC2T2_LAUNCH("brick_scan", s,
               brick_offsets_kernel<<<cgrid, 256, 0, s>>>(b.cnt, nt, g.nb, b.gsum));
  const int RS = rec_floats(C);
  if (n > 0)
    FC2T2_LAUNCH("brick_scatter", s,
                 brick_scatter_kernel<<<blocks13, 32 * nw, sm13, s>>>(pts, w, C, RS, n, level,
                                                                      tile, nt, b.cnt, b.rec,
                                                                      b.cib));
  auto launch4 = [&](auto kern, int cb) -> cudaError_t {
    const size_t sm = cb >= 512 ? k4_smem<512>() : k4_smem<256>();
    static unsigned long long a4[2] = {0, 0};
    if (attr_needed(a4[cb >= 512])) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)sm);
      if (e != cudaSuccess) return e;
    }
    FC2T2_LAUNCH("brick_p2m", s,
                 kern<<<(unsigned)g.nb, cb, sm, s>>>(b.rec, b.cib, C, RS, level, b.bstart, M));
    return cudaSuccess;
  };
  cudaError_t e = cudaSuccess;
  FC2T2_DISPATCH_RHO(rho, {
    if (g.cb == 512) e = launch4(brick_p2m_kernel<RHO, 512>, 512);
    else e = launch4(brick_p2m_kernel<RHO, 256>, 256);
  });
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace fc2t2
