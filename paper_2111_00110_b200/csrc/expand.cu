// The FC2T2 cascade on the device: P2M (sorted, segmented), M2M, M2L, L2L.
//
// Reference: pkg/src/fc2t2/expansion.py
//   p2m   :186-198   M[cell, c, n] = sum_{i in cell} w_ic d_i^n / n!
//   m2m   :200-213   coarse += sum_children fine[child] @ K_child^T, K lower-tri
//   l2l   :215-225   fine[child] = coarse @ K_child^T, K upper-tri
//   m2l   :227-264   L[t] += A_o M[t + o] over the level's active offsets,
//                    parity restriction on +-3 offsets (:246-249)
#include "common.cuh"
#include "kernels.cuh"
#include "shift.cuh"

#include <cstdlib>

namespace fc2t2 {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int PP>
__device__ __forceinline__ void store_row(float* dst, const float (&v)[PP], bool accumulate) {
#pragma unroll
  for (int k = 0; k < PP; k += 4) {
    float4 o = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
    if (accumulate) {
      float4 a = *reinterpret_cast<const float4*>(dst + k);
      o.x += a.x; o.y += a.y; o.z += a.z; o.w += a.w;
    }
    *reinterpret_cast<float4*>(dst + k) = o;
  }
}

template <int PP>
__device__ __forceinline__ void load_row(const float* src, float (&v)[PP]) {
#pragma unroll
  for (int k = 0; k < PP; k += 4) {
    float4 a = __ldg(reinterpret_cast<const float4*>(src + k));
    v[k] = a.x; v[k + 1] = a.y; v[k + 2] = a.z; v[k + 3] = a.w;
  }
}

// ------------------------------------------------------------------ P2M ---
// One thread per (cell, channel): walk the cell's points in ascending source
// index (stable sort) and accumulate w * d^n/n! in registers -- the same
// association order as np.add.at, no atomics.  (Default.)
template <int RHO>
__global__ void __launch_bounds__(128)
p2m_sorted_kernel(const float* __restrict__ pts, const float* __restrict__ w, int C, int res,
                  const int32_t* __restrict__ order, const int32_t* __restrict__ cell_start,
                  float* __restrict__ M) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  const int64_t R = (int64_t)res * res * res;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < R * C;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / C;
    const int c = (int)(g - cell * C);
    const int b2 = (int)(cell % res), b1 = (int)((cell / res) % res), b0 = (int)(cell / res / res);
    float acc[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) acc[j] = 0.f;
    const int beg = cell_start[cell], end = cell_start[cell + 1];
    int k = beg;
    // batches of 4 points: the 4 index loads, then the 4 coordinate/weight
    // gathers are all in flight before the first contraction (the sum order
    // is unchanged: points still accumulate one by one in index order)
    for (; k + 4 <= end; k += 4) {
      int64_t ii[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) ii[u] = order ? (int64_t)order[k + u] : (int64_t)(k + u);
      float px[4], py[4], pz[4], pw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        px[u] = pts[3 * ii[u]];
        py[u] = pts[3 * ii[u] + 1];
        pz[u] = pts[3 * ii[u] + 2];
        pw[u] = w[ii[u] * C + c];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float mono[P];
        monomials<RHO>(box_offset(px[u], b0, res), box_offset(py[u], b1, res),
                       box_offset(pz[u], b2, res), mono);
#pragma unroll
        for (int j = 0; j < P; ++j) acc[j] = fmaf(pw[u], mono[j], acc[j]);
      }
    }
    for (; k < end; ++k) {
      const int64_t i = order ? (int64_t)order[k] : (int64_t)k;  // no order: pre-sorted inputs
      const float dx = box_offset(pts[3 * i], b0, res);
      const float dy = box_offset(pts[3 * i + 1], b1, res);
      const float dz = box_offset(pts[3 * i + 2], b2, res);
      const float wv = w[i * C + c];
      float mono[P];
      monomials<RHO>(dx, dy, dz, mono);
#pragma unroll
      for (int j = 0; j < P; ++j) acc[j] = fmaf(wv, mono[j], acc[j]);
    }
    store_row<PP>(M + g * PP, acc, false);
  }
}

// ------------------------------------------------------------- M2M/L2L ---
// Child centre offset from the parent centre is d = (c - 1/2) * w_fine per
// axis (reference expansion.py:170-175).  The binomial shift kernel
// K[n, m] = d^(n-m) / (n-m)! (reference _shift_kernel, expansion.py:116-132)
// factorises over the axes, so the 3D shift is three exact 1D shifts; every
// intermediate index stays inside the total-degree table because a shift
// only moves weight between indices of one axis.
//
//   UP   (M2M): out[n] = sum_{m <= n_a}  in[n - m e_a] t[m]
//   DOWN (L2L): out[n] = sum_{m >= 0}    in[n + m e_a] t[m]   (|n + m e_a| <= rho)
template <int RHO>
__global__ void __launch_bounds__(128)
m2m_kernel(const float* __restrict__ fine, float* __restrict__ coarse, int C, int cres,
           float half_fine, int64_t g0, int64_t g1) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  const int fres = 2 * cres;
  for (int64_t g = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < g1;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / C;
    const int c = (int)(g - cell * C);
    const int Z = (int)(cell % cres), Y = (int)((cell / cres) % cres), X = (int)(cell / cres / cres);
    float acc[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) acc[j] = 0.f;
#pragma unroll 1
    for (int ch = 0; ch < 8; ++ch) {
      const int cx = ch >> 2, cy = (ch >> 1) & 1, cz = ch & 1;
      const int64_t fc = (((int64_t)(2 * X + cx) * fres + (2 * Y + cy)) * fres + (2 * Z + cz));
      float f[PP];
      load_row<PP>(fine + (fc * C + c) * PP, f);
      float v[P];
#pragma unroll
      for (int j = 0; j < P; ++j) v[j] = f[j];
      shift3<RHO, true>(v, cx ? half_fine : -half_fine, cy ? half_fine : -half_fine,
                        cz ? half_fine : -half_fine);
#pragma unroll
      for (int j = 0; j < P; ++j) acc[j] += v[j];
    }
    store_row<PP>(coarse + g * PP, acc, false);
  }
}

// M2M with a thread per child: the 8 children of a parent sit in 8 adjacent
// lanes (child = lane & 7, x slowest), each shifts its own row, and an xor
// butterfly over the 8 lanes forms the parent's sum -- (c0+c1)+(c2+c3) +
// (c4+c5)+(c6+c7), the same tree in every lane -- 8x the threads of the
// per-parent loop on these small grids.
template <int RHO>
__global__ void __launch_bounds__(256)
m2m_child_kernel(const float* __restrict__ fine, float* __restrict__ coarse, int C, int cres,
                 float half_fine, int64_t g0, int64_t g1) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  const int fres = 2 * cres;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int ch = (int)(t & 7);
  const int64_t gq = g0 + (t >> 3);
  const bool valid = gq < g1;
  const int64_t g = valid ? gq : g1 - 1;
  const int64_t cell = g / C;
  const int c = (int)(g - cell * C);
  const int Z = (int)(cell % cres), Y = (int)((cell / cres) % cres), X = (int)(cell / cres / cres);
  const int cx = ch >> 2, cy = (ch >> 1) & 1, cz = ch & 1;
  const int64_t fc = (((int64_t)(2 * X + cx) * fres + (2 * Y + cy)) * fres + (2 * Z + cz));
  float f[PP];
  load_row<PP>(fine + (fc * C + c) * PP, f);
  float v[P];
#pragma unroll
  for (int j = 0; j < P; ++j) v[j] = f[j];
  shift3<RHO, true>(v, cx ? half_fine : -half_fine, cy ? half_fine : -half_fine,
                    cz ? half_fine : -half_fine);
#pragma unroll
  for (int o = 1; o < 8; o <<= 1)
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
  if (valid && ch == 0) {
    float out[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) out[j] = j < P ? v[j] : 0.f;
    store_row<PP>(coarse + g * PP, out, false);
  }
}

template <int RHO>
__global__ void __launch_bounds__(128)
l2l_kernel(const float* __restrict__ coarse, float* __restrict__ fine, int C, int cres,
           float half_fine, int accumulate, int64_t g0, int64_t g1) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  const int fres = 2 * cres;
  for (int64_t g = g0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < g1;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / C;
    const int c = (int)(g - cell * C);
    const int z = (int)(cell % fres), y = (int)((cell / fres) % fres), x = (int)(cell / fres / fres);
    const int64_t pc = ((int64_t)(x >> 1) * cres + (y >> 1)) * cres + (z >> 1);
    float a[PP];
    load_row<PP>(coarse + (pc * C + c) * PP, a);
    float v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = a[j];
    shift3<RHO, false>(v, (x & 1) ? half_fine : -half_fine, (y & 1) ? half_fine : -half_fine,
                       (z & 1) ? half_fine : -half_fine);
    float out[PP];
#pragma unroll
    for (int j = 0; j < PP; ++j) out[j] = j < P ? v[j] : 0.f;
    store_row<PP>(fine + g * PP, out, accumulate != 0);
  }
}

// ------------------------------------------------------------------ M2L ---
// Implicit GEMM on FP32 FFMA.  A CTA owns ROWS = 128*RPL (target, channel)
// rows of one target parity class and walks that class's interaction list;
// per entry it stages the gathered source rows M[t + o] (cp.async with
// zero-fill for out-of-domain sources = the reference's slice clipping,
// expansion.py:135-151) and the PPxPP table B[n][k] = A_o[k][n] in shared
// memory (double buffered) and does a rank-PP update of its register tile.
constexpr int M2L_THREADS = 128;

template <int RHO, int RPL>
__global__ void __launch_bounds__(M2L_THREADS, (RHO <= 4 ? 2 : 1))
m2l_ffma_kernel(const float* __restrict__ M, float* __restrict__ L, int C, int res, int stride,
                int nu, const int4* __restrict__ entries, const int* __restrict__ cls_start,
                const float* __restrict__ coef, int accumulate, float* __restrict__ part,
                int64_t part_stride, int64_t u_begin, int64_t u_end) {
  constexpr int PP = MI<RHO>::PP;
  constexpr int NQ = PP / 4;
  constexpr int ROWS = M2L_THREADS * RPL;
  extern __shared__ __align__(16) float smem[];
  float* As = smem;                                   // [2][ROWS][PP]
  float* Bs = smem + 2 * ROWS * PP;                   // [2][PP][PP]
  int4* rowinfo = reinterpret_cast<int4*>(Bs + 2 * PP * PP);  // [ROWS]

  const int cls = blockIdx.y;
  const int ox = stride == 2 ? (cls >> 2) & 1 : 0;
  const int oy = stride == 2 ? (cls >> 1) & 1 : 0;
  const int oz = stride == 2 ? cls & 1 : 0;
  const int tpt = ROWS / C;
  const int64_t ntgt = u_end;
  const int64_t t0 = u_begin + (int64_t)blockIdx.x * tpt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int r = tid; r < ROWS; r += M2L_THREADS) {
    int4 info = make_int4(0, 0, 0, -1);
    const int tl = r / C, c = r - tl * C;
    const int64_t u = t0 + tl;
    if (tl < tpt && u < ntgt) {
      const int uz = (int)(u % nu), uy = (int)((u / nu) % nu), ux = (int)(u / nu / nu);
      info = make_int4(ux * stride + ox, uy * stride + oy, uz * stride + oz, c);
    }
    rowinfo[r] = info;
  }
  __syncthreads();

  // split-K over the interaction list (blockIdx.z); each split writes its own
  // partial grid, summed in split order by m2l_reduce_kernel (deterministic)
  int lb = cls_start[cls], nl = cls_start[cls + 1] - lb;
  if (gridDim.z > 1) {
    const int chunk = (nl + gridDim.z - 1) / gridDim.z;
    const int b = min(nl, (int)blockIdx.z * chunk);
    nl = min(nl, b + chunk) - b;
    lb += b;
    L = part + blockIdx.z * part_stride;
    accumulate = 0;
  }

  auto stage = [&](int li, int buf) {
    const int4 e = __ldg(entries + lb + li);
    float* Ad = As + buf * ROWS * PP;
    for (int q = tid; q < ROWS * NQ; q += M2L_THREADS) {
      const int r = q / NQ, ch = q - r * NQ;
      const int4 info = rowinfo[r];
      const int sx = info.x + e.x, sy = info.y + e.y, sz = info.z + e.z;
      const bool ok = info.w >= 0 && (unsigned)sx < (unsigned)res && (unsigned)sy < (unsigned)res &&
                      (unsigned)sz < (unsigned)res;
      const float* src =
          ok ? M + ((((int64_t)sx * res + sy) * res + sz) * C + info.w) * PP + ch * 4 : M;
      cp_async16(Ad + r * PP + ch * 4, src, ok ? 16 : 0);
    }
    const float* Bsrc = coef + (int64_t)e.w * PP * PP;
    float* Bd = Bs + buf * PP * PP;
    for (int q = tid; q < PP * NQ; q += M2L_THREADS) cp_async16(Bd + q * 4, Bsrc + q * 4, 16);
    cp_async_commit();
  };

  float acc[RPL][PP];
#pragma unroll
  for (int i = 0; i < RPL; ++i)
#pragma unroll
    for (int k = 0; k < PP; ++k) acc[i][k] = 0.f;

  if (nl > 0) stage(0, 0);
  for (int li = 0; li < nl; ++li) {
    const int buf = li & 1;
    if (li + 1 < nl) {
      stage(li + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const float* Ab = As + buf * ROWS * PP + (warp * 32 * RPL + lane) * PP;
    const float* Bb = Bs + buf * PP * PP;
#pragma unroll 1
    for (int n4 = 0; n4 < NQ; ++n4) {
      float4 a[RPL];
#pragma unroll
      for (int i = 0; i < RPL; ++i)
        a[i] = *reinterpret_cast<const float4*>(Ab + i * 32 * PP + n4 * 4);
#pragma unroll
      for (int nn = 0; nn < 4; ++nn) {
        const float* brow = Bb + (n4 * 4 + nn) * PP;
#pragma unroll
        for (int k4 = 0; k4 < NQ; ++k4) {
          const float4 b = *reinterpret_cast<const float4*>(brow + k4 * 4);
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const float av = nn == 0 ? a[i].x : nn == 1 ? a[i].y : nn == 2 ? a[i].z : a[i].w;
            acc[i][4 * k4 + 0] = fmaf(av, b.x, acc[i][4 * k4 + 0]);
            acc[i][4 * k4 + 1] = fmaf(av, b.y, acc[i][4 * k4 + 1]);
            acc[i][4 * k4 + 2] = fmaf(av, b.z, acc[i][4 * k4 + 2]);
            acc[i][4 * k4 + 3] = fmaf(av, b.w, acc[i][4 * k4 + 3]);
          }
        }
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = warp * 32 * RPL + i * 32 + lane;
    const int4 info = rowinfo[r];
    if (info.w < 0) continue;
    const int64_t cell = ((int64_t)info.x * res + info.y) * res + info.z;
    store_row<PP>(L + (cell * C + info.w) * PP, acc[i], accumulate != 0);
  }
}

__global__ void m2l_reduce_kernel(float4* __restrict__ L, const float4* __restrict__ part,
                                  int64_t i0, int64_t n4, int64_t stride4, int splits,
                                  int accumulate) {
  for (int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 s = accumulate ? L[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int z = 0; z < splits; ++z) {
      const float4 v = part[z * stride4 + i];
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    L[i] = s;
  }
}

template <int RHO>
constexpr int m2l_rpl() { return MI<RHO>::PP <= 36 ? 2 : 1; }

template <int RHO>
size_t m2l_smem() {
  constexpr int PP = MI<RHO>::PP;
  constexpr int ROWS = M2L_THREADS * m2l_rpl<RHO>();
  return (size_t)(2 * ROWS * PP + 2 * PP * PP) * sizeof(float) + ROWS * sizeof(int4);
}

}  // namespace

cudaError_t p2m_sorted(int rho, int level, int C, const float* pts, const float* w,
                       const int32_t* order, const int32_t* cell_start, float* M,
                       cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int64_t n = (int64_t)res * res * res * C;
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("p2m", s,
      p2m_sorted_kernel<RHO><<<grid_blocks(n, 128, 148 * 64), 128, 0, s>>>(
          pts, w, C, res, order, cell_start, M)));
  return cudaGetLastError();
}

cudaError_t m2m(int rho, int fine_level, int C, const float* fine, float* coarse,
                cudaStream_t s, int cx_begin, int cx_end) {
  const int cres = 1 << fine_level;  // res of fine_level - 1
  if (cx_end < 0) cx_end = cres;
  const int64_t plane = (int64_t)cres * cres * C;
  const int64_t g0 = cx_begin * plane, g1 = cx_end * plane;
  if (g1 <= g0) return cudaSuccess;
  const float half_fine = (float)(0.5 * 2.0 / (double)(2 * cres));
  // grids of up to 64^3 parents: a thread per child (latency bound otherwise)
  if (cres <= 64) {
    const int64_t threads = (g1 - g0) * 8;
    FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("m2m", s,
        m2m_child_kernel<RHO><<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
            fine, coarse, C, cres, half_fine, g0, g1)));
    return cudaGetLastError();
  }
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("m2m", s,
      m2m_kernel<RHO><<<grid_blocks(g1 - g0, 128, 148 * 64), 128, 0, s>>>(fine, coarse, C, cres,
                                                                          half_fine, g0, g1)));
  return cudaGetLastError();
}

cudaError_t l2l(int rho, int coarse_level, int C, const float* coarse, float* fine,
                int accumulate, cudaStream_t s, int fx_begin, int fx_end) {
  const int cres = 1 << (coarse_level + 1);
  const int fres = 2 * cres;
  if (fx_end < 0) fx_end = fres;
  const int64_t plane = (int64_t)fres * fres * C;
  const int64_t g0 = fx_begin * plane, g1 = fx_end * plane;
  if (g1 <= g0) return cudaSuccess;
  const float half_fine = (float)(0.5 * 2.0 / (double)(2 * cres));
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("l2l", s,
      l2l_kernel<RHO><<<grid_blocks(g1 - g0, 128, 148 * 64), 128, 0, s>>>(
          coarse, fine, C, cres, half_fine, accumulate, g0, g1)));
  return cudaGetLastError();
}

int m2l_splits(int rho, int C, const M2LLaunch& plan) {
  const int res = 1 << (plan.level + 1);
  const int nu = res / plan.stride;
  const int rows = 128 * (index_count(rho) <= 35 ? 2 : 1);
  const int tpt = std::max(1, rows / C);
  const int64_t ctas = ((int64_t)nu * nu * nu + tpt - 1) / tpt * plan.ncls;
  // two waves of CTAs, at most 32 splits (measured at config 2 level 3, 16
  // CTAs per split: 19 splits 45 us, 16 splits 54 us, 32 splits 56 us)
  constexpr int waves = 2, cap = 32;
  const int64_t want = (waves * 148 + ctas - 1) / ctas;
  return (int)std::max<int64_t>(1, std::min<int64_t>({want, (int64_t)cap, (int64_t)plan.max_list}));
}

cudaError_t m2l(int rho, int C, const M2LLaunch& plan, const float* coef, const float* M,
                float* L, int accumulate, cudaStream_t s, float* part, int splits, int x_begin,
                int x_end) {
  const int res = 1 << (plan.level + 1);
  const int nu = res / plan.stride;
  if (x_end < 0) x_end = res;
  // targets with x in [x_begin, x_end): class-lattice x in [x_begin, x_end) / stride
  if (x_begin % plan.stride || x_end % plan.stride) return cudaErrorInvalidValue;
  const int64_t u_begin = (int64_t)(x_begin / plan.stride) * nu * nu;
  const int64_t u_end = (int64_t)(x_end / plan.stride) * nu * nu;
  if (u_end <= u_begin) return cudaSuccess;
  if (!part) splits = 1;
  const int64_t grid_f = (int64_t)res * res * res * C * pad4(index_count(rho));
  FC2T2_DISPATCH_RHO(rho, {
    constexpr int RPL = m2l_rpl<RHO>();
    constexpr int ROWS = M2L_THREADS * RPL;
    if (C > ROWS) return cudaErrorNotSupported;
    const int tpt = ROWS / C;
    const size_t smem = m2l_smem<RHO>();
    auto kern = m2l_ffma_kernel<RHO, RPL>;
    static unsigned long long attr = 0;   // devices configured (per instantiation)
    if (attr_needed(attr)) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
    }
    dim3 grid((unsigned)((u_end - u_begin + tpt - 1) / tpt), (unsigned)plan.ncls, (unsigned)splits);
    FC2T2_LAUNCH(plan.level_name, s,
                 kern<<<grid, M2L_THREADS, smem, s>>>(M, L, C, res, plan.stride, nu, plan.entries,
                                                      plan.cls_start, coef, accumulate, part,
                                                      grid_f, u_begin, u_end));
  });
  if (splits > 1) {
    // the slab's rows are contiguous: cells x in [x_begin, x_end)
    const int64_t row4 = (int64_t)res * res * C * pad4(index_count(rho)) / 4;
    const int64_t i0 = x_begin * row4, i1 = x_end * row4;
    FC2T2_LAUNCH("m2l_reduce", s,
                 m2l_reduce_kernel<<<grid_blocks(i1 - i0, 256, 148 * 16), 256, 0, s>>>(
                     (float4*)L, (const float4*)part, i0, i1, grid_f / 4, splits, accumulate));
  }
  return cudaGetLastError();
}

}  // namespace fc2t2
