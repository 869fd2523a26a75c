// M2L on the 5th-generation tensor cores: tcgen05.mma kind::f16, two-term fp16 split.
//
// Reference: Engine.m2l (expansion.py:227-264).  For a target parity class pi
// the level's interaction list is a GEMM
//     L[t, k] = sum_{delta, n} M[t + delta, n] * A_delta[k, n]
// (rows = targets t, K = (delta, n), N = k).  Split by the *source* parity
// sigma = (pi + delta) mod 2, every delta is a shift s = (pi + delta - sigma)/2
// in {-1, 0, 1}^3 of the sigma-lattice, and the source rows of (sigma, s) for a
// target tile are the SAME for every target class pi (lattice index u + s).  So
// one MMA serves CLS target classes at once: B = the CLS tables of
// delta_pi = 2 s + sigma - pi side by side (zero where delta_pi is not in pi's
// list), A = one shifted view of the staged sigma-window.  The loop over
// (sigma, s, K step) is dense and static (8 x 27 x KS); no entry lists.
//
// Why: a tcgen05.mma with SS operands costs max(N/2, 32 + N/4) cycles at
// M = 128 (measured, scripts/ubench/mma_rate2.cu): the 4 KB A tile and the
// N x 32 B B tile are read from shared memory at 128 B/clk.  Below N = 128 the
// MMA is operand-bandwidth bound; pairing classes lifts rho = 4 from N = 96/48
// (one class) to N = 160/80.
//
// Precision: both operands are split x = hi + lo so that D = Ahi Bhi +
// (Ahi Blo + Alo Bhi) carries ~22 significant bits (3 products; Alo Blo is
// below fp32 resolution): fp16 hi = rn(x'), lo = rn((x' - hi) * 2^11) on
// power-of-two scaled operands -- moments A' = M / (g_c s_n) with static
// per-coefficient scales s_n = (h/2)^|n| / n! (|M_n| <= sum|w| s_n), a
// per-call per-channel power of two g_c (device abs-max, max|A'| <= 2^13),
// tables B' = B s_n / r_k with static per-output-column r_k.  The cross
// products are 2^11 too large and the output is L = g_c r_k (D_hh +
// 2^-11 D_s).  A kind::f16 instruction takes K = 16 at the cycle cost of a
// kind::tf32 K = 8, so a K step covers twice the coefficients (3xTF32 was
// the first version of this kernel).
// Tensor-core accumulation into TMEM truncates, so the large hi*hi products
// of each source class sigma go to their own TMEM set (double buffered,
// drained into fp32 registers with RN adds and re-zeroed), while the small
// terms (2^-11 smaller) accumulate in one persistent set.  TMEM per tile:
// [hh1 | s | hh0], W = CLS*NC columns each.  Even sigma: B rows [lo | hi] and
// the main MMA A_hi*B writes [s | hh0]; odd sigma: B rows [hi | lo], main
// writes [hh1 | s]; the cross MMA A_lo*B_hi always writes s.  All MMAs
// accumulate (TMEM is zeroed by the drain warps).
//
// CTA (16 warps): 0 MMA issuer (warp-uniform loop, elect-one per MMA),
// 1 B producer (one cp.async.bulk per 9-slot stage), 2-7 window gatherers
// (cp.async, zero-fill = the reference's domain clipping, expansion.py:135-151),
// 8-15 TMEM drain (warp % 4 = TMEM lane quarter, two column halves).
// TILES 1 x 16 x 8 target tiles stacked along x share one
// (TILES + 2) x 18 x 10 window.
#include <cuda_fp16.h>
#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

constexpr int pow2_at_least(int v) {
  int p = 32;
  while (p < v) p *= 2;
  return p;
}

template <class T>
struct Tag {
  using type = T;
};

// TL > 0 overrides the tiles per CTA.
template <int RHO, int TL = 0>
struct TC {
  static constexpr int RHO_ = RHO;
  static constexpr int TL_ = TL;
  static constexpr int P = index_count(RHO);
  static constexpr int PP = pad4(P);
  static constexpr int KI = 16;                         // K per MMA instruction (32 B rows)
  static constexpr int KPAD = (P + KI - 1) / KI * KI;   // K per offset
  static constexpr int KS = KPAD / KI;
  static constexpr int ESZ = 2;                         // bytes per operand element (fp16)
  static constexpr int CLS = 4 * ((P + 7) / 8 * 8) <= 256 ? 2 : 1;   // target classes per CTA
  static constexpr int NC = CLS == 2 ? (P + 7) / 8 * 8 : (P + 15) / 16 * 16;  // N per class
  static constexpr int W = CLS * NC;                   // one TMEM set; cross MMA N
  // Two target tiles per CTA halve the table traffic.  With the hi*hi set
  // double buffered a tile needs 3W columns ([hh1 | s | hh0]); when two such
  // tiles do not fit in 512 columns (rho >= 5) the set is single buffered,
  // [s | hh] per tile, and the MMA waits for each source-class drain (~3 % of
  // a group's MMA time).
  static constexpr bool SB = 6 * W > 512 && 4 * W <= 512;
  static constexpr int NSETS = SB ? 1 : 2;
  static constexpr int TW = (SB ? 2 : 3) * W;          // TMEM columns per tile
  static constexpr int TILES = TL > 0 ? TL : ((6 * W <= 512 || SB) ? 2 : 1);
  static constexpr int TMEM_COLS = pow2_at_least(TILES * TW);
  static constexpr int TY = 16, TZ = 8;
  static constexpr int WX = TILES + 2, WY = TY + 2, WZ = TZ + 2;
  static constexpr int WROWS = WX * WY * WZ;
  static constexpr int WSLICE = 2 * 2 * WROWS * 16;   // [part hi/lo][kchunk][row][16 B]
  static constexpr int SLOTS = 27, DPS = 9, CHUNKS = 3;
  // table rows one CTA stages per slot: both halves of B
  static constexpr int BROWS = 2 * W;
  static constexpr int BSLOT = 2 * BROWS * 16;        // [kchunk][row][16 B]
  static constexpr int BSTAGE = DPS * BSLOT;
  static constexpr int NS = 2 * WSLICE + 3 * BSTAGE + 1024 <= 232448 ? 3 : 2;
  static constexpr int THREADS = 512;
  static constexpr int GATHER_WARP0 = 2, GATHER_WARPS = 6;
  static constexpr int GATHER_THREADS = 32 * GATHER_WARPS;
  static constexpr int DRAIN_WARP0 = 8, DW = 2;
  static constexpr int DRAIN_THREADS = 32 * 4 * DW;
  static constexpr int CW = TILES * W / DW;           // accumulator columns per drain thread
  // The last K step holds P - (KS-1)*KI real inputs; when they fit in one
  // chunk (KI/2), its A operand is [A_hi chunk | A_lo chunk] (descriptor LBO
  // spanning the two window parts) against table rows [B_hi | B_lo] and
  // [0 | B_hi]: one main MMA yields all three products, no cross MMA.
  static constexpr bool MERGE_LAST = P - (KS - 1) * KI <= KI / 2;
  static constexpr size_t SMEM = 2 * (size_t)WSLICE + (size_t)NS * BSTAGE + 512;
  // instruction descriptor: D f32; A/B f16 (0); K-major; N >> 3; M >> 4
  static constexpr uint32_t idesc(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  }
  static constexpr uint32_t IDESC_MAIN = idesc(2 * W);
  static constexpr uint32_t IDESC_CROSS = idesc(W);
  static_assert(2 * W <= 256 && W % 16 == 0, "MMA N out of range");
  static_assert(CW % 8 == 0 && (TILES == 1 || CW == W), "drain split");
  static_assert(TILES * TW <= 512, "TMEM");
};

constexpr float kLoScale = 2048.f;   // fp16 lo parts carry the residual * 2^11
constexpr int kGExp = 13;            // max |A'| <= 2^13

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version for sm_100; base offset 0; SWIZZLE_NONE
  return d;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity));
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes));
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(dst), "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void cp_async16_zfill(uint32_t dst, const void* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes));
}

__device__ __forceinline__ void umma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n" ::"r"(d_tmem), "l"(a),
               "l"(b), "r"(idesc));
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}

// per-channel max over cells and n of |M[cell, c, n]| / s_n, as float bits
// (non-negative floats order like their bit patterns: atomicMax is exact and
// order independent).  grid.y = channel; one atomic per block.
template <int RHO>
__global__ void __launch_bounds__(256)
absmax_kernel(const float* __restrict__ M, const float* __restrict__ s_inv, int64_t cells, int C,
              uint32_t* __restrict__ gbits) {
  constexpr int PP = pad4(index_count(RHO)), Q = PP / 4;
  const int c = blockIdx.y;
  const int64_t n = cells * Q;
  float m = 0.f;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t cell = g / Q;
    const int q = (int)(g - cell * Q);
    const float4 v = *reinterpret_cast<const float4*>(M + (cell * C + c) * PP + 4 * q);
    const float* si = s_inv + 4 * q;
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x) * si[0], fabsf(v.y) * si[1]),
                       fmaxf(fabsf(v.z) * si[2], fabsf(v.w) * si[3])));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ float wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float b = wm[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) b = fmaxf(b, wm[i]);
    atomicMax(gbits + c, __float_as_uint(b));
  }
}

// exponent e with max |M/s| <= 2^e (0 for an all-zero channel)
__device__ __forceinline__ int gexp_of(uint32_t bits) {
  return bits == 0u ? 0 : (int)((bits >> 23) & 0xFF) - 127 + 1;
}

// fp16 two-term split of A' = M / (g_c s_n): (C, res^3, KPAD) halves
template <int RHO>
__global__ void __launch_bounds__(256)
split_f16_kernel(const float* __restrict__ M, const float* __restrict__ s_inv,
                 const uint32_t* __restrict__ gbits, uint2* __restrict__ hi,
                 uint2* __restrict__ lo, int64_t cells, int C) {
  using Cfg = TC<RHO>;
  constexpr int Q = Cfg::KPAD / 4;
  const int64_t n = cells * C * Q;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(g % Q);
    const int64_t cc = g / Q;  // (channel, cell) in output order
    const int c = (int)(cc / cells);
    const int64_t cell = cc - (int64_t)c * cells;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (4 * q < Cfg::PP) {
      const float4 m4 = *reinterpret_cast<const float4*>(M + (cell * C + c) * Cfg::PP + 4 * q);
      const float sc = ldexpf(1.f, kGExp - gexp_of(gbits[c]));
      v[0] = m4.x * s_inv[4 * q] * sc;
      v[1] = m4.y * s_inv[4 * q + 1] * sc;
      v[2] = m4.z * s_inv[4 * q + 2] * sc;
      v[3] = m4.w * s_inv[4 * q + 3] * sc;
    }
    uint16_t h[4], l[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __half hh = __float2half_rn(v[i]);
      h[i] = __half_as_ushort(hh);
      l[i] = __half_as_ushort(__float2half_rn((v[i] - __half2float(hh)) * kLoScale));
    }
    hi[g] = make_uint2((uint32_t)h[0] | ((uint32_t)h[1] << 16), (uint32_t)h[2] | ((uint32_t)h[3] << 16));
    lo[g] = make_uint2((uint32_t)l[0] | ((uint32_t)l[1] << 16), (uint32_t)l[2] | ((uint32_t)l[3] << 16));
  }
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %1, %1, %1, %1, %1, %1, %1};\n" ::"r"(taddr),
      "r"(0u)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "elect.sync _|P1, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

// ------------------------------------------------------------ M2L (tc) ---
template <int RHO, int TL>
__global__ void __launch_bounds__(512, 1)
m2l_tc_kernel(const uint8_t* __restrict__ Mhi, const uint8_t* __restrict__ Mlo,
              const uint8_t* __restrict__ Btab, const float* __restrict__ rk,
              const uint32_t* __restrict__ gbits, float* __restrict__ L, int res, int nu, int C,
              int accumulate, int ux_begin) {
  using T = TC<RHO, TL>;
  constexpr int W = T::W, NS = T::NS, KS = T::KS, TILES = T::TILES, CW = T::CW;
  constexpr int WROWS = T::WROWS, WY = T::WY, WZ = T::WZ;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* win = smem;                                  // [2][WSLICE]
  uint8_t* bring = smem + 2 * T::WSLICE;                // [NS][BSTAGE]
  uint64_t* bars = reinterpret_cast<uint64_t*>(bring + NS * T::BSTAGE);
  // bars: bfull[NS], bempty[NS], winready[2], winfree[2], accfull[2], accfree[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 8);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cg = blockIdx.y;     // class group: classes cg*CLS .. cg*CLS + CLS-1
  const int chan = blockIdx.z;
  const int nyb = nu / T::TY, nzb = nu / T::TZ;
  const int bid = blockIdx.x;
  const int ux0 = ux_begin + (bid / (nyb * nzb)) * TILES;
  const int uy0 = ((bid / nzb) % nyb) * T::TY;
  const int uz0 = (bid % nzb) * T::TZ;

  const uint32_t bar0 = smem_u32(bars);
  auto bfull = [&](int s) { return bar0 + 8u * s; };
  auto bempty = [&](int s) { return bar0 + 8u * (NS + s); };
  auto winready = [&](int b) { return bar0 + 8u * (2 * NS + b); };
  auto winfree = [&](int b) { return bar0 + 8u * (2 * NS + 2 + b); };
  auto accfull = [&](int b) { return bar0 + 8u * (2 * NS + 4 + b); };
  auto accfree = [&](int b) { return bar0 + 8u * (2 * NS + 6 + b); };
  if (warp == T::DRAIN_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(T::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bfull(s), 1);
      mbar_init(bempty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(winready(b), T::GATHER_THREADS);
      mbar_init(winfree(b), 1);
      mbar_init(accfull(b), 1);
      mbar_init(accfree(b), T::DRAIN_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- MMA issuer: warp-uniform loop, elect-one per MMA ----------------
    const uint32_t wb0 = smem_u32(win), bb0 = smem_u32(bring);
    int n = 0, q = 0;
    for (int sg = 0; sg < 8; ++sg) {
      const int set = T::SB ? 0 : (sg & 1);
      mbar_wait(accfree(set), (sg / T::NSETS) & 1);
      tc_fence_after();
      // main D: [hh1 | s] (odd) or [s | hh0] (even); single buffered: [s | hh]
      const uint32_t mcol = (T::SB || set) ? 0u : (uint32_t)W;
      // B_hi rows: second half for even sigma and always when single buffered
      const uint64_t xoff = (T::SB || !set) ? (uint64_t)W : 0u;
      const uint32_t scol = T::SB ? 0u : (uint32_t)W;   // small-term set
      for (int ks = 0; ks < KS; ++ks, ++q) {
        const int buf = q & 1;
        mbar_wait(winready(buf), (q >> 1) & 1);
        tc_fence_after();
        const uint64_t ahi = sdesc(wb0 + buf * T::WSLICE, WROWS * 16, WZ * 16);
        const uint64_t alo = ahi + (uint64_t)(2 * WROWS);
        const bool merged = T::MERGE_LAST && ks == KS - 1;
        // merged last step: K chunk 1 = the lo part's chunk 0, 2 WROWS rows on
        const uint64_t amain = merged ? sdesc(wb0 + buf * T::WSLICE, 2 * WROWS * 16, WZ * 16) : ahi;
#pragma unroll
        for (int ch = 0; ch < T::CHUNKS; ++ch, ++n) {
          const int s = n % NS;
          mbar_wait(bfull(s), (n / NS) & 1);
          tc_fence_after();
          const uint64_t b0 = sdesc(bb0 + s * T::BSTAGE, T::BROWS * 16, 128);
#pragma unroll
          for (int j = 0; j < T::DPS; ++j) {
            const int slot = ch * T::DPS + j;
            const uint64_t ex = (uint64_t)((slot / 9) * WY * WZ + ((slot / 3) % 3) * WZ + slot % 3);
            const uint64_t bd = b0 + (uint64_t)(j * T::BSLOT / 16);
#pragma unroll
            for (int t = 0; t < TILES; ++t) {
              const uint64_t arow = ex + (uint64_t)(t * WY * WZ);
              const uint32_t dt = tmem + (uint32_t)(t * T::TW);
              if (elect_one()) umma(dt + mcol, amain + arow, bd, T::IDESC_MAIN);
              if (!merged && elect_one()) umma(dt + scol, alo + arow, bd + xoff, T::IDESC_CROSS);
            }
          }
          if (elect_one()) umma_commit(bempty(s));
          __syncwarp();
        }
        if (elect_one()) umma_commit(winfree(buf));
        __syncwarp();
      }
      if (elect_one()) umma_commit(accfull(set));
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- B producer: one bulk copy per 9-slot stage ----------------
    if (lane == 0) {
      // table layout [cg][sigma][ks][slot][BSLOT]
      const uint8_t* tb = Btab + (size_t)cg * 8 * KS * T::SLOTS * T::BSLOT;
      int n = 0;
      for (int sg = 0; sg < 8; ++sg)
        for (int ks = 0; ks < KS; ++ks)
          for (int ch = 0; ch < T::CHUNKS; ++ch, ++n) {
            const int s = n % NS;
            if (n >= NS) mbar_wait(bempty(s), ((n / NS) - 1) & 1);
            mbar_expect_tx(bfull(s), T::BSTAGE);
            bulk_g2s(smem_u32(bring + s * T::BSTAGE),
                     tb + (((size_t)sg * KS + ks) * T::SLOTS + ch * T::DPS) * T::BSLOT, T::BSTAGE,
                     bfull(s));
          }
    }
  } else if (warp < T::DRAIN_WARP0) {
    // ---------------- window gatherers ----------------
    const int gt = tid - 32 * T::GATHER_WARP0;
    const size_t cells = (size_t)res * res * res;
    const uint8_t* hi_c = Mhi + (size_t)chan * cells * T::KPAD * T::ESZ;
    const uint8_t* lo_c = Mlo + (size_t)chan * cells * T::KPAD * T::ESZ;
    int q = 0;
    for (int sg = 0; sg < 8; ++sg) {
      const int sx = (sg >> 2) & 1, sy = (sg >> 1) & 1, sz = sg & 1;
      for (int ks = 0; ks < KS; ++ks, ++q) {
        const int buf = q & 1;
        if (q >= 2) mbar_wait(winfree(buf), ((q - 2) >> 1) & 1);
        uint8_t* wb = win + buf * T::WSLICE;
        for (int r = gt; r < WROWS; r += T::GATHER_THREADS) {
          const int wx = r / (WY * WZ), wy = (r / WZ) % WY, wz = r % WZ;
          const int cx = 2 * (ux0 - 1 + wx) + sx;
          const int cy = 2 * (uy0 - 1 + wy) + sy;
          const int cz = 2 * (uz0 - 1 + wz) + sz;
          const bool ok = (unsigned)cx < (unsigned)res && (unsigned)cy < (unsigned)res &&
                          (unsigned)cz < (unsigned)res;
          const size_t off =
              ok ? ((((size_t)cx * res + cy) * res + cz) * T::KPAD + ks * T::KI) * T::ESZ : 0;
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const uint8_t* src = (part ? lo_c : hi_c) + off;
#pragma unroll
            for (int kc = 0; kc < 2; ++kc)
              cp_async16_zfill(smem_u32(wb + ((part * 2 + kc) * WROWS + r) * 16), src + kc * 16,
                               ok ? 16 : 0);
          }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(winready(buf));
      }
    }
  } else {
    // ---------------- TMEM drain + epilogue ----------------
    const int dq = warp & 3, d = (warp - T::DRAIN_WARP0) >> 2;
    const int t = (d * CW) / W, c0 = (d * CW) % W;
    const uint32_t tb = tmem + ((uint32_t)(dq * 32) << 16) + (uint32_t)(t * T::TW + c0);
#pragma unroll
    for (int o = 0; o < T::TW / W; ++o)
#pragma unroll
      for (int c = 0; c < CW; c += 8) tmem_zero8(tb + o * W + c);
    tmem_wait_st();
    tc_fence_before();
    mbar_arrive(accfree(0));
    mbar_arrive(accfree(1));
    float acc[CW];
#pragma unroll
    for (int c = 0; c < CW; ++c) acc[c] = 0.f;
    for (int sg = 0; sg < 8; ++sg) {
      const int set = T::SB ? 0 : (sg & 1);
      mbar_wait(accfull(set), (sg / T::NSETS) & 1);
      tc_fence_after();
      const uint32_t hb = tb + (T::SB ? (uint32_t)W : (set ? 0u : (uint32_t)(2 * W)));
#pragma unroll
      for (int c = 0; c < CW; c += 8) {
        float v[8];
        tmem_ld8(hb + c, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[c + i] += v[i];
        tmem_zero8(hb + c);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(accfree(set));
    }
    // the small-term set is complete once the last group's commit has fired
    const float sfac = 1.f / kLoScale;
#pragma unroll
    for (int c = 0; c < CW; c += 8) {
      float v[8];
      tmem_ld8(tb + (T::SB ? 0u : (uint32_t)W) + c, v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[c + i] += v[i] * sfac;
    }
    {
      // undo the operand scaling: L = g_c r_k (D_hh + 2^-11 D_s)
      const float g = ldexpf(1.f, gexp_of(gbits[chan]) - kGExp);
#pragma unroll
      for (int c = 0; c < CW; ++c) acc[c] *= g * rk[(c0 + c) % T::NC];
    }
    const int row = dq * 32 + lane;
    const int ux = ux0 + t, uy = uy0 + row / T::TZ, uz = uz0 + row % T::TZ;
#pragma unroll
    for (int c = 0; c < CW; c += 4) {
      const int col = c0 + c, ci = col / T::NC, k = col % T::NC;
      if (k >= T::PP) continue;
      const int cls = cg * T::CLS + ci;
      const int px = (cls >> 2) & 1, py = (cls >> 1) & 1, pz = cls & 1;
      const int64_t cell = (((int64_t)(2 * ux + px) * res + (2 * uy + py)) * res + (2 * uz + pz));
      float* dst = L + (cell * C + chan) * T::PP + k;
      float4 o = make_float4(k + 0 < T::P ? acc[c] : 0.f, k + 1 < T::P ? acc[c + 1] : 0.f,
                             k + 2 < T::P ? acc[c + 2] : 0.f, k + 3 < T::P ? acc[c + 3] : 0.f);
      if (accumulate) {
        const float4 a = *reinterpret_cast<const float4*>(dst);
        o.x += a.x; o.y += a.y; o.z += a.z; o.w += a.w;
      }
      *reinterpret_cast<float4*>(dst) = o;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == T::DRAIN_WARP0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(T::TMEM_COLS));
}

}  // namespace

int tc_geometry(int rho, int* cls, int* nc, int* ks, int* bslot, int* sb, int* tiles) {
  FC2T2_DISPATCH_RHO(rho, {
    auto fill = [&](auto tag) {
      using T = typename decltype(tag)::type;
      *cls = T::CLS;
      *nc = T::NC;
      *ks = T::KS;
      *bslot = T::BSLOT;
      *sb = (T::SB ? 1 : 0) | (T::MERGE_LAST ? 2 : 0);
      *tiles = T::TILES;
    };
    fill(Tag<TC<RHO>>{});
    return 0;
  });
  return -1;
}

double tc_issued_flops(int rho, int level, int C) {
  const int nu = (1 << (level + 1)) / 2;
  FC2T2_DISPATCH_RHO(rho, {
    auto count = [&](auto tag) -> double {
      using T = typename decltype(tag)::type;
      int tiles = T::TILES;
      const double ctas2 = (double)(nu / T::TILES) * (nu / T::TY) * (nu / T::TZ) * (8 / T::CLS) * C;
      if (T::TILES == 2 && ctas2 < 148) tiles = 1;   // m2l_tc's small-grid variant
      const double tile_slots = (double)nu * (nu / T::TY) * (nu / T::TZ) * (8 / T::CLS) * C * 8 * 27;
      (void)tiles;
      const int cross_steps = T::MERGE_LAST ? T::KS - 1 : T::KS;
      const double k = T::KI, m = 128;
      return tile_slots * (T::KS * 2.0 * m * (2 * T::W) * k + cross_steps * 2.0 * m * T::W * k);
    };
    return count(Tag<TC<RHO>>{});
  });
  return 0.0;
}

int tc_moment_scales(int rho, int level, double* s) {
  const double half = 1.0 / (double)(1 << (level + 1));   // half the cell width 2/res
  FC2T2_DISPATCH_RHO(rho, {
    constexpr MI<RHO> mi{};
    for (int j = 0; j < MI<RHO>::P; ++j) {
      const int e[3] = {mi.e0[j], mi.e1[j], mi.e2[j]};
      double v = 1.0;
      for (int a = 0; a < 3; ++a)
        for (int t = 1; t <= e[a]; ++t) v *= half / t;
      s[j] = v;
    }
    return 0;
  });
  return -1;
}

namespace {
template <int RHO>
size_t plane_bytes(int level, int C) {
  const size_t res = (size_t)1 << (level + 1);
  return res * res * res * (size_t)C * TC<RHO>::KPAD * TC<RHO>::ESZ;
}
size_t gbits_bytes(int C) { return ((size_t)C * 4 + 255) / 256 * 256; }
}  // namespace

size_t tc_workspace_bytes(int rho, int level, int C) {
  FC2T2_DISPATCH_RHO(rho, return gbits_bytes(C) + 2 * plane_bytes<RHO>(level, C));
  return 0;
}

cudaError_t tc_prepare(int rho, int C, const TCPlan& plan, const float* M, void* ws,
                       cudaStream_t s) {
  const int64_t res = (int64_t)1 << (plan.level + 1);
  const int64_t cells = res * res * res;
  uint8_t* w = (uint8_t*)ws;
  uint32_t* gbits = (uint32_t*)w;
  FC2T2_DISPATCH_RHO(rho, {
    {
      using T = TC<RHO>;
      uint8_t* hi = w + gbits_bytes(C);
      uint8_t* lo = hi + plane_bytes<RHO>(plan.level, C);
      cudaError_t e = cudaMemsetAsync(gbits, 0, (size_t)C * 4, s);
      if (e != cudaSuccess) return e;
      const int64_t n4 = cells * (T::PP / 4);
      dim3 ag((unsigned)grid_blocks(n4, 256, 148 * 4), (unsigned)C);
      FC2T2_LAUNCH("m2l_absmax", s, absmax_kernel<RHO><<<ag, 256, 0, s>>>(M, plan.s_inv, cells, C,
                                                                            gbits));
      const int64_t n = cells * C * (T::KPAD / 4);
      FC2T2_LAUNCH("m2l_split", s, split_f16_kernel<RHO><<<grid_blocks(n, 256, 148 * 16), 256, 0, s>>>(
                                       M, plan.s_inv, gbits, (uint2*)hi, (uint2*)lo, cells, C));
    }
  });
  return cudaGetLastError();
}

cudaError_t m2l_tc(int rho, int C, const TCPlan& plan, const void* ws, float* L, int accumulate,
                   cudaStream_t s, int x_begin, int x_end) {
  const int res = 1 << (plan.level + 1);
  const int nu = res / 2;
  if (x_end < 0) x_end = res;
  // target cells with x in [x_begin, x_end): class-lattice planes [x_begin/2, x_end/2)
  if (nu % 16 != 0 || x_begin < 0 || x_end > res || x_begin % 4 || x_end % 4)
    return cudaErrorInvalidValue;
  if (x_end <= x_begin) return cudaSuccess;
  const int ux_begin = x_begin / 2, ux_count = (x_end - x_begin) / 2;
  const uint8_t* w = (const uint8_t*)ws;
  const uint32_t* gbits = (const uint32_t*)w;
  auto launch = [&](auto tag) -> cudaError_t {
    using T = typename decltype(tag)::type;
    auto kern = m2l_tc_kernel<T::RHO_, T::TL_>;
    static unsigned long long attr = 0;   // devices configured (per instantiation)
    if (attr_needed(attr)) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)T::SMEM);
      if (e != cudaSuccess) return e;
    }
    const uint8_t* hi = w + gbits_bytes(C);
    const uint8_t* lo = hi + plane_bytes<T::RHO_>(plan.level, C);
    dim3 grid((unsigned)((ux_count / T::TILES) * (nu / T::TY) * (nu / T::TZ)),
              (unsigned)(8 / T::CLS), (unsigned)C);
    FC2T2_LAUNCH(plan.level_name, s,
                 kern<<<grid, T::THREADS, T::SMEM, s>>>(hi, lo, plan.btab, plan.rk, gbits, L, res,
                                                        nu, C, accumulate, ux_begin));
    return cudaGetLastError();
  };
  // grids that cannot fill the machine with two-tile CTAs (small levels, thin
  // slabs) use one tile per CTA: twice the CTAs, same tables
  auto ctas = [&](auto tag) -> int64_t {
    using T = typename decltype(tag)::type;
    return (int64_t)(ux_count / T::TILES) * (nu / T::TY) * (nu / T::TZ) * (8 / T::CLS) * C;
  };
  FC2T2_DISPATCH_RHO(rho, {
    if (TC<RHO>::TILES == 2 && ctas(Tag<TC<RHO>>{}) < 148) return launch(Tag<TC<RHO, 1>>{});
    return launch(Tag<TC<RHO>>{});
  });
  return cudaGetLastError();
}

}  // namespace fc2t2
