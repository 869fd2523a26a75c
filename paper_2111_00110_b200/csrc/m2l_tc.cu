// M2L on the 5th-generation tensor cores: tcgen05.mma kind::tf32, 3xTF32.
//
// Reference: Engine.m2l (expansion.py:227-264).  For one target parity class
// pi the level's interaction list is a GEMM
//     L[t, k] = sum_{delta, n} M[t + delta, n] * A_delta[k, n]
// (rows = targets, K = (delta, n), N = k).  Split by the parity of the
// *source*, sigma = (pi + delta) mod 2, every delta of a group is a shift
// s = (pi + delta - sigma) / 2 in {-1, 0, 1}^3 of the source-class lattice, so
// the A operands of all 27 deltas of a group are shifted views of ONE staged
// window of the sigma-lattice around the target tile ("M2L on
// tcgen05").  The window is stored K-chunk-major ([kchunk][row][16 B]) so any
// row shift is a valid no-swizzle K-major UMMA descriptor; the tile is a
// 1 x 16 x 8 line block so the 8-row core-matrix groups have a uniform stride.
//
// Precision: fp32 operands are split x = hi + lo with hi = rn_tf32(x),
// lo = rn_tf32(x - hi); D += Ahi*Bhi + Ahi*Blo + Alo*Bhi accumulates in fp32 in
// TMEM (3xTF32, rel-L2 ~1e-7; plain TF32 fails the 1e-5 gate).
//
// CTA: 8 warps, TILES target tiles (M = 128 rows each).  warp 0 lane 0 issues
// the MMAs and streams the per-offset B tables (cp.async.bulk into an NS-stage
// ring, mbarrier complete_tx); warps 1-3 gather the window slices (cp.async,
// zero-fill for out-of-domain sources); warps 4-7 drain finished TMEM
// accumulator sets into fp32 registers and write the L rows.  Loop order: source class sigma -> K step (8 tf32) -> offset, so
// each B slice is loaded once per CTA and reused by TILES tiles.
#include "common.cuh"
#include "kernels.cuh"

namespace fc2t2 {

namespace {

// SMALL = one tile per CTA and a 2-stage x 6-offset B ring: ~105 KB of shared
// memory, two CTAs per SM -- for levels whose tile count cannot fill 148 SMs.
template <int RHO, bool SMALL = false>
struct TCCfg {
  static constexpr int RHO_ = RHO;
  static constexpr bool SMALL_ = SMALL;
  static constexpr int P = index_count(RHO);
  static constexpr int PP = pad4(P);
  static constexpr int KPAD = (P + 7) / 8 * 8;      // K per offset (tf32 MMA K = 8)
  static constexpr int NPAD = (P + 15) / 16 * 16;   // MMA N (M = 128 needs N % 16 == 0)
  static constexpr int KSTEPS = KPAD / 8;
  static constexpr int TILES = (NPAD <= 64 && !SMALL) ? 2 : 1;  // accumulators fit 512 TMEM cols
  static constexpr int PLOAD = (P + 15) / 16 * 16;   // accumulator columns drained
  static constexpr int TY = 16, TZ = 8;             // tile = 1 x TY x TZ targets
  static constexpr int WX = 3, WY = TY + 2, WZ = TZ + 2;
  static constexpr int WROWS = WX * WY * WZ;        // 540
  static constexpr int WSLICE = TILES * 2 * 2 * WROWS * 16;   // [tile][part][kc][row][16B]
  static constexpr int BSTAGE = 2 * 2 * NPAD * 16;  // [kc][row: hi 0..NPAD-1, lo NPAD..][16B]
  static constexpr int DPS = SMALL ? 6 : 9;         // offsets per B stage
  static constexpr int NS = (RHO <= 4 && !SMALL) ? 3 : 2;  // B stages (DPS tables each)
  static constexpr int ACC = NPAD <= 64 ? 128 : 256;          // [hi*hi | cross] per tile
  static constexpr int TMEM_COLS = 2 * TILES * ACC;           // sets x tiles
  static constexpr int THREADS = 384;                         // 12 warps
  static constexpr int GATHER_WARP0 = 2, GATHER_WARPS = 6;    // warps 2..7
  static constexpr int GATHER_THREADS = 32 * GATHER_WARPS;
  static constexpr int DRAIN_WARP0 = 8;                       // warps 8..11 (TMEM quarters)
  static constexpr int MAXE = 256;                            // entries of one target class
  static constexpr size_t SMEM =
      2 * (size_t)WSLICE + (size_t)NS * DPS * BSTAGE + 256 + MAXE * 8 + 64;
  static constexpr uint32_t idesc(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
  }
  static constexpr uint32_t IDESC1 = idesc(NPAD);      // A x B_hi
  static constexpr uint32_t IDESC2 = idesc(2 * NPAD);  // A_hi x [B_hi; B_lo]
};

template <class T>
struct CfgTag {
  using type = T;
};

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

__device__ __forceinline__ void umma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
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

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float rn_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ------------------------------------------------------------ pre-split ---
// (res^3, C, PP) fp32 grid -> per-channel hi / lo grids (C, res^3, KPAD),
// zero-padded from P to KPAD.
template <int RHO>
__global__ void __launch_bounds__(256)
split_tf32_kernel(const float* __restrict__ M, float4* __restrict__ hi, float4* __restrict__ lo,
                  int64_t cells, int C) {
  using Cfg = TCCfg<RHO>;
  constexpr int Q = Cfg::KPAD / 4;
  const int64_t n = cells * C * Q;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int q = (int)(g % Q);
    const int64_t cc = g / Q;  // (channel, cell) in output order
    const int c = (int)(cc / cells);
    const int64_t cell = cc - (int64_t)c * cells;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * q < Cfg::PP) v = *reinterpret_cast<const float4*>(M + (cell * C + c) * Cfg::PP + 4 * q);
    float4 h, l;
    h.x = rn_tf32(v.x); l.x = rn_tf32(v.x - h.x);
    h.y = rn_tf32(v.y); l.y = rn_tf32(v.y - h.y);
    h.z = rn_tf32(v.z); l.z = rn_tf32(v.z - h.z);
    h.w = rn_tf32(v.w); l.w = rn_tf32(v.w - h.w);
    hi[g] = h;
    lo[g] = l;
  }
}

// ------------------------------------------------------------ M2L (tc) ---
// Precision note: tensor-core accumulation into TMEM does not round to
// nearest, so a single accumulator over all ~3000 MMAs of a tile drifts
// (measured 2-4e-5 rel-L2).  Each source-class group therefore accumulates
// into its own TMEM set (double buffered), with the hi*hi products and the two
// small cross products in separate accumulators; drain warps fold every
// finished set into float32 registers with round-to-nearest adds.
//
// Warp roles (12 warps): 0 MMA issuer (warp-uniform loop, elect-one issue),
// 1 B-table producer (cp.async.bulk ring), 2-7 window gatherers, 8-11 TMEM
// drain + epilogue (warp % 4 = TMEM lane quarter).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "elect.sync _|P1, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}\n"
      : "=r"(pred));
  return pred != 0;
}

template <int RHO, bool SMALL>
__global__ void __launch_bounds__(384, SMALL ? 2 : 1)
m2l_tc_kernel(const float* __restrict__ Mhi, const float* __restrict__ Mlo,
              const uint8_t* __restrict__ Btab, const int2* __restrict__ entries,
              const int* __restrict__ grp_start, float* __restrict__ L, int res, int nu, int C,
              int accumulate) {
  using Cfg = TCCfg<RHO, SMALL>;
  constexpr int WROWS = Cfg::WROWS, NS = Cfg::NS, KS = Cfg::KSTEPS, TILES = Cfg::TILES;
  constexpr int P = Cfg::P, PP = Cfg::PP, PL = Cfg::PLOAD;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* win = smem;                                   // [2][WSLICE]
  uint8_t* bring = smem + 2 * Cfg::WSLICE;               // [NS][DPS][BSTAGE]
  uint64_t* bars = reinterpret_cast<uint64_t*>(bring + NS * Cfg::DPS * Cfg::BSTAGE);
  // bars: bfull[NS], bempty[NS], winready[2], winfree[2], accfull[2], accfree[2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 8);
  int* sgrp = reinterpret_cast<int*>(tmem_slot + 4);     // [9] group starts (class-local)
  int2* sent = reinterpret_cast<int2*>(sgrp + 12);       // [MAXE] class entries

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cls = blockIdx.y;  // target class
  const int px = (cls >> 2) & 1, py = (cls >> 1) & 1, pz = cls & 1;
  const int chan = blockIdx.z;
  const int nyb = (nu + Cfg::TY - 1) / Cfg::TY, nzb = (nu + Cfg::TZ - 1) / Cfg::TZ;
  const int ntiles = nu * nyb * nzb;
  const int tile0 = blockIdx.x * TILES;
  auto tile_xyz = [&](int t, int& ux, int& uy, int& uz) {
    const int id = min(tile0 + t, ntiles - 1);
    ux = id / (nyb * nzb);
    uy = ((id / nzb) % nyb) * Cfg::TY;
    uz = (id % nzb) * Cfg::TZ;
  };
  const uint32_t bar0 = smem_u32(bars);
  auto bfull = [&](int s) { return bar0 + 8u * s; };
  auto bempty = [&](int s) { return bar0 + 8u * (NS + s); };
  auto winready = [&](int b) { return bar0 + 8u * (2 * NS + b); };
  auto winfree = [&](int b) { return bar0 + 8u * (2 * NS + 2 + b); };
  auto accfull = [&](int b) { return bar0 + 8u * (2 * NS + 4 + b); };
  auto accfree = [&](int b) { return bar0 + 8u * (2 * NS + 6 + b); };

  // stage this class's interaction list (class-local group starts) in smem
  const int gb0 = grp_start[cls * 8];
  const int nent = grp_start[cls * 8 + 8] - gb0;
  if (tid < 9) sgrp[tid] = grp_start[cls * 8 + tid] - gb0;
  for (int k = tid; k < nent && k < Cfg::MAXE; k += blockDim.x) sent[k] = entries[gb0 + k];

  if (warp == Cfg::DRAIN_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(bfull(s), 1);
      mbar_init(bempty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(winready(b), Cfg::GATHER_THREADS);
      mbar_init(winfree(b), 1);
      mbar_init(accfull(b), 1);
      mbar_init(accfree(b), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const size_t cells = (size_t)res * res * res;
  const float* hi_c = Mhi + (size_t)chan * cells * Cfg::KPAD;
  const float* lo_c = Mlo + (size_t)chan * cells * Cfg::KPAD;
  // accumulator columns of (set, tile): [0, NPAD) hi*hi, [NPAD, 2 NPAD) cross terms
  auto acc_col = [](int set, int t, int kind) {
    return (set * TILES + t) * Cfg::ACC + kind * Cfg::NPAD;
  };

  if (warp == 0) {
    // ---------------- MMA issuer (whole warp, uniform control flow) ----------------
    // B stages walk (sigma, ks, chunk of <= DPS offsets); one wait + one
    // commit per stage.  Descriptors are built once and advanced by adding
    // byte offsets / 16 to their start-address field.
    const uint64_t bdesc0 = sdesc(smem_u32(bring), 2 * Cfg::NPAD * 16, 128);
    const uint64_t wdesc0 = sdesc(smem_u32(win), WROWS * 16, Cfg::WZ * 16);
    int n = 0, q = 0, g = 0;
    for (int sg = 0; sg < 8; ++sg) {
      const int gb = sgrp[sg], ne = sgrp[sg + 1] - gb;
      if (ne == 0) continue;
      const int set = g & 1;
      if (g >= 2) mbar_wait(accfree(set), ((g - 2) >> 1) & 1);
      for (int ks = 0; ks < KS; ++ks, ++q) {
        const int buf = q & 1;
        mbar_wait(winready(buf), (q >> 1) & 1);
        tc_fence_after();
        const uint64_t wd = wdesc0 + (uint64_t)((buf * Cfg::WSLICE) >> 4);
        for (int j0 = 0; j0 < ne; j0 += Cfg::DPS, ++n) {
          const int s = n % NS, cnt = min(Cfg::DPS, ne - j0);
          mbar_wait(bfull(s), (n / NS) & 1);
          tc_fence_after();
          if (elect_one()) {
            for (int jj = 0; jj < cnt; ++jj) {
              const int ex = sent[gb + j0 + jj].x;
              const uint64_t bd = bdesc0 + (uint64_t)(((s * Cfg::DPS + jj) * Cfg::BSTAGE) >> 4);
              const uint32_t acc_in = (ks == 0 && j0 + jj == 0) ? 0u : 1u;
#pragma unroll
              for (int t = 0; t < TILES; ++t) {
                const uint64_t dah = wd + (uint64_t)(((t * 4 + 0) * WROWS + ex));
                const uint64_t dal = wd + (uint64_t)(((t * 4 + 2) * WROWS + ex));
                // D[:, 0:N) += Ahi Bhi and D[:, N:2N) += Ahi Blo in one N = 2 NPAD MMA
                umma_tf32(tmem + acc_col(set, t, 0), dah, bd, Cfg::IDESC2, acc_in);
                umma_tf32(tmem + acc_col(set, t, 1), dal, bd, Cfg::IDESC1, 1u);
              }
            }
            umma_commit(bempty(s));
          }
          __syncwarp();
        }
        if (elect_one()) umma_commit(winfree(buf));
        __syncwarp();
      }
      if (elect_one()) umma_commit(accfull(set));
      __syncwarp();
      ++g;
    }
  } else if (warp == 1) {
    // ---------------- B-table producer ----------------
    if (lane == 0) {
      int n = 0;
      for (int sg = 0; sg < 8; ++sg) {
        const int gb = sgrp[sg], ne = sgrp[sg + 1] - gb;
        for (int ks = 0; ks < KS; ++ks)
          for (int j0 = 0; j0 < ne; j0 += Cfg::DPS, ++n) {
            const int s = n % NS, cnt = min(Cfg::DPS, ne - j0);
            if (n >= NS) mbar_wait(bempty(s), ((n / NS) - 1) & 1);
            mbar_expect_tx(bfull(s), cnt * Cfg::BSTAGE);
            for (int jj = 0; jj < cnt; ++jj) {
              const uint8_t* src =
                  Btab + ((size_t)sent[gb + j0 + jj].y * KS + ks) * Cfg::BSTAGE;
              bulk_g2s(smem_u32(bring + (s * Cfg::DPS + jj) * Cfg::BSTAGE), src, Cfg::BSTAGE,
                       bfull(s));
            }
          }
      }
    }
  } else if (warp < Cfg::DRAIN_WARP0) {
    // ---------------- window gatherers ----------------
    const int gt = tid - 32 * Cfg::GATHER_WARP0;
    int q = 0;
    for (int sg = 0; sg < 8; ++sg) {
      const int ne = sgrp[sg + 1] - sgrp[sg];
      if (ne == 0) continue;
      const int sx = (sg >> 2) & 1, sy = (sg >> 1) & 1, sz = sg & 1;
      for (int ks = 0; ks < KS; ++ks, ++q) {
        const int buf = q & 1;
        if (q >= 2) mbar_wait(winfree(buf), ((q - 2) >> 1) & 1);
        uint8_t* wb = win + buf * Cfg::WSLICE;
        for (int r = gt; r < TILES * WROWS; r += Cfg::GATHER_THREADS) {
          const int t = r / WROWS, wr = r - t * WROWS;
          int ux, uy, uz;
          tile_xyz(t, ux, uy, uz);
          const int wx = wr / (Cfg::WY * Cfg::WZ), wy = (wr / Cfg::WZ) % Cfg::WY, wz = wr % Cfg::WZ;
          const int cx = 2 * (ux - 1 + wx) + sx;
          const int cy = 2 * (uy - 1 + wy) + sy;
          const int cz = 2 * (uz - 1 + wz) + sz;
          const bool ok = tile0 + t < ntiles && (unsigned)cx < (unsigned)res &&
                          (unsigned)cy < (unsigned)res && (unsigned)cz < (unsigned)res;
          const size_t off = ok ? (((size_t)cx * res + cy) * res + cz) * Cfg::KPAD + ks * 8 : 0;
#pragma unroll
          for (int part = 0; part < 2; ++part) {
            const float* src = (part ? lo_c : hi_c) + off;
#pragma unroll
            for (int kc = 0; kc < 2; ++kc) {
              const uint32_t dst =
                  smem_u32(wb + ((((t * 2 + part) * 2 + kc) * WROWS) + wr) * 16);
              cp_async16_zfill(dst, src + kc * 4, ok ? 16 : 0);
            }
          }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(winready(buf));
      }
    }
  } else {
    // ---------------- drain + epilogue (TMEM quarters 0..3) ----------------
    const int dq = warp & 3;
    float accr[TILES][PL];
#pragma unroll
    for (int t = 0; t < TILES; ++t)
#pragma unroll
      for (int j = 0; j < PL; ++j) accr[t][j] = 0.f;
    int g = 0;
    for (int sg = 0; sg < 8; ++sg) {
      if (sgrp[sg + 1] == sgrp[sg]) continue;
      const int set = g & 1;
      mbar_wait(accfull(set), (g >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
#pragma unroll
        for (int c0 = 0; c0 < PL; c0 += 16) {
          float a[16], b[16];
          const uint32_t lanes = (uint32_t)(dq * 32) << 16;
          tmem_ld16(tmem + lanes + acc_col(set, t, 0) + c0, a);
          tmem_ld16(tmem + lanes + acc_col(set, t, 1) + c0, b);
#pragma unroll
          for (int j = 0; j < 16; ++j) accr[t][c0 + j] += a[j] + b[j];
        }
      }
      tc_fence_before();
      mbar_arrive(accfree(set));
      ++g;
    }
    const int row = dq * 32 + lane;
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      int ux, uy0, uz0;
      tile_xyz(t, ux, uy0, uz0);
      const int uy = uy0 + row / Cfg::TZ, uz = uz0 + row % Cfg::TZ;
      if (tile0 + t >= ntiles || uy >= nu || uz >= nu) continue;
      const int64_t cell = (((int64_t)(2 * ux + px) * res + (2 * uy + py)) * res + (2 * uz + pz));
      float* dst = L + (cell * C + chan) * PP;
#pragma unroll
      for (int k = 0; k < PP; k += 4) {
        float4 o = make_float4(k + 0 < P ? accr[t][k] : 0.f, k + 1 < P ? accr[t][k + 1] : 0.f,
                               k + 2 < P ? accr[t][k + 2] : 0.f, k + 3 < P ? accr[t][k + 3] : 0.f);
        if (accumulate) {
          const float4 a = *reinterpret_cast<const float4*>(dst + k);
          o.x += a.x; o.y += a.y; o.z += a.z; o.w += a.w;
        }
        *reinterpret_cast<float4*>(dst + k) = o;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == Cfg::DRAIN_WARP0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "n"(Cfg::TMEM_COLS));
}

}  // namespace

int tc_kpad(int rho) { return (index_count(rho) + 7) / 8 * 8; }
int tc_npad(int rho) { return (index_count(rho) + 15) / 16 * 16; }
int tc_bstage(int rho) { return 2 * 2 * tc_npad(rho) * 16; }
int tc_window_start(int sx, int sy, int sz) {
  // window dims are rho independent: 3 x 18 x 10
  return ((sx + 1) * 18 + (sy + 1)) * 10 + (sz + 1);
}

cudaError_t split_tf32(int rho, int level, int C, const float* M, float* hi, float* lo,
                       cudaStream_t s) {
  const int64_t res = (int64_t)1 << (level + 1);
  const int64_t cells = res * res * res;
  const int64_t n = cells * C * (tc_kpad(rho) / 4);
  FC2T2_DISPATCH_RHO(rho, FC2T2_LAUNCH("m2l_split", s,
      split_tf32_kernel<RHO><<<grid_blocks(n, 256, 148 * 16), 256, 0, s>>>(
          M, (float4*)hi, (float4*)lo, cells, C)));
  return cudaGetLastError();
}

cudaError_t m2l_tc(int rho, int C, const TCPlan& plan, const float* Mhi, const float* Mlo,
                   float* L, int accumulate, cudaStream_t s) {
  const int res = 1 << (plan.level + 1);
  const int nu = res / 2;
  auto launch = [&](auto cfg_tag) -> cudaError_t {
    using Cfg = typename decltype(cfg_tag)::type;
    auto kern = m2l_tc_kernel<Cfg::RHO_, Cfg::SMALL_>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Cfg::SMEM);
    if (e != cudaSuccess) return e;
    const int nyb = (nu + Cfg::TY - 1) / Cfg::TY, nzb = (nu + Cfg::TZ - 1) / Cfg::TZ;
    const int ntiles = nu * nyb * nzb;
    dim3 grid((unsigned)((ntiles + Cfg::TILES - 1) / Cfg::TILES), 8u, (unsigned)C);
    FC2T2_LAUNCH(plan.level_name, s,
                 kern<<<grid, Cfg::THREADS, Cfg::SMEM, s>>>(Mhi, Mlo, plan.btab, plan.entries,
                                                   plan.grp_start, L, res, nu, C, accumulate));
    return cudaGetLastError();
  };
  // big CTAs (2 tiles, 1 per SM) only when they fill the machine
  const int ntiles_big = nu * ((nu + 15) / 16) * ((nu + 7) / 8);
  const bool small = false && (int64_t)((ntiles_big + 1) / 2) * 8 * C < 2 * 148;  // measured slower (issuer-bound)
  FC2T2_DISPATCH_RHO(rho, {
    if (small) return launch(CfgTag<TCCfg<RHO, true>>{});
    return launch(CfgTag<TCCfg<RHO, false>>{});
  });
  return cudaGetLastError();
}

}  // namespace fc2t2
