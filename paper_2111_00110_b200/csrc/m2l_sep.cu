// M2L through the per-axis factors of the reference's tables: the finest
// level (far + near) as three 1-D convolutions between two per-axis
// triangular transforms, coarse levels' far tables as three such pieces.
//
// Reference: Engine.m2l (expansion.py:227-264) over the finest far table
// (parity stencil, :246-249) plus the near table, with the tables of
// kernel.py:180-204 (LSQ) or :169-177 (Taylor).  The Gaussian factors per
// axis, so every finest table does too (paper_2111_00110_b200/kernel.py,
// separable_factors): coeffs(o) = post_S . (K(o_x) (x) K(o_y) (x) K(o_z))_S .
// pre_S, and far + near give every target the full 6 x 6 x 6 box of source
// offsets ({-2..3} per axis for an even target index, {-3..2} for an odd
// one).  So, per channel:
//
//   pre    M'(a,b,c)  = sum pre[a'][a] pre[b'][b] pre[c'][c] M      (lower tri)
//   z pass Z(a,b,c')  = sum_{dz, c} K(dz)[c'][c]  M'(a,b,c)(z+dz)
//   y pass Y(a,b',c') = sum_{dy, b} K(dy)[b'][b]  Z(a,b,c')(y+dy)
//   x pass X(a',b',c')= sum_{dx, a} K(dx)[a'][a]  Y(a,b',c')(x+dx)
//   post   L          = post (x) post (x) post  X                  (upper tri)
//
// with every index set truncated to what the next step can use (total degree
// <= rho at the end; the triangular transforms never need more).  At rho = 4
// that is ~4e3 multiply-adds per cell instead of the dense 216 x 35 x 35.
// Sources outside the grid contribute nothing (the reference's clipped
// slices).  The factor matrices are kernel parameters (__grid_constant__),
// and every loop over them unrolls, so each FFMA reads its coefficient from
// the constant bank.
//
// Layouts (one channel block after another; x fastest unless noted):
//   M' : [e in AB order][y][z][x]       AB(a,b,c) = ab(a,b) + c
//   Z  : [e = pair(a,b)*R1 + c'][y][z][x]
//   Y  : [e = a*NAB + pair(b',c')][y][z][x]
//   X  : [e = graded-lex (a',b',c')][x][y][z]   (z fastest)
// Each pass CTA stages a 14/16-deep window (8 outputs + the 3/3 halo) of 32
// lines of the entries one partition needs (lanes along the contiguous
// axis); warp g computes one output group for all 8 positions of its lane's
// line with the accumulators in registers (see "passes" below).
//
// Coarse levels (expansion.py:272-275) apply the parity stencil minus the
// 3 x 3 x 3 hole.  Their tables factor the same way with the level's own
// K(d), and box^3 - hole is the disjoint union of three products of per-axis
// tap sets (A = the parity box, F = {|d| >= 2}, N = {|d| <= 1}):
//   F x A x A  +  N x F x A  +  N x N x F              (x, y, z)
// so a far table is the same passes with tap subsets (TAPS), the two-term
// pieces as one pass over two staged windows (TAPS1): m2l_sep(far_only).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.cuh"
#include "shift.cuh"

#include <cstring>
#include <mutex>

namespace fc2t2 {

namespace {

template <int RHO>
struct SepIdx {
  static constexpr int R1 = RHO + 1;
  static constexpr int NAB = R1 * (R1 + 1) / 2;  // pairs (a, b) with a + b <= RHO
  static constexpr int T = NAB * R1;             // entries of Z and Y
  static constexpr int P = MI<RHO>::P;
  static constexpr int pair(int a, int b) { return a * R1 - a * (a - 1) / 2 + b; }
  static constexpr int ab(int a, int b) {
    int o = 0;
    for (int i = 0; i < a; ++i) o += (R1 - i) * (R1 - i + 1) / 2;
    for (int j = 0; j < b; ++j) o += R1 - a - j;
    return o;
  }
  static constexpr int zoff(int a, int b, int c) { return pair(a, b) * R1 + c; }
  static constexpr int yoff(int a, int b, int c) { return a * NAB + pair(b, c); }
};

constexpr int kLines = 32;
// POS = 8 output positions per tile; the z/y window holds POS + 6 positions,
// the x window POS + 8 (16-byte aligned runs)
constexpr int win_of(int POS) { return POS + 6; }


// ------------------------------------------------------------ pre / post ---

// in place: v(a',..) = sum_{a <= a'} m[a'][a] v(a,..) along `axis`, on S
template <int RHO, int AXIS>
__device__ __forceinline__ void lower_axis(float (&v)[MI<RHO>::P], const float (&m)[RHO + 1][RHO + 1]) {
  constexpr MI<RHO> mi{};
#pragma unroll
  for (int j = MI<RHO>::P - 1; j >= 0; --j) {
    const int e[3] = {mi.e0[j], mi.e1[j], mi.e2[j]};
    float s = 0.f;
#pragma unroll
    for (int a = 0; a <= e[AXIS]; ++a) {
      const int i = MI<RHO>::index(AXIS == 0 ? a : e[0], AXIS == 1 ? a : e[1], AXIS == 2 ? a : e[2]);
      s = fmaf(m[e[AXIS]][a], v[i], s);
    }
    v[j] = s;  // entries with a larger AXIS degree were already rewritten
  }
}

// in place: v(a',..) = sum_{a >= a'} m[a'][a] v(a,..) along `axis`, on S
template <int RHO, int AXIS>
__device__ __forceinline__ void upper_axis(float (&v)[MI<RHO>::P], const float (&m)[RHO + 1][RHO + 1]) {
  constexpr MI<RHO> mi{};
#pragma unroll
  for (int j = 0; j < MI<RHO>::P; ++j) {
    const int e[3] = {mi.e0[j], mi.e1[j], mi.e2[j]};
    const int top = RHO - (e[0] + e[1] + e[2] - e[AXIS]);
    float s = 0.f;
#pragma unroll
    for (int a = e[AXIS]; a <= top; ++a) {
      const int i = MI<RHO>::index(AXIS == 0 ? a : e[0], AXIS == 1 ? a : e[1], AXIS == 2 ? a : e[2]);
      s = fmaf(m[e[AXIS]][a], v[i], s);
    }
    v[j] = s;  // reads only entries of equal or higher AXIS degree: not yet rewritten
  }
}

}  // namespace

template <int RHO>
struct SepParams {
  float pre[RHO + 1][RHO + 1];
  float post[RHO + 1][RHO + 1];
  float conv[7][RHO + 1][RHO + 1];  // K(d) for d = -3..3, [out][in]
  float kt[RHO + 1][7][8];          // the passes' shared-memory layout: kt[i][d][j] = conv[d][j][i]
};

namespace {

// M (res^3, C, PP) rows -> M' (AB order, x fastest).  Thread per cell,
// lanes along x.
template <int RHO>
__global__ void __launch_bounds__(256)
sep_pre_kernel(const float* __restrict__ M, float* __restrict__ Mp, int res, int lres, int C,
               int x_lo, int nx, const __grid_constant__ SepParams<RHO> prm) {
  using I = SepIdx<RHO>;
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  constexpr MI<RHO> mi{};
  // grid (cells / 256, C); 32-bit index arithmetic (cells <= 2^24), res = 2^lres
  const unsigned cells = (unsigned)nx << (2 * lres);
  const unsigned r = blockIdx.x * 256u + threadIdx.x;
  if (r >= cells) return;
  const int ch = (int)blockIdx.y;
  const unsigned yz = r / (unsigned)nx;
  const int x = x_lo + (int)(r - yz * (unsigned)nx);
  const int z = (int)(yz & (unsigned)(res - 1)), y = (int)(yz >> lres);
  const float* row = M + ((((int64_t)x * res + y) * res + z) * C + ch) * PP;
  float v[P];
#pragma unroll
  for (int k = 0; k < PP; k += 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(row + k));
    if (k < P) v[k] = q.x;
    if (k + 1 < P) v[k + 1] = q.y;
    if (k + 2 < P) v[k + 2] = q.z;
    if (k + 3 < P) v[k + 3] = q.w;
  }
  lower_axis<RHO, 0>(v, prm.pre);
  lower_axis<RHO, 1>(v, prm.pre);
  lower_axis<RHO, 2>(v, prm.pre);
  const int64_t plane = (int64_t)res * res * res;
  float* out = Mp + (int64_t)ch * P * plane + ((int64_t)y * res + z) * res + x;
#pragma unroll
  for (int j = 0; j < P; ++j) out[(int64_t)I::ab(mi.e0[j], mi.e1[j]) * plane + mi.e2[j] * plane] = v[j];
}

// X (graded-lex, z fastest) -> L rows.  Thread per cell, lanes along z.
// With `coarse` (the level above's L grid) the L2L of the cascade
// (ref expansion.py:215-225, 276-277) is fused: L = L2L(coarse) + M2L, the
// same float32 sum the separate accumulate-L2L launch forms.
template <int RHO>
__global__ void __launch_bounds__(256)
sep_post_kernel(const float* __restrict__ X, float* __restrict__ L, int res, int lres, int C,
                int x_lo, int nx, const float* __restrict__ coarse, float half_fine,
                const __grid_constant__ SepParams<RHO> prm) {
  constexpr int P = MI<RHO>::P, PP = MI<RHO>::PP;
  // grid (cells / 256, C); shifts and masks only (res = 2^lres)
  const unsigned cells = (unsigned)nx << (2 * lres);
  const unsigned r = blockIdx.x * 256u + threadIdx.x;
  if (r >= cells) return;
  const int ch = (int)blockIdx.y;
  const int z = (int)(r & (unsigned)(res - 1));
  const unsigned xy = r >> lres;
  const int y = (int)(xy & (unsigned)(res - 1)), x = x_lo + (int)(xy >> lres);
  const int64_t plane = (int64_t)res * res * res;
  const float* in = X + (int64_t)ch * P * plane + ((int64_t)x * res + y) * res + z;
  float v[P];
#pragma unroll
  for (int j = 0; j < P; ++j) v[j] = in[(int64_t)j * plane];
  upper_axis<RHO, 0>(v, prm.post);
  upper_axis<RHO, 1>(v, prm.post);
  upper_axis<RHO, 2>(v, prm.post);
  if (coarse) {
    const int cres = res >> 1;
    const float* prow =
        coarse + ((((int64_t)(x >> 1) * cres + (y >> 1)) * cres + (z >> 1)) * C + ch) * PP;
    float pv[P];
#pragma unroll
    for (int k = 0; k < PP; k += 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(prow + k));
      if (k < P) pv[k] = q.x;
      if (k + 1 < P) pv[k + 1] = q.y;
      if (k + 2 < P) pv[k + 2] = q.z;
      if (k + 3 < P) pv[k + 3] = q.w;
    }
    shift3<RHO, false>(pv, (x & 1) ? half_fine : -half_fine, (y & 1) ? half_fine : -half_fine,
                       (z & 1) ? half_fine : -half_fine);
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = pv[j] + v[j];
  }
  if constexpr (8 * 32 * (PP + 1) * 4 <= 48 * 1024) if (C == 1) {
    // one channel: the warp's 32 rows (consecutive cells) are one contiguous
    // 32 * PP float block -- transpose through shared memory and write it with
    // fully coalesced stores instead of 16-byte pieces 144 bytes apart
    __shared__ float tile[8][32 * (PP + 1)];
    float* t = tile[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < PP; ++j) t[lane * (PP + 1) + j] = j < P ? v[j] : 0.f;
    __syncwarp();
    // (cells is a multiple of 256, so warps are whole)
    float* blk = L + ((int64_t)x_lo * res * res + (int64_t)(r - lane)) * PP;
#pragma unroll
    for (int i = 0; i < PP; ++i) {
      const int idx = i * 32 + lane, rr = idx / PP;
      blk[idx] = t[idx + rr];   // rr * (PP + 1) + (idx - rr * PP)
    }
    return;
  }
  float* row = L + ((((int64_t)x * res + y) * res + z) * C + ch) * PP;
#pragma unroll
  for (int k = 0; k < PP; k += 4) {
    float4 q;
    q.x = k < P ? v[k] : 0.f;
    q.y = k + 1 < P ? v[k + 1] : 0.f;
    q.z = k + 2 < P ? v[k + 2] : 0.f;
    q.w = k + 3 < P ? v[k + 3] : 0.f;
    *reinterpret_cast<float4*>(row + k) = q;
  }
}

// ------------------------------------------------------------------ passes ---
//
// A pass CTA owns 32 lines x 8 consecutive output positions (even first
// position, so output w has parity w & 1) of one partition of the entries;
// warp g computes group g of that partition for all 8 positions of its
// lane's line, holding the 8 x n_out accumulators in registers and reading
// each staged input once (a 14/16-deep window: 8 outputs + the 3/3 halo).
//   z pass, partition a = A, group b:  in  M'(A,b,c)  c <= RHO-A-b
//                                      out Z(A,b,c')  c' <= RHO
//   y pass, partition a = A, group c': in  Z(A,b,c')  b <= RHO-A
//                                      out Y(A,b',c') b' <= RHO-c'
//   x pass, partition b' = B, group c': in Y(a,B,c')  a <= RHO
//                                      out X(a',B,c') a' <= RHO-B-c'
// Every contraction is sum_{d, i} K(d)[j][i] in_i(pos + d).

enum { PASS_Z = 0, PASS_Y = 1, PASS_X = 2 };
enum { TAPS_ALL = 0, TAPS_FAR = 1, TAPS_NEAR = 2, TAPS_NONE = 3 };

template <int RHO, int PASS, int PART>
struct Part {
  using I = SepIdx<RHO>;
  static constexpr int R1 = RHO + 1;
  static constexpr int NE = PASS == PASS_Z ? (R1 - PART) * (R1 - PART + 1) / 2
                                           : (PASS == PASS_Y ? (R1 - PART) * R1 : R1 * (R1 - PART));
  static constexpr int EBASE = PASS == PASS_Z ? I::ab(PART, 0)
                                              : (PASS == PASS_Y ? I::pair(PART, 0) * R1 : 0);
  // global entry of local window entry le (x pass: le = a * (R1 - B) + c')
  static constexpr int entry(int le) {
    return PASS == PASS_X ? (le / (R1 - PART)) * I::NAB + I::pair(PART, le % (R1 - PART))
                          : EBASE + le;
  }
};

// z/y window: [q][le NE][lane 32] (q = position - pos0 + 3), filled by
// 16-byte copies of the 32-float x-runs.  x window: [le][lane][xs] (q =
// position - pos0 + 4), filled by 16-byte copies of x-runs and read back with
// 128-bit loads; an odd number of 16-byte chunks per lane row puts the 8 lanes
// of a quarter-warp on distinct bank quads.

// One output group for 8 positions of this lane's line: NOUT outputs,
// `nin` inputs at window entries in_base + i * in_stride.  Only NOUT (and the
// pass's window layout) is compile-time, so the whole pass is a handful of
// small code paths (instruction-cache resident); the K(d)[.][i] column of an
// input comes from shared memory (Kt[i][d][j], warp-uniform broadcast).
template <int RHO, int PASS, int POS, int NL, int TAPS, int NOUT>
__device__ __forceinline__ void accum_input(float (&acc)[POS][NOUT], const float* sm,
                                            const float* Kt, int lane, int nin, int in_base,
                                            int in_stride) {
  constexpr int OFF = PASS == PASS_X ? 4 : 3;
  constexpr int NQ = PASS == PASS_X ? POS + 8 : win_of(POS);
#pragma unroll 1
  for (int i = 0; i < nin; ++i) {
    const int le = in_base + i * in_stride;
    float v[NQ];
    if constexpr (PASS == PASS_X) {
      // [le][lane][16], 16-byte chunk c of lane l in slot c ^ ((l >> 1) & 3)
      // (the TMA 64-byte swizzle): conflict-free 128-bit reads
      const float4* r4 = reinterpret_cast<const float4*>(sm + (le * NL + lane) * 16);
      const int sw = (lane >> 1) & 3;
#pragma unroll
      for (int q = 0; q < NQ / 4; ++q) {
        const float4 t = r4[q ^ sw];
        v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
      }
    } else {
      // [le][q][lane]
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = sm[(le * NQ + q) * NL + lane];
    }
    // K(d) columns one d at a time (NOUT live coefficient registers); per
    // accumulator the FMAs still run over d ascending (unchanged sums)
    const float4* kc = reinterpret_cast<const float4*>(Kt + i * 56);
#pragma unroll
    for (int d = -3; d <= 3; ++d) {
      // the tap subset of a far-table piece: F = {|d| >= 2}, N = {|d| <= 1}
      if ((TAPS == TAPS_FAR && d >= -1 && d <= 1) || (TAPS == TAPS_NEAR && (d < -1 || d > 1)))
        continue;
      float k[NOUT];
      const float4 lo = kc[2 * (d + 3)];
      const float lo_[4] = {lo.x, lo.y, lo.z, lo.w};
#pragma unroll
      for (int j = 0; j < NOUT && j < 4; ++j) k[j] = lo_[j];
      if constexpr (NOUT > 4) {
        const float4 hi = kc[2 * (d + 3) + 1];
        const float hi_[4] = {hi.x, hi.y, hi.z, hi.w};
#pragma unroll
        for (int j = 4; j < NOUT; ++j) k[j] = hi_[j - 4];
      }
#pragma unroll
      for (int w = 0; w < POS; ++w) {
        // even positions take d in -2..3, odd ones -3..2
        if (d < -2 - (w & 1) || d > 3 - (w & 1)) continue;
        const float x = v[w + OFF + d];
#pragma unroll
        for (int j = 0; j < NOUT; ++j) acc[w][j] = fmaf(k[j], x, acc[w][j]);
      }
    }
  }
}

// TAPS1 != TAPS_NONE: a second window (sm1, same layout) contributes with its
// own tap subset to the same outputs -- the two-term pieces of a far table.
template <int RHO, int PASS, int POS, int NL, int TAPS0, int TAPS1, int NOUT>
__device__ __forceinline__ void group_body(const float* sm0, const float* sm1, const float* Kt,
                                           int lane, int nin, int in_base, int in_stride,
                                           const int (&oe)[RHO + 1], float* out,
                                           int64_t pos_stride, int64_t plane, int nvalid) {
  float acc[POS][NOUT];
#pragma unroll
  for (int w = 0; w < POS; ++w)
#pragma unroll
    for (int j = 0; j < NOUT; ++j) acc[w][j] = 0.f;
  accum_input<RHO, PASS, POS, NL, TAPS0, NOUT>(acc, sm0, Kt, lane, nin, in_base, in_stride);
  if constexpr (TAPS1 != TAPS_NONE)
    accum_input<RHO, PASS, POS, NL, TAPS1, NOUT>(acc, sm1, Kt, lane, nin, in_base, in_stride);
  // one 64-bit pointer per output entry, advanced by the (uniform) position
  // stride: two integer adds + STG per store
  char* pb[NOUT];
#pragma unroll
  for (int j = 0; j < NOUT; ++j) pb[j] = reinterpret_cast<char*>(out + (int64_t)oe[j] * plane);
  const int64_t psb = pos_stride * (int64_t)sizeof(float);
#pragma unroll
  for (int w = 0; w < POS; ++w) {
    if (w < nvalid) {
#pragma unroll
      for (int j = 0; j < NOUT; ++j) *reinterpret_cast<float*>(pb[j]) = acc[w][j];
    }
#pragma unroll
    for (int j = 0; j < NOUT; ++j) pb[j] += psb;
  }
}

// Partitions are very unequal (z pass at rho = 4: 15, 10, 6, 3, 1 inputs), and
// every CTA pays the same fixed cost (window copy, barrier, index set-up), so
// the light tail shares one CTA: slot s < TAIL is partition s, slot TAIL is
// partitions TAIL .. RHO one after the other, their windows back to back in
// the shared memory sized for partition 0.  TAIL = the first partition from
// which the rest together has no more work and no more window entries than
// partition 0.
template <int RHO, int PASS>
struct Slots {
  static constexpr int R1 = RHO + 1;
  static constexpr int ne(int p) {
    return PASS == PASS_Z ? (R1 - p) * (R1 - p + 1) / 2
                          : (PASS == PASS_Y ? (R1 - p) * R1 : R1 * (R1 - p));
  }
  static constexpr int work(int p) {
    return PASS == PASS_Y ? (R1 - p) : (R1 - p) * (R1 - p + 1) / 2;
  }
  static constexpr int tail() {
    for (int t = 1; t < R1; ++t) {
      int w = 0, e = 0;
      for (int p = t; p < R1; ++p) {
        w += work(p);
        e += ne(p);
      }
      if (w <= work(0) && e <= ne(0)) return t;
    }
    return R1 - 1;
  }
  static constexpr int TAIL = tail();
  static constexpr int NSLOT = TAIL + 1;
};

// tile geometry from the 3-D grid: x = line tile, y = position tile,
// z = (channel * NSLOT + slot) * res + fixed plane (res = 2^lres)
struct Tile {
  int ch, part, fixed, line0, pos0;
};
template <int NSLOT>
__device__ __forceinline__ Tile decode_tile(int lres, int line_lo, int pos_lo, int POS, int NL) {
  Tile r;
  r.line0 = line_lo + (int)blockIdx.x * NL;
  r.pos0 = pos_lo + (int)blockIdx.y * POS;
  const int z = (int)blockIdx.z;
  r.fixed = z & ((1 << lres) - 1);
  const int cp = z >> lres;
  r.part = cp % NSLOT;   // the slot; the kernel walks its partitions
  r.ch = cp / NSLOT;
  return r;
}

template <int RHO, int PASS, int POS, int NL, int TAPS, int TAPS1>
__device__ __forceinline__ void compute_tile(const float* sm, const float* sm1, const float* Kt,
                                             float* dst, int res, int pos_end, const Tile& T) {
  using I = SepIdx<RHO>;
  constexpr int R1 = RHO + 1;
  const int64_t plane = (int64_t)res * res * res;
  const int g = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P_ = T.part;
  int ng, ne, nin, in_base, in_stride, nout;
  int oe[R1];
  if (PASS == PASS_Z) {            // partition a = P_, group b = g
    ng = R1 - P_;
    ne = (R1 - P_) * (R1 - P_ + 1) / 2;
    nin = R1 - P_ - g;
    in_base = I::ab(P_, g) - I::ab(P_, 0);
    in_stride = 1;
    nout = R1;
#pragma unroll
    for (int j = 0; j < R1; ++j) oe[j] = I::zoff(P_, g, j);
  } else if (PASS == PASS_Y) {     // partition a = P_, group c' = g
    ng = R1;
    ne = (R1 - P_) * R1;
    nin = R1 - P_;
    in_base = g;
    in_stride = R1;
    nout = R1 - g;
#pragma unroll
    for (int j = 0; j < R1; ++j) oe[j] = I::yoff(P_, j, g);
  } else {                         // partition b' = P_, group c' = g
    ng = R1 - P_;
    ne = R1 * (R1 - P_);
    nin = R1;
    in_base = g;
    in_stride = R1 - P_;
    nout = R1 - P_ - g;
#pragma unroll
    for (int j = 0; j < R1; ++j) oe[j] = MI<RHO>::index(j, P_, g) < 0 ? 0 : MI<RHO>::index(j, P_, g);
  }
  if (g >= ng || lane >= NL) return;
  float* o;
  int64_t pos_stride;
  if (PASS == PASS_Z) {
    o = dst + ((int64_t)T.fixed * res + T.pos0) * res + T.line0 + lane;
    pos_stride = res;
  } else {
    o = dst + ((int64_t)T.pos0 * res + T.fixed) * res + T.line0 + lane;
    pos_stride = (int64_t)res * res;
  }
  const int nvalid = min(POS, pos_end - T.pos0);
#define FC2T2_SEP_N(Q)                                                                     \
  case Q:                                                                                  \
    if constexpr (Q <= R1)                                                                 \
      group_body<RHO, PASS, POS, NL, TAPS, TAPS1, Q>(sm, sm1, Kt, lane, nin, in_base,          \
                                                     in_stride, oe, o, pos_stride, plane,     \
                                                     nvalid);                                 \
    break;
  switch (nout) {
    FC2T2_SEP_N(1)
    FC2T2_SEP_N(2)
    FC2T2_SEP_N(3)
    FC2T2_SEP_N(4)
    FC2T2_SEP_N(5)
    FC2T2_SEP_N(6)
    default:
      break;
  }
#undef FC2T2_SEP_N
}

template <int RHO, int PASS, int POS, int NL>
constexpr int pass_win_floats() {
  constexpr int R1 = RHO + 1;
  return PASS == PASS_X ? R1 * R1 * NL * 16
                        : win_of(POS) * (PASS == PASS_Z ? R1 * (R1 + 1) / 2 : R1 * R1) * NL;
}
template <int RHO, int PASS, int POS, int NL, int NWIN = 1>
constexpr int pass_smem_floats() {  // window(s) + Kt[i][d][8] + mbarrier + 1 KB alignment slack
  return NWIN * pass_win_floats<RHO, PASS, POS, NL>() + 7 * 8 * (RHO + 1) + 2 + 256;
}

// TMA: one tensor map per partition (box = the partition's window); the
// out-of-range halo positions come back zero-filled (the reference's clipped
// source slices).  Dims, x fastest: z/y passes (x, z, y, channel * entries,
// 1); x pass (x, z, y, pair(b', c'), channel * (rho + 1) + a) with the
// 64-byte swizzle.
struct SepMaps {
  CUtensorMap m[6];
};

__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, int c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
      : "memory");
}

template <int RHO, int PASS, int POS, int NL>
__device__ __forceinline__ uint32_t window_bytes(int part) {
  constexpr int R1 = RHO + 1;
  const int ne = PASS == PASS_Z ? (R1 - part) * (R1 - part + 1) / 2
                                : (PASS == PASS_Y ? (R1 - part) * R1 : R1 * (R1 - part));
  return (uint32_t)(PASS == PASS_X ? 16 * NL * ne * 4 : win_of(POS) * NL * ne * 4);
}

// One pass.  Tile = 32 lines x 8 output positions of one partition/channel:
//   z pass: lines x, positions z, fixed y      (in M', out Z)
//   y pass: lines x, positions y, fixed z      (in Z,  out Y)
//   x pass: lines z, positions x, fixed y      (in Y,  out X)
// The window comes from one TMA tensor copy issued by thread 0.
template <int RHO, int PASS, int POS, int NL, int TAPS, int TAPS1>
__global__ void __launch_bounds__(32 * (RHO + 1), (PASS == PASS_Z && TAPS1 == TAPS_NONE ? 5 : 1))
sep_pass_kernel(float* __restrict__ out, int res, int lres, int line_lo, int pos_lo, int pos_end,
                const __grid_constant__ SepParams<RHO> prm, const __grid_constant__ SepMaps maps,
                const __grid_constant__ SepMaps maps1) {
  using I = SepIdx<RHO>;
  extern __shared__ __align__(16) unsigned char smraw[];
  float* sm = reinterpret_cast<float*>(
      smraw + ((1024 - ((unsigned)__cvta_generic_to_shared(smraw) & 1023)) & 1023));
  constexpr int R1 = RHO + 1;
  constexpr int NWIN = TAPS1 == TAPS_NONE ? 1 : 2;
  float* sm1 = sm + pass_win_floats<RHO, PASS, POS, NL>();
  float* Kt = sm + NWIN * pass_win_floats<RHO, PASS, POS, NL>();
  uint64_t* bar = reinterpret_cast<uint64_t*>(Kt + 7 * 8 * R1);
  const int64_t plane = (int64_t)res * res * res;
  const int out_entries = PASS == PASS_X ? I::P : I::T;
  using SL = Slots<RHO, PASS>;
  Tile T = decode_tile<SL::NSLOT>(lres, line_lo, pos_lo, POS, NL);
  const int p_first = T.part, p_last = T.part < SL::TAIL ? T.part : R1 - 1;
  const uint32_t bar_s = (uint32_t)__cvta_generic_to_shared(bar);
  {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar_s));
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
      uint32_t bytes = 0;
      for (int part = p_first; part <= p_last; ++part)
        bytes += window_bytes<RHO, PASS, POS, NL>(part);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s),
                   "r"(NWIN * bytes));
      uint32_t off = 0;   // bytes into the window area
      for (int part = p_first; part <= p_last; ++part) {
#pragma unroll
        for (int wi = 0; wi < NWIN; ++wi) {
          const uint32_t dst = (uint32_t)__cvta_generic_to_shared(wi ? sm1 : sm) + off;
          const CUtensorMap* mp = wi ? &maps1.m[part] : &maps.m[part];
          if (PASS == PASS_Z)
            tma_load_5d(dst, mp, T.line0, T.pos0 - 3, T.fixed, T.ch * I::P + I::ab(part, 0), 0,
                        bar_s);
          else if (PASS == PASS_Y)
            tma_load_5d(dst, mp, T.line0, T.fixed, T.pos0 - 3,
                        T.ch * I::T + I::pair(part, 0) * R1, 0, bar_s);
          else
            tma_load_5d(dst, mp, T.pos0 - 4, T.line0, T.fixed, I::pair(part, 0), T.ch * R1,
                        bar_s);
        }
        off += window_bytes<RHO, PASS, POS, NL>(part);
      }
    }
  }
  // Kt[i][d][j] = K(d - 3)[j][i], rows padded to 8 (two 128-bit loads),
  // laid out on the host
  for (int t = threadIdx.x; t < 7 * 8 * R1; t += 32 * R1) Kt[t] = (&prm.kt[0][0][0])[t];
  {
    __syncthreads();   // the barrier init is visible before anyone waits on it
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t"
        "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar_s)
        : "memory");
  }
  __syncthreads();
  uint32_t off = 0;   // floats into the window area
#pragma unroll 1
  for (int part = p_first; part <= p_last; ++part) {
    T.part = part;
    compute_tile<RHO, PASS, POS, NL, TAPS, TAPS1>(sm + off, sm1 + off, Kt,
                                                  out + (int64_t)T.ch * out_entries * plane, res,
                                                  pos_end, T);
    off += window_bytes<RHO, PASS, POS, NL>(part) / 4;
  }
}

template <int RHO>
SepParams<RHO> to_params(const double* pre, const double* post, const double* conv) {
  SepParams<RHO> p;
  constexpr int R1 = RHO + 1;
  for (int i = 0; i < R1; ++i)
    for (int j = 0; j < R1; ++j) {
      p.pre[i][j] = (float)pre[i * R1 + j];
      p.post[i][j] = (float)post[i * R1 + j];
      for (int d = 0; d < 7; ++d) p.conv[d][i][j] = (float)conv[(d * R1 + i) * R1 + j];
    }
  for (int i = 0; i < R1; ++i)
    for (int d = 0; d < 7; ++d)
      for (int j = 0; j < 8; ++j) p.kt[i][d][j] = j < R1 ? p.conv[d][j][i] : 0.f;
  return p;
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// tensor maps of one pass over `base` (one per partition); false on failure
template <int RHO, int PASS, int POS, int NL>
bool encode_maps(SepMaps& maps, const float* base, int res, int C) {
  using I = SepIdx<RHO>;
  constexpr int R1 = RHO + 1;
  auto enc = tmap_encoder();
  if (!enc) return false;
  const cuuint64_t r = (cuuint64_t)res, f = sizeof(float);
  for (int part = 0; part < R1; ++part) {
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
    dims[0] = dims[1] = dims[2] = r;
    strides[0] = r * f;
    strides[1] = r * r * f;
    strides[2] = r * r * r * f;
    if (PASS == PASS_X) {
      dims[3] = I::NAB;
      dims[4] = (cuuint64_t)C * R1;
      strides[3] = (cuuint64_t)I::NAB * r * r * r * f;
      box[0] = 16; box[1] = NL; box[2] = 1; box[3] = R1 - part; box[4] = R1;
      sw = CU_TENSOR_MAP_SWIZZLE_64B;
    } else {
      const int ent = PASS == PASS_Z ? I::P : I::T;
      const int ne = PASS == PASS_Z ? (R1 - part) * (R1 - part + 1) / 2 : (R1 - part) * R1;
      dims[3] = (cuuint64_t)C * ent;
      dims[4] = 1;
      strides[3] = dims[3] * r * r * r * f;
      box[0] = NL;
      box[1] = PASS == PASS_Z ? win_of(POS) : 1;
      box[2] = PASS == PASS_Z ? 1 : win_of(POS);
      box[3] = ne;
      box[4] = 1;
    }
    if (enc(&maps.m[part], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

// tensor maps of (base, res, C): workspaces come back at the same address
// call after call, so keep the last few encodings per instantiation
template <int RHO, int PASS, int POS, int NL>
bool cached_maps(SepMaps& maps, const float* in, int res, int C) {
  struct Cached {
    const float* base = nullptr;
    int res = 0, C = 0;
    SepMaps maps;
  };
  static std::mutex mu;
  static Cached cache[8];
  static unsigned next = 0;
  std::lock_guard<std::mutex> lock(mu);
  const Cached* hit = nullptr;
  for (const Cached& c : cache)
    if (c.base == in && c.res == res && c.C == C) hit = &c;
  if (!hit) {
    Cached& c = cache[next++ % 8];
    c.base = nullptr;
    std::memset(&c.maps, 0, sizeof(c.maps));
    if (!encode_maps<RHO, PASS, POS, NL>(c.maps, in, res, C)) return false;
    c.base = in;
    c.res = res;
    c.C = C;
    hit = &c;
  }
  maps = hit->maps;
  return true;
}

// one pass over `in` with tap subset TAPS; with TAPS1 != TAPS_NONE a second
// input `in1` (same layout) adds its TAPS1 taps to the same outputs
template <int RHO, int PASS, int POS, int NL, int TAPS, int TAPS1>
cudaError_t launch_pass_pos(const float* in, const float* in1, float* out, int res, int C,
                            int line_lo, int line_hi, int pos_lo, int pos_hi,
                            const SepParams<RHO>& prm, const char* name, cudaStream_t s) {
  const int nlt = (line_hi - line_lo + NL - 1) / NL;
  const int npt = (pos_hi - pos_lo + POS - 1) / POS;
  if ((int64_t)nlt * npt * res * (RHO + 1) * C <= 0) return cudaSuccess;
  int lres = 0;
  while ((1 << lres) < res) ++lres;
  const dim3 grid((unsigned)nlt, (unsigned)npt,
                  (unsigned)(res * Slots<RHO, PASS>::NSLOT * C));
  constexpr int NWIN = TAPS1 == TAPS_NONE ? 1 : 2;
  constexpr int smem = pass_smem_floats<RHO, PASS, POS, NL, NWIN>() * (int)sizeof(float);
  static unsigned long long configured = 0;
  if (smem > 48 * 1024 && attr_needed(configured))
    cudaFuncSetAttribute(sep_pass_kernel<RHO, PASS, POS, NL, TAPS, TAPS1>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  SepMaps maps, maps1;
  if (!cached_maps<RHO, PASS, POS, NL>(maps, in, res, C)) return cudaErrorNotSupported;
  if (NWIN == 2) {
    if (!cached_maps<RHO, PASS, POS, NL>(maps1, in1, res, C)) return cudaErrorNotSupported;
  } else {
    maps1 = maps;
  }
  FC2T2_LAUNCH(name, s,
               (sep_pass_kernel<RHO, PASS, POS, NL, TAPS, TAPS1>
                <<<grid, 32 * (RHO + 1), smem, s>>>(out, res, lres, line_lo, pos_lo, pos_hi, prm,
                                                    maps, maps1)));
  return cudaGetLastError();
}

// 32 lines per tile, or 16 on a 16-cell grid (the far table of a coarse level)
template <int RHO, int PASS, int TAPS = TAPS_ALL, int TAPS1 = TAPS_NONE>
cudaError_t launch_pass(const float* in, float* out, int res, int C, int line_lo, int line_hi,
                        int pos_lo, int pos_hi, const SepParams<RHO>& prm, const char* name,
                        cudaStream_t s, const float* in1 = nullptr) {
  if (res >= kLines)
    return launch_pass_pos<RHO, PASS, 8, kLines, TAPS, TAPS1>(in, in1, out, res, C, line_lo,
                                                              line_hi, pos_lo, pos_hi, prm, name, s);
  return launch_pass_pos<RHO, PASS, 8, 16, TAPS, TAPS1>(in, in1, out, res, C, line_lo, line_hi,
                                                        pos_lo, pos_hi, prm, name, s);
}

// the pre transform over cells with x in [xl, xh)
template <int RHO>
void launch_pre(const char* name, const float* M, float* Mp, int res, int lres, int C, int xl,
                int xh, const SepParams<RHO>& prm, cudaStream_t s) {
  const int64_t n = (int64_t)(xh - xl) * res * res;
  if (n <= 0) return;
  FC2T2_LAUNCH(name, s,
               sep_pre_kernel<RHO><<<dim3((unsigned)((n + 255) / 256), (unsigned)C), 256, 0, s>>>(
                   M, Mp, res, lres, C, xl, xh - xl, prm));
}

template <int RHO>
cudaError_t m2l_sep_rho(int level, int C, const double* pre, const double* post,
                        const double* conv, const float* M, float* L, float* wa, float* wb,
                        int x_begin, int x_end, int stages, const float* coarse, bool far_only,
                        cudaStream_t s) {
  const int res = 1 << (level + 1);
  const int nl = std::min(res, kLines);
  if (res % nl || res < 16) return cudaErrorInvalidValue;
  const int lres = level + 1;
  const SepParams<RHO> prm = to_params<RHO>(pre, post, conv);
  // x range the z/y passes must cover: the slab plus the x pass's halo,
  // widened to whole line tiles
  const int xl = std::max(0, x_begin - 3) / nl * nl;
  const int xh = std::min(res, (x_end + 3 + nl - 1) / nl * nl);
  cudaError_t err;
  if ((stages & SEP_FRONT) && far_only) {
    // The far table of a coarse level: the parity box minus the hole
    // {-1,0,1}^3 as three disjoint separable pieces (no cancellation against
    // the large hole terms).  With the per-axis tap sets A = parity box,
    // F = {|d| >= 2}, N = {|d| <= 1} over (x, y, z):
    //   F x A x A  +  N x F x A  +  N x N x F
    // z passes A and F of M'; y passes A(Z_A) and [F(Z_A) + N(Z_F)] (one
    // kernel over two windows); x pass [F(Y_AA) + N(Y_FA+NF)] likewise.
    const size_t tb = (size_t)SepIdx<RHO>::T * res * res * res * C;
    float *b0 = wa, *b1 = wb, *b2 = wb + tb, *b3 = wb + 2 * tb;
    launch_pre<RHO>("m2l_sepfar_pre", M, b0, res, lres, C, xl, xh, prm, s);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    if ((err = launch_pass<RHO, PASS_Z, TAPS_ALL>(b0, b1, res, C, xl, xh, 0, res, prm,
                                                  "m2l_sepfar_z", s)))
      return err;
    if ((err = launch_pass<RHO, PASS_Z, TAPS_FAR>(b0, b2, res, C, xl, xh, 0, res, prm,
                                                  "m2l_sepfar_z", s)))
      return err;
    if ((err = launch_pass<RHO, PASS_Y, TAPS_ALL>(b1, b0, res, C, xl, xh, 0, res, prm,
                                                  "m2l_sepfar_y", s)))
      return err;
    if ((err = launch_pass<RHO, PASS_Y, TAPS_FAR, TAPS_NEAR>(b1, b3, res, C, xl, xh, 0, res, prm,
                                                             "m2l_sepfar_y", s, b2)))
      return err;
    if ((err = launch_pass<RHO, PASS_X, TAPS_FAR, TAPS_NEAR>(b0, b1, res, C, 0, res, x_begin,
                                                             x_end, prm, "m2l_sepfar_x", s, b3)))
      return err;
  } else if (stages & SEP_FRONT) {
    launch_pre<RHO>("m2l_sep_pre", M, wa, res, lres, C, xl, xh, prm, s);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    if ((err = launch_pass<RHO, PASS_Z>(wa, wb, res, C, xl, xh, 0, res, prm, "m2l_sep_z", s)))
      return err;
    if ((err = launch_pass<RHO, PASS_Y>(wb, wa, res, C, xl, xh, 0, res, prm, "m2l_sep_y", s)))
      return err;
    if ((err = launch_pass<RHO, PASS_X>(wa, wb, res, C, 0, res, x_begin, x_end, prm, "m2l_sep_x",
                                        s)))
      return err;
  }
  if (stages & SEP_POST) {
    const int64_t n = (int64_t)(x_end - x_begin) * res * res;
    const float half_fine = (float)(1.0 / (double)res);
    if (n > 0) {
      FC2T2_LAUNCH(far_only ? "m2l_sepfar_post" : (coarse ? "m2l_sep_post_l2l" : "m2l_sep_post"), s,
                   sep_post_kernel<RHO><<<dim3((unsigned)((n + 255) / 256), (unsigned)C), 256, 0,
                                          s>>>(wb, L, res, lres, C, x_begin, x_end - x_begin, coarse,
                                               half_fine, prm));
      if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
  }
  return cudaSuccess;
}

}  // namespace

void* tensor_map_encoder() { return reinterpret_cast<void*>(tmap_encoder()); }

size_t m2l_sep_workspace_floats(int rho, int level, int C, bool far_only) {
  const int64_t res = 1 << (level + 1);
  const int64_t R1 = rho + 1, T = R1 * (R1 + 1) / 2 * R1;
  return (size_t)((far_only ? 4 : 2) * T * res * res * res * C);
}

cudaError_t m2l_sep(int rho, int level, int C, const double* pre, const double* post,
                    const double* conv, const float* M, float* L, float* ws, int x_begin,
                    int x_end, cudaStream_t s, int stages, const float* coarse, bool far_only) {
  const int64_t res = 1 << (level + 1);
  if (x_end < 0) x_end = (int)res;
  float* wa = ws;
  float* wb = ws + m2l_sep_workspace_floats(rho, level, C, false) / 2;
#define FC2T2_SEP_RHO(R)                                                                   \
  case R:                                                                                  \
    return m2l_sep_rho<R>(level, C, pre, post, conv, M, L, wa, wb, x_begin, x_end, stages, \
                          coarse, far_only, s);
  switch (rho) {
    FC2T2_SEP_RHO(1)
    FC2T2_SEP_RHO(2)
    FC2T2_SEP_RHO(3)
    FC2T2_SEP_RHO(4)
    FC2T2_SEP_RHO(5)
    default: return cudaErrorNotSupported;
  }
#undef FC2T2_SEP_RHO
}

}  // namespace fc2t2
