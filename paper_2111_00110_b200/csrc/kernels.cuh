// Internal launcher declarations (C++ side of the C ABI in abi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

namespace fc2t2 {

// sort.cu ----------------------------------------------------------------
size_t cell_sort_workspace(int level, int64_t n);
cudaError_t cell_sort(int level, const float* pts, int64_t n, int32_t* order,
                      int32_t* cell_start, int32_t* flag, void* ws, size_t ws_bytes,
                      cudaStream_t s);
cudaError_t find_box(int level, const float* pts, int64_t n, int32_t* box, int32_t* flag,
                     cudaStream_t s);
// stable sort of precomputed cell keys (key >= res^3 = "no cell", sorted last)
size_t key_sort_workspace(int level, int64_t n);
cudaError_t key_sort(int level, const uint32_t* keys, int64_t n, int32_t* order,
                     int32_t* cell_start, void* ws, size_t ws_bytes, cudaStream_t s);
size_t scan_ws_words(int64_t n);
cudaError_t exclusive_scan(const uint32_t* in, uint32_t* out, int64_t n, uint32_t* ws,
                           cudaStream_t s);

// p2m_brick.cu -------------------------------------------------------------
// P2M straight from unsorted points: deterministic stable partition into
// 8 x 8 x (4|8) cell bricks + one CTA per brick (levels 2..6, C <= 8)
bool p2m_brick_supported(int level, int C);
size_t p2m_brick_workspace(int level, int64_t n, int C);
// phases: P2M_PREPARE (partition counts, points only) and P2M_FINISH (records,
// per-brick sums; needs the weights and the prepared workspace)
enum { P2M_PREPARE = 1, P2M_FINISH = 2, P2M_ALL = 3 };
cudaError_t p2m_brick(int rho, int level, int C, const float* pts, const float* w, int64_t n,
                      float* M, int32_t* flag, void* ws, size_t ws_bytes, cudaStream_t s,
                      int phase = P2M_ALL);

// expand.cu --------------------------------------------------------------
// float32 sums of each cell's points in the stable sort's index order
cudaError_t p2m_sorted(int rho, int level, int C, const float* pts, const float* w,
                       const int32_t* order, const int32_t* cell_start, float* M,
                       cudaStream_t s);
// x ranges (cells of the output level, x_end < 0 = all) restrict the
// outputs to one x-slab (the multi-GPU cascade)
cudaError_t m2m(int rho, int fine_level, int C, const float* fine, float* coarse, cudaStream_t s,
                int cx_begin = 0, int cx_end = -1);
cudaError_t l2l(int rho, int coarse_level, int C, const float* coarse, float* fine,
                int accumulate, cudaStream_t s, int fx_begin = 0, int fx_end = -1);

// One M2L launch: every target class (8 parity classes, or 1 for a
// parity-free stencil) walks its own interaction list.
struct M2LLaunch {
  int level;
  int stride;            // 2 with parity classes, 1 without
  int ncls;              // 8 or 1
  const int4* entries;   // device, {dx, dy, dz, slot}
  const int* cls_start;  // device, ncls + 1
  int max_list;          // host copy of the longest list (0 -> nothing to do)
  const char* level_name;  // profiling label, e.g. "m2l_L5"
};
// splits > 1 (with a workspace ``part`` of splits * grid floats) splits each
// class's interaction list across CTAs for small levels; m2l_splits picks it.
int m2l_splits(int rho, int C, const M2LLaunch& plan);
// targets restricted to cells with x in [x_begin, x_end) (multiples of the
// stencil stride; x_end < 0 = all)
cudaError_t m2l(int rho, int C, const M2LLaunch& plan, const float* coef, const float* M,
                float* L, int accumulate, cudaStream_t s, float* part = nullptr, int splits = 1,
                int x_begin = 0, int x_end = -1);

// m2l_tc.cu --------------------------------------------------------------
// tcgen05 M2L for parity levels.  btab is the plan's dense table:
// [class group][source class 8][K step][slot 27][kchunk 2][row 2W][16 B]
// (see tc_geometry and abi.cu build_tc_table), the scaled two-term fp16 split
// (rk: per-output-column scales, s_inv: 1/s_n per coefficient).
struct TCPlan {
  int level;
  const uint8_t* btab;
  const char* level_name;
  const float* rk = nullptr;
  const float* s_inv = nullptr;
};
// classes per CTA, N per class, K steps, bytes per slot table, flags (bit 0:
// single-buffered layout, B rows always [lo | hi]; bit 1: merged last K step,
// see TC::MERGE_LAST); 0 on success
int tc_geometry(int rho, int* cls, int* nc, int* ks, int* bslot, int* sb, int* tiles);
// tensor-core FLOPs one m2l_tc launch issues (2 M N K per MMA, padding and
// split terms included) for a whole level
double tc_issued_flops(int rho, int level, int C);
// s_n = (h/2)^|n| / n! at a level, graded-lex order (P doubles)
int tc_moment_scales(int rho, int level, double* s);
// scratch of one M2L launch: per-channel scale bits + hi/lo operand planes
size_t tc_workspace_bytes(int rho, int level, int C);
cudaError_t tc_prepare(int rho, int C, const TCPlan& plan, const float* M, void* ws,
                       cudaStream_t s);
// targets restricted to cells with x in [x_begin, x_end) (multiples of 4; x_end < 0 = res)
cudaError_t m2l_tc(int rho, int C, const TCPlan& plan, const void* ws, float* L, int accumulate,
                   cudaStream_t s, int x_begin = 0, int x_end = -1);

// m2l_sep.cu -------------------------------------------------------------
// Finest-level far + near M2L through the per-axis factors of the tables
// (kernel.py separable_factors): pre/post (R1 x R1) and conv (7 x R1 x R1),
// [out][in] float64 row-major, R1 = rho + 1 <= 6.  Writes L (no accumulate)
// for cells with x in [x_begin, x_end); ws = m2l_sep_workspace_floats.
// stages: SEP_FRONT (pre + z/y/x passes into the workspace), SEP_POST (post
// transform into L; with `coarse` = L of the level above, the L2L is fused:
// L = L2L(coarse) + M2L).  The two may run on different streams.
enum { SEP_FRONT = 1, SEP_POST = 2, SEP_ALL = 3 };
// far_only: the far table of a coarse level (grids of >= 16 cells): the parity
// box minus the hole as three disjoint separable pieces (5 passes, 4 scratch
// buffers instead of 2); pre/post/conv are that level's factors.
size_t m2l_sep_workspace_floats(int rho, int level, int C, bool far_only = false);
cudaError_t m2l_sep(int rho, int level, int C, const double* pre, const double* post,
                    const double* conv, const float* M, float* L, float* ws, int x_begin,
                    int x_end, cudaStream_t s, int stages = SEP_ALL,
                    const float* coarse = nullptr, bool far_only = false);

// cuTensorMapEncodeTiled from the driver (nullptr when unavailable)
void* tensor_map_encoder();

// l2p.cu -----------------------------------------------------------------
enum L2PMode : int {
  L2P_VALUE = 1,   // (n, C)
  L2P_GRAD = 2,    // (n, C, 3)
  L2P_HESS = 4,    // (n, C, 6)  xx yy zz xy xz yz
  L2P_WGRAD = 8,   // (n, 3) = sum_c wts[n, c] * grad f_c
};
// out (n, 3) = sum_c w (n, C) * grad (n, C, 3): L2P_WGRAD from stored gradients
cudaError_t weighted_grad(const float* grad, const float* w, int64_t n, int C, float* out,
                          cudaStream_t s);
cudaError_t l2p(int rho, int level, int C, const float* L, const float* q, int64_t n, int mode,
                const int32_t* order, const float* wts, float* value, float* grad, float* hess,
                float* wgrad, int32_t* flag, cudaStream_t s);

}  // namespace fc2t2

// rays.cu -----------------------------------------------------------------
namespace fc2t2 {
cudaError_t traverse_count(int level, const double* org, const double* dir, int64_t R,
                           uint32_t* counts, cudaStream_t s);
cudaError_t traverse_fill(int level, const double* org, const double* dir, int64_t R,
                          const uint32_t* offsets, int32_t* ray_id, double* t0, double* t1,
                          int32_t* box, cudaStream_t s);
cudaError_t depth_walk(int rho, int level, const float* L, const double* org, const double* dir,
                       int64_t R, double bias, double* lengths, uint8_t* hit, double* points,
                       float* grads, float* hess, float* denom, cudaStream_t s);
cudaError_t root_payload(int rho, int level, const double* dir, int64_t R, const uint8_t* hit,
                         const double* points, const float* grads, const float* hess,
                         const float* denom, const float* y_len, const float* y_grad,
                         uint32_t* keys, float* payload, int32_t* n_clamped, cudaStream_t s);
cudaError_t line_integral(int rho, int level, int C, const float* L, const double* org,
                          const double* dir, int64_t R, float* values, cudaStream_t s);
cudaError_t line_payload(int rho, int level, int C, const double* org, const double* dir,
                         int64_t R, const uint32_t* offsets, const float* y, const double* gl_x,
                         const double* gl_w, int G, uint32_t* keys, float* payload,
                         cudaStream_t s);
cudaError_t insert_sorted(int rho, int level, int C, const float* payload, const int32_t* order,
                          const int32_t* cell_start, float* M, cudaStream_t s);
}  // namespace fc2t2

// volume.cu ---------------------------------------------------------------
namespace fc2t2 {
int vol_gauss_nodes(int rho);
cudaError_t vol_forward(int rho, int level, int CC, const float* L, const double* org,
                        const double* dir, int64_t R, const double* efit, const double* bg,
                        float* rgb, double* depth_final, const uint32_t* seg_offsets,
                        uint8_t* seg_alive, cudaStream_t s, uint32_t* n_alive = nullptr,
                        double* totals = nullptr);
cudaError_t vol_totals(int rho, int level, int CC, const float* L, const double* org,
                       const double* dir, int64_t R, const double* efit, uint32_t* n_alive,
                       double* totals, double* depth_final, cudaStream_t s);
// segment records (vol_record_floats(CC) floats each) expanded and summed per
// cell in the key sort's order into M (res^3, 1 + CC, PP)
int vol_record_floats(int CC);
cudaError_t vol_insert(int rho, int level, int CC, const float* rec, const int32_t* order,
                       const int32_t* cell_start, float* M, cudaStream_t s);
cudaError_t vol_payload(int rho, int level, int CC, const float* L, const double* org,
                        const double* dir, int64_t R, const double* efit, const double* bg,
                        const float* ybar, const uint32_t* alive_offsets, const double* totals,
                        const double* depth_final, const double* gl_x, const double* gl_w,
                        uint32_t* keys, float* payload, cudaStream_t s);
// train.cu ----------------------------------------------------------------
size_t loss_workspace_bytes(int64_t n, int cols);
// stats (3 doubles): count, loss, sum(tangent)
cudaError_t loss_tangent(const float* pred, const float* target, const uint8_t* mask, int64_t n,
                         int cols, float bias, int mse, float* tangent, double* stats, void* ws,
                         cudaStream_t s);
cudaError_t nonfinite(const float* x, int64_t n, int32_t* flag, cudaStream_t s);
cudaError_t opt_step(float* x, const float* g, float* m, float* v, int64_t n, int adam, float lr,
                     float c1, float c2, float l1, int clip, const int32_t* flag, cudaStream_t s);

}  // namespace fc2t2
