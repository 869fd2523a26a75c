/*
 * fc2t2_b200.h -- C ABI of the B200-native FC2T2 hot path.
 *
 * The reference (pkg/src/fc2t2, pure NumPy) has no native boundary; its hot
 * path is the Python call surface of expansion.py / layers.py / ray.py.  This
 * header is the drop-in replacement underneath that surface: every entry point
 * below names the reference function it replaces (file:line, paths relative to
 * pkg/src/fc2t2/).  The Python shim paper_2111_00110_b200 binds it with ctypes
 * (INTEGRATION.md shows the same binding for the reference package).
 *
 * Conventions
 *   - plain pointers and sizes only; every pointer argument named d_* is
 *     DEVICE memory owned by the caller (the library never allocates or frees
 *     caller memory in a hot call; scratch comes from the caller's workspace,
 *     sized by the matching *_workspace_size query);
 *   - stream is a cudaStream_t passed as void*; all work is stream ordered,
 *     no call synchronises except fc2t2_engine_upload;
 *   - d_flag (int32, may be NULL) accumulates FLAG_* bits; the shim reads it
 *     once per layer call and raises the reference exception;
 *   - coefficient grids are (res, res, res, C, PP) float32, graded-lex order,
 *     PP = index_count(rho) rounded up to a multiple of 4 (pad entries 0);
 *     res = 2^(level+1).  Points are (n, 3) float32, weights (n, C) float32.
 *   - return value: FC2T2_OK or an FC2T2_E* code; fc2t2_last_error() gives text.
 */
#ifndef FC2T2_B200_H
#define FC2T2_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the shim maps them to the reference exception classes */
#define FC2T2_OK 0
#define FC2T2_EDOMAIN 1    /* expansion.py:23-24 DomainError           */
#define FC2T2_ESTAGE 2     /* expansion.py:27-28 StageError            */
#define FC2T2_EORDER 3     /* multiindex.py:20-21 OrderError           */
#define FC2T2_ECUDA 4      /* CUDA runtime failure                     */
#define FC2T2_EWORKSPACE 5 /* workspace too small                       */
#define FC2T2_EVALUE 6     /* ValueError (bad shapes / arguments)      */

#define FC2T2_FLAG_DOMAIN 1

/* M2L table selector for fc2t2_m2l */
#define FC2T2_TABLE_FAR 0      /* the level's far table (kernel.py:280-290)   */
#define FC2T2_TABLE_NEAR 1     /* finest-level near table (kernel.py:295-299) */
#define FC2T2_TABLE_FARNEAR 2  /* far + near merged (finest level only)       */

/* L2P output selector bits for fc2t2_l2p */
#define FC2T2_L2P_VALUE 1 /* Accessor.value    expansion.py:348-355 */
#define FC2T2_L2P_GRAD 2  /* Accessor.partials expansion.py:367-369 */
#define FC2T2_L2P_HESS 4  /* Accessor.partials2 expansion.py:371-373 */
#define FC2T2_L2P_WGRAD 8 /* sum_c wts_c * grad f_c (layers.py:183, :186-187) */

typedef struct fc2t2_engine fc2t2_engine;

int fc2t2_version(void);
const char* fc2t2_last_error(void);

/* ---- instrumentation (no reference counterpart; used by bench.py) ----
 * launch_count: kernels launched by this library since load.
 * profile_enable(1): bracket every launch with CUDA events on its stream
 * (clears previous records); profile_read syncs them and returns per-kernel
 * totals: names (32 bytes each), ms, launch counts; returns #entries. */
int64_t fc2t2_launch_count(void);
int fc2t2_profile_enable(int on);
int fc2t2_profile_read(int max_entries, char* names, double* ms, int64_t* counts);
/* The recorded launches one by one, in issue order: names (32 bytes each) and
 * the begin / end event times in ms relative to the first launch's begin
 * event (a device timeline across the library's streams).  Returns the count. */
int fc2t2_profile_timeline(int max_entries, char* names, double* begin_ms, double* end_ms);

/* ---- engine: replaces Engine.__init__ table state (expansion.py:157-177) ---- */
int fc2t2_engine_create(int rho, int levels, fc2t2_engine** out);
void fc2t2_engine_destroy(fc2t2_engine* e);
/* Hand one fitted M2LTable to the engine (host arrays, kernel.py:124-141):
 * offsets (K,3) int64, active (K,) uint8, coeffs (K,P,P) float64 [k][n]. */
int fc2t2_engine_set_table(fc2t2_engine* e, int level, int nearfield, int64_t n_offsets,
                           const int64_t* offsets, const uint8_t* active,
                           const double* coeffs);
/* On-device table fitting (replaces _build_offset_matrices / the LSQ fit of
 * kernel.py:180-204).  For `count` offsets (d_offsets (count,3)
 * int32, source - target) at one level: coeffs[o] = (pinv(V) Psi(o)
 * pinv(V)^T)^T as (count, P, P) float64 [k_local][n_moment], and d_resid[o] =
 * max |V A V^T - Psi(o)| (kernel.py:202).  d_pinv (P, nodes^3) and d_v
 * (nodes^3, P) float64 are pinv(V) and V over the nodes^3 Chebyshev grid with
 * per-axis coordinates d_nodes (nodes,) (already scaled by width/2); only
 * nodes == 6 (the reference default) is supported.  All pointers are device
 * memory; stream-ordered, no host sync.  EVALUE for bad sizes. */
int fc2t2_fit_tables(int rho, int nodes, const double* d_pinv, const double* d_v,
                     const double* d_nodes, double alpha, double width, const int32_t* d_offsets,
                     int64_t count, double* d_coeffs, double* d_resid, void* stream);
/* dynamic shared memory one fit CTA uses (bytes) */
size_t fc2t2_fit_tables_smem(int rho);
/* ---- data formats: dataio.py ----
 * Interleaved float64 rows (x, y, z, v1..vC) of an FCPT payload
 * (dataio.py:99-104) or a checkpoint's p block (C = 0) -> float32 columns
 * d_p (m, 3) and d_v (m, C), one coalesced pass.  With d_first_bad (one
 * uint64, caller-initialised to UINT64_MAX) the smallest row index with a
 * coordinate outside (-1, 1) (or NaN) is recorded: the point PointSampleSet
 * rejects (dataio.py:49-51). */
int fc2t2_unpack_rows(const double* d_rows, int64_t m, int c, float* d_p, float* d_v,
                      uint64_t* d_first_bad, void* stream);

/* Sets FLAG_DOMAIN in *d_flag if any coordinate of d_pts (n, 3) float32
 * (16-byte aligned) is not strictly inside (-1, 1) -- the check of
 * Accessor._local / SourceSet (expansion.py:45-46, :337-338) as a
 * stand-alone read, so a layer can test its inputs early. */
int fc2t2_domain_check(const float* d_pts, int64_t n, int32_t* d_flag, void* stream);

/* Build the per-parity interaction lists and upload fp32 tables (once). */
int fc2t2_engine_upload(fc2t2_engine* e, void* stream);
/* number of (level, class) interaction-list entries, for diagnostics */
int64_t fc2t2_engine_list_entries(const fc2t2_engine* e, int level, int table);
/* copy a level's interaction list to host: (n, 4) int32 {dx,dy,dz,slot} and
 * the class start offsets (ncls+1); returns ncls or -1 */
int fc2t2_engine_get_list(const fc2t2_engine* e, int level, int table, int32_t* entries,
                          int32_t* cls_start);

/* ---- point -> cell: find_box (expansion.py:85-93) ---- */
int fc2t2_find_box(int level, const float* d_pts, int64_t n, int32_t* d_box, int32_t* d_flag,
                   void* stream);
/* Stable sort of points by finest cell + per-cell ranges (the np.add.at key
 * of expansion.py:195).  d_order (n) int32, d_cell_start (res^3 + 1) int32. */
size_t fc2t2_cell_sort_workspace_size(int level, int64_t n);
int fc2t2_cell_sort(int level, const float* d_pts, int64_t n, int32_t* d_order,
                    int32_t* d_cell_start, int32_t* d_flag, void* d_ws, size_t ws_bytes,
                    void* stream);
/* ---- P2M from unsorted points (Engine.p2m, expansion.py:186-198) ----
 * d_pts (n, 3), d_w (n, C) in the caller's order; no sort object.  A
 * deterministic stable partition of the points into bricks of 8 x 8 x 4
 * cells (8 x 8 x 8 at level 6), then one CTA per brick sums every cell's
 * points in index order (the np.add.at order) -- no atomics, bit-reproducible.
 * Sets FLAG_DOMAIN for points outside (-1, 1)^3.  Levels >= 7 fall back to
 * the stable cell sort + gather P2M below (same results). */
size_t fc2t2_p2m_points_workspace_size(const fc2t2_engine* e, int channels, int64_t n);
int fc2t2_p2m_points(const fc2t2_engine* e, int channels, const float* d_pts, const float* d_w,
                     int64_t n, float* d_m_finest, int32_t* d_flag, void* d_ws, size_t ws_bytes,
                     void* stream);
/* The same in two phases on one workspace: phase 1 = the partition of the
 * points (counts and brick starts; reads only d_pts, sets FLAG_DOMAIN),
 * phase 2 = records + per-brick sums (needs d_w and a workspace prepared by
 * phase 1 for the same points); 3 = both.  Lets a caller partition points
 * early (the explicit backward's queries, beside the forward's tail). */
int fc2t2_p2m_points_phase(const fc2t2_engine* e, int channels, const float* d_pts,
                           const float* d_w, int64_t n, float* d_m_finest, int32_t* d_flag,
                           void* d_ws, size_t ws_bytes, int phase, void* stream);

/* ---- stages (expansion.py:186-264) ---- */
/* d_order NULL: d_pts / d_w are already in cell-sorted order */
int fc2t2_p2m(const fc2t2_engine* e, int channels, const float* d_pts, const float* d_w,
              const int32_t* d_order, const int32_t* d_cell_start, float* d_m_finest,
              void* stream);
int fc2t2_m2m(const fc2t2_engine* e, int channels, int fine_level, const float* d_fine,
              float* d_coarse, void* stream);
int fc2t2_l2l(const fc2t2_engine* e, int channels, int coarse_level, const float* d_coarse,
              float* d_fine, int accumulate, void* stream);
/* M2L of one table.  With a workspace of fc2t2_m2l_workspace_size bytes the
 * parity levels run the tcgen05 3xTF32 kernel; without one, FP32 FFMA. */
size_t fc2t2_m2l_workspace_size(const fc2t2_engine* e, int channels, int level, int table);
/* Tensor-core FLOPs (2 M N K per tcgen05.mma, K/N padding and the split's
 * cross products included) one M2L launch of this table issues; 0 when the
 * table runs on FFMA.  The algorithmic count is pairs * C * P^2 * 2. */
double fc2t2_m2l_issued_flops(const fc2t2_engine* e, int channels, int level, int table);
int fc2t2_m2l(const fc2t2_engine* e, int channels, int level, int table, const float* d_m,
              float* d_l, int accumulate, void* d_ws, size_t ws_bytes, void* stream);

/* ---- cascade: Engine.expand_from_moments (expansion.py:268-281) ---- */
/* Separable finest-level M2L.  The finest far (parity stencil) + near tables
 * of a Gaussian engine factor per axis (kernel.py separable_factors; the LSQ
 * fit of ref kernel.py:180-204 and the Taylor tables of :169-177):
 * coeffs(o) = post_S (K(o_x) (x) K(o_y) (x) K(o_z))_S pre_S.  With the
 * factors set, fc2t2_expand runs the finest far + near M2L
 * (ref expansion.py:276-279) as three 1-D convolutions (m2l_sep.cu) instead
 * of the dense tables; valid only when every stencil offset of that level is
 * active (the caller checks: kernel.py separable_eligible).  pre, post
 * (rho+1)^2 and conv 7 (rho+1)^2 float64, [out][in], d = -3..3; NULL
 * pointers switch back to the dense path.  rho <= 5, finest res >= 32. */
int fc2t2_engine_set_separable(fc2t2_engine* e, const double* pre, const double* post,
                               const double* conv);
int fc2t2_engine_separable(const fc2t2_engine* e);
/* The far table of a coarse level (kCoarsest < level < levels, >= 16 cells per
 * axis) through that level's per-axis factors: the parity stencil minus the
 * hole {-1,0,1}^3 (ref expansion.py:246-249, kernel.py:257-300) as three
 * disjoint separable pieces, F x A x A + N x F x A + N x N x F with the axis tap
 * sets A = parity box, F = {|d| >= 2}, N = {|d| <= 1} -- seven 1-D passes
 * instead of 189 dense tables per target.  Offsets the reference prunes (peak
 * interaction below 1e-16, kernel.py:275) are included; the caller checks
 * eligibility (kernel.py separable_far_eligible).  Same argument layout as
 * fc2t2_engine_set_separable; NULL pointers restore the dense path. */
int fc2t2_engine_set_separable_far(fc2t2_engine* e, int level, const double* pre,
                                   const double* post, const double* conv);
/* 1 (default): the separable M2L's post transform runs after the coarse chain
 * with the finest L2L fused into it (one pass over the finest L grid fewer);
 * 0: separate accumulate-L2L launch.  Results are bit-identical. */
int fc2t2_engine_set_sep_fusion(fc2t2_engine* e, int fuse_l2l);
size_t fc2t2_expand_workspace_size(const fc2t2_engine* e, int channels);
int fc2t2_expand(const fc2t2_engine* e, int channels, const float* d_m_finest,
                 float* d_l_finest, void* d_ws, size_t ws_bytes, void* stream);
/* Same cascade, but only finest-level cells with x in [x_begin, x_end) are
 * produced (multiples of 4; x_end < 0 = res): one rank's x-slab (SURVEY
 * 8(e)).  The coarse M2L and L2L run only on the slab's cells at every level
 * where the slab maps to whole cells (else on the whole level); the M2M chain
 * runs on the whole grid (d_m_finest must be complete).  Other finest cells
 * of d_l_finest are left unspecified.  Same workspace. */
int fc2t2_expand_slab(const fc2t2_engine* e, int channels, const float* d_m_finest,
                      float* d_l_finest, int x_begin, int x_end, void* d_ws, size_t ws_bytes,
                      void* stream);
/* The slab cascade in two phases for a reduce-scattered finest M (the
 * multi-GPU cascade: no level is replicated).
 *   expand_up:   M2M chain on the slab only (d_m_finest valid on the slab),
 *                coarse M grids written into the workspace at
 *                fc2t2_expand_grid_offset(level) (x-slowest, so the slab's
 *                cells are contiguous); the caller all-gathers every coarse
 *                level in [fc2t2_expand_lowest, levels) in place;
 *   expand_down: coarse M2L + L2L on the slab at every level, the finest M2L
 *                on the slab (d_m_finest valid on [x_begin - 3, x_end + 3):
 *                the M2L reach, ref kernel.py:39) and the last L2L.
 * fc2t2_expand_slab_split(x_begin, x_end) = 1 when every coarse level maps
 * the slab to whole cells (else use fc2t2_expand_slab on a complete M). */
int fc2t2_expand_up(const fc2t2_engine* e, int channels, const float* d_m_finest, int x_begin,
                    int x_end, void* d_ws, size_t ws_bytes, void* stream);
int fc2t2_expand_down(const fc2t2_engine* e, int channels, const float* d_m_finest,
                      float* d_l_finest, int x_begin, int x_end, void* d_ws, size_t ws_bytes,
                      void* stream);
int fc2t2_expand_lowest(const fc2t2_engine* e);
int64_t fc2t2_expand_grid_offset(const fc2t2_engine* e, int channels, int level);
int fc2t2_expand_slab_split(const fc2t2_engine* e, int x_begin, int x_end);

/* ---- L2P: Accessor (expansion.py:335-373) ----
 * d_order (optional, n int32): evaluate the points in this (cell-sorted) order;
 * outputs are still indexed by point. */
int fc2t2_l2p(int rho, int level, int channels, const float* d_l, const float* d_q, int64_t n,
              int mode, const int32_t* d_order, const float* d_wts, float* d_value,
              float* d_grad, float* d_hess, float* d_wgrad, int32_t* d_flag, void* stream);
/* q_bar recycling (explicit_jvp, ref layers.py:183): d_out (n, 3) =
 * sum_c d_w[n, c] * d_grad[n, c, :] from the gradient a VALUE | GRAD L2P
 * stored in the forward -- bit-identical to an FC2T2_L2P_WGRAD launch. */
int fc2t2_weighted_grad(const float* d_grad, const float* d_w, int64_t n, int channels,
                        float* d_out, void* stream);

/* ---- rays: traversal (ray.py:101-157), layers (layers.py:193-402) ----
 * Rays are (R, 3) float64 origins / directions on the device.  Traversal:
 * count segments per ray, exclusive-scan the counts (fc2t2_scan_u32), fill
 * ray_id (S) int32, t0/t1 (S) float64, box (S, 3) int32. */
const char* fc2t2_ray_last_error(void);
size_t fc2t2_scan_workspace_size(int64_t n);
int fc2t2_scan_u32(const uint32_t* d_in, uint32_t* d_out, int64_t n, void* d_ws, size_t ws_bytes,
                   void* stream);
int fc2t2_traverse_count(int level, const double* d_org, const double* d_dir, int64_t R,
                         uint32_t* d_counts, void* stream);
int fc2t2_traverse_fill(int level, const double* d_org, const double* d_dir, int64_t R,
                        const uint32_t* d_offsets, int32_t* d_ray_id, double* d_t0, double* d_t1,
                        int32_t* d_box, void* stream);
/* depth_forward + _first_root_per_ray (layers.py:208-272) fused with the
 * gradient (and optional Hessian, xx yy zz xy xz yz) at the hit. */
int fc2t2_depth_forward(int rho, int level, const float* d_l, const double* d_org,
                        const double* d_dir, int64_t R, double bias, double* d_lengths,
                        uint8_t* d_hit, double* d_points, float* d_grads, float* d_hess,
                        float* d_denom, void* stream);
/* depth_jvp / surface_gradient_jvp insertion payloads (layers.py:275-356);
 * either tangent may be NULL; both given = one fused insertion. */
int fc2t2_root_payload(int rho, int level, const double* d_dir, int64_t R, const uint8_t* d_hit,
                       const double* d_points, const float* d_grads, const float* d_hess,
                       const float* d_denom, const float* d_y_len, const float* d_y_grad,
                       uint32_t* d_keys, float* d_payload, int32_t* d_n_clamped, void* stream);
/* line_integral_forward (layers.py:371-386) and the jvp's segment payloads
 * y_c * line2taylor (layers.py:389-402, ray.py:213-246). */
int fc2t2_line_integral(int rho, int level, int channels, const float* d_l, const double* d_org,
                        const double* d_dir, int64_t R, float* d_values, void* stream);
int fc2t2_line_payload(int rho, int level, int channels, const double* d_org, const double* d_dir,
                       int64_t R, const uint32_t* d_offsets, const float* d_y,
                       const double* d_gl_x, const double* d_gl_w, int G, uint32_t* d_keys,
                       float* d_payload, void* stream);
/* generic insertion (_insert_moments, layers.py:144-153): stable sort of
 * precomputed cell keys (key res^3 = no cell), then per-cell sums of the
 * (n, C, PP) payload rows in sorted order into the finest M grid. */
size_t fc2t2_key_sort_workspace_size(int level, int64_t n);
int fc2t2_key_sort(int level, const uint32_t* d_keys, int64_t n, int32_t* d_order,
                   int32_t* d_cell_start, void* d_ws, size_t ws_bytes, void* stream);
int fc2t2_insert(int rho, int level, int channels, const float* d_payload, const int32_t* d_order,
                 const int32_t* d_cell_start, float* d_m, void* stream);

/* ---- integral-implicit radiance layer (layers.py:405-544), rho = 4 ----
 * grid channels = 1 (density, relu'd weights) + colors; efit = the 5
 * coefficients of the exp(-x) fit (poly1d.py:224-242), bg (colors,).
 * forward: rgb (R, colors), depth_final (R) float64, optional per-segment
 * alive flags (with traversal offsets).  backward: pass A (alive counts,
 * totals (R, colors) float64, depth_final), exclusive scan of the counts,
 * pass B (keys + (n_alive, 1+colors, PP) payload rows) -> fc2t2_insert. */
int fc2t2_vol_gauss_nodes(int rho);
int fc2t2_vol_forward(int rho, int level, int colors, const float* d_l, const double* d_org,
                      const double* d_dir, int64_t R, const double* d_efit, const double* d_bg,
                      float* d_rgb, double* d_depth_final, const uint32_t* d_seg_offsets,
                      uint8_t* d_seg_alive, void* stream);
/* forward that also returns pass A's outputs (n_alive (R), totals (R, colors)),
 * bit-identical to fc2t2_vol_totals: the backward then skips pass A */
int fc2t2_vol_forward_ex(int rho, int level, int colors, const float* d_l, const double* d_org,
                         const double* d_dir, int64_t R, const double* d_efit, const double* d_bg,
                         float* d_rgb, double* d_depth_final, uint32_t* d_n_alive,
                         double* d_totals, void* stream);
int fc2t2_vol_totals(int rho, int level, int colors, const float* d_l, const double* d_org,
                     const double* d_dir, int64_t R, const double* d_efit, uint32_t* d_n_alive,
                     double* d_totals, double* d_depth_final, void* stream);
/* Backward pass B (volumetric_jvp, layers.py:483-544): per alive segment its
 * cell key and a segment record of fc2t2_vol_record_floats(colors) floats
 * (d_payload (A, rec)): line base + direction and the (1 + colors) x 5 power
 * moments of the node-weighted adjoint densities.  fc2t2_vol_insert expands
 * the records of every cell, in the stable key order of fc2t2_key_sort, and
 * sums them into the moment grid (res^3, 1 + colors, PP) -- the
 * _insert_moments of layers.py:144-153 without payload rows in memory. */
int fc2t2_vol_payload(int rho, int level, int colors, const float* d_l, const double* d_org,
                      const double* d_dir, int64_t R, const double* d_efit, const double* d_bg,
                      const float* d_ybar, const uint32_t* d_alive_offsets,
                      const double* d_totals, const double* d_depth_final, const double* d_gl_x,
                      const double* d_gl_w, uint32_t* d_keys, float* d_payload, void* stream);
int fc2t2_vol_record_floats(int colors);
int fc2t2_vol_insert(int rho, int level, int colors, const float* d_rec, const int32_t* d_order,
                     const int32_t* d_cell_start, float* d_m, void* stream);

/* ---- training glue: trainer.py (reference trainer.py:70-152) ----
 * Losses (loss_and_tangent, trainer.py:70-105): diff = pred + bias - target
 * over valid entries (d_mask (n) uint8, optional, broadcast over the `cols`
 * columns); d_tangent (n, cols) = d loss / d pred; d_stats (3 doubles) =
 * count, loss, sum(tangent) (the bias tangent of cli.py fit loops).
 * Deterministic float64 reductions. */
#define FC2T2_LOSS_MAE 0
#define FC2T2_LOSS_MSE 1
size_t fc2t2_loss_workspace_size(int64_t n, int cols);
int fc2t2_loss(const float* d_pred, const float* d_target, const uint8_t* d_mask, int64_t n,
               int cols, float bias, int kind, float* d_tangent, double* d_stats, void* d_ws,
               size_t ws_bytes, void* stream);
/* sets *d_flag |= 1 when d_x holds a NaN or Inf (Optimizer.step's check) */
int fc2t2_nonfinite(const float* d_x, int64_t n, int32_t* d_flag, void* stream);
/* Optimizer.step for one tensor (trainer.py:122-152): grad + l1 sign(x)
 * (l1_term, trainer.py:108-112); Adam (t = step count, bias-corrected, betas
 * 0.9/0.999, eps 1e-8; d_m/d_v state) or SGD; x -= lr d; clip (positions) to
 * [-1 + 1e-6, 1 - 1e-6].  No-op while *d_flag != 0 (non-finite gradient). */
#define FC2T2_OPT_SGD 0
#define FC2T2_OPT_ADAM 1
int fc2t2_opt_step(float* d_x, const float* d_grad, float* d_m, float* d_v, int64_t n,
                   int optimizer, float lr, int64_t t, float l1, int clip, const int32_t* d_flag,
                   void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FC2T2_B200_H */
