// extern "C" entry points of the ray layers (include/fc2t2_b200.h, "rays").
#include <string>

#include "../../include/fc2t2_b200.h"
#include "common.cuh"
#include "kernels.cuh"

namespace {
thread_local std::string g_ray_error;
int rfail(int code, const char* msg) {
  g_ray_error = msg;
  return code;
}
int rstatus(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return FC2T2_OK;
  g_ray_error = std::string(where) + ": " + cudaGetErrorString(e);
  return FC2T2_ECUDA;
}
bool bad_level(int level) { return level < 2 || level > 8; }
}  // namespace

extern "C" {

const char* fc2t2_ray_last_error(void) { return g_ray_error.c_str(); }

size_t fc2t2_scan_workspace_size(int64_t n) {
  return (fc2t2::scan_ws_words(n) + 4) * sizeof(uint32_t);
}

int fc2t2_scan_u32(const uint32_t* d_in, uint32_t* d_out, int64_t n, void* d_ws, size_t ws_bytes,
                   void* stream) {
  if (ws_bytes < fc2t2_scan_workspace_size(n)) return rfail(FC2T2_EWORKSPACE, "scan workspace");
  return rstatus(fc2t2::exclusive_scan(d_in, d_out, n, (uint32_t*)d_ws, (cudaStream_t)stream),
                 "scan");
}

int fc2t2_traverse_count(int level, const double* d_org, const double* d_dir, int64_t R,
                         uint32_t* d_counts, void* stream) {
  if (bad_level(level) || R < 0) return rfail(FC2T2_EVALUE, "bad traverse arguments");
  return rstatus(fc2t2::traverse_count(level, d_org, d_dir, R, d_counts, (cudaStream_t)stream),
                 "traverse_count");
}

int fc2t2_traverse_fill(int level, const double* d_org, const double* d_dir, int64_t R,
                        const uint32_t* d_offsets, int32_t* d_ray_id, double* d_t0, double* d_t1,
                        int32_t* d_box, void* stream) {
  if (bad_level(level) || R < 0) return rfail(FC2T2_EVALUE, "bad traverse arguments");
  return rstatus(fc2t2::traverse_fill(level, d_org, d_dir, R, d_offsets, d_ray_id, d_t0, d_t1,
                                      d_box, (cudaStream_t)stream),
                 "traverse_fill");
}

int fc2t2_depth_forward(int rho, int level, const float* d_l, const double* d_org,
                        const double* d_dir, int64_t R, double bias, double* d_lengths,
                        uint8_t* d_hit, double* d_points, float* d_grads, float* d_hess,
                        float* d_denom, void* stream) {
  if (rho < 1 || rho > 4) return rfail(FC2T2_EORDER, "root layers need rho <= 4");
  if (bad_level(level) || R < 0) return rfail(FC2T2_EVALUE, "bad depth arguments");
  return rstatus(fc2t2::depth_walk(rho, level, d_l, d_org, d_dir, R, bias, d_lengths, d_hit,
                                   d_points, d_grads, d_hess, d_denom, (cudaStream_t)stream),
                 "depth_forward");
}

int fc2t2_root_payload(int rho, int level, const double* d_dir, int64_t R, const uint8_t* d_hit,
                       const double* d_points, const float* d_grads, const float* d_hess,
                       const float* d_denom, const float* d_y_len, const float* d_y_grad,
                       uint32_t* d_keys, float* d_payload, int32_t* d_n_clamped, void* stream) {
  if (rho < 1 || rho > 6) return rfail(FC2T2_EORDER, "bad rho");
  if (d_y_grad && !d_hess) return rfail(FC2T2_EVALUE, "surface payload needs the Hessians");
  return rstatus(fc2t2::root_payload(rho, level, d_dir, R, d_hit, d_points, d_grads, d_hess,
                                     d_denom, d_y_len, d_y_grad, d_keys, d_payload, d_n_clamped,
                                     (cudaStream_t)stream),
                 "root_payload");
}

int fc2t2_line_integral(int rho, int level, int channels, const float* d_l, const double* d_org,
                        const double* d_dir, int64_t R, float* d_values, void* stream) {
  if (rho < 1 || rho > 6 || channels < 1) return rfail(FC2T2_EVALUE, "bad line_integral args");
  return rstatus(fc2t2::line_integral(rho, level, channels, d_l, d_org, d_dir, R, d_values,
                                      (cudaStream_t)stream),
                 "line_integral");
}

int fc2t2_line_payload(int rho, int level, int channels, const double* d_org, const double* d_dir,
                       int64_t R, const uint32_t* d_offsets, const float* d_y,
                       const double* d_gl_x, const double* d_gl_w, int G, uint32_t* d_keys,
                       float* d_payload, void* stream) {
  if (rho < 1 || rho > 6 || channels < 1 || G < 1) return rfail(FC2T2_EVALUE, "bad line_payload");
  return rstatus(fc2t2::line_payload(rho, level, channels, d_org, d_dir, R, d_offsets, d_y, d_gl_x,
                                     d_gl_w, G, d_keys, d_payload, (cudaStream_t)stream),
                 "line_payload");
}

size_t fc2t2_key_sort_workspace_size(int level, int64_t n) {
  return fc2t2::key_sort_workspace(level, n);
}

int fc2t2_key_sort(int level, const uint32_t* d_keys, int64_t n, int32_t* d_order,
                   int32_t* d_cell_start, void* d_ws, size_t ws_bytes, void* stream) {
  if (bad_level(level) || n < 0 || n > INT32_MAX) return rfail(FC2T2_EVALUE, "bad key_sort args");
  if (ws_bytes < fc2t2::key_sort_workspace(level, n))
    return rfail(FC2T2_EWORKSPACE, "key_sort workspace too small");
  return rstatus(fc2t2::key_sort(level, d_keys, n, d_order, d_cell_start, d_ws, ws_bytes,
                                 (cudaStream_t)stream),
                 "key_sort");
}

int fc2t2_insert(int rho, int level, int channels, const float* d_payload, const int32_t* d_order,
                 const int32_t* d_cell_start, float* d_m, void* stream) {
  if (rho < 1 || rho > 6 || channels < 1) return rfail(FC2T2_EVALUE, "bad insert args");
  return rstatus(fc2t2::insert_sorted(rho, level, channels, d_payload, d_order, d_cell_start, d_m,
                                      (cudaStream_t)stream),
                 "insert");
}

int fc2t2_vol_gauss_nodes(int rho) { return fc2t2::vol_gauss_nodes(rho); }

int fc2t2_vol_record_floats(int colors) { return fc2t2::vol_record_floats(colors); }

int fc2t2_vol_insert(int rho, int level, int colors, const float* d_rec, const int32_t* d_order,
                     const int32_t* d_cell_start, float* d_m, void* stream) {
  if (rho != 4) return rfail(FC2T2_EORDER, "the radiance layer is built for rho = 4");
  if (colors < 1 || colors > 4) return rfail(FC2T2_EVALUE, "1..4 colour channels supported");
  return rstatus(fc2t2::vol_insert(rho, level, colors, d_rec, d_order, d_cell_start, d_m,
                                   (cudaStream_t)stream),
                 "vol_insert");
}

int fc2t2_vol_forward(int rho, int level, int colors, const float* d_l, const double* d_org,
                      const double* d_dir, int64_t R, const double* d_efit, const double* d_bg,
                      float* d_rgb, double* d_depth_final, const uint32_t* d_seg_offsets,
                      uint8_t* d_seg_alive, void* stream) {
  if (rho != 4) return rfail(FC2T2_EORDER, "the radiance layer is built for rho = 4");
  if (colors < 1 || colors > 4) return rfail(FC2T2_EVALUE, "1..4 colour channels supported");
  return rstatus(fc2t2::vol_forward(rho, level, colors, d_l, d_org, d_dir, R, d_efit, d_bg, d_rgb,
                                    d_depth_final, d_seg_offsets, d_seg_alive,
                                    (cudaStream_t)stream),
                 "vol_forward");
}

int fc2t2_vol_forward_ex(int rho, int level, int colors, const float* d_l, const double* d_org,
                         const double* d_dir, int64_t R, const double* d_efit, const double* d_bg,
                         float* d_rgb, double* d_depth_final, uint32_t* d_n_alive,
                         double* d_totals, void* stream) {
  if (rho != 4) return rfail(FC2T2_EORDER, "the radiance layer is built for rho = 4");
  if (colors < 1 || colors > 4) return rfail(FC2T2_EVALUE, "1..4 colour channels supported");
  if (!d_n_alive || !d_totals) return rfail(FC2T2_EVALUE, "vol_forward_ex needs n_alive and totals");
  return rstatus(fc2t2::vol_forward(rho, level, colors, d_l, d_org, d_dir, R, d_efit, d_bg, d_rgb,
                                    d_depth_final, nullptr, nullptr, (cudaStream_t)stream,
                                    d_n_alive, d_totals),
                 "vol_forward_ex");
}

int fc2t2_vol_totals(int rho, int level, int colors, const float* d_l, const double* d_org,
                     const double* d_dir, int64_t R, const double* d_efit, uint32_t* d_n_alive,
                     double* d_totals, double* d_depth_final, void* stream) {
  if (rho != 4) return rfail(FC2T2_EORDER, "the radiance layer is built for rho = 4");
  if (colors < 1 || colors > 4) return rfail(FC2T2_EVALUE, "1..4 colour channels supported");
  return rstatus(fc2t2::vol_totals(rho, level, colors, d_l, d_org, d_dir, R, d_efit, d_n_alive,
                                   d_totals, d_depth_final, (cudaStream_t)stream),
                 "vol_totals");
}

int fc2t2_vol_payload(int rho, int level, int colors, const float* d_l, const double* d_org,
                      const double* d_dir, int64_t R, const double* d_efit, const double* d_bg,
                      const float* d_ybar, const uint32_t* d_alive_offsets,
                      const double* d_totals, const double* d_depth_final, const double* d_gl_x,
                      const double* d_gl_w, uint32_t* d_keys, float* d_payload, void* stream) {
  if (rho != 4) return rfail(FC2T2_EORDER, "the radiance layer is built for rho = 4");
  if (colors < 1 || colors > 4) return rfail(FC2T2_EVALUE, "1..4 colour channels supported");
  return rstatus(fc2t2::vol_payload(rho, level, colors, d_l, d_org, d_dir, R, d_efit, d_bg,
                                    d_ybar, d_alive_offsets, d_totals, d_depth_final, d_gl_x,
                                    d_gl_w, d_keys, d_payload, (cudaStream_t)stream),
                 "vol_payload");
}

}  // extern "C"
