// extern "C" entry points of the training glue (include/fc2t2_b200.h,
// "training"): losses + tangents and the optimizer step of the reference
// trainer (trainer.py:70-152), see train.cu.
#include <cmath>

#include "../../include/fc2t2_b200.h"
#include "common.cuh"
#include "kernels.cuh"

extern "C" const char* fc2t2_ray_last_error(void);

namespace {
int tstatus(cudaError_t e) { return e == cudaSuccess ? FC2T2_OK : FC2T2_ECUDA; }
}  // namespace

extern "C" {

size_t fc2t2_loss_workspace_size(int64_t n, int cols) {
  return n < 0 || cols < 1 ? 0 : fc2t2::loss_workspace_bytes(n, cols);
}

int fc2t2_loss(const float* d_pred, const float* d_target, const uint8_t* d_mask, int64_t n,
               int cols, float bias, int kind, float* d_tangent, double* d_stats, void* d_ws,
               size_t ws_bytes, void* stream) {
  if (n < 0 || cols < 1 || (kind != FC2T2_LOSS_MAE && kind != FC2T2_LOSS_MSE))
    return FC2T2_EVALUE;
  if (ws_bytes < fc2t2::loss_workspace_bytes(n, cols)) return FC2T2_EWORKSPACE;
  return tstatus(fc2t2::loss_tangent(d_pred, d_target, d_mask, n, cols, bias,
                                     kind == FC2T2_LOSS_MSE ? 1 : 0, d_tangent, d_stats, d_ws,
                                     (cudaStream_t)stream));
}

int fc2t2_nonfinite(const float* d_x, int64_t n, int32_t* d_flag, void* stream) {
  if (n < 0) return FC2T2_EVALUE;
  return tstatus(fc2t2::nonfinite(d_x, n, d_flag, (cudaStream_t)stream));
}

int fc2t2_opt_step(float* d_x, const float* d_grad, float* d_m, float* d_v, int64_t n,
                   int optimizer, float lr, int64_t t, float l1, int clip, const int32_t* d_flag,
                   void* stream) {
  if (n < 0 || t < 1 || (optimizer != FC2T2_OPT_SGD && optimizer != FC2T2_OPT_ADAM))
    return FC2T2_EVALUE;
  const bool adam = optimizer == FC2T2_OPT_ADAM;
  if (adam && (!d_m || !d_v)) return FC2T2_EVALUE;
  const float c1 = (float)(1.0 - std::pow(0.9, (double)t));
  const float c2 = (float)(1.0 - std::pow(0.999, (double)t));
  return tstatus(fc2t2::opt_step(d_x, d_grad, d_m, d_v, n, adam ? 1 : 0, lr, c1, c2, l1, clip,
                                 d_flag, (cudaStream_t)stream));
}

}  // extern "C"
