// Measured compute peaks on this B200 for the roofline denominators
// (FFMA and TF32 peaks were never measured).
//   FFMA : 8 independent FMA chains per thread, 1024 threads x 4 blocks/SM
//          (full occupancy), timed with CUDA events -> TFLOP/s (2 flop / FMA).
// The TF32 / bf16 tensor peaks are measured by scripts/ubench/peaks.py
// through cuBLAS (torch.matmul), the library figure MEASURED_PEAKS.json uses.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) ffma_peak(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678f) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  ffma_peak<<<blocks, threads>>>(out, 64, 0.999f, 1e-3f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    ffma_peak<<<blocks, threads>>>(out, iters, 0.999f, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fma = (double)blocks * threads * iters * 16 * 8;
  printf("{\"ffma_tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %d, \"ms\": %.3f, "
         "\"nominal_ffma_tflops_at_max_clock\": %.2f}\n",
         2 * fma / (best * 1e-3) / 1e12, sms, clk / 1000, best,
         2.0 * sms * 128 * (clk * 1e3) / 1e12);
  return 0;
}
