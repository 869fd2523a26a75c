// Standalone check of the CTA-pair (cta_group::2) primitives used by the
// M2L kernel: cluster launch, pair TMEM alloc, one M=256 kind::f16 MMA whose
// A rows come from each CTA's smem (128 each) and B from both CTAs (N/2 each,
// assumed), multicast commit to both CTAs' mbarriers, remote arrive, readback.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t mapa0(uint32_t a) { uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(a)); return r; }

constexpr int N = 64, K = 16;   // per MMA: M=256 (128 per CTA), N total, K=16 halves

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
pair_kernel(float* out, int mode) {
  __shared__ __align__(1024) uint16_t A[128 * K];      // [kc 2][row 128][8 halves]
  __shared__ __align__(1024) uint16_t B[N * K];        // [kc 2][row N][8 halves] (rows used: N/2)
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bar2;
  const uint32_t r = crank();
  const int warp = threadIdx.x >> 5;
  // A[m][k] = (r*128 + m) % 7 + 1 ; B[n][k] = (n + 1) (rank r holds n in [r*N/2, (r+1)*N/2) when split)
  for (int i = threadIdx.x; i < 128 * K; i += blockDim.x) {
    const int kc = i / (128 * 8), row = (i / 8) % 128;
    (void)kc;
    A[i] = __half_as_ushort(__float2half((float)((r * 128 + row) % 7 + 1)));
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int row = (i / 8) % N;
    // mode 0: each rank stores rows 0..N/2-1 = its half (global n = r*N/2 + row)
    const int n = mode == 0 ? r * (N / 2) + row : row;
    B[i] = __half_as_ushort(__float2half((float)(n + 1)));
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) printf("rank %u tmem %u\n", r, tmem);
  // both CTAs signal the leader's bar2 (remote arrive)
  if (threadIdx.x == 0) {
    const uint32_t rb = mapa0(smem_u32(&bar2));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
  }
  if (r == 0 && warp == 0) {
    // wait for both CTAs' data
    asm volatile("{\n.reg .pred p;\nW1: mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n@!p bra W1;\n}" ::"r"(smem_u32(&bar2)));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) {
      const uint64_t ad = sdesc(smem_u32(A), 128 * 16, 128);
      const uint64_t bd = sdesc(smem_u32(B), N * 16, 128);
      const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      asm volatile("tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, 0;" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc));
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
      printf("leader issued\n");
    }
    __syncwarp();
  }
  // every CTA: wait for its local bar (multicast commit), read its 128 rows
  asm volatile("{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int lane_q = warp;   // warp w reads lanes 32w..32w+31
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + ((uint32_t)(lane_q * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = r * 128 + threadIdx.x;
    for (int i = 0; i < 8; ++i) out[m * N + c0 + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  float* d; cudaMalloc(&d, 256 * N * sizeof(float));
  static float h[256 * N];
  for (int mode = 0; mode < 1; ++mode) {
    cudaMemset(d, 0, 256 * N * sizeof(float));
    pair_kernel<<<2, 128>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // expected with B split by N halves: D[m][n] = K * a(m) * (n+1)
    int bad = 0; double maxerr = 0;
    for (int m = 0; m < 256; ++m) for (int n = 0; n < N; ++n) {
      const double a = (m % 7) + 1, ex = K * a * (n + 1);
      const double err = fabs(h[m * N + n] - ex);
      if (err > 1e-3 * ex) { if (bad < 6) printf("  m %d n %d got %g expect %g\n", m, n, h[m * N + n], ex); ++bad; }
      maxerr = err > maxerr ? err : maxerr;
    }
    printf("mode %d: %d mismatches (B split by N across the pair%s)\n", mode, bad, bad ? " NOT confirmed" : " confirmed");
  }
  return 0;
}
