// Microbenchmark: cycles per tcgen05.mma (cta_group::1, M = 128, SS operands,
// SWIZZLE_NONE K-major) as a function of N, kind (tf32 / f16) and the number
// of independent TMEM accumulators the MMAs rotate over.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

template <int KIND, bool UNIFORM>
__global__ void __launch_bounds__(128, 1) mma_rate(int n, int nacc, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  // f16: a/b format 0 (f16), K = 16 (32 B per row); tf32: format 2, K = 8.
  const uint32_t fmt = KIND == 0 ? 2u : 0u;
  const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t ad = sdesc(smem_u32(smem), 128 * 16, 128);
  const uint64_t bd = sdesc(smem_u32(smem + 32768), 256 * 16, 128);
  long long t0 = 0, t1 = 0;
  if (UNIFORM ? warp == 0 : threadIdx.x == 0) {
    uint32_t leader = 1;
    if (UNIFORM)
      asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n" : "=r"(leader));
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tmem + (uint32_t)((i % nacc) * ((512 / nacc) & ~7));
      if (KIND == 0)
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 e, %5, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(i >= nacc ? 1 : 0), "r"(leader));
      else
        asm volatile("{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 e, %5, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(i >= nacc ? 1 : 0), "r"(leader));
    }
    if (leader) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    if (UNIFORM) __syncwarp();
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(smem_u32(&bar)));
    t1 = clock64();
    if (leader) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

int main() {
  long long* d; cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  cudaFuncSetAttribute(mma_rate<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(mma_rate<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(mma_rate<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(mma_rate<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const int iters = 4096;
  for (int uni = 0; uni < 2; ++uni)
  for (int kind = 0; kind < 2; ++kind)
    for (int nacc : {1, 4})
      for (int n : {16, 32, 48, 64, 96, 128, 256}) {
        if (n * nacc > 512) continue;
        for (int rep = 0; rep < 2; ++rep) {
          if (uni) {
            if (kind == 0) mma_rate<0, true><<<148, 128, 64 * 1024>>>(n, nacc, iters, d);
            else mma_rate<1, true><<<148, 128, 64 * 1024>>>(n, nacc, iters, d);
          } else {
            if (kind == 0) mma_rate<0, false><<<148, 128, 64 * 1024>>>(n, nacc, iters, d);
            else mma_rate<1, false><<<148, 128, 64 * 1024>>>(n, nacc, iters, d);
          }
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
        printf("MMA %s kind=%s nacc=%d N=%3d : %.1f cyc/mma (floor %d)\n", uni ? "uniform  " : "divergent", kind ? "f16 " : "tf32", nacc, n,
               s / 148 / iters, 128 * n / 256);
        fflush(stdout);
      }
  return 0;
}
