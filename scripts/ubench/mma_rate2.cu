// Microbenchmark 2: cycles per tcgen05.mma (cta_group::1, M = 128, kind::tf32,
// SS operands) for three issue styles:
//   0  one divergent thread runs the loop
//   1  whole warp runs the loop, CUTLASS style `if (elect_one) mma` per MMA
//   2  whole warp, elect once, all MMAs of an unrolled group under one branch
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
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P1;\n\telect.sync _|P1, 0xffffffff;\n\tselp.b32 %0, 1, 0, P1;\n\t}\n" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int MODE, int W = 1>
__global__ void __launch_bounds__(128, 1) mma_rate(int n, int iters, long long* out,
                                                   int a_off = 0, int a_sbo = 128) {
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
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t ad = sdesc(smem_u32(smem) + a_off, 128 * 16 * 2, a_sbo);
  const uint64_t bd = sdesc(smem_u32(smem + 40000), 256 * 16, 128);
  const uint32_t stride = (uint32_t)((512 / 4) & ~7);
  if (MODE == 0 ? threadIdx.x == 0 : warp < W) {
    const uint32_t tm = tmem + (uint32_t)(warp * (512 / W));
    long long t0 = clock64();
    for (int i = 0; i < iters; i += 4) {
      const uint32_t acc = i > 0;
      if (MODE == 0) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mma(tm + u * (stride / W), ad + u, bd + u, idesc, acc);
      } else if (MODE == 1) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (elect_one()) mma(tm + u * (stride / W), ad + u, bd + u, idesc, acc);
      } else {
        if (elect_one()) {
#pragma unroll
          for (int u = 0; u < 4; ++u) mma(tm + u * (stride / W), ad + u, bd + u, idesc, acc);
        }
        __syncwarp();
      }
    }
    if (W > 1) asm volatile("bar.sync 1, %0;" :: "r"(32 * W));
    if ((MODE == 0 || elect_one()) && warp == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    if (MODE != 0) __syncwarp();
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}


// Kernel-like issue pattern: stages of 9 offsets; per offset an smem entry
// (row shift), 2 tiles x (N = 96 main + N = 48 cross) MMAs.
template <int MODE>
__global__ void __launch_bounds__(128, 1) mma_pattern(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int2 sent[32];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x < 32) sent[threadIdx.x] = make_int2((threadIdx.x * 7) % 27, threadIdx.x);
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
  const uint32_t id1 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(48 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t id2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t wd = sdesc(smem_u32(smem), 540 * 16, 160);
  const uint64_t bdesc0 = sdesc(smem_u32(smem + 40000), 96 * 16, 128);
  if (MODE == 3 || warp == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE == 3) {
        if (elect_one()) {
          for (int jj = 0; jj < 9; ++jj) {
            const int ex = sent[jj + (it & 15)].x;
            const uint64_t bd = bdesc0 + (uint64_t)((jj * 3072) >> 4);
            const uint32_t acc_in = (it == 0 && jj == 0) ? 0u : 1u;
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              mma(tmem + t * 128, wd + (uint64_t)((t * 4 + 0) * 540 + ex), bd, id2, acc_in);
              mma(tmem + t * 128 + 48, wd + (uint64_t)((t * 4 + 2) * 540 + ex), bd, id1, 1u);
            }
          }
        }
        __syncwarp();
      } else {
        for (int jj = 0; jj < 9; ++jj) {
          const int ex = sent[jj + (it & 15)].x;
          const uint64_t bd = bdesc0 + (uint64_t)((jj * 3072) >> 4);
          const uint32_t acc_in = (it == 0 && jj == 0) ? 0u : 1u;
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (elect_one()) mma(tmem + t * 128, wd + (uint64_t)((t * 4 + 0) * 540 + ex), bd, id2, acc_in);
            if (elect_one()) mma(tmem + t * 128 + 48, wd + (uint64_t)((t * 4 + 2) * 540 + ex), bd, id1, 1u);
          }
        }
      }
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar)) : "memory");
    __syncwarp();
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int MODE>
void runp(long long* d) {
  long long h[148];
  const int iters = 512;
  cudaFuncSetAttribute(mma_pattern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) mma_pattern<MODE><<<148, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); fflush(stdout); return; }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("PATTERN mode=%d : %.1f cyc per offset (2 tiles x [N96 + N48]; tight-loop estimate 200)\n", MODE, s / 148 / iters / 9);
  fflush(stdout);
}

template <int MODE, int W = 1>
void run(int n, long long* d, int a_off = 0, int a_sbo = 128) {
  long long h[148];
  const int iters = 4096;
  cudaFuncSetAttribute(mma_rate<MODE, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) mma_rate<MODE, W><<<148, 128, 100 * 1024>>>(n, iters, d, a_off, a_sbo);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); fflush(stdout); return; }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("MMA mode=%d warps=%d N=%3d a_off=%d a_sbo=%d : %.1f cyc/mma total (floor %d)\n", MODE, W, n, a_off, a_sbo, s / 148 / iters / W, 128 * n / 256);
  fflush(stdout);
}

int main() {
  long long* d; cudaMalloc(&d, 148 * sizeof(long long));
  for (int n : {80, 160}) {
    run<1, 1>(n, d, 0, 128);     // aligned, contiguous groups
    run<1, 1>(n, d, 0, 256);     // aligned groups, 256 B stride
    run<1, 1>(n, d, 0, 160);     // the window's 160 B group stride
    run<1, 1>(n, d, 16, 160);    // + 16 B shift
    run<1, 1>(n, d, 32, 160);
    run<1, 1>(n, d, 16, 128);    // misaligned by 16 B, contiguous
  }
  return 0;
}
