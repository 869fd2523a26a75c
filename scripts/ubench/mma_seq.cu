// The M2L kernel's MMA sequence without barriers or data movement: per slot,
// 2 tiles x (main N=160 + cross N=80) kind::f16 MMAs, A descriptors shifted by
// the slot's window row offset (as in m2l_tc), B from a 9-slot stage.
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
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;" ::"r"(d), "l"(a), "l"(b), "r"(idesc));
}
constexpr int WROWS = 720, WZ = 10, WY = 18, W = 80;

template <int MODE>
__global__ void __launch_bounds__(128, 1) seq(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];   // window 2*2*720*16 = 46 KB + B 9*5 KB
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (46080 + 46080) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t IDM = (1u << 4) | ((uint32_t)(160 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t IDC = (1u << 4) | ((uint32_t)(80 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (warp == 0) {
    const uint64_t ahi = sdesc(smem_u32(smem), WROWS * 16, WZ * 16);
    const uint64_t alo = ahi + 2 * WROWS;
    const uint64_t b0 = sdesc(smem_u32(smem + 46080), 2 * W * 16, 128);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 9; ++j) {
        const int slot = (it % 3) * 9 + j;
        const uint64_t exk = (uint64_t)((slot / 9) * WY * WZ + ((slot / 3) % 3) * WZ + slot % 3);
        const uint64_t ex = MODE == 1 ? 0
                          : MODE == 3 ? (exk & ~7ull)                 // shifts rounded to 8 rows (128 B)
                          : MODE == 4 ? (uint64_t)(slot * 8)          // varying, 128-B aligned
                          : MODE == 5 ? (uint64_t)(slot % 3)          // z shifts only (0/16/32 B)
                          : MODE == 6 ? (uint64_t)((slot % 3) * 8)    // 3 aligned addresses
                          : exk;
        const uint64_t bd = b0 + (uint64_t)(j * 5120 / 16);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const uint64_t arow = ex + (uint64_t)(t * WY * WZ);
          const uint32_t dt = tmem + t * 240;
          if (elect_one()) mma(dt + W, ahi + arow, bd, IDM);
          if (MODE != 2 && elect_one()) mma(dt + W, alo + arow, bd + W, IDC);
        }
      }
    }
    if (elect_one()) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
    __syncwarp();
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)));
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int MODE>
void run(long long* d, const char* what, double floor_per_slot) {
  long long h[148];
  const int iters = 300;
  cudaFuncSetAttribute(seq<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) seq<MODE><<<148, 128, 100 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return; }
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < 148; ++i) s += h[i];
  printf("SEQ %-40s %.1f cycles per slot (2 tiles), model %.0f\n", what, s / 148 / iters / 9, floor_per_slot);
}

int main() {
  long long* d; cudaMalloc(&d, 148 * sizeof(long long));
  run<0>(d, "shifted A, main N160 + cross N80", 2 * (80 + 52));
  run<1>(d, "fixed A, main N160 + cross N80", 2 * (80 + 52));
  run<2>(d, "shifted A, main N160 only", 2 * 80);
  run<3>(d, "shifts rounded to 8 rows", 2 * (80 + 52));
  run<4>(d, "varying A, 128-B aligned (slot*8 rows)", 2 * (80 + 52));
  run<5>(d, "z shifts only (0/16/32 B)", 2 * (80 + 52));
  run<6>(d, "3 aligned addresses", 2 * (80 + 52));
  return 0;
}
