// Sustained dense int8 tensor-core throughput on the whole GPU (the roofline denominator for
// the tensor-bound configuration): 148 persistent CTAs, one thread each issuing
// tcgen05.mma.cta_group::1.kind::i8 (M=128, N=256, K=32 B per instruction, operands in smem,
// two TMEM accumulators alternating) back to back for ~0.5 s; wall time by CUDA events,
// clocks sampled by the caller (tools/micro/i8_peak.sh). Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_peak i8_peak.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  } while (!ok);
}

__global__ void k(int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[2];
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01030507u * (i & 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) {
    const uint32_t a = su32(base), b = su32(base + 16384);
    const uint32_t idesc = idesc_i8(128, 256);
    for (int it = 0; it < iters; ++it) {
      const int buf = it & 1;
      if (it >= 2) wait_bar(&bars[buf], (uint32_t)((it - 2) >> 1) & 1u);  // accumulator free
      const uint32_t d = slot + (uint32_t)(buf * 256);
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = sw128_desc(a + kk * 32), bd = sw128_desc(b + kk * 32);
        const uint32_t acc = kk > 0 ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[buf])) : "memory");
    }
    for (int it = iters - 2; it < iters; ++it)
      if (it >= 0) wait_bar(&bars[it & 1], (uint32_t)(it >> 1) & 1u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 1000000;
  int n_sm = 0;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  k<<<n_sm, 32, 50 * 1024>>>(1000);  // warm-up
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k<<<n_sm, 32, 50 * 1024>>>(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 128 * 256 * 128 * (double)iters * n_sm;  // 4 x K=32 B per iteration
    printf("{\"rep\": %d, \"sms\": %d, \"ms\": %.3f, \"int8_tops\": %.1f, \"err\": \"%s\"}\n", rep,
           n_sm, ms, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
  }
  return 0;
}
