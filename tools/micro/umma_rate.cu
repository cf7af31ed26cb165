// Microbenchmark: tcgen05.mma kind::i8 issue-to-completion rate (M=128, N=256, K=32 per
// instruction, SW128 K-major operands in smem), to size the scan kernel's MMA stage.
#include <cstdio>
#include <cstdint>
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
// kind::f16 bf16 x bf16 -> f32: c_format=1 (f32) bits 4-5, a_format=1 (bf16) bits 7-9, b_format=1 bits 10-12
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int kKind, int N, int R>
__global__ void k(int iters, long long* cyc, volatile int* stop) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bars[2];
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x01010101u * (i & 7);
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
    const uint32_t idesc = kKind == 0 ? idesc_i8(128, N) : idesc_bf16(128, N);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t ad = sw128_desc(a + kk * 32), bd = sw128_desc(b + kk * 32);
        const uint32_t acc = kk > 0 ? 1u : 0u;
        const uint32_t d = slot;
        if (kKind == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
      }
      const int b = it & 1;
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bars[b])) : "memory");
      if (it >= 1) {  // wait for the previous commit (on the other barrier)
        const int pb = b ^ 1;
        const uint32_t par = (uint32_t)((it - 1) >> 1) & 1u;
        uint32_t ok = 0;
        do {
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bars[pb])), "r"(par) : "memory");
        } while (!ok);
      }
    }
    {
      const int b = (iters - 1) & 1;
      const uint32_t par = (uint32_t)((iters - 1) >> 1) & 1u;
      uint32_t ok = 0;
      do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(su32(&bars[b])), "r"(par) : "memory");
      } while (!ok);
    }
    cyc[blockIdx.x] = clock64() - t0;
    *stop = 1;
  } else if (threadIdx.x >= 32 && threadIdx.x < 32 * (1 + R)) {
    const int w = (threadIdx.x >> 5) - 1;
    const uint32_t base = slot + ((uint32_t)((w & 3) * 32) << 16) + 256u;  // other half
    uint32_t acc = 0;
    int n = 0;
    while (*stop == 0 && n < 1000000) {
      uint32_t r[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(base + (uint32_t)((n * 32) & 255)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 32; ++j) acc ^= r[j];
      ++n;
    }
    if (acc == 0x12345) cyc[1000] = n;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
}

template <int K, int N, int R>
void run(const char* name) {
  const int iters = 2000, grid = 148;
  long long* cyc = nullptr;
  cudaError_t e = cudaMalloc(&cyc, 2000 * 8);
  printf("malloc %s\n", cudaGetErrorString(e)); fflush(stdout);
  if (e != cudaSuccess) return;
  int* stop; cudaMalloc(&stop, 4); cudaMemset(stop, 0, 4);
  cudaFuncSetAttribute(k<K, N, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
  k<K, N, R><<<grid, 32 * (1 + R), 50 * 1024>>>(iters, cyc, stop);
  cudaDeviceSynchronize();
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("readers=%2d %-10s N=%3d: %7.1f cycles per MMA instruction (M=128, K=32B)  err=%s\n",
         R, name, N, (double)c / (iters * 4), cudaGetErrorString(cudaGetLastError()));
  fflush(stdout);
}
int main() {
  printf("start\n"); fflush(stdout);
  run<0, 256, 0>("kind::i8");
  run<0, 128, 0>("kind::i8");
  run<0, 64, 0>("kind::i8");
  run<0, 256, 4>("kind::i8");
  run<0, 256, 8>("kind::i8");
  run<0, 256, 16>("kind::i8");
  return 0;
}
