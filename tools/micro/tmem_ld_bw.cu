// Microbenchmark: tcgen05.ld read throughput per SM (accumulator drain rate), by number of
// reading warps and load shape. Not part of the product; used to size the scan epilogue.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_ld_bw tmem_ld_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int kShape>  // 0: 32x32b.x32, 1: 32x32b.x32.pack::16b, 2: 16x256b.x8, 3: 32x32b.x64
__global__ void k(int iters, uint32_t* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = (uint32_t)((i * 32 + (warp >> 2) * 64) & 511);
    uint32_t r[64];
    if (kShape == 0 || kShape == 1) {
      if (kShape == 0)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(base + col));
      else
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(base + (col & 255)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[j];
    } else if (kShape == 4 || kShape == 5) {
      const int nl = kShape == 4 ? 1 : 2;
      for (int h = 0; h < nl; ++h)
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[32*h+0]), "=r"(r[32*h+1]), "=r"(r[32*h+2]), "=r"(r[32*h+3]), "=r"(r[32*h+4]), "=r"(r[32*h+5]), "=r"(r[32*h+6]), "=r"(r[32*h+7]), "=r"(r[32*h+8]), "=r"(r[32*h+9]), "=r"(r[32*h+10]), "=r"(r[32*h+11]), "=r"(r[32*h+12]), "=r"(r[32*h+13]), "=r"(r[32*h+14]), "=r"(r[32*h+15]), "=r"(r[32*h+16]), "=r"(r[32*h+17]), "=r"(r[32*h+18]), "=r"(r[32*h+19]), "=r"(r[32*h+20]), "=r"(r[32*h+21]), "=r"(r[32*h+22]), "=r"(r[32*h+23]), "=r"(r[32*h+24]), "=r"(r[32*h+25]), "=r"(r[32*h+26]), "=r"(r[32*h+27]), "=r"(r[32*h+28]), "=r"(r[32*h+29]), "=r"(r[32*h+30]), "=r"(r[32*h+31])
            : "r"(base + ((col + 32 * h) & 511)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int h = 0; h < nl; ++h) {
        uint32_t m[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int j = 7; j >= 0; --j)
#pragma unroll
          for (int p = 0; p < 4; ++p) m[p] = __funnelshift_l(r[32 * h + 8 * p + j], m[p], 1);
        acc += ~(m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24));
      }
    } else if (kShape == 2) {
      asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(base + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= r[j];
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512) : "memory");
}

template <int S>
void run(int warps, const char* name) {
  const int iters = 4096, grid = 148;
  uint32_t* out = nullptr; long long* cyc = nullptr;
  cudaError_t e = cudaMalloc(&out, grid * 1024 * 4);
  if (e != cudaSuccess) { printf("malloc: %s\n", cudaGetErrorString(e)); return; }
  cudaMalloc(&cyc, grid * 8);
  printf("start %s %d\n", name, warps); fflush(stdout);
  k<S><<<grid, warps * 32>>>(iters, out, cyc);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<S><<<grid, warps * 32>>>(iters, out, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // bytes per SM: warps * iters * 32 lanes * 32 regs * 4 B (x32 loads; 16x256b.x8 = same)
  double bytes = (double)warps * iters * 32 * 32 * 4 * (S == 5 ? 2 : 1);
  printf("%-28s warps=%2d  %8.3f ms  %7.1f B/cyc/SM (clock64)  err=%s\n", name, warps, ms,
         bytes / (double)c, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) run<0>(w, "32x32b.x32");
  for (int w : {4, 8, 12, 16}) run<4>(w, "x32+mask");
  for (int w : {4, 8, 12, 16}) run<5>(w, "2x x32+mask");
  return 0;
}
