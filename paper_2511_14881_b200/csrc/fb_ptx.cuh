// Device helpers shared by the tcgen05 scan kernels (fb_tc_kernel.cu, fb_emit_kernel.cu):
// PTX wrappers for mbarriers, named barriers, TMA, tcgen05 MMA / TMEM loads and UMMA
// shared-memory descriptors, shared-memory accessors, and the small bit / gate helpers the
// scan epilogues use. All are sm_100a-only inline functions.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fb_internal.cuh"

namespace fb {
namespace dev {
namespace {

// CNF gate: accumulators armed by the tensor core. A CNF launch starts every accumulator at
// +127*D (D = the row's "gate digits", the sum of 32 int8 digits) with one extra K=32 MMA of
// the query's digit row by a constant tile of 127s, so the score gate (score >= tau, a
// superset test: the exact key test follows) is the accumulator's sign bit. |digits| <= 127
// bounds D to [-4096, 4064]: a gate below -127*4064 (and threshold 0) becomes "every score is
// a hit", one above 127*4096 is clamped (still a superset of score >= tau).
constexpr int32_t kGateDigitsMax = 4064;
constexpr int32_t kGateDigitsMin = -4096;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

// try_wait with a suspend-time hint: the warp is parked by the hardware until the phase
// completes (or the hint expires) instead of spinning through issue slots that the other
// roles on the same scheduler need.
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = su32(b);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(0x989680)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ void mbar_wait_idle(uint64_t* b, uint32_t parity) { mbar_wait(b, parity); }

// The same on 32-bit shared-window addresses (hot loops keep only these in registers).
__device__ __forceinline__ void mbar_wait_s(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(0x989680)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mbar_arrive_s(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_s(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Producers several stages ahead of their consumers: one try_wait, then test_wait polls
// spaced by __nanosleep, so a producer blocked on a full ring gives its issue slots to the
// warps sharing its scheduler (a spinning try_wait loop does not).
#ifndef FB_BACKOFF
#define FB_BACKOFF 0
#endif
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* b, uint32_t parity) {
#if FB_BACKOFF == 1
  mbar_wait(b, parity);
  return;
#endif
  const uint32_t a = su32(b);
  uint32_t ok = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  while (!ok) {
    __nanosleep(FB_BACKOFF == 2 ? 1000 : 128);
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// Wait for a phase with a sleep between polls: for warps that run ahead of the pipeline
// (producers, builders), whose polling would otherwise take issue slots from the warps on
// the critical path of the same sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, uint32_t ns) {
  while (!mbar_test(b, parity)) __nanosleep(ns);
}

// Hardware named barriers for warp-to-warp stage handoffs (the waiting warps block in the
// barrier unit instead of polling an mbarrier): the producing warps bar.arrive on a stage's
// "full" barrier and the consumers bar.sync on it; "empty" runs the other way.
__device__ __forceinline__ void nb_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void nb_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void tma_load_2d_s(uint32_t dst, const CUtensorMap* map, int32_t c0,
                                              int32_t c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void umma_commit_s(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

// L2 prefetch of a TMA tile / of a byte range (no shared-memory destination): keeps HBM
// streaming ahead of the shared-memory stages the latency-bandwidth product would need.
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   su32(bar))
               : "memory");
}

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Asynchronous variant: issue the load now, tmem_wait32() before the first use. The wait
// names the destination registers so the compiler cannot read them ahead of it.
__device__ __forceinline__ void tmem_ld32_async(uint32_t taddr, int32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait32(int32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]),
                 "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
                 "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// 32 lanes x 32 columns <- v (every register the same value)
__device__ __forceinline__ void tmem_st32_const(uint32_t taddr, int32_t v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(v)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// one accumulator (this lane's row, column taddr) -> register
__device__ __forceinline__ int32_t tmem_ld1(uint32_t taddr) {
  int32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v) : : "memory");
  return v;
}

// K-major, SWIZZLE_128B shared-memory matrix descriptor (8-row groups 1024 B apart).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;        // SBO: 8 rows x 128 B
  d |= (uint64_t)1 << 46;                  // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;                  // SWIZZLE_128B
  return d;
}

// K-major, no-swizzle ("interleaved") smem descriptor: 8-row x 16-byte core matrices, the
// two 16-byte K halves LBO apart, 8-row groups SBO apart.
__device__ __forceinline__ uint64_t plain_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell); layout type 0 = SWIZZLE_NONE
  return d;
}

// kind::i8 instruction descriptor: s32 accumulate, s8 x s8, both K-major, M = 128, N = 256
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// ``prog`` holds n_ops (a multiple of 8) ops, 16-byte aligned (shared or global memory).
// Ops are fetched 8 at a time and the 8 leaf masks (2 words = 128 items each) are loaded
// before any is applied, so the memory latency is paid once per batch. The stack lives in
// registers.
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint2 lds64v(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}

__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t v;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(v));
  return v;
}

// ---- CNF mode helpers ---------------------------------------------------------------
// One exchange round of a warp-wide 32x32 bit transpose for a lane whose partner is
// lane ^ s: the lane keeps the bits under its keep-mask and takes the partner's word rotated
// by its lane rotation (s for the lower lane, 32 - s for the upper one) under the rest; the
// wrapped-around bits of the rotation fall outside the taken mask. SHFL + SHF + LOP3.
__device__ __forceinline__ uint32_t transpose_round(uint32_t w, int s, uint32_t keep, uint32_t rot) {
  const uint32_t y = __shfl_xor_sync(0xffffffffu, w, s);
  const uint32_t r = __funnelshift_l(y, y, rot);
  return (w & keep) | (r & ~keep);
}

// 32x32 bit-matrix transpose across a warp: lane j holds row j on entry (bit i = (j, i)),
// column j on exit (bit i = (i, j)).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int s = 16 >> k;
    const uint32_t m = masks[k];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, s);
    x = (lane & s) ? ((x & ~m) | ((y & ~m) >> s)) : ((x & m) | ((y & m) << s));
  }
  return x;
}

// Bit j = (r[j] >= 0), i.e. the sign bits of 32 accumulators pre-loaded with -tau
// (one funnel shift per score, four independent 8-bit chains).
__device__ __forceinline__ uint32_t nonneg_mask32(const int32_t (&r)[32]) {
  uint32_t m[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int j = 7; j >= 0; --j) {
#pragma unroll
    for (int p = 0; p < 4; ++p) m[p] = __funnelshift_l((uint32_t)r[8 * p + j], m[p], 1);
  }
  return ~(m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24));
}

// Bit j of the result = (r[j] >= tau), for |r| < 2^22 and tau clamped to [-2^23, 2^23]:
// the sign of (tau - 1 - r[j]) is shifted in with a funnel shift (2 instructions per
// score), in four independent 8-bit chains.
__device__ __forceinline__ uint32_t hit_mask32(const int32_t (&r)[32], int32_t tau) {
  const int32_t ntau = -tau;  // sign of r + ntau marks a miss
  uint32_t m[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int j = 7; j >= 0; --j) {
#pragma unroll
    for (int p = 0; p < 4; ++p) m[p] = __funnelshift_l((uint32_t)(r[8 * p + j] + ntau), m[p], 1);
  }
  return ~(m[0] | (m[1] << 8) | (m[2] << 16) | (m[3] << 24));
}

__device__ __forceinline__ uint64_t word_range_mask(int64_t word_slot, int64_t s0, int64_t s1) {
  const int64_t lo = s0 > word_slot ? s0 - word_slot : 0;
  const int64_t hi = s1 - word_slot < 64 ? s1 - word_slot : 64;
  if (hi <= lo) return 0ull;
  const uint64_t upto = hi >= 64 ? ~0ull : ((1ull << hi) - 1);
  return upto & ~((1ull << lo) - 1);
}

__host__ __device__ __forceinline__ int32_t floordiv127(int32_t a) {
  const int32_t q = a / 127;
  return (a % 127 != 0 && a < 0) ? q - 1 : q;
}

// gate digits of a row from its key threshold T (T == 0: no threshold -> all hits)
__device__ __forceinline__ int32_t gate_digits(uint64_t T, bool& all) {
  all = false;
  if (T == 0ull) {
    all = true;
    return 0;
  }
  const int32_t D = -floordiv127(key_score(T));  // 127 D >= -tau
  if (D > kGateDigitsMax) {
    all = true;
    return 0;
  }
  return D < kGateDigitsMin ? kGateDigitsMin : D;
}

// byte offset of (row, k) in the no-swizzle gate tiles (LBO = 128, SBO = 256)
__host__ __device__ __forceinline__ uint32_t gate_off(int row, int k) {
  return (uint32_t)((row >> 3) * 256 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

// Exact int32 dot of a query row (A tile) and an item row (B stage) from shared memory.
// Both tiles use the SWIZZLE_128B layout: 16-byte chunk c of row r sits at c ^ (r & 7).
__device__ __forceinline__ int32_t smem_dot(uint32_t a_row, uint32_t a_sw, uint32_t b_row,
                                            uint32_t b_sw) {
  int32_t acc0 = 0, acc1 = 0;
#pragma unroll
  for (uint32_t c = 0; c < 8; c += 2) {
    const uint4 x0 = lds128(a_row + ((c ^ a_sw) << 4));
    const uint4 y0 = lds128(b_row + ((c ^ b_sw) << 4));
    const uint4 x1 = lds128(a_row + (((c + 1) ^ a_sw) << 4));
    const uint4 y1 = lds128(b_row + (((c + 1) ^ b_sw) << 4));
    acc0 = __dp4a((int)x0.x, (int)y0.x, acc0);
    acc1 = __dp4a((int)x1.x, (int)y1.x, acc1);
    acc0 = __dp4a((int)x0.y, (int)y0.y, acc0);
    acc1 = __dp4a((int)x1.y, (int)y1.y, acc1);
    acc0 = __dp4a((int)x0.z, (int)y0.z, acc0);
    acc1 = __dp4a((int)x1.z, (int)y1.z, acc1);
    acc0 = __dp4a((int)x0.w, (int)y0.w, acc0);
    acc1 = __dp4a((int)x1.w, (int)y1.w, acc1);
  }
  return acc0 + acc1;
}

// CNF filter test of one (query, item) pair: every one of the query's OR-groups shares a
// literal column with the item's column bits. Window form (<= 4 groups, each group's
// columns inside one aligned u32 pair): per group a byte offset into the item row and a
// 64-bit mask, all in registers; unused groups repeat group 0.
__device__ __forceinline__ bool cnf_test_win(uint32_t row, const uint32_t (&wo)[4],
                                             const uint32_t (&lo)[4], const uint32_t (&hi)[4]) {
  uint32_t x[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const uint2 t = lds64v(row + wo[g]);
    x[g] = (t.x & lo[g]) | (t.y & hi[g]);
  }
  return min(min(x[0], x[1]), min(x[2], x[3])) != 0u;
}

}  // namespace
}  // namespace dev
}  // namespace fb
