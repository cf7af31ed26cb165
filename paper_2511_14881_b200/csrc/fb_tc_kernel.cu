// Fused Bloom-filter + int8 scan emit kernel on the 5th-gen tensor cores (sm_100a).
//
// One persistent CTA per SM walks 256-item tiles (4 validity/plane words). Per tile:
//   warp 0      TMA-loads the 256 x 128 B item rows (SWIZZLE_128B) and bulk-copies the
//               batch's referenced Bloom plane words (32 B per plane) into shared memory;
//   warp 1      issues tcgen05.mma.kind::i8 (M = 128 queries, N = 256 items, K = 4 x 32)
//               into a double-buffered int32 accumulator in TMEM (2 x 256 columns);
//   warps 2-3   AND each distinct leaf's planes into per-tile leaf masks (the paper's
//               and.b64 Bloom test, 64 items per op);
//   warps 4-11  read the scores back with tcgen05.ld (thread = query, 128 items), gate
//               on the query's running key threshold, evaluate the query's filter
//               program only where some score clears the gate, and append surviving
//               (key, slot) candidates -- filtered-out items never leave the SM.
// Semantics are those of reference ivf.search_clusters (ivf.py:285-334) restricted by
// filter_query.eval_compiled (filter_query.py:314-356): eligible = valid & range & mask &
// program; score = exact int32 dot; candidates = eligible with key >= threshold.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "fb_internal.cuh"

#include <algorithm>

namespace fb {
namespace {

constexpr int kTileItems = 256;
constexpr int kTileWords = 4;
constexpr int kBlockM = 128;
constexpr int kMaxMBlocks = 2;
constexpr int kMaxQueries = kBlockM * kMaxMBlocks;
constexpr int kKBytes = 128;
constexpr int kUmmaK = 32;
constexpr int kAccCols = 256;
constexpr int kThreads = 384;
constexpr int kLeafThreads = 64;
constexpr int kEpiWarp0 = 4;   // warps 4-11: epilogue (thread = query x 128 items)
constexpr int kEpiWarps = 8;
// CNF mode: 16 warps, 12 of them epilogue (3 per TMEM lane quadrant, chunks interleaved)
constexpr int kThreadsCnf = 512;
constexpr int kEpiWarpsCnf = 12;
constexpr int kLeafStride = 6;  // u64 per leaf in the per-tile leaf-mask stage (48 B: 4 words +
                                // pad, so 32 lanes' 16-B loads spread over 8 bank groups)
constexpr int kRegStack = 4;
constexpr uint32_t kItemBytes = kTileItems * kKBytes;  // 32 KB

struct TcArgs {
  const int8_t* queries;
  int32_t nq;
  int32_t n_mblk;
  const uint64_t* planes;
  const uint64_t* valid;
  const uint32_t* id_rank;
  const uint64_t* masks;
  int64_t n_words;
  int32_t has_prog;
  int32_t n_planes;
  int32_t n_leaves;
  int32_t k_max;
  const int16_t* plane_list;
  const int16_t* leaf_slot;
  const int32_t* rop_offset;
  const uint16_t* rops;
  const int2* work;
  int64_t n_sel;
  int64_t work_stride;
  const int64_t* ranges;
  const uint64_t* threshold;
  uint64_t* out_key;
  uint32_t* out_slot;
  uint32_t* out_cnt;
  int32_t cap;
  int32_t* dump;
  int64_t dump_ld;
  int32_t item_stages;
  int32_t plane_stages;
  int32_t rops_cap;  // ops of this launch's programs that fit the shared-memory stage
  // CNF mode
  int32_t n_cols;
  int32_t cnf_words;
  int32_t cnf_gmax;
  int32_t qm_stride;  // u32 per (query, group) in shared memory: 4 or 8
  const int16_t* col_leaf;
  const uint32_t* qmask;
  const int32_t* qgroups;
  uint32_t off_a, off_b, off_p, off_l, off_ls, off_thr, off_r, off_bar, plane_stage_bytes,
      leaf_stage_bytes, off_qm, off_qg, off_hit, off_id;
};

constexpr int kTbStride = 8;     // u32 per item row of the transposed column bits (<= 256 cols)
constexpr int kHitCap = 128;     // per-warp ring buffer of hits (score >= threshold)

// ---- PTX helpers ----------------------------------------------------------------------
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
// completes (or the hint expires) instead of spinning through issue slots that the
// epilogue warps on the same scheduler need.
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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
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
// Score gate of a query row from its key threshold, clamped so score - tau cannot
// overflow (|score| < 2^22 at dim 128); rows past the batch get an unreachable gate.
__device__ __forceinline__ int32_t gate_tau(const uint64_t* sT, int q, int nq) {
  const uint64_t T = q < nq ? sT[q] : ~0ull;
  const int32_t t = T == 0ull ? -(1 << 23) : key_score(T);
  return min(max(t, -(1 << 23)), 1 << 23);
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

// kind::i8 instruction descriptor: s32 accumulate, s8 x s8, both K-major, M = 128, N = 256
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ uint64_t word_range_mask(int64_t word_slot, int64_t s0, int64_t s1) {
  const int64_t lo = s0 > word_slot ? s0 - word_slot : 0;
  const int64_t hi = s1 - word_slot < 64 ? s1 - word_slot : 64;
  if (hi <= lo) return 0ull;
  const uint64_t upto = hi >= 64 ? ~0ull : ((1ull << hi) - 1);
  return upto & ~((1ull << lo) - 1);
}


// ---- filter program: register machine over one 64-slot word ---------------------------
__device__ __forceinline__ void rop_apply(uint32_t code, uint64_t m, uint64_t (&a)[kRegStack]) {
  if (code == FB_ROP_ORL) {
    a[0] |= m;
  } else if (code == FB_ROP_ANDL) {
    a[0] &= m;
  } else if (code <= FB_ROP_PUSHN) {
#pragma unroll
    for (int i = kRegStack - 1; i > 0; --i) a[i] = a[i - 1];
    a[0] = code == FB_ROP_PUSHN ? ~m : m;
  } else if (code == FB_ROP_NOT) {
    a[0] = ~a[0];
  } else if (code != FB_ROP_NOP) {  // ANDS / ORS
    a[0] = code == FB_ROP_ANDS ? (a[1] & a[0]) : (a[1] | a[0]);
#pragma unroll
    for (int i = 1; i < kRegStack - 1; ++i) a[i] = a[i + 1];
  }
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

// prog_s / leaf_s are 32-bit shared-memory addresses (the program staged in smem; the
// current tile's leaf-mask stage offset by this thread's half).
__device__ __forceinline__ void eval_half(uint32_t prog_s, int n_ops, uint32_t leaf_s,
                                          uint64_t& r0, uint64_t& r1) {
  uint64_t a0[kRegStack], a1[kRegStack];
#pragma unroll
  for (int i = 0; i < kRegStack; ++i) a0[i] = a1[i] = 0ull;
  for (int b = 0; b < n_ops; b += 8) {
    const uint4 w = lds128(prog_s + 2u * b);
    const uint32_t op[8] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16,
                            w.z & 0xFFFFu, w.z >> 16, w.w & 0xFFFFu, w.w >> 16};
    uint4 m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = lds128(leaf_s + (op[j] & 0x1FFFu) * (kLeafStride * 8u));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t code = op[j] >> 13;
      rop_apply(code, ((uint64_t)m[j].y << 32) | m[j].x, a0);
      rop_apply(code, ((uint64_t)m[j].w << 32) | m[j].z, a1);
    }
  }
  r0 = a0[0];
  r1 = a1[0];
}

// Same, for a program left in global memory (batch too large to stage).
__device__ __forceinline__ void eval_half_global(const uint16_t* prog, int n_ops, uint32_t leaf_s,
                                                 uint64_t& r0, uint64_t& r1) {
  uint64_t a0[kRegStack], a1[kRegStack];
#pragma unroll
  for (int i = 0; i < kRegStack; ++i) a0[i] = a1[i] = 0ull;
  for (int b = 0; b < n_ops; b += 8) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(prog + b));
    const uint32_t op[8] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16,
                            w.z & 0xFFFFu, w.z >> 16, w.w & 0xFFFFu, w.w >> 16};
    uint4 m[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[j] = lds128(leaf_s + (op[j] & 0x1FFFu) * (kLeafStride * 8u));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t code = op[j] >> 13;
      rop_apply(code, ((uint64_t)m[j].y << 32) | m[j].x, a0);
      rop_apply(code, ((uint64_t)m[j].w << 32) | m[j].z, a1);
    }
  }
  r0 = a0[0];
  r1 = a1[0];
}

// ---- CNF mode helpers ---------------------------------------------------------------
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

// Per-warp state of the CNF epilogue for the current tile. Hits and survivors are queued
// as 16-bit entries: (m-block << 15) | (row << 8) | item, so entry >> 8 is the query.
struct HitCtx {
  int64_t tile;
  uint32_t tb_s;   // shared address of this tile's transposed column bits
  uint32_t qm_s;   // shared address of the query group masks
  uint32_t a_s;    // shared address of the query tile (SW128 rows)
  uint32_t b_s;    // shared address of this tile's item stage (SW128 rows)
  uint32_t id_s;   // shared address of this tile's id ranks (same stage index)
  uint32_t qg_s;   // shared address of the groups-per-query table
  uint32_t t_s;    // shared address of the per-query thresholds
  uint32_t hit_s;  // this warp's hit ring
  uint32_t sv_s;   // this warp's survivor ring
};
// An emission whose slot reservation (atomicAdd) is in flight; stored one batch later so
// the global round trip overlaps the next tile's work.
struct PendingEmit {
  uint64_t key;
  uint32_t p;
  uint32_t slot;
  int32_t q;
};
constexpr int kSurvCap = 64;
// per item stage, written by the producer: the tile's id ranks, its four validity & range
// words and its tile index
constexpr uint32_t kMetaValid = kTileItems * 4;       // 1024
constexpr uint32_t kMetaTile = kMetaValid + 32;       // 1056
constexpr uint32_t kStageMeta = kMetaTile + 32;       // 1088 bytes per stage  // per-warp ring of filter survivors (exact key test pending)

__device__ __forceinline__ uint32_t lds32(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
  return v;
}

// Exact int32 dot of a query row (A tile) and an item row (B stage) from shared memory.
// Both tiles use the SWIZZLE_128B layout: 16-byte chunk c of row r sits at c ^ (r & 7).
__device__ __forceinline__ int32_t smem_dot(uint32_t a_row, uint32_t a_sw, uint32_t b_row,
                                            uint32_t b_sw) {
  int32_t acc = 0;
#pragma unroll
  for (uint32_t c = 0; c < 8; ++c) {
    const uint4 x = lds128(a_row + ((c ^ a_sw) << 4));
    const uint4 y = lds128(b_row + ((c ^ b_sw) << 4));
    acc = __dp4a((int)x.x, (int)y.x, acc);
    acc = __dp4a((int)x.y, (int)y.y, acc);
    acc = __dp4a((int)x.z, (int)y.z, acc);
    acc = __dp4a((int)x.w, (int)y.w, acc);
  }
  return acc;
}

__device__ __forceinline__ uint32_t lds16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts16(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void flush_pending(const TcArgs& a, PendingEmit& pd) {
  if (pd.q >= 0 && pd.p < (uint32_t)a.cap) {
    a.out_key[(int64_t)pd.q * a.cap + pd.p] = pd.key;
    if (a.out_slot) a.out_slot[(int64_t)pd.q * a.cap + pd.p] = pd.slot;
  }
  pd.q = -1;
}

// Up to 32 filter survivors from the head of the survivor ring: exact score recomputed
// from the resident query / item tiles, exact key test, slot reservation. The previous
// batch's stores are completed first (their reservations have long returned).
__device__ __forceinline__ void emit_survivors(const TcArgs& a, const HitCtx& h,
                                               uint32_t& sv_head, uint32_t sv_tail,
                                               PendingEmit& pd, int lane) {
  const uint32_t n = min(32u, sv_tail - sv_head);
  const bool mine = (uint32_t)lane < n;
  uint32_t ent = 0;
  if (mine) ent = lds16(h.sv_s + ((sv_head + (uint32_t)lane) & (kSurvCap - 1)) * 2u);
  __syncwarp();
  sv_head += n;
  flush_pending(a, pd);
  if (mine) {
    const uint32_t q = ent >> 8;
    const uint32_t item = ent & 255u;
    const uint64_t T = lds64(h.t_s + 8u * q);
    const int32_t score =
        smem_dot(h.a_s + q * kKBytes, q & 7u, h.b_s + item * kKBytes, item & 7u);
    const uint64_t key = make_key(score, lds32(h.id_s + 4u * item));
    if (key >= T) {
      pd.p = atomicAdd(a.out_cnt + q, 1u);
      pd.key = key;
      pd.slot = (uint32_t)(h.tile * kTileItems + item);
      pd.q = (int32_t)q;
    }
  }
}

// n (<= 32) hits from the head of the hit ring -- (query, item) pairs whose score cleared
// the threshold gate and whose item is valid, in range and in the query's mask -- get the
// CNF filter test (item column bits & the query's group masks); survivors are queued.
__device__ __forceinline__ void filter_hits(const TcArgs& a, const HitCtx& h, uint32_t& head,
                                            uint32_t n, uint32_t& sv_head, uint32_t& sv_tail,
                                            PendingEmit& pd, int lane) {
  const bool mine = (uint32_t)lane < n;
  uint32_t ent = 0;
  if (mine) ent = lds16(h.hit_s + ((head + (uint32_t)lane) & (kHitCap - 1)) * 2u);
  __syncwarp();
  head += n;
  bool pass = mine;
  if (mine) {
    const uint32_t q = ent >> 8;
    const uint32_t item = ent & 255u;
    const int ng = (int)lds32(h.qg_s + 4u * q);
    if (ng > 0) {
      const uint32_t tb = h.tb_s + item * (kTbStride * 4u);
      const uint4 t0 = lds128(tb);
      uint32_t qaddr = h.qm_s + q * (uint32_t)(a.cnf_gmax * a.qm_stride) * 4u;
      if (a.qm_stride == 4) {
        for (int g = 0; g < ng && pass; ++g) {
          const uint4 m0 = lds128(qaddr);
          pass = ((t0.x & m0.x) | (t0.y & m0.y) | (t0.z & m0.z) | (t0.w & m0.w)) != 0u;
          qaddr += 16u;
        }
      } else {
        const uint4 t1 = lds128(tb + 16u);
        for (int g = 0; g < ng && pass; ++g) {
          const uint4 m0 = lds128(qaddr);
          const uint4 m1 = lds128(qaddr + 16u);
          pass = ((t0.x & m0.x) | (t0.y & m0.y) | (t0.z & m0.z) | (t0.w & m0.w) |
                  (t1.x & m1.x) | (t1.y & m1.y) | (t1.z & m1.z) | (t1.w & m1.w)) != 0u;
          qaddr += 32u;
        }
      }
    }
  }
  const uint32_t b = __ballot_sync(0xffffffffu, pass);
  if (pass) sts16(h.sv_s + ((sv_tail + __popc(b & lanemask_lt())) & (kSurvCap - 1)) * 2u, ent);
  sv_tail += (uint32_t)__popc(b);
  if (sv_tail - sv_head >= 32u) {
    __syncwarp();
    emit_survivors(a, h, sv_head, sv_tail, pd, lane);
  }
}

template <bool kCnf>
__global__ void __launch_bounds__(kCnf ? kThreadsCnf : kThreads, 1)
    k_scan_tc(const __grid_constant__ CUtensorMap tmap_items, const TcArgs a) {
  constexpr int NT = kCnf ? kThreadsCnf : kThreads;
  constexpr int NE = kCnf ? kEpiWarpsCnf : kEpiWarps;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sA = smem + a.off_a;
  uint8_t* sB = smem + a.off_b;
  uint8_t* sP = smem + a.off_p;
  uint8_t* sL = smem + a.off_l;
  int16_t* sLS = reinterpret_cast<int16_t*>(smem + a.off_ls);
  uint64_t* sT = reinterpret_cast<uint64_t*>(smem + a.off_thr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  uint64_t* items_full = bars;        // [4]
  uint64_t* items_empty = bars + 4;   // [4]
  uint64_t* planes_full = bars + 8;   // [2]
  uint64_t* planes_empty = bars + 10; // [2]
  uint64_t* leaf_full = bars + 12;    // [2]
  uint64_t* leaf_empty = bars + 14;   // [2]
  uint64_t* acc_full = bars + 16;     // [2]
  uint64_t* acc_empty = bars + 18;    // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 20);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.item_stages;
  const int PS = a.plane_stages;

  // ---- prologue: queries -> swizzled smem, thresholds, leaf table, filter programs ----
  const int a_rows = a.n_mblk * kBlockM;
  for (int i = threadIdx.x; i < a_rows * 8; i += NT) {
    const int r = i >> 3, c = i & 7;
    int4 v = make_int4(0, 0, 0, 0);
    if (r < a.nq) v = __ldg(reinterpret_cast<const int4*>(a.queries + (int64_t)r * kKBytes) + c);
    *reinterpret_cast<int4*>(sA + r * kKBytes + ((c ^ (r & 7)) << 4)) = v;
  }
  for (int q = threadIdx.x; q < kMaxQueries; q += NT)
    sT[q] = (a.threshold != nullptr && q < a.nq) ? a.threshold[q] : 0ull;
  int32_t prog_off0 = 0;
  bool prog_staged = false;
  if (kCnf) {
    // column -> plane-slot table (negated columns flagged by a set bit 14 on slot 0),
    // query group masks (zero-padded to qm_stride words), group counts, zeroed TB stages
    for (int i = threadIdx.x; i < a.n_cols * a.k_max; i += NT) {
      const int c = i / a.k_max, j = i - c * a.k_max;
      const int cl = a.col_leaf[c];
      const int leaf = cl >= 0 ? cl : ~cl;
      int s = a.leaf_slot[leaf * a.k_max + j];
      if (j == 0 && cl < 0) s |= 0x4000;
      sLS[i] = (int16_t)s;
    }
    uint32_t* qm = reinterpret_cast<uint32_t*>(smem + a.off_qm);
    const int qm_words = a.nq * a.cnf_gmax * a.qm_stride;
    for (int i = threadIdx.x; i < qm_words; i += NT) {
      const int w = i % a.qm_stride, qg = i / a.qm_stride;
      qm[i] = w < a.cnf_words ? a.qmask[(int64_t)qg * a.cnf_words + w] : 0u;
    }
    int32_t* qgs = reinterpret_cast<int32_t*>(smem + a.off_qg);
    for (int q = threadIdx.x; q < kMaxQueries; q += NT) qgs[q] = q < a.nq ? a.qgroups[q] : 0;
    uint32_t* tb = reinterpret_cast<uint32_t*>(sL);
    for (int i = threadIdx.x; i < 2 * (int)(a.leaf_stage_bytes / 4); i += NT) tb[i] = 0u;
  } else if (a.has_prog) {
    for (int i = threadIdx.x; i < a.n_leaves * a.k_max; i += NT) sLS[i] = a.leaf_slot[i];
    prog_off0 = a.rop_offset[0];
    const int32_t n_ops = a.rop_offset[a.nq] - prog_off0;
    if (n_ops <= a.rops_cap) {
      uint4* dst = reinterpret_cast<uint4*>(smem + a.off_r);
      const uint4* src = reinterpret_cast<const uint4*>(a.rops + prog_off0);
      for (int i = threadIdx.x; i < n_ops / 8; i += NT) dst[i] = __ldg(src + i);
      prog_staged = true;
    }
  }
  const uint32_t prog_s = su32(smem + a.off_r);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(items_full + s, 1 + 32 + 1);  // TMA expect-tx, id-rank cp.async per lane, meta
      mbar_init(items_empty + s, 1 + NE);  // MMA commit + every epilogue warp (id stage)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(planes_full + s, 32);  // one cp.async.mbarrier.arrive per producer lane
      mbar_init(planes_empty + s, kCnf ? 2 : kLeafThreads);
      mbar_init(leaf_full + s, kCnf ? 2 : kLeafThreads);
      mbar_init(leaf_empty + s, NE);
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, NE);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (kCnf && warp >= kEpiWarp0) {
    // CNF: both accumulator buffers start as -tau of their rows; the MMA accumulates onto
    // them, so the epilogue's gate is a sign test. Buffer b holds M-block b (or 0).
    const int ew = warp - kEpiWarp0;
#pragma unroll 1
    for (int ab = 0; ab < 2; ++ab) {
      const int mb = a.n_mblk == kMaxMBlocks ? ab : 0;
      const int32_t nt = -gate_tau(sT, mb * kBlockM + (warp & 3) * 32 + lane, a.nq);
      for (int c = ew >> 2; c < 8; c += 3)
        tmem_st32_const(tmem_base + ((uint32_t)((warp & 3) * 32) << 16) +
                            (uint32_t)(ab * kAccCols + c * 32),
                        nt);
    }
    tmem_wait_st();
  }
  if (kCnf) {
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  const int64_t n_sel = a.n_sel;
  if (warp == 0) {
    // ================= producer: TMA item tile + Bloom plane words ================
    // The per-tile global reads (work item, then its validity & range words) are issued
    // one tile ahead, so their latency never sits on the producer's critical path.
    int s = 0, ps = 0;
    uint32_t ph = 0, pph = 0;
    const int64_t G = gridDim.x;
    auto load_valid = [&](int2 w) -> uint64_t {
      if (lane >= kTileWords) return 0ull;
      const int64_t s0 = a.ranges[2 * w.y], s1 = a.ranges[2 * w.y + 1];
      const int64_t gw = (int64_t)w.x * kTileWords + lane;
      return __ldg(a.valid + gw) & word_range_mask(gw * 64, s0, s1);
    };
    int2 wk_cur = make_int2(0, 0), wk_next = make_int2(0, 0);
    uint64_t v_cur = 0ull;
    if (blockIdx.x < n_sel) {
      wk_cur = a.work[(int64_t)blockIdx.x * a.work_stride];
      v_cur = load_valid(wk_cur);
      if (blockIdx.x + G < n_sel) wk_next = a.work[((int64_t)blockIdx.x + G) * a.work_stride];
    }
    for (int64_t i = blockIdx.x; i < n_sel; i += G) {
      const int tile = wk_cur.x;
      // prefetch: the next tile's validity, the tile after next's work item
      uint64_t v_next = 0ull;
      int2 wk_nn = make_int2(0, 0);
      if (i + G < n_sel) v_next = load_valid(wk_next);
      if (i + 2 * G < n_sel) wk_nn = a.work[(i + 2 * G) * a.work_stride];
      {
        // item rows by TMA; alongside, into a stage with the item stage's lifetime: the
        // tile's 256 id ranks (1 KB, 16-byte cp.async), its validity & range words and its
        // tile index (so the epilogue never waits on global memory for per-tile metadata)
        mbar_wait_idle(items_empty + s, ph ^ 1u);
        if (lane == 0) {
          mbar_expect_tx(items_full + s, kItemBytes);
          tma_load_2d(sB + (size_t)s * kItemBytes, &tmap_items, 0, tile * kTileItems,
                      items_full + s);
        }
        const uint32_t mst = su32(smem + a.off_id) + (uint32_t)s * kStageMeta;
        const uint32_t* src = a.id_rank + (int64_t)tile * kTileItems;
#pragma unroll
        for (int e = lane; e < kTileItems / 4; e += 32)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(mst + (uint32_t)e * 16u),
                       "l"(src + 4 * e)
                       : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         su32(items_full + s))
                     : "memory");
        if (lane < kTileWords)
          asm volatile("st.shared.u64 [%0], %1;" ::"r"(mst + kMetaValid + 8u * lane), "l"(v_cur)
                       : "memory");
        if (lane == 0)
          asm volatile("st.shared.u32 [%0], %1;" ::"r"(mst + kMetaTile), "r"(tile) : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(items_full + s);
      }
      if (a.has_prog && a.n_planes > 0) {
        mbar_wait_idle(planes_empty + ps, pph ^ 1u);
        // gather the referenced planes' 32-byte rows for this tile: 16-byte cp.async per
        // lane (two lanes per plane row, a warp covers 16 rows per instruction); each lane
        // arrives on planes_full once its copies land
        const uint32_t dst = su32(sP + (size_t)ps * a.plane_stage_bytes);
        const int64_t col0 = (int64_t)tile * kTileWords;
        // (plane indices fetched eight at a time ahead of the copies: the copies' memory
        // clobber would otherwise serialise each index load behind the previous copy)
        const int n2 = 2 * a.n_planes;
        for (int e0 = lane; e0 < n2; e0 += 32 * 8) {
          int pl[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + 32 * u;
            pl[u] = e < n2 ? __ldg(a.plane_list + (e >> 1)) : 0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + 32 * u;
            if (e < n2) {
              const uint64_t* src = a.planes + (int64_t)pl[u] * a.n_words + col0 + 2 * (e & 1);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                               dst + (uint32_t)e * 16u),
                           "l"(src)
                           : "memory");
            }
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         su32(planes_full + ps))
                     : "memory");
        if (++ps == PS) { ps = 0; pph ^= 1u; }
      }
      if (++s == S) { s = 0; ph ^= 1u; }
      wk_cur = wk_next;
      v_cur = v_next;
      wk_next = wk_nn;
    }
  } else if (warp == 1) {
    // ================= MMA issuer (one thread) ====================================
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_i8(kBlockM, kTileItems);
      int acc_it = 0, s = 0;
      uint32_t ph = 0;
      for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x) {
        mbar_wait(items_full + s, ph);
        tc_fence_after();
        const uint32_t b_base = su32(sB + (size_t)s * kItemBytes);
        for (int mb = 0; mb < a.n_mblk; ++mb, ++acc_it) {
          const int ab = acc_it & 1;
          const uint32_t aph = (uint32_t)(acc_it >> 1) & 1u;
          mbar_wait_idle(acc_empty + ab, aph ^ 1u);
          tc_fence_after();
          const uint32_t a_base = su32(sA + mb * kBlockM * kKBytes);
          const uint32_t d = tmem_base + (uint32_t)(ab * kAccCols);
#pragma unroll
          for (int kk = 0; kk < kKBytes / kUmmaK; ++kk)
            umma_i8(d, sw128_desc(a_base + kk * kUmmaK), sw128_desc(b_base + kk * kUmmaK), idesc,
                    (kk > 0 || kCnf) ? 1u : 0u);
          umma_commit(acc_full + ab);
        }
        umma_commit(items_empty + s);
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp < kEpiWarp0 && kCnf) {
    // ================= column builders (CNF): Bloom test per literal column, then a
    // 32x32 bit transpose so each item row holds its column bits =====================
    const int lw = warp - 2;  // 0 or 1
    int it = 0, ps = 0;
    uint32_t pph = 0;
    for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
      const int st = it & 1;
      const uint32_t ph = (uint32_t)(it >> 1) & 1u;
      mbar_wait_idle(planes_full + ps, pph);
      mbar_wait_idle(leaf_empty + st, ph ^ 1u);
      const uint32_t p_s = su32(sP + (size_t)ps * a.plane_stage_bytes);
      uint32_t* TB = reinterpret_cast<uint32_t*>(sL + (size_t)st * a.leaf_stage_bytes);
      for (int cb = lw; cb < a.cnf_words; cb += 2) {  // 32-column block
        const int col = cb * 32 + lane;
        // the column's 256 tile bits: AND of its planes' 32-byte rows (8 x u32, one per
        // 32-item block); all loads are independent
        uint32_t m[8];
#pragma unroll
        for (int ib = 0; ib < 8; ++ib) m[ib] = col < a.n_cols ? ~0u : 0u;
        if (col < a.n_cols) {
          bool neg = false;
          for (int j = 0; j < a.k_max; ++j) {
            int sl = sLS[col * a.k_max + j];
            if (j == 0) {
              neg = (sl & 0x4000) != 0;
              sl &= ~0x4000;
            }
            if (sl < 0) break;
            const uint4 lo = lds128(p_s + (uint32_t)sl * 32u);
            const uint4 hi = lds128(p_s + (uint32_t)sl * 32u + 16u);
            m[0] &= lo.x; m[1] &= lo.y; m[2] &= lo.z; m[3] &= lo.w;
            m[4] &= hi.x; m[5] &= hi.y; m[6] &= hi.z; m[7] &= hi.w;
          }
          if (neg) {
#pragma unroll
            for (int ib = 0; ib < 8; ++ib) m[ib] = ~m[ib];
          }
        }
        // eight 32x32 transposes in lockstep (independent shuffles per round)
        const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int sft = 16 >> k;
          const uint32_t mk = masks[k];
          const bool upper = (lane & sft) != 0;
          uint32_t y[8];
#pragma unroll
          for (int ib = 0; ib < 8; ++ib) y[ib] = __shfl_xor_sync(0xffffffffu, m[ib], sft);
#pragma unroll
          for (int ib = 0; ib < 8; ++ib)
            m[ib] = upper ? ((m[ib] & ~mk) | ((y[ib] & ~mk) >> sft))
                          : ((m[ib] & mk) | ((y[ib] & mk) << sft));
        }
#pragma unroll
        for (int ib = 0; ib < 8; ++ib) TB[(ib * 32 + lane) * kTbStride + cb] = m[ib];
      }
      __syncwarp();
      if (lane == 0) {  // one arrival per builder warp
        mbar_arrive(planes_empty + ps);
        mbar_arrive(leaf_full + st);
      }
      if (++ps == PS) { ps = 0; pph ^= 1u; }
    }
  } else if (warp < kEpiWarp0) {
    // ================= leaf builders: AND each leaf's planes per word =============
    if (a.has_prog) {
      const int t = threadIdx.x - 64;
      int it = 0, ps = 0;
      uint32_t pph = 0;
      for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
        const int st = it & 1;
        const uint32_t ph = (uint32_t)(it >> 1) & 1u;
        if (a.n_planes > 0) mbar_wait_idle(planes_full + ps, pph);
        mbar_wait_idle(leaf_empty + st, ph ^ 1u);
        const uint64_t* P = reinterpret_cast<const uint64_t*>(sP + (size_t)ps * a.plane_stage_bytes);
        uint64_t* L = reinterpret_cast<uint64_t*>(sL + (size_t)st * a.leaf_stage_bytes);
        for (int e = t; e < a.n_leaves * kTileWords; e += kLeafThreads) {
          const int l = e >> 2, w = e & 3;
          uint64_t m = ~0ull;
          for (int j = 0; j < a.k_max; ++j) {
            const int sl = sLS[l * a.k_max + j];
            if (sl < 0) break;
            m &= P[sl * kTileWords + w];
          }
          L[l * kLeafStride + w] = m;
        }
        if (a.n_planes > 0) mbar_arrive(planes_empty + ps);
        mbar_arrive(leaf_full + st);
        if (++ps == PS) { ps = 0; pph ^= 1u; }
      }
    }
  } else if (kCnf) {
    // ================= epilogue (CNF): TMEM scores -> threshold gate -> hit ring ->
    // per-hit filter test (transposed column bits & query group masks) -> survivor ring ->
    // exact score from the resident smem tiles -> key test -> emit. Twelve warps, three
    // per TMEM lane quadrant; a quadrant's eight 32-column chunks of each M-block are
    // dealt round-robin with a rotating start so the three warps stay balanced. =======
    const int ew = warp - kEpiWarp0;
    const int quad = warp & 3;
    const int sub = ew >> 2;
    const int row = quad * 32 + lane;
    HitCtx h;
    h.qm_s = su32(smem + a.off_qm);
    h.a_s = su32(sA);
    h.qg_s = su32(smem + a.off_qg);
    h.t_s = su32(sT);
    h.hit_s = su32(smem + a.off_hit) + (uint32_t)ew * (kHitCap * 2u);
    h.sv_s = su32(smem + a.off_hit) + (uint32_t)(NE * kHitCap * 2) + (uint32_t)ew * (kSurvCap * 2u);
    // per query row of this thread: clamped score gate (the accumulators start at -tau)
    int32_t tau[kMaxMBlocks];
#pragma unroll
    for (int mb = 0; mb < kMaxMBlocks; ++mb) tau[mb] = gate_tau(sT, mb * kBlockM + row, a.nq);
    PendingEmit pd;
    pd.q = -1;
    pd.p = 0;
    pd.key = 0;
    pd.slot = 0;
    int it = 0, acc_it = 0, s = 0;
    uint32_t iph = 0;
    for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
      // per-tile metadata staged by the producer with the item stage
      mbar_wait(items_full + s, iph);
      const uint32_t mst = su32(smem + a.off_id) + (uint32_t)s * kStageMeta;
      h.tile = (int64_t)lds32(mst + kMetaTile);
      // lane c < 8 holds the validity & range bits of the tile's chunk c (32 items)
      const uint32_t vchunk = lane < 8 ? lds32(mst + kMetaValid + 4u * lane) : 0u;
      h.b_s = su32(sB + (size_t)s * kItemBytes);
      h.id_s = mst;
      const int st = it & 1;
      mbar_wait(leaf_full + st, (uint32_t)(it >> 1) & 1u);
      h.tb_s = su32(sL + (size_t)st * a.leaf_stage_bytes);
      uint32_t head = 0, tail = 0, sv_head = 0, sv_tail = 0;  // warp-uniform ring cursors
#pragma unroll 1
      for (int mb = 0; mb < a.n_mblk; ++mb, ++acc_it) {
        const int q = mb * kBlockM + row;
        const bool qok = q < a.nq;
        const int32_t tq = mb == 0 ? tau[0] : tau[kMaxMBlocks - 1];
        const int ab = acc_it & 1;
        mbar_wait(acc_full + ab, (uint32_t)(acc_it >> 1) & 1u);
        tc_fence_after();
        const uint32_t taddr =
            tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * kAccCols);
        const uint32_t ebase = ((uint32_t)mb << 15) | ((uint32_t)row << 8);
        const int c0 = (sub + mb + it) % 3;
        int32_t r[32];
        tmem_ld32_async(taddr + (uint32_t)(c0 * 32), r);
#pragma unroll 1
        for (int c = c0; c < 8; c += 3) {
          tmem_wait32(r);
          tmem_st32_const(taddr + (uint32_t)(c * 32), -tq);  // re-arm for the buffer's next use
          if (a.dump != nullptr && qok) {
            const int64_t base = h.tile * kTileItems + c * 32;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (base + j < a.dump_ld) a.dump[(int64_t)q * a.dump_ld + base + j] = r[j] + tq;
          }
          uint32_t em = __shfl_sync(0xffffffffu, vchunk, c);
          if (!qok) em = 0u;
          if (a.masks != nullptr && em != 0u)
            em &= (uint32_t)(__ldg(a.masks + (int64_t)q * a.n_words + h.tile * kTileWords +
                                   (c >> 1)) >>
                             (32 * (c & 1)));
          uint32_t hm = nonneg_mask32(r) & em;
          if (c + 3 < 8) {
            tmem_ld32_async(taddr + (uint32_t)((c + 3) * 32), r);  // overlaps the hit handling
          } else {
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty + ab);
          }
          // append this chunk's hits to the warp's ring, up to two per lane per round
          const uint32_t eb = ebase | (uint32_t)(c * 32);
          while (true) {
            const uint32_t b1 = __ballot_sync(0xffffffffu, hm != 0u);
            if (b1 == 0u) break;
            const uint32_t rest = hm & (hm - 1u);
            const uint32_t b2 = __ballot_sync(0xffffffffu, rest != 0u);
            if (hm != 0u) {
              const uint32_t lt = lanemask_lt();
              const uint32_t pos = tail + (uint32_t)(__popc(b1 & lt) + __popc(b2 & lt));
              sts16(h.hit_s + (pos & (kHitCap - 1)) * 2u, eb + (uint32_t)(__ffs(hm) - 1));
              if (rest != 0u)
                sts16(h.hit_s + ((pos + 1u) & (kHitCap - 1)) * 2u,
                      eb + (uint32_t)(__ffs(rest) - 1));
            }
            hm = rest & (rest - 1u);
            tail += (uint32_t)(__popc(b1) + __popc(b2));
            while (tail - head >= 32u) {
              __syncwarp();
              filter_hits(a, h, head, 32u, sv_head, sv_tail, pd, lane);
            }
          }
        }
      }
      // drain: remaining hits, then the survivors (they read the item and id stages)
      if (tail != head) {
        __syncwarp();
        filter_hits(a, h, head, tail - head, sv_head, sv_tail, pd, lane);
      }
      while (sv_tail != sv_head) {
        __syncwarp();
        emit_survivors(a, h, sv_head, sv_tail, pd, lane);
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(leaf_empty + st);
        mbar_arrive(items_empty + s);
      }
      if (++s == a.item_stages) {
        s = 0;
        iph ^= 1u;
      }
    }
    flush_pending(a, pd);
  } else {
    // ================= epilogue: filter (eager) + TMEM scores + gate + emit ========
    const int ew = warp - kEpiWarp0;
    const int quad = warp & 3;  // TMEM lane quadrant accessible to this warp
    const int half = ew >> 2;   // item columns [half * 128, half * 128 + 128)
    const int row = quad * 32 + lane;
    // per M-block: this thread's query program (offset into the staged copy, length)
    int p_off[kMaxMBlocks], p_len[kMaxMBlocks];
#pragma unroll
    for (int mb = 0; mb < kMaxMBlocks; ++mb) {
      const int q = mb * kBlockM + row;
      p_off[mb] = p_len[mb] = 0;
      if (a.has_prog && q < a.nq && mb < a.n_mblk) {
        p_off[mb] = a.rop_offset[q] - prog_off0;
        p_len[mb] = a.rop_offset[q + 1] - a.rop_offset[q];
      }
    }
    int it = 0, acc_it = 0, s = 0;
    for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
      const int2 wk = a.work[i * a.work_stride];
      const int64_t tile = wk.x;
      const uint32_t id_s = su32(smem + a.off_id) + (uint32_t)s * (kTileItems * 4u) +
                            (uint32_t)(half * 128) * 4u;
      const int64_t s0 = a.ranges[2 * wk.y], s1 = a.ranges[2 * wk.y + 1];
      const int64_t wbase = tile * kTileWords + 2 * half;
      const uint64_t v0 = __ldg(a.valid + wbase) & word_range_mask(wbase * 64, s0, s1);
      const uint64_t v1 = __ldg(a.valid + wbase + 1) & word_range_mask((wbase + 1) * 64, s0, s1);
      const int st = it & 1;
      if (a.has_prog) mbar_wait(leaf_full + st, (uint32_t)(it >> 1) & 1u);
      const uint32_t leaf_s = su32(sL + (size_t)st * a.leaf_stage_bytes) + 16u * half;
#pragma unroll 1
      for (int mb = 0; mb < a.n_mblk; ++mb, ++acc_it) {
        const int q = mb * kBlockM + row;
        const bool active = q < a.nq;
        // eligibility of this thread's 128 items: validity & range & program & mask
        uint64_t f0 = active ? v0 : 0ull, f1 = active ? v1 : 0ull;
        const int plen = mb == 0 ? p_len[0] : p_len[1];
        if (plen > 0 && (f0 | f1) != 0ull) {
          const int poff = mb == 0 ? p_off[0] : p_off[1];
          uint64_t e0, e1;
          if (prog_staged)
            eval_half(prog_s + 2u * poff, plen, leaf_s, e0, e1);
          else
            eval_half_global(a.rops + prog_off0 + poff, plen, leaf_s, e0, e1);
          f0 &= e0;
          f1 &= e1;
        }
        if (a.masks != nullptr && (f0 | f1) != 0ull) {
          f0 &= __ldg(a.masks + (int64_t)q * a.n_words + wbase);
          f1 &= __ldg(a.masks + (int64_t)q * a.n_words + wbase + 1);
        }
        const uint64_t T = active ? sT[q] : ~0ull;
        const int32_t tau = T == 0ull ? INT32_MIN : key_score(T);
        // threshold 0 (sampling pass): every eligible item is emitted, so one slot
        // reservation per M-block covers all four chunks; it is issued before the scores
        // are read so the round trip overlaps the wait
        uint32_t pdense = 0u;
        if (T == 0ull && (f0 | f1) != 0ull)
          pdense = atomicAdd(a.out_cnt + q, (uint32_t)(__popcll(f0) + __popcll(f1)));
        const int ab = acc_it & 1;
        mbar_wait(acc_full + ab, (uint32_t)(acc_it >> 1) & 1u);
        tc_fence_after();
        const uint32_t taddr =
            tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * kAccCols + half * 128);
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          int32_t r[32];
          tmem_ld32(taddr + c * 32, r);
          if (a.dump != nullptr && active) {
            const int64_t base = tile * kTileItems + half * 128 + c * 32;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (base + j < a.dump_ld) a.dump[(int64_t)q * a.dump_ld + base + j] = r[j];
          }
          const uint32_t fw = (uint32_t)((c < 2 ? f0 : f1) >> (32 * (c & 1)));
          if (fw != 0u) {
            int32_t mx = r[0];
#pragma unroll
            for (int j = 1; j < 31; j += 2) mx = __vimax3_s32(mx, r[j], r[j + 1]);
            mx = max(mx, r[31]);
            if (mx >= tau) {
              uint32_t cm = 0u;
#pragma unroll
              for (int j = 0; j < 32; ++j) cm |= (r[j] >= tau ? 1u : 0u) << j;
              cm &= fw;
              if (cm != 0u && T == 0ull) {
                const uint32_t slot0 = (uint32_t)(tile * kTileItems + half * 128 + c * 32);
                uint32_t p = pdense;
                pdense += (uint32_t)__popc(cm);
                uint64_t* okp = a.out_key + (int64_t)q * a.cap;
                uint32_t* osp = a.out_slot ? a.out_slot + (int64_t)q * a.cap : nullptr;
                const uint32_t ids = id_s + (uint32_t)(c * 32) * 4u;
                const uint32_t cap = (uint32_t)a.cap;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  const bool on = ((cm >> j) & 1u) != 0u;
                  if (on && p < cap) {
                    okp[p] = make_key(r[j], lds32(ids + 4u * j));
                    if (osp != nullptr) osp[p] = slot0 + (uint32_t)j;
                  }
                  p += on ? 1u : 0u;
                }
              } else if (cm != 0u) {
                const int64_t slot0 = tile * kTileItems + half * 128 + c * 32;
                int32_t rs[32];  // dynamic indexing below: lives in local memory (rare path)
#pragma unroll
                for (int j = 0; j < 32; ++j) rs[j] = r[j];
                while (cm != 0u) {
                  const int j = __ffs(cm) - 1;
                  cm &= cm - 1u;
                  const int64_t slot = slot0 + j;
                  const uint64_t key = make_key(rs[j], lds32(id_s + (uint32_t)(c * 32 + j) * 4u));
                  if (key >= T) {
                    const uint32_t p = atomicAdd(a.out_cnt + q, 1u);
                    if (p < (uint32_t)a.cap) {
                      a.out_key[(int64_t)q * a.cap + p] = key;
                      if (a.out_slot) a.out_slot[(int64_t)q * a.cap + p] = (uint32_t)slot;
                    }
                  }
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty + ab);
      }
      __syncwarp();
      if (lane == 0) {
        if (a.has_prog) mbar_arrive(leaf_empty + st);
        mbar_arrive(items_empty + s);  // id stage read
      }
      if (++s == a.item_stages) s = 0;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
                 : "memory");
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (fn == nullptr) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// shared-memory carve-up; returns total bytes (incl. 1 KB alignment slack)
// Shared-memory carve-up; returns total bytes (incl. 1 KB alignment slack). In CNF mode
// the per-tile stage holds transposed column bits (256 items x kTbStride u32), the query
// group masks and group counts are staged, and each epilogue warp gets a hit ring buffer.
size_t layout(TcArgs& t, int n_mblk, int n_planes, int n_leaves, int k_max, int stages,
              int plane_stages, bool cnf) {
  size_t off = 0;
  t.off_a = 0;
  off = (size_t)n_mblk * kBlockM * kKBytes;
  t.off_b = (uint32_t)align_up(off, 1024);
  off = t.off_b + (size_t)stages * kItemBytes;
  t.plane_stage_bytes = (uint32_t)align_up((size_t)(n_planes > 0 ? n_planes : 1) * 32, 128);
  t.off_p = (uint32_t)align_up(off, 128);
  off = t.off_p + (size_t)plane_stages * t.plane_stage_bytes;
  t.leaf_stage_bytes =
      cnf ? (uint32_t)(kTileItems * kTbStride * 4)
          : (uint32_t)align_up((size_t)(n_leaves > 0 ? n_leaves : 1) * kLeafStride * 8, 128);
  t.off_l = (uint32_t)align_up(off, 128);
  off = t.off_l + 2ull * t.leaf_stage_bytes;
  const int rows = cnf ? t.n_cols : n_leaves;
  t.off_ls = (uint32_t)align_up(off, 16);
  off = t.off_ls + (size_t)(rows > 0 ? rows : 1) * (k_max > 0 ? k_max : 1) * 2;
  t.off_thr = (uint32_t)align_up(off, 16);
  off = t.off_thr + (size_t)kMaxQueries * 8;
  t.off_bar = (uint32_t)align_up(off, 16);
  off = t.off_bar + 21 * 8 + 16;
  if (cnf) {
    t.off_qm = (uint32_t)align_up(off, 16);
    off = t.off_qm + (size_t)kMaxQueries * t.cnf_gmax * t.qm_stride * 4;
    t.off_qg = (uint32_t)align_up(off, 16);
    off = t.off_qg + (size_t)kMaxQueries * 4;
    t.off_hit = (uint32_t)align_up(off, 16);
    off = t.off_hit + (size_t)kEpiWarpsCnf * (kHitCap + kSurvCap) * 2;
  }
  t.off_id = (uint32_t)align_up(off, 16);
  off = t.off_id + (size_t)stages * kStageMeta;
  t.off_r = (uint32_t)align_up(off, 16);
  off = t.off_r + (size_t)t.rops_cap * 2;
  return off + 1024;
}

constexpr size_t kSmemLimit = 227 * 1024;
constexpr int kMaxStagedOps = 16384;  // 32 KB; whatever is left stays L1

// Prefer 3 item stages and 2 plane stages; stage as much filter bytecode as fits.
bool pick_stages(TcArgs& t, int n_mblk, int n_planes, int n_leaves, int k_max, int n_rops,
                 bool cnf, size_t& smem) {
  const int prefs[4][2] = {{3, 2}, {3, 1}, {2, 2}, {2, 1}};
  if (cnf) n_rops = 0;  // the CNF epilogue does not read the bytecode
  // first pass: the configuration that also holds all filter bytecode; second: any
  for (int pass = 0; pass < 2; ++pass) {
    for (const auto& pr : prefs) {
      t.rops_cap = 0;
      smem = layout(t, n_mblk, n_planes, n_leaves, k_max, pr[0], pr[1], cnf);
      if (smem > kSmemLimit) continue;
      const size_t room = (kSmemLimit - smem) / 2 / 8 * 8;
      const size_t want = (size_t)std::min(n_rops > 0 ? n_rops : 0, kMaxStagedOps);
      if (pass == 0 && room < want) continue;
      t.rops_cap = (int32_t)std::min(room, want);
      smem = layout(t, n_mblk, n_planes, n_leaves, k_max, pr[0], pr[1], cnf);
      t.item_stages = pr[0];
      t.plane_stages = pr[1];
      return true;
    }
  }
  return false;
}

bool use_cnf(const ScanArgs& a) {
  // at threshold 0 every score is a hit: the word-level bytecode epilogue is cheaper than
  // per-hit tests, so the sampling pass takes it whenever the bytecode fits the kernel
  if (a.dense && a.prog.rops != nullptr && a.prog.rmax_stack <= kRegStack) return false;
  return a.has_prog && a.prog.col_leaf != nullptr && a.prog.cnf_words >= 1 &&
         a.prog.cnf_words <= 8 && a.prog.cnf_gmax >= 1 && a.prog.cnf_gmax <= 8 &&
         a.prog.n_cols <= 32 * a.prog.cnf_words;
}

void fill_cnf(TcArgs& t, const ScanArgs& a, int q0) {
  t.n_cols = a.prog.n_cols;
  t.cnf_words = a.prog.cnf_words;
  t.cnf_gmax = a.prog.cnf_gmax;
  t.qm_stride = a.prog.cnf_words <= 4 ? 4 : 8;
  t.col_leaf = a.prog.col_leaf;
  t.qmask = a.prog.qmask + (int64_t)q0 * a.prog.cnf_gmax * a.prog.cnf_words;
  t.qgroups = a.prog.qgroups + q0;
}

}  // namespace

bool scan_tc_supported(const ScanArgs& a) {
  if (a.mode != SCAN_EMIT || a.fb != nullptr) return false;
  if (a.idx.dim_pad != kKBytes) return false;
  if (a.idx.n_slots % kTileItems != 0 || a.tc_work == nullptr) return false;
  if (encode_fn() == nullptr) return false;
  if (a.has_prog) {
    const bool cnf = use_cnf(a);
    if (!cnf && (a.prog.rops == nullptr || a.prog.rmax_stack > kRegStack)) return false;
    if (a.prog.n_leaves >= (1 << 13) || a.prog.plane_list == nullptr) return false;
    TcArgs t{};
    if (cnf) fill_cnf(t, a, 0);
    size_t smem = 0;
    const int n_mblk = a.n_queries >= kBlockM ? kMaxMBlocks : 1;
    if (!pick_stages(t, n_mblk, a.prog.n_planes, a.prog.n_leaves, a.prog.k_max, 0, cnf, smem))
      return false;
  }
  return true;
}

int launch_scan_tc(const ScanArgs& a, cudaStream_t s) {
  if (!scan_tc_supported(a)) return FB_ERR_UNSUPPORTED;
  const int64_t n_sel = (a.n_tc_work + a.word_stride - 1) / a.word_stride;
  if (n_sel <= 0 || a.n_queries <= 0) return FB_OK;
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)kKBytes, (cuuint64_t)a.idx.n_slots};
  const cuuint64_t strides[1] = {(cuuint64_t)a.idx.dim_pad};
  const cuuint32_t box[2] = {(cuuint32_t)kKBytes, (cuuint32_t)kTileItems};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2,
                            const_cast<int8_t*>(a.idx.items), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(FB_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  int n_sm = 148;
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = (int)(n_sel < n_sm ? n_sel : n_sm);
  const bool cnf = use_cnf(a);
  for (int q0 = 0; q0 < a.n_queries; q0 += kMaxQueries) {
    const int nq = a.n_queries - q0 < kMaxQueries ? a.n_queries - q0 : kMaxQueries;
    TcArgs t{};
    t.queries = a.queries + (int64_t)q0 * a.idx.dim_pad;
    t.nq = nq;
    t.n_mblk = (nq + kBlockM - 1) / kBlockM;
    t.planes = a.idx.planes;
    t.valid = a.idx.valid;
    t.id_rank = a.idx.id_rank;
    t.masks = a.masks ? a.masks + (int64_t)q0 * a.idx.n_words : nullptr;
    t.n_words = a.idx.n_words;
    t.has_prog = a.has_prog;
    if (a.has_prog) {
      t.n_planes = a.prog.n_planes;
      t.n_leaves = a.prog.n_leaves;
      t.k_max = a.prog.k_max;
      t.plane_list = a.prog.plane_list;
      t.leaf_slot = a.prog.leaf_slot;
      t.rop_offset = a.prog.rop_offset + q0;
      t.rops = a.prog.rops;
      if (cnf) fill_cnf(t, a, q0);
    }
    t.work = reinterpret_cast<const int2*>(a.tc_work);
    t.n_sel = n_sel;
    t.work_stride = a.word_stride;
    t.ranges = a.ranges;
    t.threshold = a.threshold ? a.threshold + q0 : nullptr;
    t.out_key = a.out_key + (int64_t)q0 * a.cap;
    t.out_slot = a.out_slot ? a.out_slot + (int64_t)q0 * a.cap : nullptr;
    t.out_cnt = a.out_cnt + q0;
    t.cap = a.cap;
    t.dump = a.dump ? a.dump + (int64_t)q0 * a.dump_ld : nullptr;
    t.dump_ld = a.dump_ld;
    size_t smem = 0;
    if (!pick_stages(t, t.n_mblk, t.has_prog ? t.n_planes : 0, t.has_prog ? t.n_leaves : 0,
                     t.has_prog ? t.k_max : 0, t.has_prog ? a.prog.n_rops : 0, cnf, smem))
      return FB_ERR_UNSUPPORTED;
    if (cnf) {
      FB_CUDA(cudaFuncSetAttribute(k_scan_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      k_scan_tc<true><<<grid, kThreadsCnf, smem, s>>>(tmap, t);
    } else {
      FB_CUDA(cudaFuncSetAttribute(k_scan_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
      k_scan_tc<false><<<grid, kThreads, smem, s>>>(tmap, t);
    }
    FB_LAUNCH_CHECK("k_scan_tc");
  }
  return FB_OK;
}

}  // namespace fb
