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
#include "fb_ptx.cuh"

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstdio>

namespace fb {
namespace {

using namespace ::fb::dev;

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
constexpr int kLeafStride = 6;  // u64 per leaf in the per-tile leaf-mask stage (48 B: 4 words +
                                // pad, so 32 lanes' 16-B loads spread over 8 bank groups)
constexpr int kRegStack = 4;
constexpr uint32_t kItemBytes = kTileItems * kKBytes;  // 32 KB

struct TcArgs {
  const int8_t* items;    // [n_slots, 128] (survivor scores are recomputed from L2)
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
  const int32_t* plane_list;
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
  int32_t tb_stride;
  int32_t ffirst;     // CNF window form, filter first: 1 always, 0 never, -1 when the sampled
                      // eligibility of the batch is below ff_limit (see k_scan_cnf)
  const uint32_t* sample_cnt;  // [nq] eligible sampled keys per query (nullable)
  float ff_limit;              // sum of sample_cnt under which the batch goes filter-first
  int32_t dbg;        // timing experiments only (FB_SCAN_DEBUG): bit 0 no plane copies,
                      // bit 1 no hit work, bit 2 no column builds, bit 3 no dense work,
                      // bit 7 no gate arm, bit 8 no TMEM drain,
                      // bit 9 no MMA, bit 10 timeline trace (FB_TR)
  const int16_t* col_leaf;
  const uint32_t* qmask;
  const int32_t* qgroups;
  uint32_t off_a, off_b, off_p, off_l, off_ls, off_thr, off_r, off_bar, plane_stage_bytes,
      leaf_stage_bytes, off_hm, off_gate, off_sv, off_id, off_pl;
};


// Timeline trace (compile with -DFB_TRACE, run with FB_SCAN_DEBUG bit 10): CTA 0 records
// clock64 at pipeline events of its first 16 tiles and prints them at exit.
#ifdef FB_TRACE
__device__ long long g_tr[16][16];
__device__ long long g_hit_rounds[8];
#define FB_TR(a, t, e)                                                          \
  do {                                                                          \
    if (((a).dbg & 1024) && blockIdx.x == 0 && (t) < 16 && (threadIdx.x & 31) == 0) \
      g_tr[(t)][(e)] = clock64();                                               \
  } while (0)
#else
#define FB_TR(a, t, e) \
  do {                 \
  } while (0)
#endif







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


// per item stage, written by the producer: the tile's id ranks, its four validity & range
// words and its tile index
constexpr uint32_t kMetaValid = kTileItems * 4;       // 1024
constexpr uint32_t kMetaTile = kMetaValid + 32;       // 1056
constexpr uint32_t kStageMeta = kMetaTile + 32;       // 1088 bytes per stage


// CNF gate tiles (fb_ptx.cuh: gate digits armed by the tensor core)
constexpr uint32_t kGateTileBytes = kMaxQueries * 32;  // 256 rows x 32 B (no swizzle)


// An emission whose slot reservation (atomicAdd) may still be in flight; its stores are
// issued at the lane's next-but-one emission (or at the end), so the round trip overlaps
// the scan.
struct PendingEmit {
  uint64_t key;
  uint32_t p;
  uint32_t slot;
  int32_t q;
};
__device__ __forceinline__ void flush_pending(const TcArgs& a, PendingEmit& pd) {
  if (pd.q >= 0 && pd.p < (uint32_t)a.cap) {
    a.out_key[(int64_t)pd.q * a.cap + pd.p] = pd.key;
    if (a.out_slot) a.out_slot[(int64_t)pd.q * a.cap + pd.p] = pd.slot;
  }
  pd.q = -1;
}


// ---- shared-memory carve-up and barrier slots common to both scan kernels ------------
struct Smem {
  uint8_t* base;
  uint8_t* sA;
  uint8_t* sB;
  uint8_t* sP;
  uint8_t* sL;
  int16_t* sLS;
  uint64_t* sT;
  uint64_t* bars;
};
__device__ __forceinline__ Smem carve(const TcArgs& a) {
  extern __shared__ uint8_t smem_raw[];
  Smem m;
  m.base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  m.sA = m.base + a.off_a;
  m.sB = m.base + a.off_b;
  m.sP = m.base + a.off_p;
  m.sL = m.base + a.off_l;
  m.sLS = reinterpret_cast<int16_t*>(m.base + a.off_ls);
  m.sT = reinterpret_cast<uint64_t*>(m.base + a.off_thr);
  m.bars = reinterpret_cast<uint64_t*>(m.base + a.off_bar);
  return m;
}
// barrier slots (u64 index into bars)
constexpr int kBarItemsFull = 0, kBarItemsEmpty = 4, kBarPlanesFull = 8, kBarPlanesEmpty = 10,
              kBarLeafFull = 12, kBarLeafEmpty = 14, kBarAccFull = 16, kBarAccEmpty = 18,
              kBarTmemSlot = 24, kBarCount = 25;

// queries -> SW128 smem rows (zero rows past the batch), per-row key thresholds
__device__ __forceinline__ void stage_queries(const TcArgs& a, const Smem& m, int nt) {
  const int a_rows = a.n_mblk * kBlockM;
  for (int i = threadIdx.x; i < a_rows * 8; i += nt) {
    const int r = i >> 3, c = i & 7;
    int4 v = make_int4(0, 0, 0, 0);
    if (r < a.nq) v = __ldg(reinterpret_cast<const int4*>(a.queries + (int64_t)r * kKBytes) + c);
    *reinterpret_cast<int4*>(m.sA + r * kKBytes + ((c ^ (r & 7)) << 4)) = v;
  }
  for (int q = threadIdx.x; q < kMaxQueries; q += nt)
    m.sT[q] = (a.threshold != nullptr && q < a.nq) ? a.threshold[q] : 0ull;
  int32_t* pl = reinterpret_cast<int32_t*>(m.base + a.off_pl);
  for (int i = threadIdx.x; i < a.n_planes; i += nt) pl[i] = a.plane_list[i];
}

// Plane stage layout in the CNF kernels: plane slot p's 32-byte tile row as two 16-byte
// halves, swapped when bit 2 of p is set, so the builders' 16-byte loads of 32 random slots
// spread over all eight 16-byte bank groups (not just the even ones)
#ifndef FB_PLANE_SWZ
#define FB_PLANE_SWZ 1
#endif
__device__ __forceinline__ uint32_t plane_half_off(uint32_t slot, uint32_t half) {
  return (2u * slot + (half ^ (FB_PLANE_SWZ ? ((slot >> 2) & 1u) : 0u))) * 16u;
}

// ================= producer (one warp): TMA item tile + Bloom plane words ==============
// The per-tile global reads (work item, then its validity & range words) are issued one
// tile ahead, so their latency never sits on the producer's critical path.
// do_items: TMA item rows + per-tile metadata; do_planes: the plane gather (one warp can
// do both, or two warps split them so the gather never queues behind an item stage).
__device__ __forceinline__ void producer_loop(const TcArgs& a, const CUtensorMap* tmap,
                                              const Smem& m, int lane, bool do_items,
                                              bool do_planes, bool swz = false) {
  uint8_t* smem = m.base;
  uint8_t* sB = m.sB;
  uint8_t* sP = m.sP;
  uint64_t* items_full = m.bars + kBarItemsFull;
  uint64_t* items_empty = m.bars + kBarItemsEmpty;
  uint64_t* planes_full = m.bars + kBarPlanesFull;
  uint64_t* planes_empty = m.bars + kBarPlanesEmpty;
  const int S = a.item_stages;
  const int PS = a.plane_stages;
  const int64_t n_sel = a.n_sel;
  const uint32_t pl_s = su32(m.base + a.off_pl);  // plane ids, staged by stage_queries
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
      if (do_items) {
        // item rows by TMA; alongside, into a stage with the item stage's lifetime: the
        // tile's 256 id ranks (1 KB, 16-byte cp.async), its validity & range words and its
        // tile index (so the epilogue never waits on global memory for per-tile metadata)
        mbar_wait_backoff(items_empty + s, ph ^ 1u);
        FB_TR(a, (int)((i - blockIdx.x) / G), 0);
        if (lane == 0) {
          mbar_expect_tx(items_full + s, kItemBytes);
          tma_load_2d(sB + (size_t)s * kItemBytes, tmap, 0, tile * kTileItems,
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
      if (do_planes && a.has_prog && a.n_planes > 0) {
        mbar_wait_backoff(planes_empty + ps, pph ^ 1u);
        FB_TR(a, (int)((i - blockIdx.x) / G), 10);
        // gather the referenced planes' 32-byte rows for this tile: 16-byte cp.async per
        // lane (two lanes per plane row, a warp covers 16 rows per instruction); each lane
        // arrives on planes_full once its copies land
        const uint32_t dst = su32(sP + (size_t)ps * a.plane_stage_bytes);
        const int64_t col0 = (int64_t)tile * kTileWords;
        // (plane indices fetched eight at a time ahead of the copies: the copies' memory
        // clobber would otherwise serialise each index load behind the previous copy)
        const int n2 = (a.dbg & 1) ? 0 : 2 * a.n_planes;
        for (int e0 = lane; e0 < n2; e0 += 32 * 8) {
          int pl[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + 32 * u;
            pl[u] = e < n2 ? (int)lds32(pl_s + 4u * (uint32_t)(e >> 1)) : 0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int e = e0 + 32 * u;
            if (e < n2) {
              const uint64_t* src = a.planes + (int64_t)pl[u] * a.n_words + col0 + 2 * (e & 1);
              const uint32_t doff = swz ? plane_half_off((uint32_t)(e >> 1), (uint32_t)(e & 1))
                                        : (uint32_t)e * 16u;
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + doff),
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
}

// ================= MMA issuer =============================================================
// kArm: each M-block's accumulator is first set to the row's gate (digits . 127s, K = 32,
// no-swizzle descriptors; the 127 tile is one 256-byte pair of core matrices, SBO = 0).
// kNbAcc (CNF kernel): the whole warp runs the loop and lane 0 issues; an accumulator
// buffer's release by the dense warps is a hardware named barrier (bar.arrive there,
// bar.sync here), so the MMA warp blocks in the barrier unit instead of polling an
// mbarrier -- the poll loop cost ~4.6k issue slots per tile on the scheduler it shares
// with a dense and two hit warps (ncu, round 2).
constexpr int kNbAccEmpty = 9;  // + accumulator buffer (9, 10)
template <bool kArm, bool kNbAcc = false>
__device__ __forceinline__ void mma_loop(const TcArgs& a, const Smem& m, uint32_t tmem_base,
                                         int nb_acc_count = 0) {
  uint64_t* items_full = m.bars + kBarItemsFull;
  uint64_t* items_empty = m.bars + kBarItemsEmpty;
  uint64_t* acc_full = m.bars + kBarAccFull;
  uint64_t* acc_empty = m.bars + kBarAccEmpty;
  constexpr uint32_t idesc = idesc_i8(kBlockM, kTileItems);
  const uint32_t gate_s = su32(m.base + a.off_gate);
  const int S = a.item_stages;
  const bool issuer = !kNbAcc || (threadIdx.x & 31) == 0;
  int acc_it = 0, s = 0;
  uint32_t ph = 0;
  for (int64_t i = blockIdx.x; i < a.n_sel; i += gridDim.x) {
    mbar_wait(items_full + s, ph);
    tc_fence_after();
    FB_TR(a, (int)((i - blockIdx.x) / gridDim.x), 1);
    const uint32_t b_base = su32(m.sB + (size_t)s * kItemBytes);
    for (int mb = 0; mb < a.n_mblk; ++mb, ++acc_it) {
      const int ab = acc_it & 1;
      const uint32_t aph = (uint32_t)(acc_it >> 1) & 1u;
      if (kNbAcc) {
        if (acc_it >= 2) nb_sync(kNbAccEmpty + ab, nb_acc_count);
      } else {
        mbar_wait_idle(acc_empty + ab, aph ^ 1u);
      }
      tc_fence_after();
      if (issuer) {
        const uint32_t a_base = su32(m.sA + mb * kBlockM * kKBytes);
        const uint32_t d = tmem_base + (uint32_t)(ab * kAccCols);
        const bool arm = kArm && !(a.dbg & 128);
        if (arm)
          umma_i8(d, plain_desc(gate_s + (uint32_t)mb * (kBlockM / 8) * 256u, 128u, 256u),
                  plain_desc(gate_s + kGateTileBytes, 128u, 0u), idesc, 0u);
#pragma unroll
        for (int kk = 0; kk < ((a.dbg & 512) ? 0 : kKBytes / kUmmaK); ++kk)
          umma_i8(d, sw128_desc(a_base + kk * kUmmaK), sw128_desc(b_base + kk * kUmmaK), idesc,
                  (kk > 0 || arm) ? 1u : 0u);
        umma_commit(acc_full + ab);
      }
      if (kNbAcc) __syncwarp();
      if (mb == 0) FB_TR(a, (int)((i - blockIdx.x) / gridDim.x), 2);
    }
    if (issuer) umma_commit(items_empty + s);
    if (++s == S) { s = 0; ph ^= 1u; }
  }
  if (kNbAcc)  // retire the dense warps' releases of the last two buffers
    for (int t = acc_it; t < acc_it + 2; ++t)
      if (t >= 2) nb_sync(kNbAccEmpty + (t & 1), nb_acc_count);
}

// ---- CNF kernel warp layout (see k_scan_cnf) ----
constexpr int kCnfThreads = 640;
constexpr int kCnfBuilders = 5;
constexpr int kCnfDense0 = 8;
constexpr int kCnfDenseWarps = 4;
constexpr int kCnfHit0 = 12;
constexpr int kCnfHitWarps = 8;
#ifndef FB_HM_EARLY
#define FB_HM_EARLY 1  // modes 3 / 4: release the hit map right after the words are read
#endif
#ifndef FB_HIT_TAKE
#define FB_HIT_TAKE 3  // mode 3: hits taken per lane and round (with the early hit-map release: 3: 1.004 ms, 4: 1.022, 5: 1.019)
#endif
constexpr int kSurvCap = FB_HIT_TAKE >= 5 ? 192 : FB_HIT_TAKE >= 4 ? 160 : 128;  // u16 survivor entries per hit warp: (lane << 8) | item
// named barrier ids (0 is __syncthreads) and their thread counts
constexpr int kNbHmFull = 1, kNbHmEmpty = 3, kNbLeafFull = 5, kNbLeafEmpty = 7;  // + stage
constexpr int kNbHmCount = 32 * (kCnfDenseWarps + kCnfHitWarps);
constexpr int kNbAccCount = 32 * (kCnfDenseWarps + 1);  // dense warps arrive, MMA warp syncs
constexpr int kNbLeafCount = 32 * (kCnfBuilders + kCnfHitWarps);

// ================= CNF column builders (nb warps): Bloom test per literal column, then a
// 32x32 bit transpose so each item row holds its column bits ==========================

struct NoTail {
  __device__ void operator()(int) const {}
};
// tail(it) runs after the builders have published tile it + 1's column bits (and once more
// after the last tile): mode 3 drains tile it's survivors there
template <typename Tail = NoTail>
__device__ __forceinline__ void cnf_builder_loop(const TcArgs& a, const Smem& m, int lw, int nb,
                                                 int lane, bool ff, int leaf_count = kNbLeafCount,
                                                 Tail tail = Tail()) {
  constexpr bool kDrain = !std::is_same<Tail, NoTail>::value;
  uint8_t* sP = m.sP;
  uint8_t* sL = m.sL;
  const int16_t* sLS = m.sLS;
  uint64_t* planes_full = m.bars + kBarPlanesFull;
  uint64_t* planes_empty = m.bars + kBarPlanesEmpty;
  const int PS = a.plane_stages;
  const int64_t n_sel = a.n_sel;
    int it = 0, ps = 0;
    uint32_t pph = 0;
    for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
      const int st = it & 1;
      const uint32_t ph = (uint32_t)(it >> 1) & 1u;
      (void)ph;
      mbar_wait_backoff(planes_full + ps, pph);  // a plane stage lands ~1 tile ahead
      if (it >= 2) nb_sync(kNbLeafEmpty + st, leaf_count);
      if (kDrain && lw == 0) FB_TR(a, it, 12);
      const uint32_t p_s = su32(sP + (size_t)ps * a.plane_stage_bytes);
      uint32_t* TB = reinterpret_cast<uint32_t*>(sL + (size_t)st * a.leaf_stage_bytes);
      const uint32_t sls_s = su32(sLS);
      for (int cb = lw; cb < ((a.dbg & 4) ? 0 : a.cnf_words); cb += nb) {  // 32-column block
        const int col = cb * 32 + lane;
        // the column's 256 tile bits: AND of its planes' 32-byte rows (8 x u32, one per
        // 32-item block); all loads are independent
        uint32_t m[8];
#pragma unroll
        for (int ib = 0; ib < 8; ++ib) m[ib] = col < a.n_cols ? ~0u : 0u;
        if (col < a.n_cols) {
          bool neg = false;
          for (int j = 0; j < a.k_max; ++j) {
            int sl = (int)(int16_t)lds16(sls_s + 2u * (uint32_t)(col * a.k_max + j));
            if (j == 0) {
              neg = (sl & 0x4000) != 0;
              sl &= ~0x4000;
            }
            if (sl < 0) break;
            const uint4 lo = lds128(p_s + plane_half_off((uint32_t)sl, 0u));
            const uint4 hi = lds128(p_s + plane_half_off((uint32_t)sl, 1u));
            m[0] &= lo.x; m[1] &= lo.y; m[2] &= lo.z; m[3] &= lo.w;
            m[4] &= hi.x; m[5] &= hi.y; m[6] &= hi.z; m[7] &= hi.w;
          }
          if (neg) {
#pragma unroll
            for (int ib = 0; ib < 8; ++ib) m[ib] = ~m[ib];
          }
        }
        if (ff) {  // filter-first: the column's 256 tile bits, column-major
          const uint32_t cw = su32(TB) + (uint32_t)col * 32u;
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(cw), "r"(m[0]), "r"(m[1]),
                       "r"(m[2]), "r"(m[3])
                       : "memory");
          asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(cw + 16u), "r"(m[4]),
                       "r"(m[5]), "r"(m[6]), "r"(m[7])
                       : "memory");
          continue;
        }
        // eight 32x32 transposes in lockstep (independent shuffles per round). Per word and
        // round: the partner's word rotated by s (left in the lower lane of a pair, right in
        // the upper) lands its exchanged bit blocks in place, so one SHFL + one rotate + one
        // LOP3 (keep = the lane's own blocks) does the round
        const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const int sft = 16 >> k;
          const bool upper = (lane & sft) != 0;
          const uint32_t keep = upper ? ~masks[k] : masks[k];
          const uint32_t amt = upper ? (uint32_t)(32 - sft) : (uint32_t)sft;
#pragma unroll
          for (int ib = 0; ib < 8; ++ib) {
            const uint32_t y = __shfl_xor_sync(0xffffffffu, m[ib], sft);
            const uint32_t rot = __funnelshift_l(y, y, amt);
            m[ib] = (m[ib] & keep) | (rot & ~keep);
          }
        }
#pragma unroll
        for (int ib = 0; ib < 8; ++ib) TB[(ib * 32 + lane) * a.tb_stride + cb] = m[ib];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(planes_empty + ps);  // one arrival per builder warp
      nb_arrive(kNbLeafFull + st, leaf_count);
      if (++ps == PS) { ps = 0; pph ^= 1u; }
      if constexpr (kDrain) {
        if (lw == 0) FB_TR(a, it, 13);
        if (it >= 1) tail(it - 1);
        if (lw == 0 && it >= 1) FB_TR(a, it - 1, 14);
      }
    }
    if constexpr (kDrain) {
      if (it >= 1) tail(it - 1);
    }
    // retire the hit pass's releases of the last two stages (every barrier phase completes)
    for (int t = it; t < it + 2; ++t)
      if (t >= 2) nb_sync(kNbLeafEmpty + (t & 1), leaf_count);
}

// ---- tensor memory -----------------------------------------------------------------------
__device__ __forceinline__ uint32_t tmem_alloc512(const Smem& m) {
  uint32_t* slot = reinterpret_cast<uint32_t*>(m.bars + kBarTmemSlot);
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   su32(slot)),
               "r"(512)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  return 0;
}

// ======================================================================================
// Bytecode scan kernel: any filter program (stack depth <= 4) evaluated word-wise per
// (query, 128 items) from per-tile leaf masks; also the threshold-0 sampling pass.
// ======================================================================================
__global__ void __launch_bounds__(kThreads, 1)
    k_scan_tc(const __grid_constant__ CUtensorMap tmap_items, const TcArgs a) {
  constexpr int NT = kThreads;
  constexpr int NE = kEpiWarps;
  const Smem m = carve(a);
  uint8_t* smem = m.base;
  uint8_t* sA = m.sA;
  uint8_t* sB = m.sB;
  uint8_t* sP = m.sP;
  uint8_t* sL = m.sL;
  int16_t* sLS = m.sLS;
  uint64_t* sT = m.sT;
  uint64_t* bars = m.bars;
  uint64_t* items_full = bars + kBarItemsFull;
  uint64_t* items_empty = bars + kBarItemsEmpty;
  uint64_t* planes_full = bars + kBarPlanesFull;
  uint64_t* planes_empty = bars + kBarPlanesEmpty;
  uint64_t* leaf_full = bars + kBarLeafFull;
  uint64_t* leaf_empty = bars + kBarLeafEmpty;
  uint64_t* acc_full = bars + kBarAccFull;
  uint64_t* acc_empty = bars + kBarAccEmpty;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kBarTmemSlot);
  (void)sA;
  (void)sB;
  (void)items_full;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int PS = a.plane_stages;
  const int64_t n_sel = a.n_sel;

  // ---- prologue: queries, thresholds, leaf table, filter programs ----
  stage_queries(a, m, NT);
  int32_t prog_off0 = 0;
  bool prog_staged = false;
  if (a.has_prog) {
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
      mbar_init(items_empty + s, 1 + NE);     // MMA commit + every epilogue warp (id stage)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(planes_full + s, 32);  // one cp.async.mbarrier.arrive per producer lane
      mbar_init(planes_empty + s, kLeafThreads);
      mbar_init(leaf_full + s, kLeafThreads);
      mbar_init(leaf_empty + s, NE);
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, NE);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(m);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    producer_loop(a, &tmap_items, m, lane, true, true);
  } else if (warp == 1) {
    if (lane == 0) mma_loop<false>(a, m, tmem_base);
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
      const uint32_t id_s = su32(smem + a.off_id) + (uint32_t)s * kStageMeta +
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
                if (osp == nullptr && p + 32u <= cap) {
                  // the sampling pass (no slots, room for the whole word): keys only
#pragma unroll
                  for (int j = 0; j < 32; ++j) {
                    const bool on = ((cm >> j) & 1u) != 0u;
                    if (on) okp[p] = make_key(r[j], lds32(ids + 4u * j));
                    p += on ? 1u : 0u;
                  }
                } else {
#pragma unroll
                  for (int j = 0; j < 32; ++j) {
                    const bool on = ((cm >> j) & 1u) != 0u;
                    if (on && p < cap) {
                      okp[p] = make_key(r[j], lds32(ids + 4u * j));
                      if (osp != nullptr) osp[p] = slot0 + (uint32_t)j;
                    }
                    p += on ? 1u : 0u;
                  }
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

// ======================================================================================
// CNF scan kernel (every program an AND of OR-groups of literals). Twenty warps:
//   warp 0       item producer (TMA item rows, per-tile id ranks / validity / tile index)
//   warp 1       MMA: per M-block the gate-arming K=32 MMA, then 4 K-steps of kind::i8
//   warp 2       plane producer (cp.async gather of the batch's planes, 32 B per tile)
//   warps 3-7    column builders: per literal column the AND of its planes, transposed so
//                each item row holds its column bits (the paper's and.b64 Bloom test)
//   warps 8-11   dense pass, one per TMEM lane quadrant: tcgen05.ld 32 columns (double
//                buffered), the hit mask is the accumulators' sign bits (armed at +127 D),
//                & validity/range; 32-bit hit masks go to a double-buffered [chunk][query]
//                map in smem and the accumulator is released at once
//   warps 12-19  hit pass, lane = query: walks its hit bits, tests the CNF filter against
//                the item's column bits (window form: 4 groups x one u32 pair, masks in
//                registers), queues survivors per warp; survivors get their exact score
//                from the resident smem tiles (dp4a), the exact key test and an atomic
//                slot reservation -- filtered-out items never leave the SM.
// ======================================================================================
constexpr uint32_t kHmapBytes = 8u * kMaxQueries * 4u;  // [chunk][query] u32


// General-form filter test: masks read (L1-cached) from the batch's qmask rows.
__device__ __forceinline__ bool cnf_test_global(uint32_t tb_addr, const uint32_t* qm, int ng,
                                                int words) {
  const uint4 t0 = lds128(tb_addr);
  const uint4 t1 = lds128(tb_addr + 16u);
  const uint32_t t[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
  bool pass = true;
  for (int g = 0; g < ng && pass; ++g) {
    uint32_t x = 0u;
#pragma unroll
    for (int w = 0; w < 8; ++w)
      if (w < words) x |= t[w] & __ldg(qm + g * words + w);
    pass = x != 0u;
  }
  return pass;
}

// Survivors queued by one hit warp: exact score from the smem tiles, exact key test against
// the query's threshold, slot reservation (the stores trail by two emissions per lane).
struct EmitState {
  PendingEmit pa, pb;
  bool par;
};
__device__ __forceinline__ void emit_one(const TcArgs& a, EmitState& e, int q, uint64_t key,
                                         uint32_t slot) {
  if (e.par) {
    flush_pending(a, e.pa);
    e.pa.p = atomicAdd(a.out_cnt + q, 1u);
    e.pa.key = key;
    e.pa.slot = slot;
    e.pa.q = q;
  } else {
    flush_pending(a, e.pb);
    e.pb.p = atomicAdd(a.out_cnt + q, 1u);
    e.pb.key = key;
    e.pb.slot = slot;
    e.pb.q = q;
  }
  e.par = !e.par;
}
__device__ __forceinline__ void drain_survivors(const TcArgs& a, const Smem& m, EmitState& e,
                                                uint32_t sv_s, uint32_t n, int qbase,
                                                uint32_t b_s, uint32_t mst, int64_t tile,
                                                int lane) {
  if (a.dbg & 4096) return;  // timing only: survivors dropped
  for (uint32_t i = (uint32_t)lane; i < n; i += 32u) {
    const uint32_t ent = lds16(sv_s + 2u * i);
    const int q = qbase + (int)(ent >> 8);
    const uint32_t item = ent & 255u;
    const int32_t score = smem_dot(su32(m.sA) + (uint32_t)q * kKBytes, (uint32_t)q & 7u,
                                   b_s + item * kKBytes, item & 7u);
    const uint64_t key = make_key(score, lds32(mst + 4u * item));
    if (key >= m.sT[q] && !(a.dbg & 8192)) emit_one(a, e, q, key, (uint32_t)(tile * kTileItems) + item);
  }
}

// ---- mode 3 (window form, two M-blocks): 24 warps -------------------------------------
// Eight dense warps instead of four: warp (mb, quad) drains accumulator buffer mb (M-block mb
// of every tile) in TMEM lane quadrant quad, so two warps per scheduler overlap their
// tcgen05.ld round trips and each warp's per-tile chain is half as long (ncu, round 2: the
// four-warp dense pass was the critical path -- ~760 dependent instructions per warp per
// tile). The other roles are mode 1's. 768 threads = six warps per scheduler, so 80
// registers each (16K per scheduler): the dense warps load one 32-column chunk at a time
// (FB_C3_DBUF=1 builds the double-buffered variant).
// Survivors (gate hit + filter pass) of a tile are handed to the column builders, which
// are idle most of each period: the hit warps queue them per tile (double-buffered lists),
// the builders compute the exact scores and emit them after building the next tile.
#ifndef FB_C3_HANDOFF
#define FB_C3_HANDOFF 1
#endif
constexpr int kNbSvFull = 11, kNbSvEmpty = 13;  // + tile parity
constexpr int kNbSvCount = 32 * (kCnfBuilders + kCnfHitWarps);
constexpr uint32_t kSvListBytes = kSurvCap * 2u;  // per hit warp and parity
constexpr uint32_t kSvBytes = 2u * kCnfHitWarps * kSvListBytes + 2u * kCnfHitWarps * 4u;
constexpr int kCnf3Threads = 768;
constexpr int kC3DenseWarps = 8;
constexpr int kC3Builders = 5;
#ifndef FB_C3_DBUF
#define FB_C3_DBUF 0
#endif

__device__ __forceinline__ void cnf3_dense_loop(const TcArgs& a, const Smem& m, uint32_t tmem_base,
                                                uint32_t hm_s, int warp, int lane, int hm_count) {
  uint64_t* items_full = m.bars + kBarItemsFull;
  uint64_t* acc_full = m.bars + kBarAccFull;
  const int quad = warp & 3;
  const int mb = (warp - kCnfDense0) >> 2;  // dense warps 8..15
  const int row = quad * 32 + lane;
  const int q = mb * kBlockM + row;
  const bool qok = q < a.nq;
  bool all = false;
  (void)gate_digits(qok ? m.sT[q] : ~0ull, all);
  const uint32_t allmask = all ? ~0u : 0u;
  int it = 0, s = 0;
  uint32_t iph = 0;
  for (int64_t i = blockIdx.x; i < a.n_sel; i += gridDim.x, ++it) {
    mbar_wait(items_full + s, iph);
    const uint32_t mst = su32(m.base + a.off_id) + (uint32_t)s * kStageMeta;
    const int64_t tile = (int64_t)lds32(mst + kMetaTile);
    const uint32_t vchunk = lane < 8 ? lds32(mst + kMetaValid + 4u * lane) : 0u;
    if (++s == a.item_stages) {
      s = 0;
      iph ^= 1u;
    }
    const int hb = it & 1;
    if (it >= 2) nb_sync(kNbHmEmpty + hb, hm_count);
    const uint32_t hmap = hm_s + (uint32_t)hb * kHmapBytes + 4u * (uint32_t)q;
    mbar_wait(acc_full + mb, (uint32_t)it & 1u);
    tc_fence_after();
    if (quad == 0) FB_TR(a, it, mb ? 6 : 4);
    const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(mb * kAccCols);
    auto chunk_mask = [&](int c, const int32_t (&r)[32]) -> uint32_t {
      uint32_t em = __shfl_sync(0xffffffffu, vchunk, c);
      if (!qok) em = 0u;
      if (a.masks != nullptr && em != 0u)
        em &= (uint32_t)(__ldg(a.masks + (int64_t)q * a.n_words + tile * kTileWords + (c >> 1)) >>
                         (32 * (c & 1)));
      return (a.dbg & 8) ? 0u : (nonneg_mask32(r) | allmask) & em;
    };
#if FB_C3_DBUF
    int32_t ra[32], rb[32];
    tmem_ld32_async(taddr, ra);
#pragma unroll 1
    for (int c = 0; c < 8; c += 2) {
      tmem_wait32(ra);
      tmem_ld32_async(taddr + (uint32_t)((c + 1) * 32), rb);
      sts32(hmap + (uint32_t)c * (kMaxQueries * 4u), chunk_mask(c, ra));
      tmem_wait32(rb);
      if (c + 2 < 8) tmem_ld32_async(taddr + (uint32_t)((c + 2) * 32), ra);
      sts32(hmap + (uint32_t)(c + 1) * (kMaxQueries * 4u), chunk_mask(c + 1, rb));
    }
#else
#pragma unroll 1
    for (int c = 0; c < 8; ++c) {
      int32_t r[32];
      tmem_ld32_async(taddr + (uint32_t)(c * 32), r);
      tmem_wait32(r);
      sts32(hmap + (uint32_t)c * (kMaxQueries * 4u), chunk_mask(c, r));
    }
#endif
    tc_fence_before();
    nb_arrive(kNbAccEmpty + mb, kNbAccCount);  // the MMA warp bar.syncs on it
    if (quad == 0) FB_TR(a, it, mb ? 7 : 5);
    __syncwarp();
    nb_arrive(kNbHmFull + hb, hm_count);
  }
  for (int t = it; t < it + 2; ++t)
    if (t >= 2) nb_sync(kNbHmEmpty + (t & 1), hm_count);
}

// Builders' share of a mode-3 tile: the survivors the hit warps queued for tile `it`
// (item stage s). Builder warp w takes hit lists w and w + 5 (< 8) as one index space.
__device__ __forceinline__ void cnf3_builder_drain(const TcArgs& a, const Smem& m, EmitState& e,
                                                   int it, int lw, int lane) {
  const int par = it & 1;
  const int s = it % a.item_stages;
  const uint32_t sv0 = su32(m.base + a.off_sv);
  const uint32_t cnt_s = sv0 + 2u * kCnfHitWarps * kSvListBytes + (uint32_t)par * kCnfHitWarps * 4u;
  const int la = lw, lb = lw + kCnfBuilders;
  const uint32_t na = lds32(cnt_s + 4u * (uint32_t)la);
  const uint32_t nb = lb < kCnfHitWarps ? lds32(cnt_s + 4u * (uint32_t)lb) : 0u;
  const uint32_t mst = su32(m.base + a.off_id) + (uint32_t)s * kStageMeta;
  const int64_t tile = (int64_t)lds32(mst + kMetaTile);
  const uint32_t b_s = su32(m.sB + (size_t)s * kItemBytes);
  if (a.dbg & 4096) return;
  for (uint32_t i = (uint32_t)lane; i < na + nb; i += 32u) {
    const bool in_a = i < na;
    const int l = in_a ? la : lb;
    const uint32_t ent =
        lds16(sv0 + ((uint32_t)par * kCnfHitWarps + (uint32_t)l) * kSvListBytes + 2u * (in_a ? i : i - na));
    const int q = l * 32 + (int)(ent >> 8);
    const uint32_t item = ent & 255u;
    const int32_t score = smem_dot(su32(m.sA) + (uint32_t)q * kKBytes, (uint32_t)q & 7u,
                                   b_s + item * kKBytes, item & 7u);
    const uint64_t key = make_key(score, lds32(mst + 4u * item));
    if (key >= m.sT[q] && !(a.dbg & 8192)) emit_one(a, e, q, key, (uint32_t)(tile * kTileItems) + item);
  }
}

// kMode: 0 general CNF form; 1 window form. A window-form launch runs one of two hit passes,
// chosen per launch from the sampling pass (uniform across CTAs):
//  * per hit: each gate hit is tested on the item's item-major column bits;
//  * filter first (low-selectivity batches, where the score gate admits ~k / selectivity hits
//    per query): the builders leave column-major column words, each hit warp lane builds its
//    query's eligibility words AND_g OR_{c in S_qg} col_c for the tile's eight chunks and ANDs
//    them into the hit words, so only eligible hits reach the exact test.
template <int kMode>
__global__ void __launch_bounds__(kMode >= 3 ? kCnf3Threads : kCnfThreads)
    __maxnreg__(kMode >= 3 ? 80 : 96) k_scan_cnf(const __grid_constant__ CUtensorMap tmap_items, const TcArgs a) {
  constexpr bool kWin = kMode != 0;
  constexpr bool ff = kMode == 2 || kMode == 4;
  constexpr bool kL3 = kMode >= 3;  // 24-warp layout (mode 3 per-hit, mode 4 filter-first)
  if (kWin && a.ffirst < 0) {
    // both window-form instances are launched; the one the sampled eligibility does not pick
    // returns at once (uniform across CTAs: every CTA sums the same counts)
    float sum = 0.f;
    for (int q = threadIdx.x & 31; q < a.nq; q += 32) sum += (float)a.sample_cnt[q];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
    if ((sum < a.ff_limit) != ff) return;
  }
  constexpr int NT = kL3 ? kCnf3Threads : kCnfThreads;
  constexpr int kDenseN = kL3 ? kC3DenseWarps : kCnfDenseWarps;
  constexpr int kBuildN = kL3 ? kC3Builders : kCnfBuilders;
  constexpr int kDense0 = 3 + kBuildN;
  constexpr int kHit0 = kDense0 + kDenseN;
  constexpr int kHmCount = 32 * (kDenseN + kCnfHitWarps);
  constexpr int kLeafCount = 32 * (kBuildN + kCnfHitWarps);
  constexpr bool kHand = kL3 && FB_C3_HANDOFF;  // survivors drained by the builders
  static_assert(32 * (kHit0 + kCnfHitWarps) == NT, "warp layout");
  const Smem m = carve(a);
  uint8_t* smem = m.base;
  uint64_t* bars = m.bars;
  uint64_t* items_full = bars + kBarItemsFull;
  uint64_t* items_empty = bars + kBarItemsEmpty;
  uint64_t* planes_full = bars + kBarPlanesFull;
  uint64_t* planes_empty = bars + kBarPlanesEmpty;
  uint64_t* acc_full = bars + kBarAccFull;
  uint64_t* acc_empty = bars + kBarAccEmpty;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kBarTmemSlot);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_sel = a.n_sel;

  // ---- prologue: queries, thresholds, column table, zeroed column-bit stages, gate tiles
  stage_queries(a, m, NT);
  for (int i = threadIdx.x; i < a.n_cols * a.k_max; i += NT) {
    // column -> plane-slot table (negated columns flagged by bit 14 on slot 0)
    const int c = i / a.k_max, j = i - c * a.k_max;
    const int cl = a.col_leaf[c];
    const int leaf = cl >= 0 ? cl : ~cl;
    int s = a.leaf_slot[leaf * a.k_max + j];
    if (j == 0 && cl < 0) s |= 0x4000;
    m.sLS[i] = (int16_t)s;
  }
  {
    uint32_t* tb = reinterpret_cast<uint32_t*>(m.sL);
    for (int i = threadIdx.x; i < 2 * (int)(a.leaf_stage_bytes / 4); i += NT) tb[i] = 0u;
    uint8_t* gA = smem + a.off_gate;
    uint32_t* gB = reinterpret_cast<uint32_t*>(smem + a.off_gate + kGateTileBytes);
    for (int i = threadIdx.x; i < 64; i += NT) gB[i] = 0x7F7F7F7Fu;  // 256 B of 127s
    for (int r = threadIdx.x; r < kMaxQueries; r += NT) {
      bool all;
      const uint64_t T = (a.threshold != nullptr && r < a.nq) ? a.threshold[r] : 0ull;
      const int32_t D = r < a.nq ? gate_digits(T, all) : kGateDigitsMin;
      const int32_t base = D >= 0 ? D / 32 : -((-D + 31) / 32);  // floor(D / 32)
      const int32_t rem = D - 32 * base;                        // 0..31
      for (int k = 0; k < 32; ++k)
        gA[gate_off(r, k)] = (uint8_t)(int8_t)(base + (k < rem ? 1 : 0));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(items_full + s, 1 + 32 + 1);          // TMA expect-tx, id ranks, meta
      // MMA commit + hit warps (B tile, ids) [+ builders: mode 3 drains survivors there]
      mbar_init(items_empty + s, 1 + kCnfHitWarps + (kHand ? kCnfBuilders : 0));
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(planes_full + s, 32);
      mbar_init(planes_empty + s, kBuildN);
      mbar_init(acc_full + s, 1);
      mbar_init(acc_empty + s, kCnfDenseWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc512(m);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t hm_s = su32(smem + a.off_hm);

  if (warp == 0) {
    producer_loop(a, &tmap_items, m, lane, true, false);
  } else if (warp == 1) {
    mma_loop<true, true>(a, m, tmem_base, kNbAccCount);
  } else if (warp == 2) {
    producer_loop(a, &tmap_items, m, lane, false, true, true);
  } else if (warp < kDense0) {
    if constexpr (kHand) {
      EmitState be;
      be.pa.q = be.pb.q = -1;
      be.pa.p = be.pb.p = 0u;
      be.pa.key = be.pb.key = 0ull;
      be.pa.slot = be.pb.slot = 0u;
      be.par = false;
      const int lw = warp - 3;
      auto tail = [&](int t) {
        const int par = t & 1;
        nb_sync(kNbSvFull + par, kNbSvCount);
        if (lw == 0) FB_TR(a, t, 15);
        cnf3_builder_drain(a, m, be, t, lw, lane);
        __syncwarp();
        nb_arrive(kNbSvEmpty + par, kNbSvCount);
        if (lane == 0) mbar_arrive(items_empty + (t % a.item_stages));
      };
      cnf_builder_loop(a, m, lw, kBuildN, lane, ff, kLeafCount, tail);
      flush_pending(a, be.pa);
      flush_pending(a, be.pb);
    } else {
      cnf_builder_loop(a, m, warp - 3, kBuildN, lane, ff, kLeafCount);
    }
  } else if (kL3 && warp < kHit0) {
    cnf3_dense_loop(a, m, tmem_base, hm_s, warp, lane, kHmCount);
  } else if (warp < kHit0) {
    // ================= dense pass (one warp per TMEM lane quadrant) ======================
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    // per-row gate constants of both M-blocks, fixed for the whole launch
    uint32_t allm[2];
    int32_t Dm[2];
#pragma unroll
    for (int mb = 0; mb < 2; ++mb) {
      const int q = mb * kBlockM + row;
      bool all = false;
      Dm[mb] = mb < a.n_mblk ? gate_digits(q < a.nq ? m.sT[q] : ~0ull, all) : 0;
      allm[mb] = all ? ~0u : 0u;
    }
    int it = 0, acc_it = 0, s = 0;
    uint32_t iph = 0;
    for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
      mbar_wait(items_full + s, iph);
      const uint32_t mst = su32(smem + a.off_id) + (uint32_t)s * kStageMeta;
      const int64_t tile = (int64_t)lds32(mst + kMetaTile);
      // lane c < 8 holds the validity & range bits of the tile's chunk c (32 items)
      const uint32_t vchunk = lane < 8 ? lds32(mst + kMetaValid + 4u * lane) : 0u;
      if (++s == a.item_stages) {
        s = 0;
        iph ^= 1u;
      }
      const int hb = it & 1;
      if (quad == 0) FB_TR(a, it, 12);
      if (it >= 2) nb_sync(kNbHmEmpty + hb, kHmCount);
      if (quad == 0) FB_TR(a, it, 13);
      const uint32_t hmap = hm_s + (uint32_t)hb * kHmapBytes;
#pragma unroll 1
      for (int mb = 0; mb < a.n_mblk; ++mb, ++acc_it) {
        const int q = mb * kBlockM + row;
        const bool qok = q < a.nq;
        const int32_t D = mb == 0 ? Dm[0] : Dm[1];
        const uint32_t allmask = mb == 0 ? allm[0] : allm[1];
        const int ab = acc_it & 1;
        if (quad == 0 && mb == 0) FB_TR(a, it, 14);
        mbar_wait(acc_full + ab, (uint32_t)(acc_it >> 1) & 1u);
        tc_fence_after();
        if (quad == 0) FB_TR(a, it, 4 + 2 * mb);
        const uint32_t taddr =
            tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(ab * kAccCols);
        // hit mask of chunk c from its 32 accumulators (validity, range, explicit mask)
        auto chunk_mask = [&](int c, const int32_t (&r)[32]) -> uint32_t {
          uint32_t em = __shfl_sync(0xffffffffu, vchunk, c);
          if (!qok) em = 0u;
          if (a.masks != nullptr && em != 0u)
            em &= (uint32_t)(__ldg(a.masks + (int64_t)q * a.n_words + tile * kTileWords +
                                   (c >> 1)) >>
                             (32 * (c & 1)));
          if (a.dump != nullptr && qok) {
            const int64_t base = tile * kTileItems + c * 32;
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (base + j < a.dump_ld)
                a.dump[(int64_t)q * a.dump_ld + base + j] = r[j] - 127 * D;
          }
          return (a.dbg & 8) ? 0u : (nonneg_mask32(r) | allmask) & em;
        };
        // two register buffers: chunk c + 1 loads while chunk c is reduced to its mask
        int32_t ra[32], rb[32];
        tmem_ld32_async(taddr, ra);
#pragma unroll 1
        for (int c = 0; c < ((a.dbg & 256) ? 0 : 8); c += 2) {
          tmem_wait32(ra);
          tmem_ld32_async(taddr + (uint32_t)((c + 1) * 32), rb);
          sts32(hmap + (uint32_t)(c * kMaxQueries + q) * 4u, chunk_mask(c, ra));
          tmem_wait32(rb);
          if (c + 2 < 8) tmem_ld32_async(taddr + (uint32_t)((c + 2) * 32), ra);
          sts32(hmap + (uint32_t)((c + 1) * kMaxQueries + q) * 4u, chunk_mask(c + 1, rb));
        }
        tc_fence_before();
        nb_arrive(kNbAccEmpty + ab, kNbAccCount);  // the MMA warp bar.syncs on it
        if (quad == 0) FB_TR(a, it, 5 + 2 * mb);
      }
      __syncwarp();
      nb_arrive(kNbHmFull + hb, kHmCount);
    }
    for (int t = it; t < it + 2; ++t)
      if (t >= 2) nb_sync(kNbHmEmpty + (t & 1), kHmCount);
  } else {
    // ================= hit pass (lane = query) =========================================
    const int qbase = (warp - kHit0) * 32;
    const int q = qbase + lane;
    const bool qok = q < a.nq;
    const uint64_t T = qok ? m.sT[q] : ~0ull;
    (void)T;
    const int ng = qok ? a.qgroups[q] : 0;
    const bool nof = ng == 0;
    // window form: per group (byte offset of its u32 pair in an item row, 64-bit mask);
    // unused groups repeat group 0 (AND is idempotent)
    uint32_t wo[4] = {0u, 0u, 0u, 0u}, lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u};
    const uint32_t* qmg = a.qmask + (int64_t)(qok ? q : 0) * a.cnf_gmax * a.cnf_words;
    if (kWin && !nof) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const uint32_t* mg = qmg + (g < ng ? g : 0) * a.cnf_words;
        int w0 = 0;
        while (w0 < a.cnf_words - 1 && mg[w0] == 0u) ++w0;
        w0 &= ~1;
        wo[g] = 4u * (uint32_t)w0;
        lo[g] = mg[w0];
        hi[g] = w0 + 1 < a.cnf_words ? mg[w0 + 1] : 0u;
      }
    }
    const uint32_t sv_base = su32(smem + a.off_sv) + (uint32_t)(warp - kHit0) * kSvListBytes;
    EmitState e;
    e.pa.q = e.pb.q = -1;
    e.pa.p = e.pb.p = 0u;
    e.pa.key = e.pb.key = 0ull;
    e.pa.slot = e.pb.slot = 0u;
    e.par = false;
    int it = 0, s = 0;
    uint32_t iph = 0;
    for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
      mbar_wait(items_full + s, iph);
      const uint32_t mst = su32(smem + a.off_id) + (uint32_t)s * kStageMeta;
      const int64_t tile = (int64_t)lds32(mst + kMetaTile);
      const uint32_t b_s = su32(m.sB + (size_t)s * kItemBytes);
      const int st = it & 1;
      nb_sync(kNbLeafFull + st, kLeafCount);
      const uint32_t tb_s = su32(m.sL + (size_t)st * a.leaf_stage_bytes);
      const int hb = it & 1;
      nb_sync(kNbHmFull + hb, kHmCount);
      if (warp == kHit0) FB_TR(a, it, 8);
      // mode 3: this tile's survivor list (the builders drain it after building the next tile)
      const uint32_t sv_s = sv_base + (kHand ? (uint32_t)(it & 1) * kCnfHitWarps * kSvListBytes : 0u);
      if (kHand && it >= 2) nb_sync(kNbSvEmpty + (it & 1), kNbSvCount);
      const uint32_t hmap = hm_s + (uint32_t)hb * kHmapBytes + 4u * (uint32_t)q;
      // this query's nonzero chunk words
      uint32_t nzm = 0u;
      uint32_t fw[8];  // filter-first: eligibility words of the tile's eight chunks
#pragma unroll
      for (int c = 0; c < 8; ++c) fw[c] = ~0u;
      if (ff && qok && !nof && !(a.dbg & 2)) {
        // AND over the query's groups of the OR of its literal columns (window form: group g's
        // columns are 8 * wo[g] + j, j < 64, flagged in lo / hi)
        const uint32_t cw0 = tb_s;
        for (int g = 0; g < ng && g < 4; ++g) {
          uint32_t acc[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] = 0u;
          const uint32_t glo = g == 0 ? lo[0] : g == 1 ? lo[1] : g == 2 ? lo[2] : lo[3];
          const uint32_t ghi = g == 0 ? hi[0] : g == 1 ? hi[1] : g == 2 ? hi[2] : hi[3];
          const uint32_t gwo = g == 0 ? wo[0] : g == 1 ? wo[1] : g == 2 ? wo[2] : wo[3];
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            uint32_t x = half ? ghi : glo;
            const uint32_t cbase = cw0 + (8u * gwo + 32u * (uint32_t)half) * 32u;
            while (x != 0u) {
              const uint32_t j = (uint32_t)(__ffs(x) - 1);
              x &= x - 1u;
              const uint4 u0 = lds128(cbase + j * 32u), u1 = lds128(cbase + j * 32u + 16u);
              acc[0] |= u0.x; acc[1] |= u0.y; acc[2] |= u0.z; acc[3] |= u0.w;
              acc[4] |= u1.x; acc[5] |= u1.y; acc[6] |= u1.z; acc[7] |= u1.w;
            }
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) fw[c] &= acc[c];
        }
      }
      uint32_t mw[8];
      if (qok && !(a.dbg & 2)) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          mw[c] = lds32(hmap + (uint32_t)c * (kMaxQueries * 4u)) & fw[c];
          nzm |= (mw[c] != 0u ? 1u : 0u) << c;
        }
      }
      if (a.dbg & 16384) nzm &= 0x0Fu;  // timing only: walk half the chunks (wrong results)
#if FB_HM_EARLY
      if constexpr (kMode >= 3) {
        // the walk reads the hit words from registers only: the hit map goes back to the
        // dense warps now, so their next drain (and the MMA after it) need not wait for it
        __syncwarp();
        nb_arrive(kNbHmEmpty + hb, kHmCount);
      }
#endif
      auto word_at = [&](int c) -> uint32_t {
        if (ff)
          return c < 4 ? (c < 2 ? (c == 0 ? mw[0] : mw[1]) : (c == 2 ? mw[2] : mw[3]))
                       : (c < 6 ? (c == 4 ? mw[4] : mw[5]) : (c == 6 ? mw[6] : mw[7]));
        return lds32(hmap + (uint32_t)c * (kMaxQueries * 4u));
      };
      uint32_t n_sv = 0;  // warp-uniform survivor count
      int n_rounds = 0;
      if constexpr (kMode == 3) {
        // one cursor over the tile's eight hit words (kept in registers), NT hits taken per
        // round wherever they are: the round count is max over lanes of ceil(hits / NT); the
        // NT filter tests of a round issue their row loads together
        constexpr int NT = FB_HIT_TAKE;
        auto word8 = [&](int c) -> uint32_t {
          return c < 4 ? (c < 2 ? (c == 0 ? mw[0] : mw[1]) : (c == 2 ? mw[2] : mw[3]))
                       : (c < 6 ? (c == 4 ? mw[4] : mw[5]) : (c == 6 ? mw[6] : mw[7]));
        };
        uint32_t rest = nzm;
        int cc8 = rest ? __ffs(rest) - 1 : 0;
        rest &= rest - 1u;
        uint32_t cur = nzm ? word8(cc8) : 0u;
        const uint32_t lt = lanemask_lt();
        const uint32_t rstride = (uint32_t)a.tb_stride * 4u;
        while (__any_sync(0xffffffffu, cur != 0u)) {
          ++n_rounds;
          bool has[NT], sv[NT];
          uint32_t itm[NT], row[NT], x[NT][4];
#pragma unroll
          for (int u = 0; u < NT; ++u) {
            has[u] = cur != 0u;
            itm[u] = has[u] ? (uint32_t)(cc8 * 32 + __ffs(cur) - 1) : 0u;
            row[u] = tb_s + itm[u] * rstride;
            cur &= cur - 1u;
            if (cur == 0u && rest != 0u) {
              cc8 = __ffs(rest) - 1;
              rest &= rest - 1u;
              cur = word8(cc8);
            }
          }
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int u = 0; u < NT; ++u) {
              const uint2 t = lds64v(row[u] + wo[g]);
              x[u][g] = (t.x & lo[g]) | (t.y & hi[g]);
            }
#pragma unroll
          for (int u = 0; u < NT; ++u) {
            sv[u] = has[u] && (nof || min(min(x[u][0], x[u][1]), min(x[u][2], x[u][3])) != 0u);
            const uint32_t bb = __ballot_sync(0xffffffffu, sv[u]);
            if (sv[u])
              sts16(sv_s + 2u * (n_sv + (uint32_t)__popc(bb & lt)), ((uint32_t)lane << 8) | itm[u]);
            n_sv += (uint32_t)__popc(bb);
          }
          if (n_sv > (uint32_t)(kSurvCap - 32 * NT)) {
            __syncwarp();
            drain_survivors(a, m, e, sv_s, n_sv, qbase, b_s, mst, tile, lane);
            __syncwarp();
            n_sv = 0;
          }
        }
      }
      int cc = nzm ? __ffs(nzm) - 1 : 0;
      uint32_t cur = (kMode != 3 && nzm) ? word_at(cc) : 0u;
      while (kMode != 3 && __any_sync(0xffffffffu, cur != 0u)) {
        ++n_rounds;
        (void)n_rounds;
        bool surv = false;
        uint32_t item = 0;
        if (cur != 0u) {
          const int j = __ffs(cur) - 1;
          cur &= cur - 1u;
          item = (uint32_t)(cc * 32 + j);
          const uint32_t tb = tb_s + item * (uint32_t)a.tb_stride * 4u;
          if (ff)
            surv = true;  // eligibility already applied
          else if (kWin)
            surv = nof || cnf_test_win(tb, wo, lo, hi);
          else
            surv = cnf_test_global(tb, qmg, ng, a.cnf_words);
          if (cur == 0u) {
            nzm &= nzm - 1u;
            if (nzm) {
              cc = __ffs(nzm) - 1;
              cur = word_at(cc);
            }
          }
        }
        const uint32_t sb = __ballot_sync(0xffffffffu, surv);
        if (surv)
          sts16(sv_s + 2u * (n_sv + (uint32_t)__popc(sb & lanemask_lt())),
                ((uint32_t)lane << 8) | item);
        n_sv += (uint32_t)__popc(sb);
        if (n_sv > (uint32_t)(kSurvCap - 32)) {
          __syncwarp();
          drain_survivors(a, m, e, sv_s, n_sv, qbase, b_s, mst, tile, lane);
          __syncwarp();
          n_sv = 0;
        }
      }
      __syncwarp();
      if (!(FB_HM_EARLY && kMode >= 3)) nb_arrive(kNbHmEmpty + hb, kHmCount);
      if (warp == kHit0) FB_TR(a, it, 11);
#ifdef FB_TRACE
      if ((a.dbg & 1024) && blockIdx.x == 0 && warp == kHit0 && lane == 0 && it < 16)
        g_tr[it][3] = (long long)n_rounds * 1000 + n_sv;
      if ((a.dbg & 1024) && blockIdx.x == 0 && lane == 0) {
        g_hit_rounds[warp - kHit0] += n_rounds;
        int hits = 0;
        for (int c = 0; c < 8; ++c) hits += 0;  // (per-lane counts are not kept)
        (void)hits;
      }
#endif
      if constexpr (kHand) {
        if (lane == 0)
          sts32(su32(smem + a.off_sv) + 2u * kCnfHitWarps * kSvListBytes +
                    ((uint32_t)(it & 1) * kCnfHitWarps + (uint32_t)(warp - kHit0)) * 4u,
                n_sv);
        __syncwarp();
        nb_arrive(kNbSvFull + (it & 1), kNbSvCount);
      } else if (n_sv) {
        drain_survivors(a, m, e, sv_s, n_sv, qbase, b_s, mst, tile, lane);
      }
      __syncwarp();
      nb_arrive(kNbLeafEmpty + st, kLeafCount);
      if (lane == 0) mbar_arrive(items_empty + s);
      if (++s == a.item_stages) {
        s = 0;
        iph ^= 1u;
      }
      if (warp == kHit0) FB_TR(a, it, 9);
    }
    if constexpr (kHand) {  // retire the builders' releases of the last two lists
      for (int t = it; t < it + 2; ++t)
        if (t >= 2) nb_sync(kNbSvEmpty + (t & 1), kNbSvCount);
    }
    flush_pending(a, e.pa);
    flush_pending(a, e.pb);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
#ifdef FB_TRACE
  if ((a.dbg & 1024) && blockIdx.x == 0 && threadIdx.x == 0) {
    const long long t0 = g_tr[0][0];
    for (int t = 0; t < 16; ++t)
      printf("tile %2d: prodI %6lld mmaSee %6lld c0 %6lld rounds*1000+surv %6lld | d0 %6lld r0 %6lld d1 %6lld "
             "r1 %6lld | h %6lld loop %6lld hdone %6lld | prodP %6lld\n",
             t, g_tr[t][0] - t0, g_tr[t][1] - t0, g_tr[t][2] - t0, g_tr[t][3],
             g_tr[t][4] - t0, g_tr[t][5] - t0, g_tr[t][6] - t0, g_tr[t][7] - t0,
             g_tr[t][8] - t0, g_tr[t][11] - t0, g_tr[t][9] - t0, g_tr[t][10] - t0);
    printf("hit rounds per warp (CTA 0, whole launch):");
    for (int w = 0; w < 8; ++w) printf(" %lld", g_hit_rounds[w]);
    printf("\n");
    for (int t = 0; t < 16; ++t)
      printf("dense %2d: top %6lld afterHmEmpty %6lld beforeAccWait %6lld d0 %6lld | ev15 %6lld\n", t,
             g_tr[t][12] - t0, g_tr[t][13] - t0, g_tr[t][14] - t0, g_tr[t][4] - t0,
             g_tr[t][15] - t0);
  }
#endif
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

// Shared-memory carve-up; returns total bytes (incl. 1 KB alignment slack). Bytecode mode:
// per-tile leaf masks and the staged register-machine programs. CNF mode: per-tile column
// bits (256 items x tb_stride u32), two [chunk][query] hit maps, the gate tiles (8 KB of
// digits + 256 B of 127s) and the hit warps' survivor lists.
size_t layout(TcArgs& t, int n_mblk, int n_planes, int n_leaves, int k_max, int stages,
              int plane_stages, int mode) {
  const bool cnf = mode != 0;
  size_t off = 0;
  t.off_a = 0;
  off = (size_t)n_mblk * kBlockM * kKBytes;
  t.off_b = (uint32_t)align_up(off, 1024);
  off = t.off_b + (size_t)stages * kItemBytes;
  t.plane_stage_bytes = (uint32_t)align_up((size_t)(n_planes > 0 ? n_planes : 1) * 32, 128);
  t.off_p = (uint32_t)align_up(off, 128);
  off = t.off_p + (size_t)plane_stages * t.plane_stage_bytes;
  t.leaf_stage_bytes =
      cnf ? (uint32_t)(kTileItems * t.tb_stride * 4)
          : (uint32_t)align_up((size_t)(n_leaves > 0 ? n_leaves : 1) * kLeafStride * 8, 128);
  t.off_l = (uint32_t)align_up(off, 128);
  off = t.off_l + 2ull * t.leaf_stage_bytes;
  const int rows = cnf ? t.n_cols : n_leaves;
  t.off_ls = (uint32_t)align_up(off, 16);
  off = t.off_ls + (size_t)(rows > 0 ? rows : 1) * (k_max > 0 ? k_max : 1) * 2;
  t.off_thr = (uint32_t)align_up(off, 16);
  off = t.off_thr + (size_t)kMaxQueries * 8;
  t.off_bar = (uint32_t)align_up(off, 16);
  off = t.off_bar + kBarCount * 8;
  t.off_pl = (uint32_t)align_up(off, 16);
  off = t.off_pl + (size_t)(n_planes > 0 ? n_planes : 1) * 4;
  if (cnf) {
    t.off_hm = (uint32_t)align_up(off, 128);
    off = t.off_hm + 2ull * kHmapBytes;
    t.off_gate = (uint32_t)align_up(off, 128);
    off = t.off_gate + kGateTileBytes + 256;
    t.off_sv = (uint32_t)align_up(off, 16);
    off = t.off_sv + (size_t)kSvBytes;  // mode 3's double-buffered lists (mode 1 uses half)
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
                 int cnf, size_t& smem) {
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

// 0: bytecode epilogue; 1: CNF fast form; 2: CNF general form
int cnf_mode(const ScanArgs& a) {
  // at threshold 0 every score is a hit: the word-level bytecode epilogue is cheaper than
  // per-hit tests, so the sampling pass takes it whenever the bytecode fits the kernel
  if (a.dense && a.prog.rops != nullptr && a.prog.rmax_stack <= kRegStack) return 0;
  const bool cnf = a.has_prog && a.prog.col_leaf != nullptr && a.prog.cnf_words >= 1 &&
                   a.prog.cnf_words <= 8 && a.prog.cnf_gmax >= 1 && a.prog.cnf_gmax <= 8 &&
                   a.prog.n_cols <= 32 * a.prog.cnf_words;
  if (!cnf) return 0;
  return (a.prog.cnf_windowed && a.prog.cnf_gmax <= 4) ? 1 : 2;
}

void fill_cnf(TcArgs& t, const ScanArgs& a, int q0, int mode) {
  t.n_cols = a.prog.n_cols;
  t.cnf_words = a.prog.cnf_words;
  t.cnf_gmax = a.prog.cnf_gmax;
  // window form: rows of an odd number of u64 (conflict-free 8-byte loads at random
  // items), at least the column words rounded up to a pair; general form: 32-byte rows
  int u64s = (a.prog.cnf_words + 1) / 2;
  if (u64s % 2 == 0) ++u64s;
  t.tb_stride = mode == 1 ? 2 * u64s : 8;
  t.col_leaf = a.prog.col_leaf;
  t.qmask = a.prog.qmask + (int64_t)q0 * a.prog.cnf_gmax * a.prog.cnf_words;
  t.qgroups = a.prog.qgroups + q0;
}

template <typename K>
int launch_kernel(K kernel, int threads, const CUtensorMap& tmap, const TcArgs& t, int grid,
                  size_t smem, cudaStream_t s) {
  FB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kernel<<<grid, threads, smem, s>>>(tmap, t);
  FB_LAUNCH_CHECK("k_scan_tc");
  return FB_OK;
}

// window form, mode chosen on the device from the sampling pass: per-hit and filter-first
// instances back to back, the one not chosen returns at its first instruction
bool use_mode3(const TcArgs& t) {  // (and mode 4, its filter-first twin)
  const char* v1 = getenv("FB_CNF_V1");  // A/B: the 20-warp organisation
  return t.n_mblk == 2 && !(v1 != nullptr && atoi(v1) != 0);
}

int launch_win(const TcArgs& t, const CUtensorMap& tmap, int grid, size_t smem, cudaStream_t s) {
  return use_mode3(t) ? launch_kernel(k_scan_cnf<3>, kCnf3Threads, tmap, t, grid, smem, s)
                      : launch_kernel(k_scan_cnf<1>, kCnfThreads, tmap, t, grid, smem, s);
}

int launch_ff(const TcArgs& t, const CUtensorMap& tmap, int grid, size_t smem, cudaStream_t s) {
  return use_mode3(t) ? launch_kernel(k_scan_cnf<4>, kCnf3Threads, tmap, t, grid, smem, s)
                      : launch_kernel(k_scan_cnf<2>, kCnfThreads, tmap, t, grid, smem, s);
}

int launch_both(const TcArgs& t, const CUtensorMap& tmap, int grid, size_t smem, cudaStream_t s) {
  const int rc = launch_win(t, tmap, grid, smem, s);
  return rc ? rc : launch_ff(t, tmap, grid, smem, s);
}

}  // namespace

bool scan_tc_supported(const ScanArgs& a) {
  if (a.mode != SCAN_EMIT || a.fb != nullptr) return false;
  if (a.idx.dim_pad != kKBytes) return false;
  if (a.idx.n_slots % kTileItems != 0 || a.tc_work == nullptr) return false;
  if (encode_fn() == nullptr) return false;
  if (a.has_prog) {
    const int cnf = cnf_mode(a);
    if (!cnf && (a.prog.rops == nullptr || a.prog.rmax_stack > kRegStack)) return false;
    if (a.prog.n_leaves >= (1 << 13) || a.prog.plane_list == nullptr) return false;
    TcArgs t{};
    if (cnf) fill_cnf(t, a, 0, cnf);
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
  const int cnf = cnf_mode(a);
  if (cnf == 1 && emit_win_supported(a)) return launch_emit_win(a, tmap, grid, s);
  for (int q0 = 0; q0 < a.n_queries; q0 += kMaxQueries) {
    const int nq = a.n_queries - q0 < kMaxQueries ? a.n_queries - q0 : kMaxQueries;
    TcArgs t{};
    t.items = a.idx.items;
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
      if (cnf) fill_cnf(t, a, q0, cnf);
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
    if (const char* d = getenv("FB_SCAN_DEBUG")) t.dbg = atoi(d);
    // filter-first below ~3 % sampled eligibility (config-4 sweep: it wins at 1 and 2 %, the
    // per-hit pass at 5 % and above); FB_CNF_FFIRST = 0 / 1 forces either, _FRAC moves the cut
    t.ffirst = cnf == 1 ? -1 : 0;
    if (const char* f = getenv("FB_CNF_FFIRST")) t.ffirst = cnf == 1 ? atoi(f) : 0;
    double ff_frac = 0.03;
    if (const char* f = getenv("FB_CNF_FFIRST_FRAC")) ff_frac = atof(f);
    t.sample_cnt = a.sample_cnt ? a.sample_cnt + q0 : nullptr;
    t.ff_limit = (float)(ff_frac * a.sampled_slots * (double)nq);
    if (t.ffirst < 0 && t.sample_cnt == nullptr) t.ffirst = 0;
    size_t smem = 0;
    if (!pick_stages(t, t.n_mblk, t.has_prog ? t.n_planes : 0, t.has_prog ? t.n_leaves : 0,
                     t.has_prog ? t.k_max : 0, t.has_prog ? a.prog.n_rops : 0, cnf, smem))
      return FB_ERR_UNSUPPORTED;
    const int rc =
        cnf == 1 && t.ffirst > 0 ? launch_ff(t, tmap, grid, smem, s)
        : cnf == 1 && t.ffirst == 0 ? launch_win(t, tmap, grid, smem, s)
        : cnf == 1 ? launch_both(t, tmap, grid, smem, s)
        : cnf == 2 ? launch_kernel(k_scan_cnf<0>, kCnfThreads, tmap, t, grid, smem, s)
                   : launch_kernel(k_scan_tc, kThreads, tmap, t, grid, smem, s);
    if (rc) return rc;
  }
  return FB_OK;
}

}  // namespace fb
