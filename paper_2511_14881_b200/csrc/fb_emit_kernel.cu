// Emit pass of the co-designed filtered top-k for CNF filter batches in the window form
// (every program an AND of <= 4 OR-groups whose literal columns share one aligned 64-column
// window -- the "f in S" groups of the 4-attribute filter), on sm_100a.
//
// One persistent CTA per SM walks 256-item tiles with warp-specialised roles:
//   * item producer: TMA of the 256 x 128 B item rows (SWIZZLE_128B) plus the tile's id ranks,
//     validity & range words and index, into three item stages;
//   * plane producer: cp.async gather of the batch's referenced Bloom plane words (32 B per
//     plane per tile), one commit group per tile;
//   * five column builders: AND each literal column's planes (the paper's and.b64 Bloom test,
//     32 items per op), then bit-transpose so each item row holds its literal columns;
//   * MMA issuer: gate-armed int32 scores of every (query, item) pair with
//     tcgen05.mma.kind::i8, M = 128 queries x N = 128 items per sub-tile, in four 128-column
//     TMEM accumulators;
//   * eight scan warps (TMEM lane quadrant x item half; lane = query): tcgen05.ld 32x32b.x32,
//     hit word of 32 items = sign bits of the gate-armed accumulators & validity & range; the
//     buffer goes back to the MMA as soon as the words are in registers; the warp's hits are
//     compacted into a per-warp list (one (query, item) pair per entry) and tested lane-
//     parallel against the query's CNF window on the item's column bits; survivors are
//     re-scored exactly from the resident tiles before the exact key test and the append.
// SIMT warps hand off through hardware named barriers where the waiting side would otherwise
// poll; the asynchronous producers (TMA, cp.async, tcgen05.commit) signal mbarriers.
// Filtered-out items never leave the SM. Semantics: reference ivf.search_clusters
// (ivf.py:285-334) restricted by filter_query.eval_compiled (filter_query.py:314-356):
// eligible = valid & range & mask & program; candidates = eligible pairs with key >= T.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <unistd.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fb_internal.cuh"
#include "fb_ptx.cuh"

namespace fb {
namespace {

using namespace ::fb::dev;

constexpr int kTile = 256;           // items per tile
constexpr int kTileW = 4;            // 64-slot words per tile
constexpr int kBM = 128;             // queries per M-block
constexpr int kMaxQ = 256;           // queries per launch
constexpr int kRow = 128;            // bytes per item / query row (dim_pad)
constexpr int kSubN = 128;           // items per MMA sub-tile = accumulator columns
constexpr uint32_t kItemStage = kTile * kRow;  // 32 KB
constexpr uint32_t kGateBytes = kMaxQ * 32;     // gate digit tile (no swizzle) + 256 B of 127s
constexpr uint32_t kWinBytes = kMaxQ * 48u;     // CNF windows [query][12] u32
// per item stage, written by the item producer: 256 id ranks, 4 validity & range words, the
// tile index
constexpr uint32_t kMetaValid = kTile * 4;
constexpr uint32_t kMetaTile = kMetaValid + 32;
constexpr uint32_t kMetaBytes = kMetaTile + 32;
constexpr int kItemStages = 3;

// warp roles (16 warps; each SM sub-partition gets two scan warps and one or two builders)
constexpr int kThreads = 512;
constexpr int kWItems = 0, kWMma = 1, kWPlanes = 2, kWBuild0 = 3, kNBuild = 5;
constexpr int kWScan0 = 8, kNScan = 8;
constexpr int kSurvCap = 64;         // u16 survivors per scan warp: (query << 8) | item
constexpr int kHitCap = 192;         // u16 hits per scan warp per batch: (lane << 7) | item
// Named barriers (0 is __syncthreads; "+ stage"). The waiting side blocks in the barrier
// unit: column-bit stages (scan warps release -> builders), plane stages (plane producer <->
// builders), item stages (scan warps release -> item producer).
constexpr int kNbCbEmpty = 1, kNbPlFull = 3, kNbPlEmpty = 5, kNbItEmpty = 7;
constexpr int kNbCbCount = 32 * (kNBuild + kNScan);
constexpr int kNbPlCount = 32 * (1 + kNBuild);
constexpr int kNbItCount = 32 * (1 + kNScan);
// mbarrier slots: item stages full (TMA + id ranks + meta), accumulators full / empty, column
// bits full (every builder warp; the scan warps test it once per tile, so a slow scan warp
// never holds the others up)
constexpr int kBarItemsFull = 0, kBarAccFull = 3, kBarAccEmpty = 7, kBarCbFull = 11,
              kBarTmem = 13, kBarCount = 14;

struct EmitArgs {
  const int8_t* queries;  // [nq, 128]
  int32_t nq;
  int32_t n_mblk;
  const uint64_t* planes;
  const uint64_t* valid;
  const uint32_t* id_rank;
  const uint64_t* masks;  // [nq, n_words] nullable
  int64_t n_words;
  int32_t n_planes;
  int32_t k_max;
  int32_t n_cols;
  int32_t cnf_words;
  int32_t tb_stride;      // u32 per item row of the column-bit stage
  const int32_t* plane_list;
  const int16_t* leaf_slot;
  const int16_t* col_leaf;
  const uint32_t* qrec;   // [nq][12]: lo[4], hi[4], window byte offsets (packed), unfiltered
  const int2* work;
  int64_t n_sel;
  int64_t work_stride;
  const int64_t* ranges;
  const uint64_t* threshold;
  uint64_t* out_key;
  uint32_t* out_slot;
  uint32_t* out_cnt;
  int32_t cap;
  int32_t plane_stages;
  long long* trace;  // timeline (FB_EMIT_TRACE): CTA 0, tiles 16..31, [tile][event] clock64
  uint32_t* prog;    // hang triage (FB_EMIT_PROGRESS): per (CTA, warp) last reached point
  int32_t dbg;       // timing experiments only (FB_SCAN_DEBUG, wrong results): bit 0 no plane
                     // copies, bit 1 no hit tests, bit 2 no column builds
  uint32_t off_a, off_b, off_meta, off_p, off_cb, off_ls, off_thr, off_bar, off_pl, off_gate,
      off_win, off_list, off_sv, plane_stage_bytes, cb_stage_bytes;
};

// hang triage: record (tile counter << 8 | point) of this warp in host-mapped memory
#define FB_PROG(a, t, pt)                                                               \
  do {                                                                                  \
    if ((a).prog != nullptr && (threadIdx.x & 31) == 0) {                               \
      *(volatile uint32_t*)((a).prog + blockIdx.x * 32 + (threadIdx.x >> 5)) =          \
          ((uint32_t)(t) << 8) | (pt);                                                  \
      __threadfence_system();                                                           \
    }                                                                                   \
  } while (0)
// timeline: CTA 0 records clock64 at pipeline events of its tiles 16..31 (steady state)
#define FB_EV(a, t, ev)                                                                 \
  do {                                                                                  \
    if ((a).trace != nullptr && blockIdx.x == 0 && (t) >= 16 && (t) < 32 &&             \
        (threadIdx.x & 31) == 0)                                                        \
      (a).trace[((t)-16) * 32 + (ev)] = clock64();                                      \
  } while (0)

// 32-bit shared-window address of the 1 KB-aligned dynamic shared memory
__device__ __forceinline__ uint32_t smem_base() {
  extern __shared__ uint8_t smem_raw[];
  return (su32(smem_raw) + 1023u) & ~1023u;
}

// ---- item producer: TMA rows + per-tile metadata (one tile of global reads ahead) -----
__device__ __forceinline__ void items_loop(const EmitArgs& a, const CUtensorMap* tmap,
                                           uint32_t sb, int lane) {
  const uint32_t full0 = sb + a.off_bar + 8u * kBarItemsFull;
  const uint32_t rows0 = sb + a.off_b, meta0 = sb + a.off_meta;
  const int64_t G = gridDim.x, n_sel = a.n_sel, wstride = a.work_stride;
  const int2* work = a.work;
  auto load_valid = [&](int2 w) -> uint64_t {
    if (lane >= kTileW) return 0ull;
    const int64_t s0 = a.ranges[2 * w.y], s1 = a.ranges[2 * w.y + 1];
    const int64_t gw = (int64_t)w.x * kTileW + lane;
    return __ldg(a.valid + gw) & word_range_mask(gw * 64, s0, s1);
  };
  int2 wk_cur = make_int2(0, 0), wk_next = make_int2(0, 0);
  uint64_t v_cur = 0ull;
  if (blockIdx.x < n_sel) {
    wk_cur = work[(int64_t)blockIdx.x * wstride];
    v_cur = load_valid(wk_cur);
    if (blockIdx.x + G < n_sel) wk_next = work[((int64_t)blockIdx.x + G) * wstride];
  }
  int s = 0, t = 0;
  for (int64_t i = blockIdx.x; i < n_sel; i += G, ++t) {
    const int tile = wk_cur.x;
    uint64_t v_next = 0ull;
    int2 wk_nn = make_int2(0, 0);
    if (i + G < n_sel) v_next = load_valid(wk_next);
    if (i + 2 * G < n_sel) wk_nn = work[(i + 2 * G) * wstride];
    FB_PROG(a, t, 1);
    if (t >= kItemStages) nb_sync(kNbItEmpty + s, kNbItCount);  // scan warps done with t - 3
    FB_PROG(a, t, 2);
    FB_EV(a, t, 0);
    const uint32_t full = full0 + 8u * (uint32_t)s;
    if (lane == 0) {
      mbar_expect_tx_s(full, kItemStage);
      tma_load_2d_s(rows0 + (uint32_t)s * kItemStage, tmap, 0, tile * kTile, full);
    }
    const uint32_t mst = meta0 + (uint32_t)s * kMetaBytes;
    const uint32_t* src = a.id_rank + (int64_t)tile * kTile;
#pragma unroll
    for (int e = lane; e < kTile / 4; e += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(mst + (uint32_t)e * 16u),
                   "l"(src + 4 * e)
                   : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(full) : "memory");
    if (lane < kTileW)
      asm volatile("st.shared.u64 [%0], %1;" ::"r"(mst + kMetaValid + 8u * lane), "l"(v_cur)
                   : "memory");
    if (lane == 0)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(mst + kMetaTile), "r"(tile) : "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive_s(full);
    if (++s == kItemStages) s = 0;
    wk_cur = wk_next;
    v_cur = v_next;
    wk_next = wk_nn;
  }
  for (int u = t; u < t + kItemStages; ++u)  // consume the scan warps' last releases
    if (u >= kItemStages) nb_sync(kNbItEmpty + u % kItemStages, kNbItCount);
  FB_PROG(a, t, 4);
}

// ---- plane producer: 16-byte cp.async gather of the referenced planes' 32-byte rows, one
// commit group per tile; a stage is handed to the builders once its group has landed ------
__device__ __forceinline__ void cp_async_wait_stages(int pending) {
  if (pending >= 2)
    asm volatile("cp.async.wait_group 2;" ::: "memory");
  else if (pending == 1)
    asm volatile("cp.async.wait_group 1;" ::: "memory");
  else
    asm volatile("cp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void planes_loop(const EmitArgs& a, uint32_t sb, int lane) {
  const uint32_t pl_s = sb + a.off_pl, p0 = sb + a.off_p, psb = a.plane_stage_bytes;
  const int n2 = (a.dbg & 1) ? 0 : 2 * a.n_planes;
  const int S = a.plane_stages;
  const uint64_t* planes = a.planes;
  const int64_t n_words = a.n_words, n_sel = a.n_sel, wstride = a.work_stride;
  int t = 0;
  for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++t) {
    const int ps = t % S;
    const int tile = a.work[i * wstride].x;
    FB_PROG(a, t, 1);
    if (t >= S) nb_sync(kNbPlEmpty + ps, kNbPlCount);  // builders finished tile t - S
    FB_PROG(a, t, 2);
    const uint32_t dst = p0 + (uint32_t)ps * psb;
    const int64_t col0 = (int64_t)tile * kTileW;
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
        if (e < n2)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (uint32_t)e * 16u),
                       "l"(planes + (int64_t)pl[u] * n_words + col0 + 2 * (e & 1))
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (t >= S - 1) {  // tile t - S + 1 has landed once at most S - 1 groups are pending
      cp_async_wait_stages(S - 1);
      FB_EV(a, t - S + 1, 1);
      nb_arrive(kNbPlFull + (t - S + 1) % S, kNbPlCount);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  for (int u = (t - S + 1 > 0 ? t - S + 1 : 0); u < t; ++u) nb_arrive(kNbPlFull + u % S, kNbPlCount);
  for (int u = t; u < t + S; ++u)  // consume the builders' releases of the last stages
    if (u >= S) nb_sync(kNbPlEmpty + u % S, kNbPlCount);
  FB_PROG(a, t, 4);
}

// ---- MMA issuer: per sub-tile (M-block mb, item half h) the gate-arming K = 32 MMA
// (query digit row x a tile of 127s), then 4 K-steps of kind::i8, into TMEM buffer seq % 4
__device__ __forceinline__ void mma_loop(const EmitArgs& a, uint32_t sb, uint32_t tmem_base) {
  const uint32_t full0 = sb + a.off_bar + 8u * kBarItemsFull;
  const uint32_t accf0 = sb + a.off_bar + 8u * kBarAccFull;
  const uint32_t acce0 = sb + a.off_bar + 8u * kBarAccEmpty;
  constexpr uint32_t idesc = idesc_i8(kBM, kSubN);
  const uint32_t gate_s = sb + a.off_gate, a_s = sb + a.off_a, b0 = sb + a.off_b;
  const int n_mblk = a.n_mblk;
  const int64_t n_sel = a.n_sel;
  int s = 0, t = 0;
  uint32_t ph = 0, seq = 0;
  for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++t) {
    FB_PROG(a, t, 1);
    mbar_wait_s(full0 + 8u * (uint32_t)s, ph);
    FB_PROG(a, t, 2);
    FB_EV(a, t, 2);
    tc_fence_after();
    const uint32_t b_s = b0 + (uint32_t)s * kItemStage;
    for (int mb = 0; mb < n_mblk; ++mb) {
      const uint32_t a_base = a_s + (uint32_t)mb * kBM * kRow;
#pragma unroll
      for (int h = 0; h < 2; ++h, ++seq) {
        const uint32_t buf = seq & 3u;
        mbar_wait_s(acce0 + 8u * buf, ((seq >> 2) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * kSubN;
        umma_i8(d, plain_desc(gate_s + (uint32_t)mb * (kBM / 8) * 256u, 128u, 256u),
                plain_desc(gate_s + kGateBytes, 128u, 0u), idesc, 0u);
        // item half h starts 128 rows (16 KB, a whole number of 1 KB swizzle atoms) in
#pragma unroll
        for (int kk = 0; kk < kRow / 32; ++kk)
          umma_i8(d, sw128_desc(a_base + kk * 32), sw128_desc(b_s + h * 16384u + kk * 32), idesc,
                  1u);
        umma_commit_s(accf0 + 8u * buf);
        FB_EV(a, t, 3 + 2 * mb + h);
      }
    }
    if (++s == kItemStages) { s = 0; ph ^= 1u; }
  }
}

// ---- column builders: per literal column the AND of its planes' 256 tile bits, then eight
// 32 x 32 bit transposes so item row i holds bit c of every column c. The column's plane
// slots are read once as 8 x i16 (padded with an all-ones row), so the plane loads issue
// back to back. -----------------------------------------------------------------------------
__device__ __forceinline__ void build_loop(const EmitArgs& a, uint32_t sb, int lw, int lane) {
  const uint32_t ls_s = sb + a.off_ls, p0 = sb + a.off_p, psb = a.plane_stage_bytes;
  const uint32_t cb0 = sb + a.off_cb, cbsb = a.cb_stage_bytes;
  const uint32_t cbf0 = sb + a.off_bar + 8u * kBarCbFull;
  const int words = (a.dbg & 4) ? 0 : a.cnf_words, n_cols = a.n_cols, kmax = a.k_max;
  const uint32_t tb4 = 4u * (uint32_t)a.tb_stride;
  const int S = a.plane_stages;
  const int64_t n_sel = a.n_sel;
  int it = 0;
  for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
    const int st = it & 1;
    const int ps = it % S;
    FB_PROG(a, it, 1);
    if (it >= 2) nb_sync(kNbCbEmpty + st, kNbCbCount);
    nb_sync(kNbPlFull + ps, kNbPlCount);
    FB_PROG(a, it, 3);
    if (lw == 0) FB_EV(a, it, 7);
    const uint32_t p_s = p0 + (uint32_t)ps * psb;
    const uint32_t tb = cb0 + (uint32_t)st * cbsb;
    for (int cb = lw; cb < words; cb += kNBuild) {
      const int col = cb * 32 + lane;
      uint32_t w[8];
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) w[ib] = ~0u;
      // the column's plane slots (offsets of 32-byte rows in the stage; bit 15 of slot 0
      // marks a negated literal; missing positions point at the stage's all-ones row)
      const uint4 sl = lds128(ls_s + 16u * (uint32_t)(col < n_cols ? col : n_cols));
      const uint32_t sls[8] = {sl.x & 0x7FFFu, sl.x >> 16, sl.y & 0xFFFFu, sl.y >> 16,
                               sl.z & 0xFFFFu, sl.z >> 16, sl.w & 0xFFFFu, sl.w >> 16};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < kmax) {
          const uint4 lo = lds128(p_s + sls[j]);
          const uint4 hi = lds128(p_s + sls[j] + 16u);
          w[0] &= lo.x; w[1] &= lo.y; w[2] &= lo.z; w[3] &= lo.w;
          w[4] &= hi.x; w[5] &= hi.y; w[6] &= hi.z; w[7] &= hi.w;
        }
      }
      const uint32_t neg = (sl.x & 0x8000u) ? ~0u : 0u;
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) w[ib] ^= neg;
      // eight 32x32 transposes in lockstep (per round: SHFL + SHF + LOP3 per word)
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        const int sft = 16 >> k;
        const uint32_t mk = k == 0 ? 0x0000FFFFu : k == 1 ? 0x00FF00FFu : k == 2 ? 0x0F0F0F0Fu
                          : k == 3 ? 0x33333333u : 0x55555555u;
        const bool upper = (lane & sft) != 0;
        const uint32_t keep = upper ? ~mk : mk;
        const uint32_t rot = upper ? (uint32_t)(32 - sft) : (uint32_t)sft;
#pragma unroll
        for (int ib = 0; ib < 8; ++ib) w[ib] = transpose_round(w[ib], sft, keep, rot);
      }
#pragma unroll
      for (int ib = 0; ib < 8; ++ib)
        sts32(tb + (uint32_t)(ib * 32 + lane) * tb4 + 4u * (uint32_t)cb, w[ib]);
    }
    __syncwarp();
    if (lw == 0) FB_EV(a, it, 8);
    nb_arrive(kNbPlEmpty + ps, kNbPlCount);
    if (lane == 0) mbar_arrive_s(cbf0 + 8u * (uint32_t)st);
  }
  for (int t = it; t < it + 2; ++t)
    if (t >= 2) nb_sync(kNbCbEmpty + (t & 1), kNbCbCount);
  FB_PROG(a, it, 4);
}

// ---- survivors: exact score, exact key test, slot reservation -------------------------
struct Pending {
  uint64_t key;
  uint32_t p;
  uint32_t slot;
  int32_t q;
};
// Queued survivors (filter passed): exact score from the resident query / item tiles, exact
// key test against the query's threshold, slot reservation; an emission's stores trail by
// two emissions per lane so the atomic's round trip overlaps the next ones. (Off the hot
// path: everything is re-derived from the parameters here.)
__device__ __forceinline__ void flush(const EmitArgs& a, Pending& pd) {
  if (pd.q >= 0 && pd.p < (uint32_t)a.cap) {
    a.out_key[(int64_t)pd.q * a.cap + pd.p] = pd.key;
    if (a.out_slot) a.out_slot[(int64_t)pd.q * a.cap + pd.p] = pd.slot;
  }
  pd.q = -1;
}
__device__ __noinline__ void drain(const EmitArgs& a, uint32_t sb, Pending (&pd)[2], int& par,
                                   uint32_t sv_s, uint32_t n, int s, int64_t tile, int lane) {
  const uint32_t a_s = sb + a.off_a, b_s = sb + a.off_b + (uint32_t)s * kItemStage;
  const uint32_t mst = sb + a.off_meta + (uint32_t)s * kMetaBytes, thr_s = sb + a.off_thr;
  for (uint32_t i = (uint32_t)lane; i < n; i += 32u) {
    const uint32_t ent = lds16(sv_s + 2u * i);
    const uint32_t q = ent >> 8;
    const uint32_t item = ent & 255u;
    const int32_t score = smem_dot(a_s + q * kRow, q & 7u, b_s + item * kRow, item & 7u);
    const uint64_t key = make_key(score, lds32(mst + 4u * item));
    if (key >= lds64(thr_s + 8u * q)) {
      const uint32_t slot = (uint32_t)(tile * kTile) + item;
      if (par) {
        flush(a, pd[1]);
        pd[1].p = atomicAdd(a.out_cnt + q, 1u);
        pd[1].key = key;
        pd[1].slot = slot;
        pd[1].q = (int32_t)q;
      } else {
        flush(a, pd[0]);
        pd[0].p = atomicAdd(a.out_cnt + q, 1u);
        pd[0].key = key;
        pd[0].slot = slot;
        pd[0].q = (int32_t)q;
      }
      par ^= 1;
    }
  }
}

// ---- scan warps: warp (TMEM lane quadrant, item half h) drains its 32 lanes x 128 columns
// of every sub-tile (mb, h); lane = query --------------------------------------------------
template <bool kMasks>
__device__ __forceinline__ void scan_loop(const EmitArgs& a, uint32_t sb, uint32_t tmem_base,
                                          int warp, int lane) {
  const uint32_t full0 = sb + a.off_bar + 8u * kBarItemsFull;
  const uint32_t accf0 = sb + a.off_bar + 8u * kBarAccFull;
  const uint32_t acce0 = sb + a.off_bar + 8u * kBarAccEmpty;
  const uint32_t cbf0 = sb + a.off_bar + 8u * kBarCbFull;
  const int quad = warp & 3;
  const int dw = warp - kWScan0;
  const int h = dw >> 2;
  const int n_mblk = a.n_mblk, nq = a.nq, n_sub = 2 * n_mblk;
  const uint32_t meta0 = sb + a.off_meta, thr_s = sb + a.off_thr, win_s = sb + a.off_win;
  const uint32_t cb0 = sb + a.off_cb, cbsb = a.cb_stage_bytes, tb4 = 4u * (uint32_t)a.tb_stride;
  const uint32_t sv_s = sb + a.off_sv + (uint32_t)dw * (kSurvCap * 2u);
  const uint32_t hl_s = sb + a.off_list + (uint32_t)dw * (kHitCap * 2u);
  const int64_t n_sel = a.n_sel;
  const bool skip_hits = (a.dbg & 2) != 0;
  // gate constants of this lane's rows in both M-blocks
  uint32_t allm[2];
  for (int mb = 0; mb < 2; ++mb) {
    const int q = mb * kBM + quad * 32 + lane;
    bool all = false;
    if (mb < n_mblk) gate_digits(q < nq ? lds64(thr_s + 8u * (uint32_t)q) : ~0ull, all);
    allm[mb] = all ? ~0u : 0u;
  }
  Pending pd[2];
  pd[0].q = pd[1].q = -1;
  pd[0].p = pd[1].p = 0u;
  pd[0].key = pd[1].key = 0ull;
  pd[0].slot = pd[1].slot = 0u;
  int par = 0;
  int it = 0, s = 0;
  uint32_t iph = 0;
  for (int64_t i = blockIdx.x; i < n_sel; i += gridDim.x, ++it) {
    FB_PROG(a, it, 1);
    mbar_wait_s(full0 + 8u * (uint32_t)s, iph);
    FB_PROG(a, it, 2);
    const uint32_t mst = meta0 + (uint32_t)s * kMetaBytes;
    const int64_t tile = (int64_t)lds32(mst + kMetaTile);
    // lane c < 4: validity & range bits of chunk 4h + c
    const uint32_t vchunk = lane < 4 ? lds32(mst + kMetaValid + 4u * (uint32_t)(4 * h + lane)) : 0u;
    const int st = it & 1;
    const uint32_t cbs = cb0 + (uint32_t)st * cbsb;
    bool cb_ready = false;
    uint32_t n_sv = 0;
#pragma unroll 1
    for (int mb = 0; mb < n_mblk; ++mb) {
      const uint32_t seq = (uint32_t)(it * n_sub + 2 * mb + h);
      const uint32_t buf = seq & 3u;
      const int qbase = mb * kBM + quad * 32;
      const int q = qbase + lane;
      const bool qok = q < nq;
      const uint32_t am = mb == 0 ? allm[0] : allm[1];
      uint64_t m01[2] = {~0ull, ~0ull};
      if (kMasks) {
        const uint64_t* mw = a.masks + (int64_t)(qok ? q : 0) * a.n_words + tile * kTileW + 2 * h;
        m01[0] = __ldg(mw);
        m01[1] = __ldg(mw + 1);
      }
      FB_PROG(a, it * 4 + mb, 3);
      mbar_wait_s(accf0 + 8u * buf, (seq >> 2) & 1u);
      FB_PROG(a, it * 4 + mb, 4);
      if (quad == 0) FB_EV(a, it, 9 + 2 * mb + h);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * kSubN;
      auto word_of = [&](int c, const int32_t (&r)[32]) -> uint32_t {
        uint32_t em = __shfl_sync(0xffffffffu, vchunk, c);  // whole warp (never predicated)
        if (!qok) em = 0u;
        if (kMasks) em &= (uint32_t)(m01[c >> 1] >> (32 * (c & 1)));
        return (nonneg_mask32(r) | am) & em;
      };
      uint32_t w0, w1, w2, w3;
      {
        int32_t ra[32], rb[32];
        tmem_ld32_async(taddr, ra);
        tmem_wait32(ra);
        tmem_ld32_async(taddr + 32u, rb);
        w0 = word_of(0, ra);
        tmem_wait32(rb);
        tmem_ld32_async(taddr + 64u, ra);
        w1 = word_of(1, rb);
        tmem_wait32(ra);
        tmem_ld32_async(taddr + 96u, rb);
        w2 = word_of(2, ra);
        tmem_wait32(rb);
        // the accumulator buffer is free once its last columns are in registers
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_s(acce0 + 8u * buf);
        w3 = word_of(3, rb);
      }
      if (quad == 0) FB_EV(a, it, 13 + 2 * mb + h);
      if (skip_hits) continue;
      if (!cb_ready) {  // column bits of this tile (the builders run a tile ahead)
        mbar_wait_s(cbf0 + 8u * (uint32_t)st, (uint32_t)((it >> 1) & 1));
        cb_ready = true;
      }
      // compact the warp's hits into (lane, item) entries, then one filter test per lane
      const uint32_t nh = (uint32_t)(__popc(w0) + __popc(w1) + __popc(w2) + __popc(w3));
      uint32_t incl = nh;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t tt = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += tt;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - nh;
      for (uint32_t b0e = 0; b0e < total; b0e += (uint32_t)kHitCap) {
        // entries of global index [b0e, b0e + kHitCap); more than one batch only when a
        // batch holds nearly every pair (threshold 0 / unfiltered)
        if (nh != 0u && excl < b0e + (uint32_t)kHitCap && excl + nh > b0e) {
          uint32_t pos = excl;
          uint32_t cur = w0, cc = 0;
          for (;;) {
            while (cur == 0u && cc < 3u) {
              ++cc;
              cur = cc == 1u ? w1 : cc == 2u ? w2 : w3;
            }
            if (cur == 0u || pos >= b0e + (uint32_t)kHitCap) break;
            const uint32_t j = (uint32_t)(__ffs(cur) - 1);
            cur &= cur - 1u;
            if (pos >= b0e) sts16(hl_s + 2u * (pos - b0e), ((uint32_t)lane << 7) | (cc * 32u + j));
            ++pos;
          }
        }
        __syncwarp();
        const uint32_t n = min(total - b0e, (uint32_t)kHitCap);
        for (uint32_t r0 = 0; r0 < n; r0 += 32u) {
          const uint32_t e = r0 + (uint32_t)lane;
          bool surv = false;
          uint32_t qe = 0, item = 0;
          if (e < n) {
            const uint32_t ent = lds16(hl_s + 2u * e);
            qe = (uint32_t)qbase + (ent >> 7);
            item = (uint32_t)(h * kSubN) + (ent & 127u);
            const uint32_t wq = win_s + qe * 48u;
            const uint4 L = lds128(wq), H = lds128(wq + 16u), W = lds128(wq + 32u);
            const uint32_t lo[4] = {L.x, L.y, L.z, L.w}, hi[4] = {H.x, H.y, H.z, H.w};
            const uint32_t wo[4] = {W.x & 255u, (W.x >> 8) & 255u, (W.x >> 16) & 255u, W.x >> 24};
            surv = W.y != 0u || cnf_test_win(cbs + item * tb4, wo, lo, hi);
          }
          const uint32_t sbal = __ballot_sync(0xffffffffu, surv);
          if (surv) sts16(sv_s + 2u * (n_sv + (uint32_t)__popc(sbal & lanemask_lt())), (qe << 8) | item);
          n_sv += (uint32_t)__popc(sbal);
          if (n_sv > (uint32_t)(kSurvCap - 32)) {
            __syncwarp();
            drain(a, sb, pd, par, sv_s, n_sv, s, tile, lane);
            __syncwarp();
            n_sv = 0;
          }
        }
        __syncwarp();
      }
    }
    if (!cb_ready) mbar_wait_s(cbf0 + 8u * (uint32_t)st, (uint32_t)((it >> 1) & 1));
    __syncwarp();
    nb_arrive(kNbCbEmpty + st, kNbCbCount);  // column bits consumed
    if (n_sv) drain(a, sb, pd, par, sv_s, n_sv, s, tile, lane);
    __syncwarp();
    nb_arrive(kNbItEmpty + s, kNbItCount);  // item rows and id ranks read
    if (quad == 0) FB_EV(a, it, 17 + h);
    FB_PROG(a, it, 7);
    if (++s == kItemStages) { s = 0; iph ^= 1u; }
  }
  flush(a, pd[0]);
  flush(a, pd[1]);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_emit_win(const __grid_constant__ CUtensorMap tmap_items, const EmitArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t sb = smem_base();
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + a.off_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- prologue: queries (SW128), thresholds, plane ids, column table, windows, gates ----
  {
    uint8_t* sA = smem + a.off_a;
    for (int i = threadIdx.x; i < a.n_mblk * kBM * 8; i += kThreads) {
      const int r = i >> 3, c = i & 7;
      int4 v = make_int4(0, 0, 0, 0);
      if (r < a.nq) v = __ldg(reinterpret_cast<const int4*>(a.queries + (int64_t)r * kRow) + c);
      *reinterpret_cast<int4*>(sA + r * kRow + ((c ^ (r & 7)) << 4)) = v;
    }
    uint64_t* sT = reinterpret_cast<uint64_t*>(smem + a.off_thr);
    for (int q = threadIdx.x; q < kMaxQ; q += kThreads)
      sT[q] = (a.threshold != nullptr && q < a.nq) ? a.threshold[q] : 0ull;
    int32_t* pl = reinterpret_cast<int32_t*>(smem + a.off_pl);
    for (int i = threadIdx.x; i < a.n_planes; i += kThreads) pl[i] = a.plane_list[i];
    // column -> 8 plane-row byte offsets in a plane stage (negated literal: bit 15 of entry
    // 0; missing positions, and the padding column n_cols, point at the all-ones row)
    uint16_t* sLS = reinterpret_cast<uint16_t*>(smem + a.off_ls);
    const uint16_t ones = (uint16_t)(32 * a.n_planes);
    for (int i = threadIdx.x; i < (a.n_cols + 1) * 8; i += kThreads) {
      const int c = i >> 3, j = i & 7;
      uint16_t v = ones;
      if (c < a.n_cols && j < a.k_max) {
        const int cl = a.col_leaf[c];
        const int leaf = cl >= 0 ? cl : ~cl;
        const int sl = a.leaf_slot[leaf * a.k_max + j];
        if (sl >= 0) v = (uint16_t)(32 * sl);
        if (j == 0 && cl < 0) v |= 0x8000;
      }
      sLS[i] = v;
    }
    // the all-ones 32-byte row after every plane stage's rows
    for (int ps = 0; ps < a.plane_stages; ++ps)
      for (int i = threadIdx.x; i < 8; i += kThreads)
        reinterpret_cast<uint32_t*>(smem + a.off_p + (size_t)ps * a.plane_stage_bytes +
                                    32 * a.n_planes)[i] = ~0u;
    uint32_t* win = reinterpret_cast<uint32_t*>(smem + a.off_win);
    for (int i = threadIdx.x; i < kMaxQ * 12; i += kThreads)
      win[i] = i < a.nq * 12 ? a.qrec[i] : 0u;
    uint32_t* cb = reinterpret_cast<uint32_t*>(smem + a.off_cb);
    for (int i = threadIdx.x; i < 2 * (int)(a.cb_stage_bytes / 4); i += kThreads) cb[i] = 0u;
    uint8_t* gA = smem + a.off_gate;
    uint32_t* gB = reinterpret_cast<uint32_t*>(smem + a.off_gate + kGateBytes);
    for (int i = threadIdx.x; i < 64; i += kThreads) gB[i] = 0x7F7F7F7Fu;  // 256 B of 127s
    for (int r = threadIdx.x; r < kMaxQ; r += kThreads) {
      bool all;
      const uint64_t T = (a.threshold != nullptr && r < a.nq) ? a.threshold[r] : 0ull;
      const int32_t D = r < a.nq ? gate_digits(T, all) : kGateDigitsMin;
      const int32_t base = D >= 0 ? D / 32 : -((-D + 31) / 32);  // floor(D / 32)
      const int32_t rem = D - 32 * base;                        // 0..31
      for (int k = 0; k < 32; ++k) gA[gate_off(r, k)] = (uint8_t)(int8_t)(base + (k < rem ? 1 : 0));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    for (int s = 0; s < kItemStages; ++s)
      mbar_init(bars + kBarItemsFull + s, 1 + 32 + 1);  // TMA expect-tx, id-rank cp.async, meta
    for (int b = 0; b < 4; ++b) {
      mbar_init(bars + kBarAccFull + b, 1);
      mbar_init(bars + kBarAccEmpty + b, 4);  // the four scan warps of the buffer's half
    }
    for (int s = 0; s < 2; ++s) mbar_init(bars + kBarCbFull + s, kNBuild);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kBarTmem);
  if (warp == kWMma) {
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

  if (warp == kWItems) {
    items_loop(a, &tmap_items, sb, lane);
  } else if (warp == kWMma) {
    if (lane == 0) mma_loop(a, sb, tmem_base);
  } else if (warp == kWPlanes) {
    planes_loop(a, sb, lane);
  } else if (warp < kWScan0) {
    build_loop(a, sb, warp - kWBuild0, lane);
  } else if (a.masks != nullptr) {
    scan_loop<true>(a, sb, tmem_base, warp, lane);
  } else {
    scan_loop<false>(a, sb, tmem_base, warp, lane);
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kWMma)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
                 : "memory");
}

// Per-query window records of a CNF batch: for each of the (<= 4) groups, the byte offset of
// its aligned u32 pair in an item's column-bit row and the pair's two masks; unused groups
// repeat group 0 (AND is idempotent); a query without groups is unfiltered.
__global__ void k_window_records(const uint32_t* qmask, const int32_t* qgroups, int nq, int gmax,
                                 int words, uint32_t* rec) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int ng = qgroups[q];
  uint32_t lo[4] = {0u, 0u, 0u, 0u}, hi[4] = {0u, 0u, 0u, 0u}, wo = 0u;
  for (int g = 0; g < 4; ++g) {
    const uint32_t* mg = qmask + ((size_t)q * gmax + (g < ng ? g : 0)) * words;
    int w0 = 0;
    if (ng > 0)
      while (w0 < words - 1 && mg[w0] == 0u) ++w0;
    w0 &= ~1;
    wo |= (uint32_t)(4 * w0) << (8 * g);
    lo[g] = ng > 0 ? mg[w0] : 0u;
    hi[g] = (ng > 0 && w0 + 1 < words) ? mg[w0 + 1] : 0u;
  }
  uint32_t* r = rec + (size_t)q * 12;
  for (int g = 0; g < 4; ++g) {
    r[g] = lo[g];
    r[4 + g] = hi[g];
  }
  r[8] = wo;
  r[9] = ng == 0 ? 1u : 0u;
  r[10] = r[11] = 0u;
}

size_t align_up(size_t x, size_t al) { return (x + al - 1) / al * al; }

size_t layout(EmitArgs& t, int plane_stages) {
  size_t off = 0;
  t.off_a = 0;
  off = (size_t)t.n_mblk * kBM * kRow;
  t.off_b = (uint32_t)align_up(off, 1024);
  off = t.off_b + (size_t)kItemStages * kItemStage;
  // plane rows of the batch + one all-ones row (missing Bloom positions AND with it)
  t.plane_stage_bytes = (uint32_t)align_up((size_t)(t.n_planes + 1) * 32, 128);
  t.off_p = (uint32_t)align_up(off, 128);
  off = t.off_p + (size_t)plane_stages * t.plane_stage_bytes;
  t.cb_stage_bytes = (uint32_t)(kTile * t.tb_stride * 4);
  t.off_cb = (uint32_t)align_up(off, 128);
  off = t.off_cb + 2ull * t.cb_stage_bytes;
  t.off_win = (uint32_t)align_up(off, 128);
  off = t.off_win + kWinBytes;
  t.off_ls = (uint32_t)align_up(off, 16);
  off = t.off_ls + (size_t)(t.n_cols + 1) * 16;
  t.off_thr = (uint32_t)align_up(off, 16);
  off = t.off_thr + (size_t)kMaxQ * 8;
  t.off_bar = (uint32_t)align_up(off, 16);
  off = t.off_bar + kBarCount * 8;
  t.off_pl = (uint32_t)align_up(off, 16);
  off = t.off_pl + (size_t)(t.n_planes > 0 ? t.n_planes : 1) * 4;
  t.off_gate = (uint32_t)align_up(off, 128);
  off = t.off_gate + kGateBytes + 256;
  t.off_list = (uint32_t)align_up(off, 16);
  off = t.off_list + (size_t)kNScan * kHitCap * 2;
  t.off_sv = (uint32_t)align_up(off, 16);
  off = t.off_sv + (size_t)kNScan * kSurvCap * 2;
  t.off_meta = (uint32_t)align_up(off, 16);
  off = t.off_meta + (size_t)kItemStages * kMetaBytes;
  return off + 1024;  // alignment slack of the dynamic shared-memory base
}

constexpr size_t kSmemLimit = 227 * 1024;

bool pick(EmitArgs& t, size_t& smem) {
  int want = 2;
  if (const char* e = getenv("FB_EMIT_PLANE_STAGES")) want = atoi(e);  // experiments
  for (int ps = want < 1 ? 1 : (want > 3 ? 3 : want); ps >= 1; --ps) {
    smem = layout(t, ps);
    if (smem <= kSmemLimit) {
      t.plane_stages = ps;
      return true;
    }
  }
  return false;
}

void fill(EmitArgs& t, const ScanArgs& a) {
  t.n_planes = a.prog.n_planes;
  t.k_max = a.prog.k_max;
  t.n_cols = a.prog.n_cols;
  t.cnf_words = a.prog.cnf_words;
  // rows of an odd number of u64 (conflict-free 8-byte loads at random items), at least the
  // column words rounded up to a pair
  int u64s = (a.prog.cnf_words + 1) / 2;
  if (u64s % 2 == 0) ++u64s;
  t.tb_stride = 2 * u64s;
}

}  // namespace

bool emit_win_supported(const ScanArgs& a) {
  if (a.mode != SCAN_EMIT || a.fb != nullptr || a.dense || a.dump != nullptr) return false;
  if (!a.has_prog || a.prog.col_leaf == nullptr || !a.prog.cnf_windowed || a.prog.cnf_gmax > 4)
    return false;
  if (a.prog.cnf_words < 1 || a.prog.cnf_words > 8 || a.prog.n_cols > 32 * a.prog.cnf_words)
    return false;
  if (a.idx.dim_pad != kRow || a.idx.n_slots % kTile != 0 || a.tc_work == nullptr) return false;
  if (a.tc_qrec == nullptr || a.prog.plane_list == nullptr || a.prog.leaf_slot == nullptr)
    return false;
  // plane-row offsets are 15-bit (bit 15 flags a negated literal), <= 8 positions per leaf
  if (a.prog.n_planes > 1023 || a.prog.k_max > 8) return false;
  // opt-in while it is slower than k_scan_cnf<1> (FB_EMIT_V2=1)
  {
    const char* e = getenv("FB_EMIT_V2");
    if (e == nullptr || atoi(e) == 0) return false;
  }
  EmitArgs t{};
  fill(t, a);
  t.n_mblk = a.n_queries > kBM ? 2 : 1;
  size_t smem = 0;
  return pick(t, smem);
}

int launch_emit_win(const ScanArgs& a, const CUtensorMap& tmap, int grid, cudaStream_t s) {
  const int64_t n_sel = (a.n_tc_work + a.word_stride - 1) / a.word_stride;
  if (n_sel <= 0 || a.n_queries <= 0) return FB_OK;
  // window records of the whole batch (one tiny launch)
  k_window_records<<<(a.n_queries + 127) / 128, 128, 0, s>>>(a.prog.qmask, a.prog.qgroups,
                                                             a.n_queries, a.prog.cnf_gmax,
                                                             a.prog.cnf_words, a.tc_qrec);
  FB_LAUNCH_CHECK("k_window_records");
  FB_CUDA(cudaFuncSetAttribute(k_emit_win, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kSmemLimit));
  for (int q0 = 0; q0 < a.n_queries; q0 += kMaxQ) {
    const int nq = a.n_queries - q0 < kMaxQ ? a.n_queries - q0 : kMaxQ;
    EmitArgs t{};
    fill(t, a);
    t.queries = a.queries + (int64_t)q0 * kRow;
    t.nq = nq;
    t.n_mblk = (nq + kBM - 1) / kBM;
    t.planes = a.idx.planes;
    t.valid = a.idx.valid;
    t.id_rank = a.idx.id_rank;
    t.masks = a.masks ? a.masks + (int64_t)q0 * a.idx.n_words : nullptr;
    t.n_words = a.idx.n_words;
    t.plane_list = a.prog.plane_list;
    t.leaf_slot = a.prog.leaf_slot;
    t.col_leaf = a.prog.col_leaf;
    t.qrec = a.tc_qrec + (size_t)q0 * 12;
    t.work = reinterpret_cast<const int2*>(a.tc_work);
    t.n_sel = n_sel;
    t.work_stride = a.word_stride;
    t.ranges = a.ranges;
    t.threshold = a.threshold ? a.threshold + q0 : nullptr;
    t.out_key = a.out_key + (int64_t)q0 * a.cap;
    t.out_slot = a.out_slot ? a.out_slot + (int64_t)q0 * a.cap : nullptr;
    t.out_cnt = a.out_cnt + q0;
    t.cap = a.cap;
    if (const char* d = getenv("FB_SCAN_DEBUG")) t.dbg = atoi(d);
    size_t smem = 0;
    if (!pick(t, smem)) return FB_ERR_UNSUPPORTED;
    static uint32_t* h_prog = nullptr;
    const char* pe = getenv("FB_EMIT_PROGRESS");
    if (pe != nullptr && atoi(pe) != 0) {
      if (h_prog == nullptr) FB_CUDA(cudaHostAlloc(&h_prog, 148 * 32 * 4, cudaHostAllocMapped));
      memset(h_prog, 0xff, 148 * 32 * 4);
      FB_CUDA(cudaHostGetDevicePointer(&t.prog, h_prog, 0));
    }
    static long long* d_trace = nullptr;
    if (const char* te = getenv("FB_EMIT_TRACE")) {
      if (atoi(te) != 0) {
        if (d_trace == nullptr) FB_CUDA(cudaMalloc(&d_trace, 16 * 32 * sizeof(long long)));
        FB_CUDA(cudaMemsetAsync(d_trace, 0, 16 * 32 * sizeof(long long), s));
        t.trace = d_trace;
      }
    }
    k_emit_win<<<grid, kThreads, smem, s>>>(tmap, t);
    FB_LAUNCH_CHECK("k_emit_win");
    if (t.trace != nullptr) {
      long long h[16 * 32];
      FB_CUDA(cudaMemcpyAsync(h, d_trace, sizeof(h), cudaMemcpyDeviceToHost, s));
      FB_CUDA(cudaStreamSynchronize(s));
      const long long t0 = h[0];
      fprintf(stderr, "tile: rowsIss planeLd mmaSee m00 m01 m10 m11 | bld0s bld0e | "
                      "acc00 acc01 acc10 acc11 rel00 rel01 rel10 rel11 | done0 done1\n");
      for (int r = 0; r < 16; ++r) {
        const long long* e = h + r * 32;
        fprintf(stderr, "%2d:", r + 16);
        for (int k = 0; k < 19; ++k) fprintf(stderr, " %6lld", e[k] ? e[k] - t0 : -1);
        fprintf(stderr, "\n");
      }
    }
    if (t.prog != nullptr) {  // watchdog: dump every warp's last point if it does not finish
      for (int w = 0; w < 100 && cudaStreamQuery(s) == cudaErrorNotReady; ++w) usleep(50000);
      if (cudaStreamQuery(s) == cudaErrorNotReady) {
        fprintf(stderr, "k_emit_win hung: n_sel %lld grid %d nq %d n_mblk %d plane stages %d\n",
                (long long)n_sel, grid, t.nq, t.n_mblk, t.plane_stages);
        for (int b = 0; b < 4 && b < grid; ++b) {
          fprintf(stderr, "cta %d:", b);
          for (int w = 0; w < kThreads / 32; ++w) {
            const uint32_t v = ((volatile uint32_t*)h_prog)[b * 32 + w];
            fprintf(stderr, " w%d=%u.%u", w, v >> 8, v & 255u);
          }
          fprintf(stderr, "\n");
        }
        fflush(stderr);
        abort();
      }
    }
  }
  return FB_OK;
}

}  // namespace fb
