// Emit pass of the co-designed filtered top-k for CNF filter batches in the window form
// (every program an AND of <= 4 OR-groups whose literal columns share one aligned 64-column
// window -- the "f in S" groups of the 4-attribute filter), on sm_100a.
//
// One persistent CTA per SM walks 256-item tiles. Per tile:
//   * TMA brings the 256 x 128 B item rows (SWIZZLE_128B) and a plane producer gathers the
//     batch's referenced Bloom plane words (32 B per plane per tile);
//   * column builders AND each literal column's planes (the paper's and.b64 Bloom test, 32
//     items per op) and transpose the bits so each item row holds its literal columns;
//   * the tensor core computes the gate-armed int32 scores of every (query, item) pair
//     (tcgen05.mma.kind::i8, M = 128 queries x N = 128 items per sub-tile, accumulators in
//     four 128-column TMEM buffers, so the MMA runs up to three sub-tiles ahead of the drain);
//   * eight scan warps drain TMEM (tcgen05.ld 32x32b.x32, lane = query): the hit mask of 32
//     scores is their sign bits & validity & range; each hit is tested against the query's
//     CNF window (4 x 64-bit masks held in registers) on the item's column bits, and the
//     survivors are re-scored exactly from the resident tiles and appended as (key, slot).
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
// per item stage, written by the item producer: 256 id ranks, 4 validity & range words,
// the tile index
constexpr uint32_t kMetaValid = kTile * 4;
constexpr uint32_t kMetaTile = kMetaValid + 32;
constexpr uint32_t kMetaBytes = kMetaTile + 32;

// warp roles (16 warps; each SM sub-partition gets two scan warps and one or two builders)
constexpr int kThreads = 512;
constexpr int kWItems = 0, kWMma = 1, kWPlanes = 2, kWBuild0 = 3, kNBuild = 5;
constexpr int kWDense0 = 8, kNDense = 8;
constexpr int kSurvCap = 64;         // u16 survivors per scan warp: (query << 8) | item
constexpr int kHitCap = 128;         // u16 hits per scan warp per batch: (lane << 7) | item
// Named barriers (0 is __syncthreads; "+ stage"). Warp-to-warp handoffs block in the
// barrier unit instead of polling: column bits (builders -> scan warps, double-buffered),
// plane stages (plane producer -> builders, up to 3), item stages (scan warps -> item
// producer: a tile's scan warps finish after its last MMA, which read the stage).
constexpr int kNbCbFull = 1, kNbCbEmpty = 3, kNbPlFull = 5, kNbPlEmpty = 8, kNbItEmpty = 11;
constexpr int kNbCbCount = 32 * (kNBuild + kNDense);
constexpr int kNbPlCount = 32 * (1 + kNBuild);
constexpr int kNbItCount = 32 * (1 + kNDense);
// mbarrier slots
constexpr int kBarItemsFull = 0, kBarAccFull = 3, kBarAccEmpty = 7, kBarTmem = 11, kBarCount = 12;

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
  const int16_t* plane_list;
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
  int32_t item_stages;
  int32_t plane_stages;
  uint32_t* prog;  // hang triage (FB_EMIT_PROGRESS): per (CTA, warp) last reached point
  int32_t dbg;  // timing experiments only (FB_SCAN_DEBUG, wrong results): bit 0 no plane
                // copies, bit 1 no hit tests, bit 2 no column builds
  uint32_t off_a, off_b, off_p, off_cb, off_ls, off_thr, off_bar, off_pl, off_gate, off_sv,
      off_hl, off_meta, plane_stage_bytes, cb_stage_bytes;
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

struct Sm {
  uint8_t* base;
  uint64_t* bars;
  uint64_t* sT;
};
__device__ __forceinline__ Sm carve(const EmitArgs& a) {
  extern __shared__ uint8_t smem_raw[];
  Sm m;
  m.base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                      ~uintptr_t(1023));
  m.bars = reinterpret_cast<uint64_t*>(m.base + a.off_bar);
  m.sT = reinterpret_cast<uint64_t*>(m.base + a.off_thr);
  return m;
}

// ---- item producer: TMA rows + per-tile metadata (one tile of global reads ahead) -----
__device__ __forceinline__ void items_loop(const EmitArgs& a, const CUtensorMap* tmap,
                                           const Sm& m, int lane) {
  uint64_t* full = m.bars + kBarItemsFull;
  const int64_t G = gridDim.x;
  const int S = a.item_stages;
  auto load_valid = [&](int2 w) -> uint64_t {
    if (lane >= kTileW) return 0ull;
    const int64_t s0 = a.ranges[2 * w.y], s1 = a.ranges[2 * w.y + 1];
    const int64_t gw = (int64_t)w.x * kTileW + lane;
    return __ldg(a.valid + gw) & word_range_mask(gw * 64, s0, s1);
  };
  int2 wk_cur = make_int2(0, 0), wk_next = make_int2(0, 0);
  uint64_t v_cur = 0ull;
  if (blockIdx.x < a.n_sel) {
    wk_cur = a.work[(int64_t)blockIdx.x * a.work_stride];
    v_cur = load_valid(wk_cur);
    if (blockIdx.x + G < a.n_sel) wk_next = a.work[((int64_t)blockIdx.x + G) * a.work_stride];
  }
  int s = 0, t = 0;
  for (int64_t i = blockIdx.x; i < a.n_sel; i += G, ++t) {
    const int tile = wk_cur.x;
    uint64_t v_next = 0ull;
    int2 wk_nn = make_int2(0, 0);
    if (i + G < a.n_sel) v_next = load_valid(wk_next);
    if (i + 2 * G < a.n_sel) wk_nn = a.work[(i + 2 * G) * a.work_stride];
    FB_PROG(a, t, 1);
    if (t >= S) nb_sync(kNbItEmpty + s, kNbItCount);  // the scan warps finished tile t - S
    FB_PROG(a, t, 2);
    if (lane == 0) {
      mbar_expect_tx(full + s, kItemStage);
      tma_load_2d(m.base + a.off_b + (size_t)s * kItemStage, tmap, 0, tile * kTile, full + s);
    }
    const uint32_t mst = su32(m.base + a.off_meta) + (uint32_t)s * kMetaBytes;
    const uint32_t* src = a.id_rank + (int64_t)tile * kTile;
#pragma unroll
    for (int e = lane; e < kTile / 4; e += 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(mst + (uint32_t)e * 16u),
                   "l"(src + 4 * e)
                   : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(full + s))
                 : "memory");
    if (lane < kTileW)
      asm volatile("st.shared.u64 [%0], %1;" ::"r"(mst + kMetaValid + 8u * lane), "l"(v_cur)
                   : "memory");
    if (lane == 0)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(mst + kMetaTile), "r"(tile) : "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(full + s);
    if (++s == S) s = 0;
    wk_cur = wk_next;
    v_cur = v_next;
    wk_next = wk_nn;
  }
  for (int u = t; u < t + S; ++u)  // consume the scan warps' releases of the last stages
    if (u >= S) { FB_PROG(a, u, 3); nb_sync(kNbItEmpty + u % S, kNbItCount); }
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
__device__ __forceinline__ void planes_loop(const EmitArgs& a, const Sm& m, int lane) {
  const uint32_t pl_s = su32(m.base + a.off_pl);
  const int n2 = (a.dbg & 1) ? 0 : 2 * a.n_planes;
  const int S = a.plane_stages;
  int t = 0;
  for (int64_t i = blockIdx.x; i < a.n_sel; i += gridDim.x, ++t) {
    const int ps = t % S;
    const int tile = a.work[i * a.work_stride].x;
    FB_PROG(a, t, 1);
    if (t >= S) nb_sync(kNbPlEmpty + ps, kNbPlCount);  // builders finished tile t - S
    FB_PROG(a, t, 2);
    const uint32_t dst = su32(m.base + a.off_p + (size_t)ps * a.plane_stage_bytes);
    const int64_t col0 = (int64_t)tile * kTileW;
    for (int e0 = lane; e0 < n2; e0 += 32 * 8) {
      int pl[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 32 * u;
        pl[u] = e < n2 ? (int)lds16(pl_s + 2u * (uint32_t)(e >> 1)) : 0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 32 * u;
        if (e < n2)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (uint32_t)e * 16u),
                       "l"(a.planes + (int64_t)pl[u] * a.n_words + col0 + 2 * (e & 1))
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (t >= S - 1) {  // tile t - S + 1 has landed once at most S - 1 groups are pending
      FB_PROG(a, t, 5);
      cp_async_wait_stages(S - 1);
      FB_PROG(a, t, 6);
      nb_arrive(kNbPlFull + (t - S + 1) % S, kNbPlCount);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  for (int u = (t - S + 1 > 0 ? t - S + 1 : 0); u < t; ++u) nb_arrive(kNbPlFull + u % S, kNbPlCount);
  for (int u = t; u < t + S; ++u)  // consume the builders' releases of the last stages
    if (u >= S) { FB_PROG(a, u, 3); nb_sync(kNbPlEmpty + u % S, kNbPlCount); }
  FB_PROG(a, t, 4);
}

// ---- MMA issuer: per sub-tile (M-block mb, item half h) the gate-arming K = 32 MMA
// (query digit row x a tile of 127s), then 4 K-steps of kind::i8, into TMEM buffer seq % 4
__device__ __forceinline__ void mma_loop(const EmitArgs& a, const Sm& m, uint32_t tmem_base) {
  uint64_t* items_full = m.bars + kBarItemsFull;
  uint64_t* acc_full = m.bars + kBarAccFull;
  uint64_t* acc_empty = m.bars + kBarAccEmpty;
  constexpr uint32_t idesc = idesc_i8(kBM, kSubN);
  const uint32_t gate_s = su32(m.base + a.off_gate);
  const uint32_t a_s = su32(m.base + a.off_a);
  int s = 0;
  uint32_t ph = 0, seq = 0;
  for (int64_t i = blockIdx.x; i < a.n_sel; i += gridDim.x) {
    FB_PROG(a, i, 1);
    mbar_wait(items_full + s, ph);
    FB_PROG(a, i, 2);
    tc_fence_after();
    const uint32_t b_s = su32(m.base + a.off_b + (size_t)s * kItemStage);
    for (int mb = 0; mb < a.n_mblk; ++mb) {
      const uint32_t a_base = a_s + (uint32_t)mb * kBM * kRow;
#pragma unroll
      for (int h = 0; h < 2; ++h, ++seq) {
        const uint32_t buf = seq & 3u;
        FB_PROG(a, seq, 3);
        mbar_wait(acc_empty + buf, ((seq >> 2) & 1u) ^ 1u);
        FB_PROG(a, seq, 4);
        tc_fence_after();
        const uint32_t d = tmem_base + buf * kSubN;
        umma_i8(d, plain_desc(gate_s + (uint32_t)mb * (kBM / 8) * 256u, 128u, 256u),
                plain_desc(gate_s + kGateBytes, 128u, 0u), idesc, 0u);
        // item half h starts 128 rows (16 KB, a whole number of 1 KB swizzle atoms) in
#pragma unroll
        for (int kk = 0; kk < kRow / 32; ++kk)
          umma_i8(d, sw128_desc(a_base + kk * 32), sw128_desc(b_s + h * 16384u + kk * 32), idesc,
                  1u);
        umma_commit(acc_full + buf);
      }
    }
    if (++s == a.item_stages) { s = 0; ph ^= 1u; }
  }
}

// ---- column builders: per literal column the AND of its planes' 256 tile bits, then eight
// 32 x 32 bit transposes so item row i holds bit c of every column c ---------------------
__device__ __forceinline__ void build_loop(const EmitArgs& a, const Sm& m, int lw, int lane) {
  const int16_t* sLS = reinterpret_cast<const int16_t*>(m.base + a.off_ls);
  int it = 0;
  for (int64_t i = blockIdx.x; i < a.n_sel; i += gridDim.x, ++it) {
    const int st = it & 1;
    const int ps = it % a.plane_stages;
    FB_PROG(a, it, 1);
    if (it >= 2) nb_sync(kNbCbEmpty + st, kNbCbCount);
    FB_PROG(a, it, 2);
    nb_sync(kNbPlFull + ps, kNbPlCount);
    FB_PROG(a, it, 3);
    const uint32_t p_s = su32(m.base + a.off_p + (size_t)ps * a.plane_stage_bytes);
    uint32_t* TB = reinterpret_cast<uint32_t*>(m.base + a.off_cb + (size_t)st * a.cb_stage_bytes);
    for (int cb = lw; cb < ((a.dbg & 4) ? 0 : a.cnf_words); cb += kNBuild) {
      const int col = cb * 32 + lane;
      uint32_t w[8];
#pragma unroll
      for (int ib = 0; ib < 8; ++ib) w[ib] = col < a.n_cols ? ~0u : 0u;
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
          w[0] &= lo.x; w[1] &= lo.y; w[2] &= lo.z; w[3] &= lo.w;
          w[4] &= hi.x; w[5] &= hi.y; w[6] &= hi.z; w[7] &= hi.w;
        }
        if (neg) {
#pragma unroll
          for (int ib = 0; ib < 8; ++ib) w[ib] = ~w[ib];
        }
      }
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
      for (int ib = 0; ib < 8; ++ib) TB[(ib * 32 + lane) * a.tb_stride + cb] = w[ib];
    }
    __syncwarp();
    nb_arrive(kNbPlEmpty + ps, kNbPlCount);
    nb_arrive(kNbCbFull + st, kNbCbCount);
  }
  for (int t = it; t < it + 2; ++t)
    if (t >= 2) { FB_PROG(a, t, 4); nb_sync(kNbCbEmpty + (t & 1), kNbCbCount); }
}

// ---- survivors: exact score, exact key test, slot reservation -------------------------
struct Pending {
  uint64_t key;
  uint32_t p;
  uint32_t slot;
  int32_t q;
};
__device__ __forceinline__ void flush(const EmitArgs& a, Pending& pd) {
  if (pd.q >= 0 && pd.p < (uint32_t)a.cap) {
    a.out_key[(int64_t)pd.q * a.cap + pd.p] = pd.key;
    if (a.out_slot) a.out_slot[(int64_t)pd.q * a.cap + pd.p] = pd.slot;
  }
  pd.q = -1;
}
// Queued survivors (filter passed): exact score from the resident query / item tiles, exact
// key test against the query's threshold, slot reservation; the stores of an emission trail
// by two emissions per lane so the atomic's round trip overlaps the next ones.
__device__ __forceinline__ void drain(const EmitArgs& a, const Sm& m, Pending (&pd)[2], int& par,
                                      uint32_t sv_s, uint32_t n, uint32_t b_s, uint32_t mst,
                                      int64_t tile, int lane) {
  const uint32_t a_s = su32(m.base + a.off_a);
  for (uint32_t i = (uint32_t)lane; i < n; i += 32u) {
    const uint32_t ent = lds16(sv_s + 2u * i);
    const int q = (int)(ent >> 8);
    const uint32_t item = ent & 255u;
    const int32_t score = smem_dot(a_s + (uint32_t)q * kRow, (uint32_t)q & 7u,
                                   b_s + item * kRow, item & 7u);
    const uint64_t key = make_key(score, lds32(mst + 4u * item));
    if (key >= m.sT[q]) {
      const uint32_t slot = (uint32_t)(tile * kTile) + item;
      if (par) {
        flush(a, pd[1]);
        pd[1].p = atomicAdd(a.out_cnt + q, 1u);
        pd[1].key = key;
        pd[1].slot = slot;
        pd[1].q = q;
      } else {
        flush(a, pd[0]);
        pd[0].p = atomicAdd(a.out_cnt + q, 1u);
        pd[0].key = key;
        pd[0].slot = slot;
        pd[0].q = q;
      }
      par ^= 1;
    }
  }
}

// ---- scan epilogue: warp (TMEM lane quadrant, item half h) drains its 32 lanes x 128
// columns of every sub-tile (mb, h) -- lane = query. The hit word of 32 items is the sign
// bits of the gate-armed accumulators & validity & range (& explicit mask); once the four
// words are in registers the accumulator buffer goes back to the MMA, and every hit bit is
// tested against the query's CNF window (4 x (u32 pair offset, 64-bit mask), loaded once per
// sub-tile) on the item's column bits. Survivors queue per warp for the exact test. --------
template <bool kMasks>
__device__ __forceinline__ void scan_loop(const EmitArgs& a, const Sm& m, uint32_t tmem_base,
                                          int warp, int lane) {
  uint64_t* items_full = m.bars + kBarItemsFull;
  uint64_t* acc_full = m.bars + kBarAccFull;
  uint64_t* acc_empty = m.bars + kBarAccEmpty;
  const int quad = warp & 3;
  const int dw = warp - kWDense0;
  const int h = dw >> 2;
  const int n_sub = 2 * a.n_mblk;
  // gate constants of this lane's rows in both M-blocks
  uint32_t allm[2];
  for (int mb = 0; mb < 2; ++mb) {
    const int q = mb * kBM + quad * 32 + lane;
    bool all = false;
    if (mb < a.n_mblk) gate_digits(q < a.nq ? m.sT[q] : ~0ull, all);
    allm[mb] = all ? ~0u : 0u;
  }
  const uint32_t cb0 = su32(m.base + a.off_cb);
  const uint32_t sv_s = su32(m.base + a.off_sv) + (uint32_t)dw * (kSurvCap * 2u);
  const uint32_t hl_s = su32(m.base + a.off_hl) + (uint32_t)dw * (kHitCap * 2u);
  const uint32_t lt = lanemask_lt();
  Pending pd[2];
  pd[0].q = pd[1].q = -1;
  pd[0].p = pd[1].p = 0u;
  pd[0].key = pd[1].key = 0ull;
  pd[0].slot = pd[1].slot = 0u;
  int par = 0;
  int it = 0, s = 0;
  uint32_t iph = 0;
  for (int64_t i = blockIdx.x; i < a.n_sel; i += gridDim.x, ++it) {
    FB_PROG(a, it, 1);
    mbar_wait(items_full + s, iph);
    FB_PROG(a, it, 2);
    const uint32_t mst = su32(m.base + a.off_meta) + (uint32_t)s * kMetaBytes;
    const int64_t tile = (int64_t)lds32(mst + kMetaTile);
    const uint32_t b_s = su32(m.base + a.off_b + (size_t)s * kItemStage);
    // lane c < 4: validity & range bits of chunk 4h + c
    const uint32_t vchunk = lane < 4 ? lds32(mst + kMetaValid + 4u * (uint32_t)(4 * h + lane)) : 0u;
    const int st = it & 1;
    const uint32_t cbs = cb0 + (uint32_t)st * a.cb_stage_bytes;
    bool cb_ready = false;
    uint32_t n_sv = 0;
#pragma unroll 1
    for (int mb = 0; mb < a.n_mblk; ++mb) {
      const uint32_t seq = (uint32_t)(it * n_sub + 2 * mb + h);
      const uint32_t buf = seq & 3u;
      const int q = mb * kBM + quad * 32 + lane;
      const bool qok = q < a.nq;
      const uint32_t am = mb == 0 ? allm[0] : allm[1];
      // this query's CNF window (L1-resident records), fetched while the MMA runs
      uint4 L = make_uint4(0u, 0u, 0u, 0u), H = L, W = L;
      if (qok) {
        const uint4* rec = reinterpret_cast<const uint4*>(a.qrec + (size_t)q * 12);
        L = __ldg(rec);
        H = __ldg(rec + 1);
        W = __ldg(rec + 2);
      }
      FB_PROG(a, it * 4 + mb, 3);
      mbar_wait(acc_full + buf, (seq >> 2) & 1u);
      FB_PROG(a, it * 4 + mb, 4);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * kSubN;
      // eligibility word of chunk c: validity & range (& explicit mask)
      uint64_t m01[2] = {~0ull, ~0ull};
      if (kMasks) {
        const uint64_t* mw = a.masks + (int64_t)(qok ? q : 0) * a.n_words + tile * kTileW + 2 * h;
        m01[0] = __ldg(mw);
        m01[1] = __ldg(mw + 1);
      }
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
        if (lane == 0) mbar_arrive(acc_empty + buf);
        w3 = word_of(3, rb);
      }
      if (a.dbg & 2) continue;
      if (!cb_ready) {  // column bits of this tile (the builders run a tile ahead)
        FB_PROG(a, it, 5);
        nb_sync(kNbCbFull + st, kNbCbCount);
        FB_PROG(a, it, 6);
        cb_ready = true;
      }
      // compact the warp's hits: lane = query, (chunk, bit) per hit -> a per-warp list of
      // (query lane, item) entries, then one filter test per lane per round
      const uint32_t nh = (uint32_t)(__popc(w0) + __popc(w1) + __popc(w2) + __popc(w3));
      uint32_t incl = nh;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - nh;
      for (uint32_t b0 = 0; b0 < total; b0 += (uint32_t)kHitCap) {
        // entries of global index [b0, b0 + kHitCap); more only when a batch holds nearly
        // every pair (threshold 0 / unfiltered)
        if (nh != 0u && excl < b0 + (uint32_t)kHitCap && excl + nh > b0) {
          uint32_t pos = excl;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t x = c == 0 ? w0 : c == 1 ? w1 : c == 2 ? w2 : w3;
            while (x != 0u) {
              const uint32_t j = (uint32_t)(__ffs(x) - 1);
              x &= x - 1u;
              if (pos >= b0 && pos < b0 + (uint32_t)kHitCap)
                sts16(hl_s + 2u * (pos - b0), ((uint32_t)lane << 7) | ((uint32_t)c * 32u + j));
              ++pos;
            }
          }
        }
        __syncwarp();
        const uint32_t n = min(total - b0, (uint32_t)kHitCap);
        for (uint32_t r0 = 0; r0 < n; r0 += 32u) {
          const uint32_t e = r0 + (uint32_t)lane;
          const uint32_t ent = e < n ? lds16(hl_s + 2u * e) : 0u;
          const int ql = (int)(ent >> 7);
          const uint32_t item = (uint32_t)(h * kSubN) + (ent & 127u);
          // the hit's query window from the lane that owns the query
          uint32_t lo[4], hi[4], wo[4];
          lo[0] = __shfl_sync(0xffffffffu, L.x, ql); lo[1] = __shfl_sync(0xffffffffu, L.y, ql);
          lo[2] = __shfl_sync(0xffffffffu, L.z, ql); lo[3] = __shfl_sync(0xffffffffu, L.w, ql);
          hi[0] = __shfl_sync(0xffffffffu, H.x, ql); hi[1] = __shfl_sync(0xffffffffu, H.y, ql);
          hi[2] = __shfl_sync(0xffffffffu, H.z, ql); hi[3] = __shfl_sync(0xffffffffu, H.w, ql);
          const uint32_t wp = __shfl_sync(0xffffffffu, W.x, ql);
          const bool nof = __shfl_sync(0xffffffffu, W.y, ql) != 0u;
          wo[0] = wp & 255u; wo[1] = (wp >> 8) & 255u; wo[2] = (wp >> 16) & 255u; wo[3] = wp >> 24;
          const bool surv = e < n &&
              (nof || cnf_test_win(cbs + item * (uint32_t)a.tb_stride * 4u, wo, lo, hi));
          const uint32_t sb = __ballot_sync(0xffffffffu, surv);
          if (surv)
            sts16(sv_s + 2u * (n_sv + (uint32_t)__popc(sb & lt)),
                  ((uint32_t)(mb * kBM + quad * 32 + ql) << 8) | item);
          n_sv += (uint32_t)__popc(sb);
          if (n_sv > (uint32_t)(kSurvCap - 32)) {
            __syncwarp();
            drain(a, m, pd, par, sv_s, n_sv, b_s, mst, tile, lane);
            __syncwarp();
            n_sv = 0;
          }
        }
        __syncwarp();
      }
    }
    if (!cb_ready) nb_sync(kNbCbFull + st, kNbCbCount);
    __syncwarp();
    nb_arrive(kNbCbEmpty + st, kNbCbCount);  // column bits consumed
    if (n_sv) drain(a, m, pd, par, sv_s, n_sv, b_s, mst, tile, lane);
    __syncwarp();
    nb_arrive(kNbItEmpty + s, kNbItCount);  // item rows and id ranks read
    FB_PROG(a, it, 7);
    if (++s == a.item_stages) { s = 0; iph ^= 1u; }
  }
  flush(a, pd[0]);
  flush(a, pd[1]);
}

__global__ void __launch_bounds__(kThreads, 1)
    k_emit_win(const __grid_constant__ CUtensorMap tmap_items, const EmitArgs a) {
  const Sm m = carve(a);
  uint8_t* smem = m.base;
  uint64_t* bars = m.bars;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- prologue: queries (SW128), thresholds, plane ids, column table, gate tiles ----
  {
    uint8_t* sA = smem + a.off_a;
    for (int i = threadIdx.x; i < a.n_mblk * kBM * 8; i += kThreads) {
      const int r = i >> 3, c = i & 7;
      int4 v = make_int4(0, 0, 0, 0);
      if (r < a.nq) v = __ldg(reinterpret_cast<const int4*>(a.queries + (int64_t)r * kRow) + c);
      *reinterpret_cast<int4*>(sA + r * kRow + ((c ^ (r & 7)) << 4)) = v;
    }
    for (int q = threadIdx.x; q < kMaxQ; q += kThreads)
      m.sT[q] = (a.threshold != nullptr && q < a.nq) ? a.threshold[q] : 0ull;
    int16_t* pl = reinterpret_cast<int16_t*>(smem + a.off_pl);
    for (int i = threadIdx.x; i < a.n_planes; i += kThreads) pl[i] = a.plane_list[i];
    int16_t* sLS = reinterpret_cast<int16_t*>(smem + a.off_ls);
    for (int i = threadIdx.x; i < a.n_cols * a.k_max; i += kThreads) {
      // column -> plane-slot table (negated columns flagged by bit 14 on slot 0)
      const int c = i / a.k_max, j = i - c * a.k_max;
      const int cl = a.col_leaf[c];
      const int leaf = cl >= 0 ? cl : ~cl;
      int sl = a.leaf_slot[leaf * a.k_max + j];
      if (j == 0 && cl < 0) sl |= 0x4000;
      sLS[i] = (int16_t)sl;
    }
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
    for (int s = 0; s < 3; ++s)
      mbar_init(bars + kBarItemsFull + s, 1 + 32 + 1);  // TMA expect-tx, id-rank cp.async, meta
    for (int b = 0; b < 4; ++b) {
      mbar_init(bars + kBarAccFull + b, 1);
      mbar_init(bars + kBarAccEmpty + b, 4);  // the four dense warps of the buffer's half
    }
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
    items_loop(a, &tmap_items, m, lane);
  } else if (warp == kWMma) {
    if (lane == 0) mma_loop(a, m, tmem_base);
  } else if (warp == kWPlanes) {
    planes_loop(a, m, lane);
  } else if (warp < kWDense0) {
    build_loop(a, m, warp - kWBuild0, lane);
  } else if (a.masks != nullptr) {
    scan_loop<true>(a, m, tmem_base, warp, lane);
  } else {
    scan_loop<false>(a, m, tmem_base, warp, lane);
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

size_t layout(EmitArgs& t, int item_stages, int plane_stages) {
  size_t off = 0;
  t.off_a = 0;
  off = (size_t)t.n_mblk * kBM * kRow;
  t.off_b = (uint32_t)align_up(off, 1024);
  off = t.off_b + (size_t)item_stages * kItemStage;
  t.plane_stage_bytes = (uint32_t)align_up((size_t)(t.n_planes > 0 ? t.n_planes : 1) * 32, 128);
  t.off_p = (uint32_t)align_up(off, 128);
  off = t.off_p + (size_t)plane_stages * t.plane_stage_bytes;
  t.cb_stage_bytes = (uint32_t)(kTile * t.tb_stride * 4);
  t.off_cb = (uint32_t)align_up(off, 128);
  off = t.off_cb + 2ull * t.cb_stage_bytes;
  t.off_ls = (uint32_t)align_up(off, 16);
  off = t.off_ls + (size_t)(t.n_cols > 0 ? t.n_cols : 1) * (t.k_max > 0 ? t.k_max : 1) * 2;
  t.off_thr = (uint32_t)align_up(off, 16);
  off = t.off_thr + (size_t)kMaxQ * 8;
  t.off_bar = (uint32_t)align_up(off, 16);
  off = t.off_bar + kBarCount * 8;
  t.off_pl = (uint32_t)align_up(off, 16);
  off = t.off_pl + (size_t)(t.n_planes > 0 ? t.n_planes : 1) * 2;
  t.off_gate = (uint32_t)align_up(off, 128);
  off = t.off_gate + kGateBytes + 256;
  t.off_sv = (uint32_t)align_up(off, 16);
  off = t.off_sv + (size_t)kNDense * kSurvCap * 2;
  t.off_hl = (uint32_t)align_up(off, 16);
  off = t.off_hl + (size_t)kNDense * kHitCap * 2;
  t.off_meta = (uint32_t)align_up(off, 16);
  off = t.off_meta + (size_t)item_stages * kMetaBytes;
  return off + 1024;  // alignment slack of the dynamic shared-memory base
}

constexpr size_t kSmemLimit = 227 * 1024;

bool pick(EmitArgs& t, size_t& smem) {
  const int prefs[4][2] = {{3, 3}, {3, 2}, {2, 2}, {3, 1}};
  const char* e = getenv("FB_EMIT_STAGES");  // experiments: "items,planes"
  if (e != nullptr) {
    int si = 0, sp = 0;
    if (sscanf(e, "%d,%d", &si, &sp) == 2 && si >= 2 && si <= 3 && sp >= 1 && sp <= 3) {
      smem = layout(t, si, sp);
      if (smem <= kSmemLimit) {
        t.item_stages = si;
        t.plane_stages = sp;
        return true;
      }
    }
  }
  for (const auto& p : prefs) {
    smem = layout(t, p[0], p[1]);
    if (smem <= kSmemLimit) {
      t.item_stages = p[0];
      t.plane_stages = p[1];
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
    k_emit_win<<<grid, kThreads, smem, s>>>(tmap, t);
    FB_LAUNCH_CHECK("k_emit_win");
    if (t.prog != nullptr) {  // watchdog: dump every warp's last point if it does not finish
      for (int w = 0; w < 100 && cudaStreamQuery(s) == cudaErrorNotReady; ++w) usleep(50000);
      if (cudaStreamQuery(s) == cudaErrorNotReady) {
        fprintf(stderr, "k_emit_win hung: n_sel %lld grid %d nq %d n_mblk %d stages %d/%d\n",
                (long long)n_sel, grid, t.nq, t.n_mblk, t.item_stages, t.plane_stages);
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
