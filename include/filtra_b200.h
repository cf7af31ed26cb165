/*
 * filtra_b200 -- C-ABI of the B200-native filtered int8 top-k hot path.
 *
 * Plain pointers and sizes only (no torch types). Device pointers are
 * caller-owned; every call is asynchronous on the given cudaStream_t (passed as
 * void*) unless documented otherwise. Return codes: 0 = ok, otherwise one of
 * FB_ERR_*; fb_last_error() returns the thread-local message of the last
 * failure. Codes map 1:1 onto the reference's Python exceptions (see
 * paper_2511_14881_b200/_native.py).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/filtra):
 *   fb_hash_leaves        <- bloom.hash_seed / positions_from_seed / hash_positions  (bloom.py:65-88)
 *   fb_bloom_build        <- bloom.build_bloom                                       (bloom.py:114-144)
 *   fb_filter_eval        <- filter_query.eval_compiled + bloom.bloom_eval_leaf      (filter_query.py:314-356, bloom.py:160-181)
 *   fb_quantize           <- quantize.quantize_vector / quantize_matrix              (quantize.py:64-76)
 *   fb_topk_plan_create /
 *   fb_topk_execute       <- ivf.search_clusters + ivf._select_topk, batched; with a
 *                            filter program this is retrieval.codesigned_search      (ivf.py:272-334, retrieval.py:110-144)
 *   fb_merge_topk         <- serve._reduce_topk over the per-shard results           (serve.py:98-121)
 *   fb_dequant_scores     <- quantize.dequantize applied to both operands of the dot (quantize.py:79-81)
 *   fb_pack_text /
 *   fb_pack_postfix       <- filter_query.parse_filter + compile_filter for a whole batch,
 *                            plus the device-form packing (filter_query.py:82-189, 280-311)
 */
#ifndef FILTRA_B200_H
#define FILTRA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FB_ABI_VERSION 5

enum fb_status {
  FB_OK = 0,
  FB_ERR_INVALID = 1,          /* ValueError: bad params, unaligned slot range, unbalanced program */
  FB_ERR_DIM_MISMATCH = 2,     /* errors.DimMismatch */
  FB_ERR_LENGTH_MISMATCH = 3,  /* errors.LengthMismatch */
  FB_ERR_DEGENERATE = 4,       /* errors.DegenerateRange */
  FB_ERR_CUDA = 5,             /* CUDA runtime failure */
  FB_ERR_UNSUPPORTED = 6,      /* outside this build's limits (documented per call) */
  FB_ERR_NO_DEVICE = 7,        /* no sm_100 device */
  FB_ERR_PARSE = 8             /* filter text not accepted: the caller re-parses it with the
                                  reference grammar to raise FilterSyntaxError / UnknownFeature /
                                  UnknownValue with the reference's message */
};

/* Opcodes of the postfix filter program (filter_query.OpCode, filter_query.py:253-257). */
enum fb_opcode { FB_OP_PUSH_LEAF = 0, FB_OP_AND = 1, FB_OP_OR = 2, FB_OP_NOT = 3 };

#define FB_MAX_K_HASHES 32     /* K per leaf (reference: unbounded; 5 by default) */
#define FB_MAX_STACK 64        /* filter program stack depth */
#define FB_MAX_LEAVES 16384    /* distinct leaves per batch (14-bit op argument) */

/*
 * Device-resident index over one shard's slot space (ivf.IvfIndex + bloom.BloomIndex).
 *   items     int8  [n_slots, dim_pad]  quantized rows in slot order; padding rows/columns are 0
 *   planes    u64   [m_bits, n_words]   transposed Bloom planes (bloom.py:91-111 layout)
 *   valid     u64   [n_words]           validity words (padding slots cleared)
 *   id_rank   u32   [n_slots]           rank of the slot's item_id among the shard's valid
 *                                       items (ascending u64); equal scores break by it
 *   item_ids  u64   [n_slots]           item id per slot
 *   row_sum   i32   [n_slots]           sum of the row's codes (dequantised-score term); may be NULL
 */
typedef struct fb_index {
  const int8_t* items;
  const uint64_t* planes;
  const uint64_t* valid;
  const uint32_t* id_rank;
  const uint64_t* item_ids;
  const int32_t* row_sum;
  int64_t n_slots;   /* multiple of 64 */
  int64_t n_words;   /* n_slots / 64 */
  int32_t dim;       /* logical embedding dimension */
  int32_t dim_pad;   /* row stride in bytes: dim rounded up to 32 */
  int32_t m_bits;
  int32_t k_hashes;
  /* Nullable inverse of id_rank (slot holding each rank) when id_rank is a permutation
   * of [0, n_slots). With it, candidates carry only their merge key and the selection
   * sorts keys alone (radix sort in shared memory). */
  const uint32_t* slot_of_rank;
  /* Nullable: item id of each rank (item_ids[slot_of_rank[r]]), so the selection gathers
   * an output id with one load instead of two dependent ones. */
  const uint64_t* id_of_rank;
  /* Dense ids: non-zero when id_of_rank[r] == id_base + r (mod 2^64) for the rank r of
   * every valid slot (a shard whose valid ids are one contiguous run, e.g. 0..n-1). The
   * selection then computes each output id from its rank instead of gathering it from
   * id_of_rank (2.56M random 8-byte reads per batch at config 2). Zero: use the table. */
  int32_t id_dense;
  uint64_t id_base;
} fb_index_t;

/*
 * A batch of compiled filters (filter_query.CompiledFilter, one per query), with the
 * leaves de-duplicated across the batch. All arrays are device pointers.
 *   leaf_pos   i32 [n_leaves * k_max]  plane indices per leaf, ascending, -1 padded
 *   op_offset  i32 [n_queries + 1]     query q's ops are ops[op_offset[q] .. op_offset[q+1])
 *   ops        u16 [...]               (opcode << 14) | leaf index
 * A query with zero ops is unfiltered (mask = validity).
 */
typedef struct fb_filter_prog {
  int32_t n_queries;
  int32_t n_leaves;
  int32_t k_max;
  int32_t max_stack;
  const int32_t* leaf_pos;
  const int32_t* op_offset;
  const uint16_t* ops;
  /* Register-machine form consumed by the tensor-core scan (all nullable; when absent
   * the SIMT scan is used). The batch's distinct planes are staged per tile in
   * plane_list order; leaf_slot holds each leaf's positions as indices into that list.
   *   rops: (ropcode << 13) | leaf, ropcodes FB_ROP_*; rmax_stack = its max depth. */
  int32_t n_planes;
  int32_t rmax_stack;
  int32_t n_rops;              /* total rops (multiple of FB_ROP_ALIGN) */
  int32_t reserved;
  const int32_t* plane_list;   /* [n_planes] plane ids (any m_bits) */
  const int16_t* leaf_slot;    /* [n_leaves * k_max] */
  const int32_t* rop_offset;   /* [n_queries + 1] */
  const uint16_t* rops;
  /* Conjunctive normal form (nullable; set when every program is an AND of ORs of
   * literals). Literal columns: col_leaf[c] = leaf, or ~leaf for a negated literal.
   * qmask[q][g][w] is the column bitmask of query q's group g (cnf_words u32 words);
   * qgroups[q] the number of groups (0 = unfiltered). A slot passes query q iff for
   * every group some column of the group holds for it. */
  int32_t n_cols;
  int32_t cnf_words;           /* <= 8 */
  int32_t cnf_gmax;            /* <= 8 */
  int32_t cnf_windowed;        /* 1: every group's columns lie in u32 words {2j, 2j+1} and
                                  cnf_gmax <= 4 (register-resident filter test) */
  const int16_t* col_leaf;     /* [n_cols] */
  const uint32_t* qmask;       /* [n_queries][cnf_gmax][cnf_words] */
  const int32_t* qgroups;      /* [n_queries] */
} fb_filter_prog_t;

/* Register-machine opcodes: PUSH l | PUSHN l (push ~leaf) | ANDL l (top &= leaf) |
 * ORL l (top |= leaf) | ANDS / ORS (pop, combine) | NOT (top = ~top). Peephole-lowered
 * from the postfix ops on the host; NOT without "& valid" is exact because the final
 * result is ANDed with validity. */
enum fb_ropcode {
  FB_ROP_PUSH = 0, FB_ROP_PUSHN = 1, FB_ROP_ANDL = 2, FB_ROP_ORL = 3,
  FB_ROP_ANDS = 4, FB_ROP_ORS = 5, FB_ROP_NOT = 6, FB_ROP_NOP = 7
};
/* Each query's rops start on an 8-op boundary (rop_offset[q] % 8 == 0) and are padded
 * with FB_ROP_NOP to a multiple of 8, so the kernel fetches them 16 bytes at a time. */
#define FB_ROP_ALIGN 8

/* Work counters (ivf.ScanStats + bloom.FilterStats), filled analytically by the plan. */
typedef struct fb_stats {
  int64_t slots_scanned;
  int64_t tiles;
  int64_t max_tile_rows;
  int64_t slots_evaluated;
  int64_t fallback_queries;   /* queries that needed the exact-threshold fallback on the last execute */
} fb_stats_t;

int fb_abi_version(void);
const char* fb_last_error(void);
/* 1 when device 0 is sm_100 and the sm_100a cubin loads; else 0 (message in fb_last_error). */
int fb_device_ok(void);

/* Host: positions of n (fid, value) leaves; pos_out[n*k_hashes] ascending, -1 padded;
 * n_pos_out[n] (nullable) = number of distinct positions. */
int fb_hash_leaves(const uint64_t* fid, const uint64_t* value, int64_t n, int32_t m_bits,
                   int32_t k_hashes, int32_t* pos_out, int32_t* n_pos_out);

/* Device: zero `planes` then set bit (p, slot) for every pair and hash position p. */
int fb_bloom_build(const uint64_t* fid, const uint64_t* value, const int64_t* slot,
                   int64_t n_pairs, int64_t n_slots, int32_t m_bits, int32_t k_hashes,
                   uint64_t* planes, void* stream);

/* Device: masks_out[q][w - w0] for words [w0, w1) of every query's program.
 * apply_valid = 1 gives eval_compiled semantics; 0 gives the raw program value
 * (bloom_eval_leaf for single-leaf programs). */
int fb_filter_eval(const fb_index_t* idx, const fb_filter_prog_t* prog, int64_t w0, int64_t w1,
                   int32_t apply_valid, uint64_t* masks_out, void* stream);

/* Device: int8 out[rows, out_stride] = clip(rint((x - gmin) * (255 / (gmax - gmin))) - 128)
 * in float64; columns [cols, out_stride) are zeroed. */
int fb_quantize(const float* x, int64_t rows, int32_t cols, double gmin, double gmax,
                int8_t* out, int32_t out_stride, void* stream);

/* Same as fb_quantize for float64 inputs (quantize_matrix / quantize_vector cast to float64). */
int fb_quantize_f64(const double* x, int64_t rows, int32_t cols, double gmin, double gmax,
                    int8_t* out, int32_t out_stride, void* stream);

/* Device: out[r] = sum of int8 row r over cols (row_sum for fb_index_t). */
int fb_row_sums(const int8_t* x, int64_t rows, int32_t cols, int32_t stride, int32_t* out,
                void* stream);

/* ---- batched filtered top-k ------------------------------------------------------ */
typedef struct fb_topk_plan fb_topk_plan_t;

enum fb_plan_flags {
  FB_PLAN_FORCE_FALLBACK = 1,  /* testing: take the exact-threshold fallback for every query */
  FB_PLAN_SIMT = 2,            /* use the SIMT scan kernel instead of the tcgen05 one */
  FB_PLAN_NO_SAMPLE = 4        /* skip the sampling pass (threshold 0 for every query) */
};

/* Plan for `n_queries` queries against `idx` over the slot ranges ranges[2*i], ranges[2*i+1]
 * (host array; starts must be 64-aligned). Allocates all device scratch once. */
int fb_topk_plan_create(const fb_index_t* idx, int32_t n_queries, int32_t k,
                        const int64_t* ranges, int32_t n_ranges, int32_t flags,
                        fb_topk_plan_t** plan_out);
int fb_topk_plan_destroy(fb_topk_plan_t* plan);
/* Fills stats analytically for one execute of this plan (host). */
int fb_topk_plan_stats(const fb_topk_plan_t* plan, fb_stats_t* stats);

/* Hot path: queries_q int8 [n_queries, dim_pad]; prog may be NULL (unfiltered);
 * masks u64 [n_queries, n_words] (nullable) is an explicit per-query slot mask ANDed
 * into eligibility (search_clusters' `mask` argument, ivf.py:285-312).
 * Outputs (device, [n_queries, k], rows sorted by (score desc, item_id asc)):
 *   out_ids u64, out_scores i32, out_count i32 [n_queries] = min(k, eligible);
 *   out_keys u64 (nullable): ((score ^ 2^31) << 32) | (~id_rank) -- the merge key;
 *   out_fscores f64 (nullable): dequantised scores (needs idx->row_sum and gmin/gmax).
 * No host synchronisation; capturable in a CUDA graph. */
int fb_topk_execute(fb_topk_plan_t* plan, const int8_t* queries_q, const fb_filter_prog_t* prog,
                    const uint64_t* masks, uint64_t* out_ids, int32_t* out_scores, int32_t* out_count,
                    uint64_t* out_keys, double* out_fscores, double gmin, double gmax,
                    void* stream);

/* Measurement hooks: total kernel launches issued by this library (process-wide), and
 * CUDA-event timing of the emit scan and the selection of a plan's last execute. */
uint64_t fb_launch_count(void);
/* 1 when the plan's last execute ran its emit pass on the tcgen05 kernel, 0 for SIMT. */
int fb_topk_scan_path(const fb_topk_plan_t* plan);
/* Testing: raw int32 scores of every (query, slot) from the tcgen05 kernel (unfiltered,
 * all slots); out [n_queries, idx->n_slots]. Synchronous. */
int fb_debug_tc_scores(const fb_index_t* idx, const int8_t* queries_q, int32_t n_queries,
                       int32_t* out, void* stream);
int fb_topk_set_timing(fb_topk_plan_t* plan, int32_t enable);
int fb_topk_last_timing(fb_topk_plan_t* plan, float* emit_ms, float* select_ms);

/* Device: merge n_lists per-query lists, each sorted by (score desc, item_id asc), into the
 * global top-k (serve._reduce_topk semantics, serve.py:98-100). Pairs are compared directly,
 * so shards need no global id ranks.
 *   in_scores i32 [n_lists, n_queries, k_in], in_ids u64 [same], in_count i32 [n_lists, n_queries],
 *   in_fscores f64 [same] (nullable); outputs [n_queries, k_out]; out_fscores nullable. */
int fb_merge_topk(const int32_t* in_scores, const uint64_t* in_ids, const double* in_fscores,
                  const int32_t* in_count, int32_t n_lists, int32_t n_queries, int32_t k_in,
                  int32_t k_out, uint64_t* out_ids, int32_t* out_scores, int32_t* out_count,
                  double* out_fscores, void* stream);

/* Device: f64 dequantised dot from the int32 dot, the item row sum and the query sum
 * (closed form of sum_j dequantize(a_j) * dequantize(b_j)). */
int fb_dequant_scores(const int32_t* scores, const int32_t* item_row_sum, const int32_t* query_sum,
                      int32_t n_queries, int32_t k, const int32_t* count, int32_t dim,
                      double gmin, double gmax, double* out, void* stream);

/* Device: out[r] = exact int32 dot of int8 row r (stride bytes) with vec (quantize.int8_dot_rows,
 * quantize.py:84-102). */
int fb_int8_dot_rows(const int8_t* rows, int64_t n_rows, int32_t dim, int32_t stride,
                     const int8_t* vec, int32_t* out, void* stream);

/* Device: out[c] = float64 dot of float32 row c with the float32 query, accumulated with
 * numpy's pairwise-summation order (vecmath.dot_rows, vecmath.py:15-24) so centroid
 * probing ties resolve exactly as in ivf.probe_centroids (ivf.py:261-269). */
int fb_dot_rows_f64(const float* rows, int64_t n_rows, int32_t dim, const float* vec,
                    double* out, void* stream);

/* Device, multi-task re-scoring (config 5; retrieval.retrieve re-rank with the identity
 * mixture-of-logits scorer, scoring.py:99-130, retrieval.py:180-186): for request b and task
 * t, out[(b * n_tasks + t) * n_cand + c] = float64 dot of cache row rows[b * n_cand + c]
 * (float32, dim wide) with users[(b * n_tasks + t) * dim ..], in numpy's pairwise order (so
 * the scores are bit-identical to the reference); c >= count[b] gives 0. */
int fb_task_dots_f64(const float* cache, int64_t n_rows, int32_t dim, const int64_t* rows,
                     const int32_t* count, int64_t n_cand, const float* users, int32_t n_req,
                     int32_t n_tasks, double* out, void* stream);

/* Device, multi-task union merge (retrieval.merge_candidates with merge="union",
 * retrieval.py:147-160): keys[(b * n_tasks + t) * k + i], i < counts[b * n_tasks + t], are
 * fb_topk_execute output keys (they carry the id rank); merged[b * n_tasks * k ..] receives
 * the distinct ids of request b in ascending id order (padded with all-ones), mcount[b] their
 * number. bitmap: n_requests * (ceil(n_slots / 64) + 8) u64 of scratch, zero on the first
 * call; the bitmap part is left zeroed. id_of_rank: fb_index_t.id_of_rank. merged_ranks
 * (nullable, same shape as merged, -1 padded) receives the id ranks. */
int fb_merge_union(const uint64_t* keys, const int32_t* counts, int32_t n_requests,
                   int32_t n_tasks, int32_t k, int64_t n_slots, const uint64_t* id_of_rank,
                   uint64_t* bitmap, uint64_t* merged, int64_t* merged_ranks, int32_t* mcount,
                   void* stream);

/* Device, OverArch value model (value_model.py:31-91 as retrieval.retrieve applies it,
 * retrieval.py:186-189): out[b * ld + i] = formula(task_scores[(b * n_tasks + t) * ld + i])
 * for every request b and candidate i < ld, in float64 with NumPy's rounding. code: postfix
 * u16 words (op | arg << 8): CONST c, TASK t, ADD, SUB, MUL, DIV, MIN, MAX, CLAMP c (consts
 * c, c + 1), IF_{LT,LE,GT,GE,EQ} (left right then else); consts: float64. A zero divisor for
 * a candidate i < count[b] sets *zero_flag to 1 (the reference raises DivByZero). */
int fb_value_model(const uint16_t* code, int32_t n_code, const double* consts,
                   const double* task_scores, int32_t n_requests, int32_t n_tasks, int64_t ld,
                   const int32_t* count, double* out, int32_t* zero_flag, void* stream);

/* Device, final ranking of multi-task retrieval (retrieval.retrieve, retrieval.py:190:
 * np.lexsort((merged, -final))[:topk]): for request b, the first count[b] values of
 * final_scores[b * ld ..] (merged candidates in ascending id order) ordered by (value desc,
 * position asc) with NumPy's float order (NaN last, -0.0 == +0.0); order[b * topk + r] is
 * the position of rank r (0 past out_count[b] = min(topk, count[b])). ld <= 24576,
 * topk <= 8192 (FB_ERR_UNSUPPORTED otherwise). */
int fb_final_topk(const double* final_scores, int64_t ld, const int32_t* count,
                  int32_t n_requests, int32_t topk, int64_t* order, int32_t* out_count,
                  void* stream);

/* Device, IVF-probed batched search (retrieval.codesigned_search with nprobe < n_clusters,
 * retrieval.py:110-144; ivf.search_clusters over the probed clusters, ivf.py:285-334): for
 * query b, probe_words[(b * nprobe + j) * 2 ..] is the 64-slot word range [w0, w1) of its
 * j-th probed cluster. Every slot there that is valid and passes the query's filter program
 * (evaluated over the probed words only, as the reference does) is scored exactly and its
 * key kept in cand_key[b * cap ..]; then the exact (score desc, item_id asc) top-k is written
 * as by fb_topk_execute. cap must be >= the largest number of slots one query probes (the
 * selection is exact only then); cand_slot may be NULL when idx->slot_of_rank is set and
 * k <= 24576. */
int fb_ivf_topk(const fb_index_t* idx, const int8_t* queries_q, int32_t n_queries,
                const fb_filter_prog_t* prog, const int64_t* probe_words, int32_t nprobe, int32_t k,
                int32_t cap, uint64_t* cand_key, uint32_t* cand_slot, uint32_t* cand_cnt,
                uint64_t* out_ids, int32_t* out_scores, int32_t* out_count, uint64_t* out_keys,
                double* out_fscores, double gmin, double gmax, void* stream);

/* ---- publish-side k-means (ivf.kmeans_pp_init / kmeans_train / kmeans_inertia,
 * ivf.py:68-145). data is float64 [n, dim] row-major on the device. ---- */

/* Device: D^2 seeding distances, best[i] = (init ? d_i : min(best[i], d_i)) with
 * d_i = np.sum((data[i] - data[center_row]) ** 2) in numpy's pairwise order (ivf.py:86, 97). */
int fb_kmeans_min_sqdist(const double* data, int64_t n, int32_t dim, int64_t center_row,
                         double* best, int32_t init, void* stream);

/* Scratch doubles fb_pairwise_sum_f64 needs for n elements. */
int64_t fb_pairwise_sum_scratch(int64_t n);

/* Device: *out = numpy's x.sum() for a contiguous float64 vector (pairwise summation tree,
 * bit-identical; ivf.py:89 best.sum(), ivf.py:135 inertia). */
int fb_pairwise_sum_f64(const double* x, int64_t n, double* out, double* scratch,
                        int64_t scratch_len, void* stream);

/* Device: the D^2 draw of ivf.py:94-96, *out_idx = min(searchsorted(cumsum(best), u * total,
 * 'right'), n - 1), exact: approx_prefix (any-order prefix sums of best) decides the crossing
 * when its error bound separates it, else the sequential cumsum is walked; exact_walks
 * (optional) counts those walks. scratch: one uint64. */
int fb_kmeans_draw(const double* best, const double* approx_prefix, int64_t n,
                   const double* total, double u, int64_t* out_idx, uint64_t* scratch,
                   int32_t* exact_walks, void* stream);

/* Device: out[i] = |x[i]|^2 (pairwise order) for float64 rows (ivf.py:70-72). */
int fb_row_sqnorm_f64(const double* x, int64_t n, int32_t dim, double* out, void* stream);

/* Device: Lloyd assignment (ivf.py:68-73, 119-120): d2 = max((data_sq - 2 x.c) + center_sq, 0)
 * in fp64, assign[i] = first argmin over the k centres, min_d2[i] its d2. */
int fb_kmeans_assign(const double* data, int64_t n, int32_t dim, const double* centers, int32_t k,
                     const double* data_sq, const double* center_sq, int64_t* assign,
                     double* min_d2, void* stream);

/* Device: centers[c] = mean of data rows order[seg_start[c] .. + seg_count[c]] (ascending row
 * index), summed sequentially per column then divided by the count, bit-identical to
 * data64[members].mean(axis=0) (ivf.py:131-133). */
int fb_kmeans_means(const double* data, int32_t dim, const int64_t* order,
                    const int64_t* seg_start, const int64_t* seg_count, int32_t k,
                    double* centers, void* stream);

/* ---------------------------------------------------------------------------------------
 * Host: batch filter compilation + packing (C++, no device work). The output arrays are
 * exactly the fb_filter_prog_t device form (upload them, then fill the struct from
 * fb_pack_meta / fb_pack_array) plus per-query push-bit counts (FilterStats.words_read).
 * Leaf positions are cached per (fid, value, M, K) across calls (bounded, thread-safe).
 * ------------------------------------------------------------------------------------- */
typedef struct fb_vocab fb_vocab_t;
typedef struct fb_pack fb_pack_t;

enum fb_pack_meta_id {
  FB_PACK_N_QUERIES = 0, FB_PACK_N_LEAVES = 1, FB_PACK_K_MAX = 2, FB_PACK_MAX_STACK = 3,
  FB_PACK_HAS_ROPS = 4, FB_PACK_N_PLANES = 5, FB_PACK_RMAX_STACK = 6, FB_PACK_N_ROPS = 7,
  FB_PACK_IS_CNF = 8, FB_PACK_N_COLS = 9, FB_PACK_CNF_WORDS = 10, FB_PACK_CNF_GMAX = 11,
  FB_PACK_CNF_WINDOWED = 12, FB_PACK_DISTINCT_LEAVES = 13, FB_PACK_DISTINCT_PLANES = 14,
  FB_PACK_META_N = 16
};
enum fb_pack_array_id {
  FB_PACK_LEAF_POS = 0,    /* i32 [n_leaves * k_max] */
  FB_PACK_OP_OFFSET = 1,   /* i32 [n_queries + 1] */
  FB_PACK_OPS = 2,         /* u16 */
  FB_PACK_PLANE_LIST = 3,  /* i32 [n_planes]            (has_rops) */
  FB_PACK_LEAF_SLOT = 4,   /* i16 [n_leaves * k_max]    (has_rops) */
  FB_PACK_ROP_OFFSET = 5,  /* i32 [n_queries + 1]       (has_rops) */
  FB_PACK_ROPS = 6,        /* u16 [n_rops]              (has_rops) */
  FB_PACK_COL_LEAF = 7,    /* i16 [n_cols]              (is_cnf) */
  FB_PACK_QMASK = 8,       /* u32 [n_queries][gmax][words] (is_cnf) */
  FB_PACK_QGROUPS = 9,     /* i32 [n_queries]           (is_cnf) */
  FB_PACK_PUSH_BITS = 10,  /* i64 [n_queries] sum of |positions| over the query's pushes */
  FB_PACK_LEAF_FID = 11,   /* u64 [distinct leaves] */
  FB_PACK_LEAF_VAL = 12    /* u64 [distinct leaves] */
};

/* Host: name dictionaries of filter_query.Vocabulary (feature name -> id, value -> id). */
int fb_vocab_create(int32_t n_feat, const char* const* feat_names, const uint64_t* feat_ids,
                    int32_t n_vals, const char* const* val_names, const uint64_t* val_ids,
                    fb_vocab_t** out);
void fb_vocab_free(fb_vocab_t* vocab);

/* Host: parse + compile + pack one filter text per query (NULL or "" = unfiltered), the
 * grammar of filter_query.parse_filter (filter_query.py:82-189). FB_ERR_PARSE sets
 * *bad_query. */
int fb_pack_text(int32_t n_queries, const char* const* texts, const fb_vocab_t* vocab,
                 int32_t m_bits, int32_t k_hashes, fb_pack_t** out, int32_t* bad_query);

/* Host: the same from postfix programs (CompiledFilter.ops with the leaves inlined): query
 * q's ops are [op_offset[q], op_offset[q+1]) (empty = unfiltered); a PUSH_LEAF op i carries
 * its leaf's (fid, value) and, when pos_offset is not NULL, the leaf's positions
 * pos[pos_offset[i] .. pos_offset[i+1]) (QueryBloom.set_bits; otherwise they are hashed).
 * Leaves are de-duplicated by (fid, value), first push wins. */
int fb_pack_postfix(int32_t n_queries, const int64_t* op_offset, const uint8_t* opcode,
                    const uint64_t* fid, const uint64_t* value, const int64_t* pos_offset,
                    const int32_t* pos, int32_t m_bits, int32_t k_hashes, fb_pack_t** out);

int fb_pack_meta(const fb_pack_t* pack, int64_t* meta /* [FB_PACK_META_N] */);
int fb_pack_array(const fb_pack_t* pack, int32_t which, const void** data, int64_t* n_elems);
void fb_pack_free(fb_pack_t* pack);

#ifdef __cplusplus
}
#endif
#endif /* FILTRA_B200_H */
