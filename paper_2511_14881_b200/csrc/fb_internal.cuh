// Internal declarations shared by the filtra_b200 translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "filtra_b200.h"

namespace fb {

// ------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define FB_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return ::fb::cuda_fail(e_, #call); \
  } while (0)

void count_launch();
// FB_DEBUG_LAUNCH=1: print every launch's name and synchronise after it (hang triage)
void debug_launch(const char* what);

#define FB_LAUNCH_CHECK(what)                           \
  do {                                                  \
    ::fb::count_launch();                               \
    ::fb::debug_launch(what);                           \
    cudaError_t e_ = cudaGetLastError();                \
    if (e_ != cudaSuccess) return ::fb::cuda_fail(e_, what); \
  } while (0)

// ------------------------------------------------------------------------------------
// hashing: FNV-1a-64 over fid||value (little endian) + K SplitMix64 mixes
// (reference bloom.py:48-88)
// ------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t fnv1a_pair(uint64_t fid, uint64_t value) {
  uint64_t h = 0xCBF29CE484222325ull;
#pragma unroll
  for (int i = 0; i < 8; ++i) { h ^= (fid >> (8 * i)) & 0xFF; h *= 0x100000001B3ull; }
#pragma unroll
  for (int i = 0; i < 8; ++i) { h ^= (value >> (8 * i)) & 0xFF; h *= 0x100000001B3ull; }
  return h;
}

// Sorted distinct positions; returns the count (<= k). k <= FB_MAX_K_HASHES.
__host__ __device__ __forceinline__ int leaf_positions(uint64_t fid, uint64_t value, int m_bits,
                                                       int k, int32_t* out) {
  const uint64_t seed = fnv1a_pair(fid, value);
  int n = 0;
  for (int i = 0; i < k; ++i) {
    const int32_t p = (int32_t)(splitmix64(seed ^ ((uint64_t)i * 0x9E3779B97F4A7C15ull)) %
                                (uint64_t)m_bits);
    // insertion into the sorted prefix, skipping duplicates
    int j = n;
    bool dup = false;
    for (int t = 0; t < n; ++t) dup |= (out[t] == p);
    if (dup) continue;
    while (j > 0 && out[j - 1] > p) { out[j] = out[j - 1]; --j; }
    out[j] = p;
    ++n;
  }
  return n;
}

// ------------------------------------------------------------------------------------
// merge key: ((score ^ 2^31) << 32) | (0xFFFFFFFF - id_rank). Larger key = better
// under (score desc, item_id asc). Key 0 never occurs for a real item.
// ------------------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t make_key(int32_t score, uint32_t id_rank) {
  return ((uint64_t)((uint32_t)score ^ 0x80000000u) << 32) | (uint64_t)(0xFFFFFFFFu - id_rank);
}
__host__ __device__ __forceinline__ int32_t key_score(uint64_t key) {
  return (int32_t)((uint32_t)(key >> 32) ^ 0x80000000u);
}

// ------------------------------------------------------------------------------------
// scan modes + shared argument block
// ------------------------------------------------------------------------------------
enum ScanMode { SCAN_EMIT = 0, SCAN_HIST = 1 };

// per-query fallback state (exact threshold by radix-narrowing over the 64-bit key)
enum QueryState : uint32_t { Q_OK = 0, Q_FLAGGED = 1, Q_RESOLVED = 2 };

struct Fallback {
  uint64_t lo;       // current key window [lo, lo + 2^(shift+12))
  uint32_t shift;    // bin width = 2^shift, 4096 bins
  uint32_t state;    // QueryState
  uint64_t above;    // keys counted above the window
  uint64_t need;     // target rank within the window
};
constexpr int kHistBins = 4096;

struct ScanArgs {
  fb_index_t idx;
  const int8_t* queries;  // [B, dim_pad]
  int32_t n_queries;
  fb_filter_prog_t prog;  // n_queries==0 / ops==nullptr: unfiltered
  int32_t has_prog;
  const uint64_t* masks;  // [B, idx.n_words] explicit per-query masks (nullable)
  // work: slot ranges (device) + prefix of word counts
  const int64_t* ranges;       // [n_ranges, 2]
  const int64_t* word_prefix;  // [n_ranges + 1]
  int32_t n_ranges;
  int64_t total_words;
  int64_t word_stride;  // visit every word_stride-th work word (sampling)
  int32_t mode;
  // emit
  const uint64_t* threshold;  // [B] key threshold (nullptr: 0)
  uint64_t* out_key;          // [B, cap]
  uint32_t* out_slot;         // [B, cap] (nullable)
  uint32_t* out_cnt;          // [B]
  uint32_t* out_elig;         // [B]
  int32_t cap;
  // fallback (hist mode and redo emits)
  const Fallback* fb;         // [B] (nullable)
  uint32_t* hist;             // [B, kHistBins]
  const uint32_t* active_count;  // early-exit when *active_count == 0 (nullable)
  uint32_t only_state;        // process only queries whose fb state == only_state (if fb != null)
  // tensor-core path: work list of (256-slot tile, range index) pairs; word_stride then
  // strides over this list
  const void* tc_work;        // int2 [n_tc_work]
  int64_t n_tc_work;
  int32_t dense;              // threshold 0 everywhere (sampling): word-level filter is cheaper
  int32_t* dump;              // testing: raw scores [B, dump_ld] (nullable)
  int64_t dump_ld;
  uint32_t* tc_qrec;          // [B, 12] scratch: CNF window records (fb_emit_kernel.cu)
  // eligible keys per query seen by the sampling pass and the slots it sampled: the emit
  // pass of a CNF window batch goes filter-first when the batch's sampled eligibility is low
  const uint32_t* sample_cnt; // [B] (nullable: no sampling pass)
  double sampled_slots;
};

// IVF-probed scan: per (query, probed cluster) pair, every eligible slot's key
constexpr int kIvfMaxDimPad = 1024;
struct IvfScanArgs {
  fb_index_t idx;
  const int8_t* queries;       // [B, dim_pad]
  int32_t n_queries;
  fb_filter_prog_t prog;
  int32_t has_prog;
  const int64_t* probe_words;  // [B, nprobe, 2] word range [w0, w1) of each probed cluster
  int32_t nprobe;
  uint64_t* out_key;           // [B, cap]
  uint32_t* out_slot;          // [B, cap] (nullable)
  uint32_t* out_cnt;           // [B] (zeroed by the caller)
  int32_t cap;
};
int launch_ivf_scan(const IvfScanArgs& a, cudaStream_t s);
int launch_value_model(const uint16_t* code, int n_code, const double* consts, const double* ts,
                       int B, int T, int64_t C, const int32_t* count, double* out,
                       int32_t* zero_flag, cudaStream_t s);
int launch_final_topk(const double* final_, int64_t ld, const int32_t* count, int n_requests,
                      int topk, int64_t* order, int32_t* out_count, cudaStream_t s);
int launch_union_merge(const uint64_t* keys, const int32_t* counts, int B, int T, int k,
                       int64_t n_words, uint64_t* bitmap, const uint64_t* id_of_rank,
                       uint64_t* merged, int64_t* merged_ranks, int32_t* mcount, cudaStream_t s);

// kernels / launchers implemented in fb_kernels.cu
int launch_scan_simt(const ScanArgs& a, cudaStream_t s);
int launch_bloom_build(const uint64_t* fid, const uint64_t* value, const int64_t* slot,
                       int64_t n_pairs, int64_t n_words, int m_bits, int k, uint64_t* planes,
                       cudaStream_t s);
int launch_filter_eval(const fb_index_t& idx, const fb_filter_prog_t& prog, int64_t w0, int64_t w1,
                       int apply_valid, uint64_t* out, cudaStream_t s);
int launch_quantize_f64(const double* x, int64_t rows, int cols, double gmin, double gmax,
                        int8_t* out, int out_stride, cudaStream_t s);
int launch_quantize(const float* x, int64_t rows, int cols, double gmin, double gmax, int8_t* out,
                    int out_stride, cudaStream_t s);
int launch_dot_rows_i8(const int8_t* rows, int64_t n, int dim, int stride, const int8_t* vec,
                       int32_t* out, cudaStream_t s);
int launch_task_dots_f64(const float* cache, int64_t n_rows, int dim, const int64_t* rows,
                         const int32_t* count, int64_t n_cand, const float* users, int n_req,
                         int n_tasks, double* out, cudaStream_t s);
int launch_dot_rows_f64(const float* rows, int64_t n, int dim, const float* vec, double* out,
                        cudaStream_t s);
int launch_row_sums(const int8_t* x, int64_t rows, int cols, int stride, int32_t* out,
                    cudaStream_t s);

// tcgen05 (sm_100a) emit scan; returns FB_ERR_UNSUPPORTED when the shape is outside
// its envelope (the caller then uses the SIMT kernel)
int launch_scan_tc(const ScanArgs& a, cudaStream_t s);
bool scan_tc_supported(const ScanArgs& a);
// the window-form CNF emit kernel (fb_emit_kernel.cu), dispatched by launch_scan_tc
bool emit_win_supported(const ScanArgs& a);
int launch_emit_win(const ScanArgs& a, const CUtensorMap& tmap, int grid, cudaStream_t s);

struct SelectArgs {
  int32_t n_queries;
  int32_t k;
  int32_t cap;
  const uint64_t* cand_key;   // [B, cap] (sorted in place chunk-wise)
  uint32_t* cand_slot;        // [B, cap]
  const uint32_t* cnt;        // [B]
  const fb_index_t* idx_dev_unused;
  const uint64_t* item_ids;   // [n_slots]
  const int32_t* row_sum;     // [n_slots] nullable
  const int8_t* queries;      // [B, dim_pad] (query sums for fscores)
  int32_t dim;
  int32_t dim_pad;
  double gmin, gmax;
  uint64_t* out_ids;
  int32_t* out_scores;
  int32_t* out_count;
  uint64_t* out_keys;         // nullable
  double* out_fscores;        // nullable
  uint64_t* scratch_key;      // [B, cap]
  uint32_t* scratch_slot;     // [B, cap]
  const uint32_t* slot_of_rank;  // [n_slots] nullable (fb_index_t.slot_of_rank)
  const uint64_t* id_of_rank;    // [n_slots] nullable (fb_index_t.id_of_rank)
  int32_t id_dense;              // fb_index_t.id_dense: id = dense_id_base + rank, no gather
  uint64_t dense_id_base;        // fb_index_t.id_base
  int64_t n_slots;               // ranks are a permutation of [0, n_slots)
};
int launch_select(const SelectArgs& a, cudaStream_t s);
// true when the key-only radix selection applies (candidates then need no slot column)
bool select_by_rank(int32_t cap, int32_t k, const uint32_t* slot_of_rank);

struct ThresholdArgs {
  int32_t n_queries;
  int32_t k;
  int32_t sample_cap;
  int32_t cap;                 // emit-pass candidate capacity per query
  const uint64_t* sample_key;  // [B, sample_cap]
  const uint32_t* sample_cnt;  // [B] eligible keys seen (may exceed cap)
  double sample_fraction;      // sampled slots / scanned slots (0 -> no sample: T = 0)
  uint64_t* threshold;         // [B] out
  uint32_t* cnt;               // [B] zeroed
  uint32_t* elig;              // [B] zeroed
};
int launch_threshold(const ThresholdArgs& a, cudaStream_t s);

struct FallbackArgs {
  ScanArgs hist;   // SCAN_HIST over the flagged queries
  ScanArgs emit;   // SCAN_EMIT of the resolved queries
  int32_t n_queries, k, cap;
  Fallback* fb;
  uint32_t* hist_buf;
  uint64_t* threshold;
  uint32_t* cnt;
  uint32_t* elig;
  uint32_t* active;  // [0] flagged & unresolved, [1] resolved
};
int launch_fallback(const FallbackArgs& f, cudaStream_t s);
// keys the exact radix selection stages / sorts in shared memory per query (larger
// candidate sets are selected from L2; k up to this many)
constexpr int32_t kSelectMaxCand = 24576;

int launch_check(int32_t n_queries, int32_t k, int32_t cap, const uint32_t* cnt,
                 const uint64_t* thr, int force, Fallback* fb, uint32_t* active_count,
                 uint32_t* total_flagged, cudaStream_t s);
int launch_resolve(int32_t n_queries, int32_t k, int32_t cap, Fallback* fb, uint32_t* hist,
                   uint64_t* threshold, uint32_t* cnt, uint32_t* elig, uint32_t* active_count,
                   int final_pass, cudaStream_t s);
int launch_zero_hist(int32_t n_queries, const Fallback* fb, uint32_t* hist,
                     const uint32_t* active_count, cudaStream_t s);

int launch_merge(const int32_t* in_scores, const uint64_t* in_ids, const double* in_fscores,
                 const int32_t* in_count, int n_lists, int n_queries, int k_in, int k_out,
                 uint64_t* out_ids, int32_t* out_scores, int32_t* out_count, double* out_fscores,
                 cudaStream_t s);
int launch_dequant(const int32_t* scores, const int32_t* item_row_sum, const int32_t* query_sum,
                   int n_queries, int k, const int32_t* count, int dim, double gmin, double gmax,
                   double* out, cudaStream_t s);

// fp64 dequantised dot: closed form of sum_j deq(a_j) deq(b_j), deq(c) = (c+128)/s + m
__host__ __device__ __forceinline__ double dequant_dot(int32_t dot, int32_t sa, int32_t sb, int dim,
                                                       double gmin, double gmax) {
  const double s = 255.0 / (gmax - gmin);
  const long long p = (long long)dot + 128LL * ((long long)sa + (long long)sb) + 16384LL * dim;
  const long long q = (long long)sa + (long long)sb + 256LL * dim;
  return (double)p / (s * s) + (gmin / s) * (double)q + (double)dim * gmin * gmin;
}

}  // namespace fb
