// extern "C" boundary of filtra_b200 (declared in include/filtra_b200.h).
//
// Validation happens here, before any launch, so error codes map 1:1 onto the
// reference's exceptions (ValueError / DimMismatch / LengthMismatch ...).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "fb_internal.cuh"

namespace fb {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void debug_launch(const char* what) {
  static const int on = [] {
    const char* e = getenv("FB_DEBUG_LAUNCH");
    return e != nullptr && atoi(e) != 0;
  }();
  if (!on) return;
  fprintf(stderr, "[fb] launch %s\n", what);
  fflush(stderr);
  cudaError_t e = cudaDeviceSynchronize();
  fprintf(stderr, "[fb]   done %s: %s\n", what, cudaGetErrorString(e));
  fflush(stderr);
}

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return FB_ERR_CUDA;
}

}  // namespace fb

using namespace fb;

struct fb_topk_plan {
  fb_index_t idx;
  int32_t B = 0;
  int32_t k = 0;
  int32_t cap = 0;
  int32_t sample_cap = 16384;
  int32_t flags = 0;
  int32_t n_ranges = 0;
  int64_t total_words = 0;
  int64_t total_slots = 0;
  int64_t max_range = 0;
  int64_t sample_stride = 0;  // 0: no sampling pass
  double sample_fraction = 0.0;
  std::vector<int64_t> h_ranges;
  // device scratch (one allocation)
  void* dev = nullptr;
  int64_t* d_ranges = nullptr;
  int64_t* d_word_prefix = nullptr;
  uint64_t* d_cand_key = nullptr;
  uint32_t* d_cand_slot = nullptr;
  uint32_t* d_cnt = nullptr;
  uint32_t* d_elig = nullptr;
  uint64_t* d_threshold = nullptr;
  uint64_t* d_sample_key = nullptr;
  uint32_t* d_sample_cnt = nullptr;
  uint32_t* d_sample_elig = nullptr;
  Fallback* d_fb = nullptr;
  uint32_t* d_hist = nullptr;
  uint32_t* d_active = nullptr;  // [0] flagged & unresolved, [1] resolved, [2] total flagged
  uint32_t* d_qrec = nullptr;    // [B, 12] CNF window records (emit kernel scratch)
  int32_t* d_tc_work = nullptr;  // (tile, range) pairs for the tensor-core scan
  int64_t n_tc_work = 0;
  int64_t tc_sample_stride = 0;
  double tc_sample_fraction = 0.0;
  int32_t last_scan_tc = 0;      // 1 when the last execute's emit pass ran on tcgen05
  // optional per-stage timing (CUDA events on the execute stream)
  bool timing = false;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

__global__ void k_probe() {}

int validate_index(const fb_index_t* idx) {
  if (idx == nullptr) return fail(FB_ERR_INVALID, "index is NULL");
  if (idx->n_slots < 0 || idx->n_slots % 64 != 0)
    return fail(FB_ERR_INVALID, "n_slots must be a non-negative multiple of 64");
  if (idx->n_words != idx->n_slots / 64) return fail(FB_ERR_INVALID, "n_words != n_slots / 64");
  if (idx->dim < 1 || idx->dim_pad < idx->dim || idx->dim_pad % 32 != 0)
    return fail(FB_ERR_INVALID, "dim_pad must be >= dim and a multiple of 32");
  if (idx->dim_pad > 2048) return fail(FB_ERR_UNSUPPORTED, "dim_pad > 2048 is not supported");
  if (idx->m_bits < 1 || idx->k_hashes < 1 || idx->k_hashes > FB_MAX_K_HASHES)
    return fail(FB_ERR_INVALID, "bad Bloom parameters");
  return FB_OK;
}

int validate_prog(const fb_filter_prog_t* prog, int n_queries) {
  if (prog == nullptr) return FB_OK;
  if (prog->n_queries != n_queries)
    return fail(FB_ERR_LENGTH_MISMATCH, "filter program count != number of queries");
  if (prog->max_stack > FB_MAX_STACK)
    return fail(FB_ERR_UNSUPPORTED, "filter program stack depth exceeds FB_MAX_STACK");
  if (prog->n_leaves > FB_MAX_LEAVES)
    return fail(FB_ERR_UNSUPPORTED, "more than FB_MAX_LEAVES distinct leaves in one batch");
  return FB_OK;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" {

int fb_abi_version(void) { return FB_ABI_VERSION; }

const char* fb_last_error(void) { return g_last_error.c_str(); }

int fb_device_ok(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_error(std::string("cudaGetDevice: ") + cudaGetErrorString(e));
    return 0;
  }
  cudaDeviceProp p;
  e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) {
    set_error(std::string("cudaGetDeviceProperties: ") + cudaGetErrorString(e));
    return 0;
  }
  if (p.major != 10 || p.minor != 0) {
    set_error("device is sm_" + std::to_string(p.major) + std::to_string(p.minor) +
              "; this build targets sm_100a only");
    return 0;
  }
  cudaFuncAttributes fa;
  e = cudaFuncGetAttributes(&fa, (const void*)k_probe);
  if (e != cudaSuccess) {
    set_error(std::string("sm_100a kernels do not load: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return 0;
  }
  return 1;
}

int fb_hash_leaves(const uint64_t* fid, const uint64_t* value, int64_t n, int32_t m_bits,
                   int32_t k_hashes, int32_t* pos_out, int32_t* n_pos_out) {
  if (m_bits < 1 || k_hashes < 1) return fail(FB_ERR_INVALID, "m_bits and k_hashes must be >= 1");
  if (k_hashes > FB_MAX_K_HASHES) return fail(FB_ERR_UNSUPPORTED, "k_hashes > FB_MAX_K_HASHES");
  for (int64_t i = 0; i < n; ++i) {
    int32_t* row = pos_out + i * k_hashes;
    const int np = leaf_positions(fid[i], value[i], m_bits, k_hashes, row);
    for (int j = np; j < k_hashes; ++j) row[j] = -1;
    if (n_pos_out) n_pos_out[i] = np;
  }
  return FB_OK;
}

int fb_bloom_build(const uint64_t* fid, const uint64_t* value, const int64_t* slot,
                   int64_t n_pairs, int64_t n_slots, int32_t m_bits, int32_t k_hashes,
                   uint64_t* planes, void* stream) {
  if (m_bits < 1 || k_hashes < 1) return fail(FB_ERR_INVALID, "m_bits and k_hashes must be >= 1");
  if (k_hashes > FB_MAX_K_HASHES) return fail(FB_ERR_UNSUPPORTED, "k_hashes > FB_MAX_K_HASHES");
  if (n_slots < 0 || n_pairs < 0) return fail(FB_ERR_INVALID, "negative size");
  const int64_t n_words = (n_slots + 63) / 64;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_words > 0)
    FB_CUDA(cudaMemsetAsync(planes, 0, (size_t)m_bits * n_words * sizeof(uint64_t), s));
  return launch_bloom_build(fid, value, slot, n_pairs, n_words, m_bits, k_hashes, planes, s);
}

int fb_filter_eval(const fb_index_t* idx, const fb_filter_prog_t* prog, int64_t w0, int64_t w1,
                   int32_t apply_valid, uint64_t* masks_out, void* stream) {
  int rc = validate_index(idx);
  if (rc) return rc;
  if (prog == nullptr) return fail(FB_ERR_INVALID, "filter program is NULL");
  rc = validate_prog(prog, prog->n_queries);
  if (rc) return rc;
  if (w0 < 0 || w1 < w0 || w1 > idx->n_words) return fail(FB_ERR_INVALID, "word range out of bounds");
  return launch_filter_eval(*idx, *prog, w0, w1, apply_valid, masks_out,
                            static_cast<cudaStream_t>(stream));
}

int fb_quantize(const float* x, int64_t rows, int32_t cols, double gmin, double gmax, int8_t* out,
                int32_t out_stride, void* stream) {
  if (!(gmax > gmin) || !std::isfinite(255.0 / (gmax - gmin)))
    return fail(FB_ERR_DEGENERATE, "degenerate quantisation range");
  if (cols < 0 || out_stride < cols) return fail(FB_ERR_INVALID, "out_stride < cols");
  return launch_quantize(x, rows, cols, gmin, gmax, out, out_stride,
                         static_cast<cudaStream_t>(stream));
}

int fb_quantize_f64(const double* x, int64_t rows, int32_t cols, double gmin, double gmax,
                    int8_t* out, int32_t out_stride, void* stream) {
  if (!(gmax > gmin) || !std::isfinite(255.0 / (gmax - gmin)))
    return fail(FB_ERR_DEGENERATE, "degenerate quantisation range");
  if (cols < 0 || out_stride < cols) return fail(FB_ERR_INVALID, "out_stride < cols");
  return launch_quantize_f64(x, rows, cols, gmin, gmax, out, out_stride,
                             static_cast<cudaStream_t>(stream));
}

int fb_row_sums(const int8_t* x, int64_t rows, int32_t cols, int32_t stride, int32_t* out,
                void* stream) {
  if (stride < cols) return fail(FB_ERR_INVALID, "stride < cols");
  return launch_row_sums(x, rows, cols, stride, out, static_cast<cudaStream_t>(stream));
}

int fb_topk_plan_create(const fb_index_t* idx, int32_t n_queries, int32_t k, const int64_t* ranges,
                        int32_t n_ranges, int32_t flags, fb_topk_plan_t** plan_out) {
  if (plan_out == nullptr) return fail(FB_ERR_INVALID, "plan_out is NULL");
  *plan_out = nullptr;
  int rc = validate_index(idx);
  if (rc) return rc;
  if (n_queries < 0) return fail(FB_ERR_INVALID, "n_queries < 0");
  if (k < 0) return fail(FB_ERR_INVALID, "k < 0");
  if (n_ranges < 0 || (n_ranges > 0 && ranges == nullptr))
    return fail(FB_ERR_INVALID, "bad slot ranges");
  fb_topk_plan* p = new fb_topk_plan();
  p->idx = *idx;
  p->B = n_queries;
  p->k = k;
  p->flags = flags;
  std::vector<int64_t> prefix(1, 0);
  for (int i = 0; i < n_ranges; ++i) {
    const int64_t s0 = ranges[2 * i], s1 = ranges[2 * i + 1];
    if (s0 % 64 != 0) {
      delete p;
      return fail(FB_ERR_INVALID, "slot range start " + std::to_string(s0) + " not 64-aligned");
    }
    if (s0 < 0 || s1 < s0 || s1 > idx->n_slots) {
      delete p;
      return fail(FB_ERR_INVALID, "slot range out of bounds");
    }
    if (s1 == s0) continue;
    p->h_ranges.push_back(s0);
    p->h_ranges.push_back(s1);
    const int64_t words = (s1 + 63) / 64 - s0 / 64;
    prefix.push_back(prefix.back() + words);
    p->total_slots += s1 - s0;
    p->max_range = std::max(p->max_range, s1 - s0);
  }
  p->n_ranges = (int32_t)(p->h_ranges.size() / 2);
  p->total_words = prefix.back();
  // tensor-core work list: (256-slot tile, range) pairs covering every range
  std::vector<int32_t> tc_work;
  if (idx->n_slots % 256 == 0) {
    for (int r = 0; r < p->n_ranges; ++r) {
      const int64_t t0 = p->h_ranges[2 * r] / 256, t1 = (p->h_ranges[2 * r + 1] + 255) / 256;
      for (int64_t t = t0; t < t1; ++t) {
        tc_work.push_back((int32_t)t);
        tc_work.push_back(r);
      }
    }
  }
  p->n_tc_work = (int64_t)tc_work.size() / 2;
  // candidate buffer: room for the sampling threshold's spread; while the exact radix
  // selection applies (k <= 10240) up to its staging capacity
  // The sampled threshold lands ~jd / f above the k-th key (jd = mu + 5 sqrt(mu) + 8,
  // mu = k f, f ~ 1/128) with a spread of ~sqrt(jd) / f; room for 5.5 sigma of it.
  int64_t want = std::max<int64_t>(2LL * k + 2048, 8192);
  // sampled share of the tiles is 1 / sdiv (FB_SAMPLE_DIV: A/B experiments only)
  const char* sdiv_env = getenv("FB_SAMPLE_DIV");
  const double sdiv = sdiv_env ? std::max(1.0, atof(sdiv_env)) : 128.0;
  {
    const double mu = (double)k / sdiv;
    const double jd = mu + 5.0 * std::sqrt(mu) + 8.0;
    const int64_t noise = (int64_t)std::ceil(sdiv * (jd + 5.5 * std::sqrt(jd)));
    // k <= 10240: stay within the selection's shared-memory staging when that is close
    want = std::max<int64_t>(want, k <= 10240 ? std::min<int64_t>(kSelectMaxCand, noise) : noise);
  }
  p->cap = (int32_t)std::max<int64_t>(1, std::min<int64_t>(p->total_slots, want));
  // sampling pass only when the candidate buffer cannot simply hold everything
  if (!(flags & FB_PLAN_NO_SAMPLE) && p->total_slots > p->cap && k > 0) {
    const int64_t target_words = std::max<int64_t>(std::min<int64_t>(p->total_words, 4096),
                                                   p->total_words / 32);
    p->sample_stride = std::max<int64_t>(1, p->total_words / target_words);
    const int64_t sampled = (p->total_words + p->sample_stride - 1) / p->sample_stride;
    p->sample_fraction = (double)sampled / (double)p->total_words;
    if (p->n_tc_work > 0) {
      // the sample pass runs at threshold 0 (every score is a hit): keep it to ~1/128 of
      // the tiles (>= 256 tiles, ~65k slots) -- enough for the rank estimate
      // (rounded to whole waves of one tile per SM so no CTA runs a tile more than others)
      const int64_t target_tiles = std::max<int64_t>(std::min<int64_t>(p->n_tc_work, 256),
                                                     (int64_t)((double)p->n_tc_work / sdiv));
      int n_sm = 148;
      cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
      const int64_t waves = std::max<int64_t>(1, (target_tiles + n_sm / 2) / n_sm);
      p->tc_sample_stride =
          std::max<int64_t>(1, (p->n_tc_work + waves * n_sm - 1) / (waves * n_sm));
      const int64_t st = (p->n_tc_work + p->tc_sample_stride - 1) / p->tc_sample_stride;
      p->tc_sample_fraction = (double)st / (double)p->n_tc_work;
    }
    // keep every eligible sampled key up to the whole sample (an unfiltered query keeps
    // ~N/128): the threshold's rank estimate stays precise at any selectivity
    const double f = p->n_tc_work > 0 ? p->tc_sample_fraction : p->sample_fraction;
    const int64_t want_s = (int64_t)((double)p->total_slots * f * 1.05) + 1024;
    p->sample_cap = (int32_t)std::min<int64_t>(std::max<int64_t>(16384, want_s), 1 << 18);
  }
  const int64_t B = std::max(1, n_queries);
  const int64_t nr = std::max(1, p->n_ranges);
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = align_up(off, 256);
    off = o + std::max<size_t>(bytes, 1);
    return o;
  };
  const size_t o_ranges = carve(sizeof(int64_t) * 2 * nr);
  const size_t o_prefix = carve(sizeof(int64_t) * (nr + 1));
  const size_t o_ckey = carve(sizeof(uint64_t) * B * p->cap);
  const size_t o_cslot = carve(sizeof(uint32_t) * B * p->cap);
  const size_t o_cnt = carve(sizeof(uint32_t) * B);
  const size_t o_elig = carve(sizeof(uint32_t) * B);
  const size_t o_thr = carve(sizeof(uint64_t) * B);
  const size_t o_skey = carve(p->sample_stride ? sizeof(uint64_t) * B * p->sample_cap : 0);
  const size_t o_scnt = carve(sizeof(uint32_t) * B);
  const size_t o_selig = carve(sizeof(uint32_t) * B);
  const size_t o_fb = carve(sizeof(Fallback) * B);
  const size_t o_hist = carve(sizeof(uint32_t) * B * kHistBins);
  const size_t o_active = carve(sizeof(uint32_t) * 4);
  const size_t o_tc = carve(sizeof(int32_t) * std::max<size_t>(2, tc_work.size()));
  const size_t o_qrec = carve(sizeof(uint32_t) * 12 * B);
  cudaError_t e = cudaMalloc(&p->dev, off);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "cudaMalloc(plan scratch)");
  }
  uint8_t* base = static_cast<uint8_t*>(p->dev);
  p->d_ranges = reinterpret_cast<int64_t*>(base + o_ranges);
  p->d_word_prefix = reinterpret_cast<int64_t*>(base + o_prefix);
  p->d_cand_key = reinterpret_cast<uint64_t*>(base + o_ckey);
  p->d_cand_slot = reinterpret_cast<uint32_t*>(base + o_cslot);
  p->d_cnt = reinterpret_cast<uint32_t*>(base + o_cnt);
  p->d_elig = reinterpret_cast<uint32_t*>(base + o_elig);
  p->d_threshold = reinterpret_cast<uint64_t*>(base + o_thr);
  p->d_sample_key = reinterpret_cast<uint64_t*>(base + o_skey);
  p->d_sample_cnt = reinterpret_cast<uint32_t*>(base + o_scnt);
  p->d_sample_elig = reinterpret_cast<uint32_t*>(base + o_selig);
  p->d_fb = reinterpret_cast<Fallback*>(base + o_fb);
  p->d_hist = reinterpret_cast<uint32_t*>(base + o_hist);
  p->d_active = reinterpret_cast<uint32_t*>(base + o_active);
  p->d_tc_work = reinterpret_cast<int32_t*>(base + o_tc);
  p->d_qrec = reinterpret_cast<uint32_t*>(base + o_qrec);
  if (p->n_ranges > 0) {
    e = cudaMemcpy(p->d_ranges, p->h_ranges.data(), sizeof(int64_t) * p->h_ranges.size(),
                   cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
      e = cudaMemcpy(p->d_word_prefix, prefix.data(), sizeof(int64_t) * prefix.size(),
                     cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !tc_work.empty())
      e = cudaMemcpy(p->d_tc_work, tc_work.data(), sizeof(int32_t) * tc_work.size(),
                     cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(p->dev);
      delete p;
      return cuda_fail(e, "cudaMemcpy(plan ranges)");
    }
  }
  *plan_out = p;
  return FB_OK;
}

int fb_topk_plan_destroy(fb_topk_plan_t* plan) {
  if (plan == nullptr) return FB_OK;
  for (auto& e : plan->ev)
    if (e) cudaEventDestroy(e);
  if (plan->dev) cudaFree(plan->dev);
  delete plan;
  return FB_OK;
}

int fb_topk_plan_stats(const fb_topk_plan_t* plan, fb_stats_t* st) {
  if (plan == nullptr || st == nullptr) return fail(FB_ERR_INVALID, "NULL argument");
  st->slots_scanned = plan->total_slots;
  st->tiles = 0;
  st->max_tile_rows = 0;
  for (int i = 0; i < plan->n_ranges; ++i) {
    const int64_t len = plan->h_ranges[2 * i + 1] - plan->h_ranges[2 * i];
    st->tiles += (len + 127) / 128;
    st->max_tile_rows = std::max<int64_t>(st->max_tile_rows, std::min<int64_t>(len, 128));
  }
  st->slots_evaluated = plan->total_words * 64;
  // queries the last execute sent through the exact fallback (synchronises the device)
  uint32_t flagged = 0;
  if (plan->d_active != nullptr &&
      cudaMemcpy(&flagged, plan->d_active + 2, sizeof(uint32_t), cudaMemcpyDeviceToHost) !=
          cudaSuccess)
    return fail(FB_ERR_CUDA, "reading the fallback counter failed");
  st->fallback_queries = flagged;
  return FB_OK;
}

int fb_topk_execute(fb_topk_plan_t* p, const int8_t* queries_q, const fb_filter_prog_t* prog,
                    const uint64_t* masks, uint64_t* out_ids, int32_t* out_scores, int32_t* out_count, uint64_t* out_keys,
                    double* out_fscores, double gmin, double gmax, void* stream) {
  if (p == nullptr) return fail(FB_ERR_INVALID, "plan is NULL");
  int rc = validate_prog(prog, p->B);
  if (rc) return rc;
  if (out_fscores && !(gmax > gmin)) return fail(FB_ERR_DEGENERATE, "fscores need gmax > gmin");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (p->B == 0) return FB_OK;
  const int k = p->k;
  if (k == 0 || p->n_ranges == 0) {
    FB_CUDA(cudaMemsetAsync(p->d_cnt, 0, sizeof(uint32_t) * p->B, s));
  }

  ScanArgs a{};
  a.idx = p->idx;
  a.queries = queries_q;
  a.n_queries = p->B;
  a.has_prog = prog != nullptr && prog->ops != nullptr ? 1 : 0;
  if (a.has_prog) a.prog = *prog;
  a.masks = masks;
  a.ranges = p->d_ranges;
  a.word_prefix = p->d_word_prefix;
  a.n_ranges = p->n_ranges;
  a.total_words = p->total_words;
  a.cap = p->cap;
  a.fb = nullptr;
  a.hist = p->d_hist;
  a.active_count = nullptr;
  a.tc_work = p->d_tc_work;
  a.n_tc_work = p->n_tc_work;
  a.tc_qrec = p->d_qrec;
  a.mode = SCAN_EMIT;
  const bool use_tc = !(p->flags & FB_PLAN_SIMT) && p->n_tc_work > 0 && scan_tc_supported(a);
  p->last_scan_tc = use_tc ? 1 : 0;

  auto emit = [&](ScanArgs& sa) -> int {
    if (use_tc) return launch_scan_tc(sa, s);
    return launch_scan_simt(sa, s);
  };

  if (k > 0 && p->n_ranges > 0) {
    FB_CUDA(cudaMemsetAsync(p->d_active, 0, sizeof(uint32_t) * 4, s));
    // 1) sampling pass: every sample_stride-th word, threshold 0, keep <= sample_cap keys
    ThresholdArgs t{};
    t.n_queries = p->B;
    t.k = k;
    t.sample_cap = p->sample_cap;
    t.cap = p->cap;
    t.sample_key = p->d_sample_key;
    t.sample_cnt = p->d_sample_cnt;
    t.sample_fraction = !p->sample_stride ? 0.0
                        : use_tc          ? p->tc_sample_fraction
                                          : p->sample_fraction;
    t.threshold = p->d_threshold;
    t.cnt = p->d_cnt;
    t.elig = p->d_elig;
    if (p->sample_stride) {
      FB_CUDA(cudaMemsetAsync(p->d_sample_cnt, 0, sizeof(uint32_t) * p->B, s));
      FB_CUDA(cudaMemsetAsync(p->d_sample_elig, 0, sizeof(uint32_t) * p->B, s));
      ScanArgs sa = a;
      sa.mode = SCAN_EMIT;
      sa.word_stride = use_tc ? p->tc_sample_stride : p->sample_stride;
      sa.threshold = nullptr;
      sa.out_key = p->d_sample_key;
      sa.out_slot = nullptr;
      sa.out_cnt = p->d_sample_cnt;
      sa.out_elig = p->d_sample_elig;
      sa.cap = p->sample_cap;
      sa.dense = 1;
      rc = emit(sa);
      if (rc) return rc;
    }
    // 2) per-query threshold (also zeroes the emit counters)
    rc = launch_threshold(t, s);
    if (rc) return rc;
    if (p->timing) FB_CUDA(cudaEventRecord(p->ev[0], s));
    // 3) emit pass
    ScanArgs ea = a;
    ea.mode = SCAN_EMIT;
    ea.word_stride = 1;
    ea.threshold = p->d_threshold;
    ea.out_key = p->d_cand_key;
    ea.out_slot = select_by_rank(p->cap, k, p->idx.slot_of_rank) ? nullptr : p->d_cand_slot;
    ea.out_cnt = p->d_cnt;
    ea.out_elig = p->d_elig;
    if (p->sample_stride && use_tc) {
      ea.sample_cnt = p->d_sample_cnt;
      ea.sampled_slots = p->tc_sample_fraction * (double)p->total_slots;
    }
    rc = emit(ea);
    if (rc) return rc;
    if (p->timing) FB_CUDA(cudaEventRecord(p->ev[1], s));
    // 4) exactness check; 5) fallback, one cooperative launch that only reads a flag
    //    unless some query was flagged: radix-narrow the key window (<= 6 grid-synchronised
    //    histogram passes), then re-emit the resolved queries
    rc = launch_check(p->B, k, p->cap, p->d_cnt, p->d_threshold,
                      (p->flags & FB_PLAN_FORCE_FALLBACK) ? 1 : 0, p->d_fb, p->d_active,
                      p->d_active + 2, s);
    if (rc) return rc;
    FallbackArgs fa{};
    fa.hist = a;
    fa.hist.mode = SCAN_HIST;
    fa.hist.word_stride = 1;
    fa.hist.fb = p->d_fb;
    fa.hist.only_state = Q_FLAGGED;
    fa.hist.active_count = nullptr;
    fa.emit = ea;
    fa.emit.fb = p->d_fb;
    fa.emit.only_state = Q_RESOLVED;
    fa.emit.active_count = nullptr;
    fa.n_queries = p->B;
    fa.k = k;
    fa.cap = p->cap;
    fa.fb = p->d_fb;
    fa.hist_buf = p->d_hist;
    fa.threshold = p->d_threshold;
    fa.cnt = p->d_cnt;
    fa.elig = p->d_elig;
    fa.active = p->d_active;
    rc = launch_fallback(fa, s);
    if (rc) return rc;
  }
  // 6) exact selection + outputs
  SelectArgs sel{};
  sel.n_queries = p->B;
  sel.k = k;
  sel.cap = p->cap;
  sel.cand_key = p->d_cand_key;
  sel.cand_slot = p->d_cand_slot;
  sel.slot_of_rank = p->idx.slot_of_rank;
  sel.id_of_rank = p->idx.id_of_rank;
  sel.id_dense = p->idx.id_dense;
  sel.dense_id_base = p->idx.id_base;
  sel.n_slots = p->idx.n_slots;
  sel.cnt = p->d_cnt;
  sel.item_ids = p->idx.item_ids;
  sel.row_sum = p->idx.row_sum;
  sel.queries = queries_q;
  sel.dim = p->idx.dim;
  sel.dim_pad = p->idx.dim_pad;
  sel.gmin = gmin;
  sel.gmax = gmax;
  sel.out_ids = out_ids;
  sel.out_scores = out_scores;
  sel.out_count = out_count;
  sel.out_keys = out_keys;
  sel.out_fscores = out_fscores;
  if (k == 0) {
    FB_CUDA(cudaMemsetAsync(out_count, 0, sizeof(int32_t) * p->B, s));
    return FB_OK;
  }
  if (p->timing) FB_CUDA(cudaEventRecord(p->ev[2], s));
  rc = launch_select(sel, s);
  if (rc) return rc;
  if (p->timing) FB_CUDA(cudaEventRecord(p->ev[3], s));
  return FB_OK;
}

int fb_merge_union(const uint64_t* keys, const int32_t* counts, int32_t n_requests,
                   int32_t n_tasks, int32_t k, int64_t n_slots, const uint64_t* id_of_rank,
                   uint64_t* bitmap, uint64_t* merged, int64_t* merged_ranks, int32_t* mcount,
                   void* stream) {
  if (n_requests < 0 || n_tasks < 0 || k < 0 || n_slots < 0) return fail(FB_ERR_INVALID, "negative size");
  if (id_of_rank == nullptr) return fail(FB_ERR_INVALID, "id_of_rank is required");
  if ((int64_t)n_tasks * k > 0x7fffffffLL) return fail(FB_ERR_INVALID, "merged width overflows");
  return launch_union_merge(keys, counts, n_requests, n_tasks, k, (n_slots + 63) / 64, bitmap,
                            id_of_rank, merged, merged_ranks, mcount,
                            static_cast<cudaStream_t>(stream));
}

int fb_value_model(const uint16_t* code, int32_t n_code, const double* consts,
                   const double* task_scores, int32_t n_requests, int32_t n_tasks, int64_t ld,
                   const int32_t* count, double* out, int32_t* zero_flag, void* stream) {
  if (n_code <= 0 || n_requests < 0 || n_tasks < 0 || ld < 0)
    return fail(FB_ERR_INVALID, "bad value-model size");
  return launch_value_model(code, n_code, consts, task_scores, n_requests, n_tasks, ld, count, out,
                            zero_flag, static_cast<cudaStream_t>(stream));
}

int fb_final_topk(const double* final_scores, int64_t ld, const int32_t* count,
                  int32_t n_requests, int32_t topk, int64_t* order, int32_t* out_count,
                  void* stream) {
  if (n_requests < 0 || topk < 0 || ld < 0) return fail(FB_ERR_INVALID, "negative size");
  if (n_requests > 0 && topk > 0 && (final_scores == nullptr || count == nullptr || order == nullptr ||
                                     out_count == nullptr))
    return fail(FB_ERR_INVALID, "null buffer");
  return launch_final_topk(final_scores, ld, count, n_requests, topk, order, out_count,
                           static_cast<cudaStream_t>(stream));
}

int fb_ivf_topk(const fb_index_t* idx, const int8_t* queries_q, int32_t n_queries,
                const fb_filter_prog_t* prog, const int64_t* probe_words, int32_t nprobe, int32_t k,
                int32_t cap, uint64_t* cand_key, uint32_t* cand_slot, uint32_t* cand_cnt,
                uint64_t* out_ids, int32_t* out_scores, int32_t* out_count, uint64_t* out_keys,
                double* out_fscores, double gmin, double gmax, void* stream) {
  int rc = validate_index(idx);
  if (rc) return rc;
  if (n_queries < 0 || nprobe < 0 || k < 0 || cap < 0) return fail(FB_ERR_INVALID, "negative size");
  if (prog != nullptr && prog->ops != nullptr) {
    rc = validate_prog(prog, n_queries);
    if (rc) return rc;
  }
  if (idx->dim_pad % 16 != 0 || idx->dim_pad > kIvfMaxDimPad)
    return fail(FB_ERR_UNSUPPORTED, "dim_pad must be a multiple of 16 and <= 1024");
  if (out_fscores && !(gmax > gmin)) return fail(FB_ERR_DEGENERATE, "fscores need gmax > gmin");
  const bool by_rank = select_by_rank(cap, k, idx->slot_of_rank);
  if (!by_rank && cand_slot == nullptr) return fail(FB_ERR_INVALID, "cand_slot needed for this k");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n_queries == 0) return FB_OK;
  FB_CUDA(cudaMemsetAsync(cand_cnt, 0, sizeof(uint32_t) * n_queries, s));
  if (k == 0) {
    FB_CUDA(cudaMemsetAsync(out_count, 0, sizeof(int32_t) * n_queries, s));
    return FB_OK;
  }
  IvfScanArgs a{};
  a.idx = *idx;
  a.queries = queries_q;
  a.n_queries = n_queries;
  a.has_prog = prog != nullptr && prog->ops != nullptr ? 1 : 0;
  if (a.has_prog) a.prog = *prog;
  a.probe_words = probe_words;
  a.nprobe = nprobe;
  a.out_key = cand_key;
  a.out_slot = by_rank ? nullptr : cand_slot;
  a.out_cnt = cand_cnt;
  a.cap = cap;
  rc = launch_ivf_scan(a, s);
  if (rc) return rc;
  SelectArgs sel{};
  sel.n_queries = n_queries;
  sel.k = k;
  sel.cap = cap;
  sel.cand_key = cand_key;
  sel.cand_slot = cand_slot;
  sel.slot_of_rank = idx->slot_of_rank;
  sel.id_of_rank = idx->id_of_rank;
  sel.id_dense = idx->id_dense;
  sel.dense_id_base = idx->id_base;
  sel.n_slots = idx->n_slots;
  sel.cnt = cand_cnt;
  sel.item_ids = idx->item_ids;
  sel.row_sum = idx->row_sum;
  sel.queries = queries_q;
  sel.dim = idx->dim;
  sel.dim_pad = idx->dim_pad;
  sel.gmin = gmin;
  sel.gmax = gmax;
  sel.out_ids = out_ids;
  sel.out_scores = out_scores;
  sel.out_count = out_count;
  sel.out_keys = out_keys;
  sel.out_fscores = out_fscores;
  return launch_select(sel, s);
}

uint64_t fb_launch_count(void) { return g_launches.load(); }

int fb_topk_scan_path(const fb_topk_plan_t* p) { return p == nullptr ? -1 : p->last_scan_tc; }

int fb_debug_tc_scores(const fb_index_t* idx, const int8_t* queries_q, int32_t n_queries,
                       int32_t* out, void* stream) {
  const int64_t full[2] = {0, idx ? idx->n_slots : 0};
  fb_topk_plan_t* p = nullptr;
  int rc = fb_topk_plan_create(idx, n_queries, 1, full, 1, FB_PLAN_NO_SAMPLE, &p);
  if (rc) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ScanArgs a{};
  a.idx = p->idx;
  a.queries = queries_q;
  a.n_queries = n_queries;
  a.ranges = p->d_ranges;
  a.word_prefix = p->d_word_prefix;
  a.n_ranges = p->n_ranges;
  a.total_words = p->total_words;
  a.mode = SCAN_EMIT;
  a.word_stride = 1;
  a.out_key = p->d_cand_key;
  a.out_slot = p->d_cand_slot;
  a.out_cnt = p->d_cnt;
  a.out_elig = p->d_elig;
  a.cap = p->cap;
  a.tc_work = p->d_tc_work;
  a.n_tc_work = p->n_tc_work;
  a.dump = out;
  a.dump_ld = idx->n_slots;
  rc = p->n_tc_work > 0 ? launch_scan_tc(a, s) : FB_ERR_UNSUPPORTED;
  if (rc == FB_ERR_UNSUPPORTED) fail(rc, "shape not supported by the tcgen05 scan");
  cudaError_t e = cudaStreamSynchronize(s);
  fb_topk_plan_destroy(p);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "fb_debug_tc_scores");
  return FB_OK;
}

int fb_topk_set_timing(fb_topk_plan_t* p, int32_t enable) {
  if (p == nullptr) return fail(FB_ERR_INVALID, "plan is NULL");
  if (enable && !p->ev[0])
    for (auto& e : p->ev) FB_CUDA(cudaEventCreate(&e));
  p->timing = enable != 0;
  return FB_OK;
}

int fb_topk_last_timing(fb_topk_plan_t* p, float* emit_ms, float* select_ms) {
  if (p == nullptr || !p->timing) return fail(FB_ERR_INVALID, "timing not enabled");
  FB_CUDA(cudaEventSynchronize(p->ev[3]));
  if (emit_ms) FB_CUDA(cudaEventElapsedTime(emit_ms, p->ev[0], p->ev[1]));
  if (select_ms) FB_CUDA(cudaEventElapsedTime(select_ms, p->ev[2], p->ev[3]));
  return FB_OK;
}

int fb_merge_topk(const int32_t* in_scores, const uint64_t* in_ids, const double* in_fscores,
                  const int32_t* in_count, int32_t n_lists, int32_t n_queries, int32_t k_in,
                  int32_t k_out, uint64_t* out_ids, int32_t* out_scores, int32_t* out_count,
                  double* out_fscores, void* stream) {
  if (n_lists < 1 || n_queries < 0 || k_in < 0 || k_out < 0)
    return fail(FB_ERR_INVALID, "bad merge shape");
  return launch_merge(in_scores, in_ids, in_fscores, in_count, n_lists, n_queries, k_in, k_out,
                      out_ids, out_scores, out_count, out_fscores,
                      static_cast<cudaStream_t>(stream));
}

int fb_int8_dot_rows(const int8_t* rows, int64_t n_rows, int32_t dim, int32_t stride,
                     const int8_t* vec, int32_t* out, void* stream) {
  if (stride < dim || dim < 0) return fail(FB_ERR_INVALID, "stride < dim");
  return launch_dot_rows_i8(rows, n_rows, dim, stride, vec, out, static_cast<cudaStream_t>(stream));
}

int fb_dot_rows_f64(const float* rows, int64_t n_rows, int32_t dim, const float* vec, double* out,
                    void* stream) {
  if (dim < 0) return fail(FB_ERR_INVALID, "dim < 0");
  return launch_dot_rows_f64(rows, n_rows, dim, vec, out, static_cast<cudaStream_t>(stream));
}

int fb_task_dots_f64(const float* cache, int64_t n_rows, int32_t dim, const int64_t* rows,
                     const int32_t* count, int64_t n_cand, const float* users, int32_t n_req,
                     int32_t n_tasks, double* out, void* stream) {
  if (dim < 0 || n_rows < 0 || n_cand < 0 || n_req < 0 || n_tasks < 0)
    return fail(FB_ERR_INVALID, "negative size");
  return launch_task_dots_f64(cache, n_rows, dim, rows, count, n_cand, users, n_req, n_tasks,
                              out, static_cast<cudaStream_t>(stream));
}

int fb_dequant_scores(const int32_t* scores, const int32_t* item_row_sum, const int32_t* query_sum,
                      int32_t n_queries, int32_t k, const int32_t* count, int32_t dim, double gmin,
                      double gmax, double* out, void* stream) {
  if (!(gmax > gmin)) return fail(FB_ERR_DEGENERATE, "degenerate quantisation range");
  return launch_dequant(scores, item_row_sum, query_sum, n_queries, k, count, dim, gmin, gmax, out,
                        static_cast<cudaStream_t>(stream));
}

}  // extern "C"
