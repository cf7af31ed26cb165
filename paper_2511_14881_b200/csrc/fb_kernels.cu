// SIMT kernels of filtra_b200: Bloom build, filter-program evaluation, quantisation,
// the SIMT masked scan (sample / emit / fallback-histogram modes), per-query
// threshold + exact selection, and the shard merge.
//
// Reference semantics (paths under /root/reference/pkg/src/filtra):
//   build_bloom           bloom.py:114-144
//   eval_compiled         filter_query.py:314-356 (NOT = ~x & valid, result & valid)
//   quantize_vector       quantize.py:72-76 (float64, rint half-to-even)
//   search_clusters       ivf.py:285-334  (eligible = valid & mask, exact int32 dot)
//   _select_topk          ivf.py:272-282  (score desc, item_id asc)
//   _reduce_topk          serve.py:98-100
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fb_internal.cuh"

namespace cg = cooperative_groups;

#include <algorithm>
#include <cstdio>

namespace fb {

namespace {

constexpr int kSelectChunk = 8192;   // keys per in-smem bitonic chunk (12 B each)
constexpr int kSelectThreads = 1024;

__device__ __forceinline__ int64_t grid_stride() { return (int64_t)gridDim.x * blockDim.x; }
__device__ __forceinline__ int64_t grid_tid() {
  return (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
}

// ------------------------------------------------------------------------------------
// Bloom build: one thread per (fid, value, slot) pair, 64-bit atomicOr into the plane word.
// ------------------------------------------------------------------------------------
__global__ void k_bloom_build(const uint64_t* __restrict__ fid, const uint64_t* __restrict__ val,
                              const int64_t* __restrict__ slot, int64_t n, int64_t n_words,
                              int m_bits, int k, unsigned long long* planes) {
  for (int64_t i = grid_tid(); i < n; i += grid_stride()) {
    int32_t pos[FB_MAX_K_HASHES];
    const int np = leaf_positions(fid[i], val[i], m_bits, k, pos);
    const int64_t s = slot[i];
    const unsigned long long bit = 1ull << (s & 63);
    for (int j = 0; j < np; ++j) atomicOr(planes + (int64_t)pos[j] * n_words + (s >> 6), bit);
  }
}

// ------------------------------------------------------------------------------------
// Filter program: postfix stack machine over one 64-slot word.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t leaf_word(const int32_t* __restrict__ pos, int k_max,
                                              const uint64_t* __restrict__ planes, int64_t n_words,
                                              int64_t w) {
  uint64_t m = ~0ull;
  for (int j = 0; j < k_max; ++j) {
    const int p = pos[j];
    if (p < 0) break;
    m &= __ldg(planes + (int64_t)p * n_words + w);
  }
  return m;
}

__device__ uint64_t eval_program_word(const fb_filter_prog_t& prog, int q,
                                      const uint64_t* __restrict__ planes, int64_t n_words,
                                      int64_t w, uint64_t valid_w) {
  const int32_t o0 = prog.op_offset[q], o1 = prog.op_offset[q + 1];
  if (o0 == o1) return valid_w;  // unfiltered query
  uint64_t stk[FB_MAX_STACK];
  int sp = 0;
  for (int o = o0; o < o1; ++o) {
    const uint32_t op = prog.ops[o];
    const uint32_t code = op >> 14, arg = op & 0x3FFF;
    if (code == FB_OP_PUSH_LEAF) {
      stk[sp++] = leaf_word(prog.leaf_pos + (int64_t)arg * prog.k_max, prog.k_max, planes,
                            n_words, w);
    } else if (code == FB_OP_NOT) {
      stk[sp - 1] = ~stk[sp - 1] & valid_w;
    } else {
      const uint64_t rhs = stk[--sp];
      stk[sp - 1] = (code == FB_OP_AND) ? (stk[sp - 1] & rhs) : (stk[sp - 1] | rhs);
    }
  }
  return stk[0];
}

// eval_program_word over leaf words already in shared memory (s_leaf[leaf]); stack of
// depth <= 4 in registers
__device__ uint64_t eval_program_leaves(const fb_filter_prog_t& prog, int q,
                                        const uint64_t* s_leaf, uint64_t v) {
  const int32_t o0 = prog.op_offset[q], o1 = prog.op_offset[q + 1];
  if (o0 == o1) return v;  // unfiltered query
  if (prog.max_stack <= 4) {
    uint64_t top = 0ull, s1 = 0ull, s2 = 0ull, s3 = 0ull;
    uint32_t n1 = prog.ops[o0], n2 = o0 + 1 < o1 ? prog.ops[o0 + 1] : 0u;
    for (int o = o0; o < o1; ++o) {
      const uint32_t op = n1;
      n1 = n2;
      n2 = o + 2 < o1 ? prog.ops[o + 2] : 0u;
      const uint32_t code = op >> 14;
      if (code == FB_OP_PUSH_LEAF) {
        s3 = s2;
        s2 = s1;
        s1 = top;
        top = s_leaf[op & 0x3FFF];
      } else if (code == FB_OP_NOT) {
        top = ~top & v;
      } else {
        top = (code == FB_OP_AND) ? (s1 & top) : (s1 | top);
        s1 = s2;
        s2 = s3;
      }
    }
    return top;
  }
  uint64_t stk[FB_MAX_STACK];
  int sp = 0;
  for (int o = o0; o < o1; ++o) {
    const uint32_t op = prog.ops[o];
    const uint32_t code = op >> 14;
    if (code == FB_OP_PUSH_LEAF) {
      stk[sp++] = s_leaf[op & 0x3FFF];
    } else if (code == FB_OP_NOT) {
      stk[sp - 1] = ~stk[sp - 1] & v;
    } else {
      const uint64_t rhs = stk[--sp];
      stk[sp - 1] = (code == FB_OP_AND) ? (stk[sp - 1] & rhs) : (stk[sp - 1] | rhs);
    }
  }
  return stk[0];
}

__global__ void k_filter_eval(fb_index_t idx, fb_filter_prog_t prog, int64_t w0, int64_t w1,
                              int apply_valid, uint64_t* __restrict__ out) {
  const int64_t width = w1 - w0;
  const int64_t total = width * prog.n_queries;
  for (int64_t i = grid_tid(); i < total; i += grid_stride()) {
    const int q = (int)(i / width);
    const int64_t w = w0 + (i - (int64_t)q * width);
    const uint64_t v = idx.valid[w];
    uint64_t m = eval_program_word(prog, q, idx.planes, idx.n_words, w, v);
    if (apply_valid) m &= v;
    out[i] = m;
  }
}

// Batched evaluation with the batch's leaves shared: a CTA takes kFeWords consecutive words;
// phase 1 evaluates every distinct leaf of the batch (leaves are de-duplicated across
// queries) once per word into shared memory, phase 2 runs each query's program over those
// leaf words (thread = (query, word), a warp = one query's 32 words: coalesced output,
// uniform program walk). Stack of depth <= 4 in registers.
constexpr int kFeWords = 64;   // words per CTA chunk
constexpr int kFeWpt = kFeWords / 32;  // words per thread (one op decode serves them all)

// program of query q over words j + 32 u (u < kFeWpt) of the chunk
__device__ __forceinline__ void eval_ops_leafwords(const fb_filter_prog_t& prog, int q,
                                                   const uint64_t* s_leaf, int j,
                                                   const uint64_t (&v)[kFeWpt],
                                                   uint64_t (&res)[kFeWpt]) {
  const int32_t o0 = prog.op_offset[q], o1 = prog.op_offset[q + 1];
  if (o0 == o1) {  // unfiltered query
#pragma unroll
    for (int u = 0; u < kFeWpt; ++u) res[u] = v[u];
    return;
  }
  if (prog.max_stack <= 4) {
    uint64_t top[kFeWpt], s1[kFeWpt], s2[kFeWpt], s3[kFeWpt];
#pragma unroll
    for (int u = 0; u < kFeWpt; ++u) top[u] = s1[u] = s2[u] = s3[u] = 0ull;
    // ops fetched two ahead of their use (the loads hide behind the current op's work)
    uint32_t n1 = prog.ops[o0], n2 = o0 + 1 < o1 ? prog.ops[o0 + 1] : 0u;
    for (int o = o0; o < o1; ++o) {
      const uint32_t op = n1;
      n1 = n2;
      n2 = o + 2 < o1 ? prog.ops[o + 2] : 0u;
      const uint32_t code = op >> 14;
      if (code == FB_OP_PUSH_LEAF) {
        const uint64_t* lw = s_leaf + (op & 0x3FFF) * kFeWords + j;
#pragma unroll
        for (int u = 0; u < kFeWpt; ++u) {
          s3[u] = s2[u];
          s2[u] = s1[u];
          s1[u] = top[u];
          top[u] = lw[32 * u];
        }
      } else if (code == FB_OP_NOT) {
#pragma unroll
        for (int u = 0; u < kFeWpt; ++u) top[u] = ~top[u] & v[u];
      } else {
        const bool is_and = code == FB_OP_AND;
#pragma unroll
        for (int u = 0; u < kFeWpt; ++u) {
          top[u] = is_and ? (s1[u] & top[u]) : (s1[u] | top[u]);
          s1[u] = s2[u];
          s2[u] = s3[u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kFeWpt; ++u) res[u] = top[u];
    return;
  }
#pragma unroll 1
  for (int u = 0; u < kFeWpt; ++u) {
    uint64_t stk[FB_MAX_STACK];
    int sp = 0;
    for (int o = o0; o < o1; ++o) {
      const uint32_t op = prog.ops[o];
      const uint32_t code = op >> 14;
      if (code == FB_OP_PUSH_LEAF) {
        stk[sp++] = s_leaf[(op & 0x3FFF) * kFeWords + j + 32 * u];
      } else if (code == FB_OP_NOT) {
        stk[sp - 1] = ~stk[sp - 1] & v[u];
      } else {
        const uint64_t rhs = stk[--sp];
        stk[sp - 1] = (code == FB_OP_AND) ? (stk[sp - 1] & rhs) : (stk[sp - 1] | rhs);
      }
    }
    res[u] = stk[0];
  }
}

// Batched evaluation with the batch's leaves shared: a CTA takes kFeWords consecutive words;
// phase 1 evaluates every distinct leaf of the batch (leaves are de-duplicated across
// queries) once per word into shared memory, phase 2 runs each query's program over those
// leaf words (a warp = one query; each lane kFeWpt words, so one op decode serves several
// words; coalesced output). Stack of depth <= 4 in registers.
__global__ void __launch_bounds__(256) k_filter_eval_shared(fb_index_t idx, fb_filter_prog_t prog,
                                                            int64_t w0, int64_t w1, int apply_valid,
                                                            uint64_t* __restrict__ out) {
  extern __shared__ uint64_t s_leaf[];  // [n_leaves][kFeWords]
  const int64_t width = w1 - w0;
  const int nl = prog.n_leaves;
  for (int64_t c0 = w0 + (int64_t)blockIdx.x * kFeWords; c0 < w1;
       c0 += (int64_t)gridDim.x * kFeWords) {
    const int nw = (int)min((int64_t)kFeWords, w1 - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < nl * kFeWords; e += blockDim.x) {
      const int leaf = e / kFeWords, jj = e - leaf * kFeWords;
      s_leaf[e] = jj < nw ? leaf_word(prog.leaf_pos + (int64_t)leaf * prog.k_max, prog.k_max,
                                      idx.planes, idx.n_words, c0 + jj)
                          : 0ull;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < prog.n_queries * 32; e += blockDim.x) {
      const int q = e >> 5, j = e & 31;
      uint64_t v[kFeWpt], m[kFeWpt];
#pragma unroll
      for (int u = 0; u < kFeWpt; ++u) v[u] = j + 32 * u < nw ? idx.valid[c0 + j + 32 * u] : 0ull;
      eval_ops_leafwords(prog, q, s_leaf, j, v, m);
#pragma unroll
      for (int u = 0; u < kFeWpt; ++u) {
        const int jj = j + 32 * u;
        if (jj < nw) out[(int64_t)q * width + (c0 + jj - w0)] = apply_valid ? (m[u] & v[u]) : m[u];
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// Quantisation: float64 (x - min) * scale, rint (half to even), -128, clip.
// ------------------------------------------------------------------------------------
template <typename T>
__global__ void k_quantize(const T* __restrict__ x, int64_t rows, int cols, double gmin,
                           double scale, int8_t* __restrict__ out, int out_stride) {
  const int64_t total = rows * out_stride;
  for (int64_t i = grid_tid(); i < total; i += grid_stride()) {
    const int64_t r = i / out_stride;
    const int c = (int)(i - r * out_stride);
    int8_t q = 0;
    if (c < cols) {
      const double v = (double)x[r * cols + c];
      double t = rint(__dmul_rn(__dsub_rn(v, gmin), scale)) - 128.0;
      t = fmin(127.0, fmax(-128.0, t));
      q = (int8_t)(int)t;
    }
    out[i] = q;
  }
}

__global__ void k_dot_rows_i8(const int8_t* __restrict__ x, int64_t rows, int dim, int stride,
                              const int8_t* __restrict__ v, int32_t* __restrict__ out) {
  for (int64_t r = grid_tid(); r < rows; r += grid_stride()) {
    int32_t s = 0;
    for (int c = 0; c < dim; ++c) s += (int32_t)x[r * stride + c] * (int32_t)v[c];
    out[r] = s;
  }
}

// numpy's pairwise summation (numpy/_core/src/umath/loops_utils.h.src, PW_BLOCKSIZE 128)
// over p[i] = (double)a[i] * (double)b[i]; 0.0 + pairwise(p) reproduces
// np.sum(rows * vec, axis=1) bit-for-bit (checked in tests/test_native_cpu.py's emulation).
__device__ double pairwise_f64(const float* __restrict__ a, const float* __restrict__ b, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, __dmul_rn((double)a[i], (double)b[i]));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dmul_rn((double)a[j], (double)b[j]);
    int i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        r[j] = __dadd_rn(r[j], __dmul_rn((double)a[i + j], (double)b[i + j]));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, __dmul_rn((double)a[i], (double)b[i]));
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_f64(a, b, n2), pairwise_f64(a + n2, b + n2, n - n2));
}

__global__ void k_dot_rows_f64(const float* __restrict__ x, int64_t rows, int dim,
                               const float* __restrict__ v, double* __restrict__ out) {
  for (int64_t r = grid_tid(); r < rows; r += grid_stride())
    out[r] = __dadd_rn(0.0, pairwise_f64(x + r * dim, v, dim));
}

// Multi-task re-scoring, dim <= 128: a block stages 128 candidates' rows (coalesced
// gathers, rows padded to dim + 1 floats so the per-thread row walks are conflict-free)
// and the request's task vectors in shared memory; one thread per candidate then runs
// numpy's pairwise float64 dot against every task.
constexpr int kTdRows = 128;
__global__ void __launch_bounds__(kTdRows) k_task_dots_f64_smem(
    const float* __restrict__ cache, int64_t n_rows, int dim, const int64_t* __restrict__ rows,
    const int32_t* __restrict__ count, int64_t n_cand, const float* __restrict__ users,
    int n_tasks, double* __restrict__ out) {
  extern __shared__ double s_td[];
  const int stride = dim + 4;  // 16-byte rows; float4 reads by 8-thread phases hit distinct banks
  double* s_users = s_td;                                       // [n_tasks][dim], widened once
  float* s_rows = reinterpret_cast<float*>(s_td + n_tasks * dim);  // [kTdRows][stride]
  const int64_t b = blockIdx.y;
  const int64_t c0 = (int64_t)blockIdx.x * kTdRows;
  const int64_t nb = count[b];
  if (c0 >= n_cand) return;
  // rows: all 16-byte chunks of the block's rows in flight at once (cp.async, zero-fill for
  // padding lanes), then the task vectors while they land
  const int q4 = dim >> 2;
  for (int e = threadIdx.x; e < kTdRows * q4; e += blockDim.x) {
    const int r = e / q4, k = e - r * q4;
    const int64_t c = c0 + r;
    const int64_t row = (c < nb && c < n_cand) ? rows[b * n_cand + c] : -1;
    const bool ok = row >= 0 && row < n_rows;
    const float* src = cache + (ok ? row * dim + 4 * k : 0);
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_rows + r * stride + 4 * k);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(ok ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  for (int i = threadIdx.x; i < n_tasks * dim; i += blockDim.x)
    s_users[i] = (double)users[b * n_tasks * dim + i];
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const int64_t c = c0 + threadIdx.x;
  if (c >= n_cand) return;
  const int64_t row = c < nb ? rows[b * n_cand + c] : -1;
  const bool ok = row >= 0 && row < n_rows;
  const float* a = s_rows + threadIdx.x * stride;
  // numpy pairwise order for 8 <= n <= 128 (see pairwise_f64): eight strided partial sums,
  // a fixed combine tree, then the tail; four tasks share each widened row element.
  const int n = dim, body = n - (n % 8);
  for (int t0 = 0; t0 < n_tasks; t0 += 4) {
    const double* u[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) u[q] = s_users + min(t0 + q, n_tasks - 1) * dim;
    double r[4][8];
    float xs0[8];
    *reinterpret_cast<float4*>(xs0) = *reinterpret_cast<const float4*>(a);
    *reinterpret_cast<float4*>(xs0 + 4) = *reinterpret_cast<const float4*>(a + 4);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double x = (double)xs0[j];
#pragma unroll
      for (int q = 0; q < 4; ++q) r[q][j] = __dmul_rn(x, u[q][j]);
    }
    for (int i = 8; i < body; i += 8) {
      float xs[8];
      *reinterpret_cast<float4*>(xs) = *reinterpret_cast<const float4*>(a + i);
      *reinterpret_cast<float4*>(xs + 4) = *reinterpret_cast<const float4*>(a + i + 4);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double x = (double)xs[j];
#pragma unroll
        for (int q = 0; q < 4; ++q) r[q][j] = __dadd_rn(r[q][j], __dmul_rn(x, u[q][i + j]));
      }
    }
    double res[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      res[q] = __dadd_rn(__dadd_rn(__dadd_rn(r[q][0], r[q][1]), __dadd_rn(r[q][2], r[q][3])),
                         __dadd_rn(__dadd_rn(r[q][4], r[q][5]), __dadd_rn(r[q][6], r[q][7])));
    for (int i = body; i < n; ++i) {
      const double x = (double)a[i];
#pragma unroll
      for (int q = 0; q < 4; ++q) res[q] = __dadd_rn(res[q], __dmul_rn(x, u[q][i]));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (t0 + q < n_tasks) out[(b * n_tasks + t0 + q) * n_cand + c] = ok ? __dadd_rn(0.0, res[q]) : 0.0;
  }
}

// Multi-task re-scoring, any dim: one thread per (request, candidate) computes the
// candidate's dot with every task's user vector (numpy pairwise order, float64).
__global__ void k_task_dots_f64(const float* __restrict__ cache, int64_t n_rows, int dim,
                                const int64_t* __restrict__ rows, const int32_t* __restrict__ count,
                                int64_t n_cand, const float* __restrict__ users, int n_req,
                                int n_tasks, double* __restrict__ out) {
  const int64_t total = (int64_t)n_req * n_cand;
  for (int64_t g = grid_tid(); g < total; g += grid_stride()) {
    const int64_t b = g / n_cand, c = g - b * n_cand;
    const int64_t r = rows[g];
    const bool ok = c < count[b] && r >= 0 && r < n_rows;
    for (int t = 0; t < n_tasks; ++t) {
      const int64_t o = (b * n_tasks + t) * n_cand + c;
      out[o] = ok ? __dadd_rn(0.0, pairwise_f64(cache + r * dim, users + (b * n_tasks + t) * dim, dim))
                  : 0.0;
    }
  }
}

__global__ void k_row_sums(const int8_t* __restrict__ x, int64_t rows, int cols, int stride,
                           int32_t* __restrict__ out) {
  for (int64_t r = grid_tid(); r < rows; r += grid_stride()) {
    int32_t s = 0;
    for (int c = 0; c < cols; ++c) s += x[r * stride + c];
    out[r] = s;
  }
}

// ------------------------------------------------------------------------------------
// SIMT masked scan. One CTA per 64-slot word (grid-stride over the work list); the 64
// item rows are staged in shared memory, each thread owns a query: program -> mask,
// then an exact dp4a dot per admitted slot.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int32_t dot_i8(const int8_t* __restrict__ a, const int8_t* b, int n) {
  int acc = 0;
  for (int j = 0; j < n; j += 16) {
    const int4 x = __ldg(reinterpret_cast<const int4*>(a + j));
    const int4 y = *reinterpret_cast<const int4*>(b + j);
    acc = __dp4a(x.x, y.x, acc);
    acc = __dp4a(x.y, y.y, acc);
    acc = __dp4a(x.z, y.z, acc);
    acc = __dp4a(x.w, y.w, acc);
  }
  return acc;
}

__device__ __forceinline__ void locate_word(const ScanArgs& a, int64_t g, int64_t& w,
                                            uint64_t& rmask) {
  // range r with word_prefix[r] <= g < word_prefix[r + 1]
  int lo = 0, hi = a.n_ranges - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.word_prefix[mid] <= g) lo = mid; else hi = mid - 1;
  }
  const int64_t s0 = a.ranges[2 * lo], s1 = a.ranges[2 * lo + 1];
  w = (s0 >> 6) + (g - a.word_prefix[lo]);
  const int64_t rem = s1 - w * 64;
  rmask = rem >= 64 ? ~0ull : ((1ull << rem) - 1);
}

constexpr int kSimtMaxSharedLeaves = 2048;  // 16 KB of leaf words per CTA
__host__ __device__ __forceinline__ bool simt_shared_leaves(const fb_filter_prog_t& p) {
  return p.n_leaves > 0 && p.n_leaves <= kSimtMaxSharedLeaves;
}
__host__ __device__ __forceinline__ size_t simt_smem(const ScanArgs& a) {
  return (size_t)64 * a.idx.dim_pad +
         (a.has_prog && simt_shared_leaves(a.prog) ? (size_t)a.prog.n_leaves * 8 : 0);
}

template <int MODE>
__device__ void scan_simt_body(const ScanArgs& a, uint8_t* smem_items) {
  const int dp = a.idx.dim_pad;
  const int64_t n_work = (a.total_words + a.word_stride - 1) / a.word_stride;
  // the batch's distinct leaves evaluated once per word (behind the staged item rows) when
  // they fit, instead of once per (query, leaf)
  const bool shared_leaves = a.has_prog && simt_shared_leaves(a.prog);
  uint64_t* s_leaf = reinterpret_cast<uint64_t*>(smem_items + (size_t)64 * dp);
  for (int64_t gi = blockIdx.x; gi < n_work; gi += gridDim.x) {
    int64_t w;
    uint64_t rmask;
    locate_word(a, gi * a.word_stride, w, rmask);
    const uint64_t vword = a.idx.valid[w] & rmask;
    const int64_t slot0 = w * 64;
    __syncthreads();
    if (vword != 0) {
      const int4* src = reinterpret_cast<const int4*>(a.idx.items + slot0 * dp);
      int4* dst = reinterpret_cast<int4*>(smem_items);
      for (int i = threadIdx.x; i < 4 * dp; i += blockDim.x) dst[i] = __ldg(src + i);
      if (shared_leaves)
        for (int l = threadIdx.x; l < a.prog.n_leaves; l += blockDim.x)
          s_leaf[l] = leaf_word(a.prog.leaf_pos + (int64_t)l * a.prog.k_max, a.prog.k_max,
                                a.idx.planes, a.idx.n_words, w);
    }
    __syncthreads();
    if (vword == 0) continue;
    for (int q = threadIdx.x; q < a.n_queries; q += blockDim.x) {
      if (a.fb != nullptr && a.fb[q].state != a.only_state) continue;
      uint64_t m = !a.has_prog     ? vword
                   : shared_leaves ? eval_program_leaves(a.prog, q, s_leaf, vword) & vword
                                   : eval_program_word(a.prog, q, a.idx.planes, a.idx.n_words, w,
                                                       vword) & vword;
      if (a.masks != nullptr) m &= a.masks[(int64_t)q * a.idx.n_words + w];
      if (m == 0) continue;
      const int8_t* qrow = a.queries + (int64_t)q * dp;
      if (MODE == SCAN_EMIT) {
        atomicAdd(a.out_elig + q, (uint32_t)__popcll(m));
        const uint64_t T = a.threshold ? a.threshold[q] : 0ull;
        while (m) {
          const int i = __ffsll((long long)m) - 1;
          m &= m - 1;
          const int32_t sc = dot_i8(qrow, reinterpret_cast<const int8_t*>(smem_items) + i * dp, dp);
          const uint64_t key = make_key(sc, a.idx.id_rank[slot0 + i]);
          if (key >= T) {
            const uint32_t p = atomicAdd(a.out_cnt + q, 1u);
            if (p < (uint32_t)a.cap) {
              a.out_key[(int64_t)q * a.cap + p] = key;
              if (a.out_slot) a.out_slot[(int64_t)q * a.cap + p] = (uint32_t)(slot0 + i);
            }
          }
        }
      } else {
        const Fallback f = a.fb[q];
        uint32_t* h = a.hist + (int64_t)q * kHistBins;
        while (m) {
          const int i = __ffsll((long long)m) - 1;
          m &= m - 1;
          const int32_t sc = dot_i8(qrow, reinterpret_cast<const int8_t*>(smem_items) + i * dp, dp);
          const uint64_t key = make_key(sc, a.idx.id_rank[slot0 + i]);
          if (key >= f.lo) {
            const uint64_t b = (key - f.lo) >> f.shift;
            if (b < (uint64_t)kHistBins) atomicAdd(h + b, 1u);
          }
        }
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(256) k_scan_simt(ScanArgs a) {
  extern __shared__ __align__(16) uint8_t smem_items[];
  if (a.active_count != nullptr && *a.active_count == 0) return;
  scan_simt_body<MODE>(a, smem_items);
}

// ------------------------------------------------------------------------------------
// IVF-probed scan (ref retrieval.codesigned_search with nprobe < n_clusters,
// retrieval.py:124-135 + ivf.search_clusters, ivf.py:285-334): one CTA per (query, probed
// cluster) pair, one thread per 64-slot word of the cluster. The thread evaluates the
// query's filter program on its word (coalesced plane loads across the warp's consecutive
// words), then scores every eligible slot with dp4a against the query staged in shared
// memory and appends its key. The caller sizes cap to the largest possible eligible count,
// so every eligible pair is kept and the selection is exact without a threshold.
// ------------------------------------------------------------------------------------
constexpr int kIvfThreads = 64;
constexpr int kIvfMaxOps = 512;    // staged ops per query (longer programs: per-word global path)
constexpr int kIvfMaxPush = 128;  // (smem per CTA bounds the resident CTAs: 17 KB -> 13 per SM)
constexpr int kIvfRing = 4;        // leaves whose plane loads are in flight ahead of the stack

// The query's program, staged per CTA: ops with leaf operands renumbered in push order,
// and the pushed leaves' plane positions (padded with -1) in the same order.
struct IvfProg {
  uint16_t ops[kIvfMaxOps];
  int32_t pos[kIvfMaxPush * 8];
  int n_ops, n_push, fast;
};

// Plane words of leaf li -> ring slot li % kIvfRing of this thread (cp.async: no register
// holds the pending words, so later loads do not wait on earlier ones); one commit group
// per leaf, empty groups past the last leaf keep the group count uniform.
template <int K>
__device__ __forceinline__ void ivf_issue(const IvfProg& P, int li, const uint64_t* __restrict__ planes,
                                          int64_t n_words, int64_t w, uint64_t* ring) {
  if (li < P.n_push) {
    const int slot = li % kIvfRing;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const int p = P.pos[li * 8 + j];
      uint64_t* dst = ring + (slot * K + j) * kIvfThreads;
      if (p >= 0) {
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d),
                     "l"(planes + (int64_t)p * n_words + w) : "memory");
      } else {
        *dst = ~0ull;
      }
    }
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

// Filter word of one query on word w: the stack machine of eval_program_word over the staged
// program, with the plane words of the next kIvfRing leaves in flight ahead of their PUSH.
template <int K>
__device__ uint64_t ivf_eval_word(const IvfProg& P, const uint64_t* __restrict__ planes,
                                  int64_t n_words, int64_t w, uint64_t v, uint64_t* ring) {
#pragma unroll
  for (int r = 0; r < kIvfRing; ++r) ivf_issue<K>(P, r, planes, n_words, w, ring);
  // stack of depth <= 4 in registers: top cached, the rest shifted on push / pop (no
  // dynamic indexing, so nothing goes to local memory)
  uint64_t top = 0ull, s1 = 0ull, s2 = 0ull, s3 = 0ull;
  int li = 0;
  for (int o = 0; o < P.n_ops; ++o) {
    const uint32_t op = P.ops[o];
    const uint32_t code = op >> 14;
    if (code == FB_OP_PUSH_LEAF) {
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kIvfRing - 1) : "memory");
      const int slot = li % kIvfRing;
      uint64_t m = ~0ull;
#pragma unroll
      for (int j = 0; j < K; ++j) m &= ring[(slot * K + j) * kIvfThreads];
      ivf_issue<K>(P, li + kIvfRing, planes, n_words, w, ring);
      ++li;
      s3 = s2;
      s2 = s1;
      s1 = top;
      top = m;
    } else if (code == FB_OP_NOT) {
      top = ~top & v;
    } else {
      top = (code == FB_OP_AND) ? (s1 & top) : (s1 | top);
      s1 = s2;
      s2 = s3;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  return top;
}

template <int K>
__global__ void __launch_bounds__(kIvfThreads) k_ivf_scan(IvfScanArgs a) {
  __shared__ __align__(16) int8_t s_q[kIvfMaxDimPad];
  __shared__ IvfProg P;
  __shared__ uint64_t s_ring[kIvfRing * K * kIvfThreads];
  const int dp = a.idx.dim_pad;
  const int64_t pairs = (int64_t)a.n_queries * a.nprobe;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t pr = blockIdx.x; pr < pairs; pr += gridDim.x) {
    const int q = (int)(pr / a.nprobe);
    const int64_t w0 = a.probe_words[2 * pr], w1 = a.probe_words[2 * pr + 1];
    __syncthreads();
    for (int i = threadIdx.x; i < dp / 16; i += blockDim.x)
      reinterpret_cast<int4*>(s_q)[i] =
          __ldg(reinterpret_cast<const int4*>(a.queries + (int64_t)q * dp) + i);
    if (warp == 0 && a.has_prog) {
      // stage the program: lanes read 32 ops at a time, PUSH operands renumbered by a
      // ballot prefix, their positions copied
      const int o0 = a.prog.op_offset[q], o1 = a.prog.op_offset[q + 1];
      const int n_ops = o1 - o0;
      int n_push = 0;
      bool fast = n_ops <= kIvfMaxOps;
      for (int b = 0; fast && b < n_ops; b += 32) {
        const int o = b + lane;
        const uint32_t op = o < n_ops ? a.prog.ops[o0 + o] : 0u;
        const bool push = o < n_ops && (op >> 14) == FB_OP_PUSH_LEAF;
        const uint32_t bal = __ballot_sync(0xffffffffu, push);
        const int li = n_push + __popc(bal & ((1u << lane) - 1u));
        if (li + (push ? 1 : 0) > kIvfMaxPush) fast = false;
        if (o < n_ops && li < kIvfMaxPush) {
          P.ops[o] = push ? (uint16_t)((FB_OP_PUSH_LEAF << 14) | (li & 0x3FFF)) : (uint16_t)op;
          if (push) {
            const int32_t* src = a.prog.leaf_pos + (int64_t)(op & 0x3FFF) * a.prog.k_max;
            for (int j = 0; j < 8; ++j) P.pos[li * 8 + j] = j < a.prog.k_max && j < K ? src[j] : -1;
          }
        }
        n_push += __popc(bal);
        fast = __all_sync(0xffffffffu, fast);
      }
      if (lane == 0) {
        P.n_ops = n_ops;
        P.n_push = n_push;
        P.fast = fast && a.prog.k_max <= K && a.prog.max_stack <= 4 ? 1 : 0;
      }
    }
    __syncthreads();
    for (int64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
      const uint64_t v = a.idx.valid[w];
      if (v == 0) continue;
      uint64_t m = v;
      if (a.has_prog) {
        if (P.n_ops == 0) {
          m = v;  // unfiltered query inside a filtered batch
        } else if (P.fast) {
          m = ivf_eval_word<K>(P, a.idx.planes, a.idx.n_words, w, v, s_ring + threadIdx.x) & v;
        } else {
          m = eval_program_word(a.prog, q, a.idx.planes, a.idx.n_words, w, v) & v;
        }
      }
      if (m == 0) continue;
      const int64_t slot0 = w * 64;
      uint32_t p = atomicAdd(a.out_cnt + q, (uint32_t)__popcll(m));
      uint64_t* ok = a.out_key + (int64_t)q * a.cap;
      uint32_t* os = a.out_slot ? a.out_slot + (int64_t)q * a.cap : nullptr;
      while (m) {  // two rows in flight per step
        const int i0 = __ffsll((long long)m) - 1;
        m &= m - 1;
        const int i1 = m ? __ffsll((long long)m) - 1 : -1;
        if (m) m &= m - 1;
        const int32_t s0 = dot_i8(a.idx.items + (slot0 + i0) * dp, s_q, dp);
        const int32_t s1 = i1 >= 0 ? dot_i8(a.idx.items + (slot0 + i1) * dp, s_q, dp) : 0;
        if (p < (uint32_t)a.cap) {
          ok[p] = make_key(s0, a.idx.id_rank[slot0 + i0]);
          if (os) os[p] = (uint32_t)(slot0 + i0);
        }
        ++p;
        if (i1 >= 0) {
          if (p < (uint32_t)a.cap) {
            ok[p] = make_key(s1, a.idx.id_rank[slot0 + i1]);
            if (os) os[p] = (uint32_t)(slot0 + i1);
          }
          ++p;
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// Multi-task union merge by id rank (ref retrieval.merge_candidates, retrieval.py:147-160):
// ranks order ids (id_rank is the rank of the slot's id among the valid ids), so the union
// of a request's T candidate lists in ascending id order is the set bits of a per-request
// rank bitmap read in order. k_union_mark sets the bits; k_union_extract (one CTA per
// request) counts bits per thread-chunk, scans, writes ids in rank order and clears the
// words it read, leaving the bitmap zeroed for the next call.
// ------------------------------------------------------------------------------------
__global__ void k_union_mark(const uint64_t* __restrict__ keys, const int32_t* __restrict__ counts,
                             int B, int T, int k, int64_t n_words,
                             unsigned long long* __restrict__ bitmap) {
  const int64_t total = (int64_t)B * T * k;
  for (int64_t g = grid_tid(); g < total; g += grid_stride()) {
    const int64_t bt = g / k;
    const int i = (int)(g - bt * k);
    if (i >= counts[bt]) continue;
    const uint32_t rank = 0xFFFFFFFFu - (uint32_t)keys[g];
    const int64_t b = bt / T;
    atomicOr(bitmap + b * n_words + (rank >> 6), 1ull << (rank & 63));
  }
}

// Extraction: each request's words split into kUnionSegs segments of one CTA each; pass 1
// counts set bits per segment, pass 2 places each segment at the prefix of the earlier ones
// and, inside it, each warp at the prefix of the earlier warps; a warp walks its words 32 at
// a time (coalesced), lanes placed by a shuffle scan of their popcounts.
constexpr int kUnionThreads = 256, kUnionSegs = 16;

__device__ __forceinline__ void union_span(int64_t n_words, int seg, int warp, int64_t& w0,
                                           int64_t& w1) {
  const int nw = kUnionThreads / 32;
  const int64_t per_seg = (n_words + kUnionSegs - 1) / kUnionSegs;
  const int64_t s0 = min(n_words, per_seg * seg), s1 = min(n_words, s0 + per_seg);
  const int64_t per_warp = ((s1 - s0 + nw - 1) / nw + 31) / 32 * 32;
  w0 = min(s1, s0 + per_warp * warp);
  w1 = min(s1, w0 + per_warp);
}

__device__ __forceinline__ uint32_t union_warp_count(const unsigned long long* bm, int64_t w0,
                                                     int64_t w1, int lane) {
  uint32_t c = 0;
  for (int64_t w = w0 + lane; w < w1; w += 32) c += (uint32_t)__popcll(bm[w]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  return c;
}

__global__ void __launch_bounds__(kUnionThreads) k_union_count(
    const unsigned long long* __restrict__ bitmap, int64_t n_words, uint32_t* __restrict__ seg_cnt) {
  __shared__ uint32_t s_c[kUnionThreads / 32];
  const int b = blockIdx.y, seg = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t w0, w1;
  union_span(n_words, seg, wid, w0, w1);
  const uint32_t c = union_warp_count(bitmap + (int64_t)b * n_words, w0, w1, lane);
  if (lane == 0) s_c[wid] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < kUnionThreads / 32; ++i) t += s_c[i];
    seg_cnt[b * kUnionSegs + seg] = t;
  }
}

__global__ void __launch_bounds__(kUnionThreads) k_union_extract(
    unsigned long long* __restrict__ bitmap, int64_t n_words, const uint32_t* __restrict__ seg_cnt,
    const uint64_t* __restrict__ id_of_rank, int out_len, uint64_t* __restrict__ merged,
    int64_t* __restrict__ merged_ranks, int32_t* __restrict__ mcount) {
  __shared__ uint32_t s_c[kUnionThreads / 32];
  const int b = blockIdx.y, seg = blockIdx.x, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long* bm = bitmap + (int64_t)b * n_words;
  int64_t w0, w1;
  union_span(n_words, seg, wid, w0, w1);
  const uint32_t c = union_warp_count(bm, w0, w1, lane);
  if (lane == 0) s_c[wid] = c;
  __syncthreads();
  uint32_t pos = 0;
  for (int i = 0; i < seg; ++i) pos += seg_cnt[b * kUnionSegs + i];
  for (int i = 0; i < wid; ++i) pos += s_c[i];
  if (seg == kUnionSegs - 1 && threadIdx.x == 0) {
    uint32_t tot = 0;
    for (int i = 0; i < kUnionSegs; ++i) tot += seg_cnt[b * kUnionSegs + i];
    mcount[b] = (int32_t)min(tot, (uint32_t)out_len);
  }
  uint64_t* out = merged + (int64_t)b * out_len;
  for (int64_t base = w0; base < w1; base += 32) {
    const int64_t w = base + lane;
    unsigned long long m = w < w1 ? bm[w] : 0ull;
    const uint32_t pc = (uint32_t)__popcll(m);
    uint32_t incl = pc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    uint32_t p = pos + incl - pc;
    if (m != 0ull) {
      bm[w] = 0ull;
      while (m) {
        const int i = __ffsll((long long)m) - 1;
        m &= m - 1;
        if (p < (uint32_t)out_len) {
          out[p] = id_of_rank[w * 64 + i];
          if (merged_ranks) merged_ranks[(int64_t)b * out_len + p] = w * 64 + i;
        }
        ++p;
      }
    }
    pos += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// ------------------------------------------------------------------------------------
// Block-wide bitonic sort (descending by key) over n = power of two elements in smem.
// ------------------------------------------------------------------------------------
template <bool kHasVal>
__device__ void bitonic_desc(uint64_t* key, uint32_t* val, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        const int i = 2 * t - (t & (stride - 1));
        const int j = i + stride;
        const bool desc = (i & size) == 0;
        const uint64_t ki = key[i], kj = key[j];
        if (desc ? (ki < kj) : (ki > kj)) {
          key[i] = kj;
          key[j] = ki;
          if (kHasVal) {
            const uint32_t t2 = val[i];
            val[i] = val[j];
            val[j] = t2;
          }
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ int pow2_ceil(int n) {
  int p = 1;
  while (p < n) p <<= 1;
  return p;
}

// Per query: radix-select the sampled key of rank jd from the top, where mu = k * f_eff is
// the expected sample rank of the true k-th key (f_eff = the sampled fraction times the
// kept share of the eligible sample keys) and jd sits between mu and the emit capacity
// with >= 5 sigma on each side when the sample allows, so the emit pass keeps every key
// of the true top-k and fits the buffer with overwhelming probability at any selectivity
// (the check/fallback keeps the answer exact regardless). Samples that fit are staged in
// shared memory; larger ones are re-read from global memory (L2) per digit pass.
// 104 KB: two 1024-thread CTAs per SM (32 registers), so a 256-query batch runs in one
// wave on 148 SMs (a filtered config-2 query keeps ~8.7k sampled keys; at 208 KB the
// 256 CTAs took two waves)
constexpr int kThrSmemKeys = 13312;
__global__ void __launch_bounds__(kSelectThreads, 2) k_threshold(ThresholdArgs a) {
  extern __shared__ __align__(16) uint64_t s_key[];
  const int q = blockIdx.x;
  if (threadIdx.x == 0) {
    a.cnt[q] = 0;
    a.elig[q] = 0;
  }
  const uint32_t ns = a.sample_cnt != nullptr ? a.sample_cnt[q] : 0u;
  if (a.sample_fraction <= 0.0 || ns == 0) {
    if (threadIdx.x == 0) a.threshold[q] = 0ull;
    return;
  }
  const int nk = (int)min(ns, (uint32_t)a.sample_cap);
  // sample rank of the threshold: 5 sigma above the true k-th key's expected sample rank
  // when that stays 5 sigma below the capacity, else the middle of [k, cap]
  const double fe = a.sample_fraction * (double)nk / (double)ns;
  const double mu = (double)a.k * fe;
  const double cf = (double)a.cap * fe;
  const double lo = mu + 5.0 * sqrt(mu) + 8.0;
  const double hi = cf - 5.0 * sqrt(cf);
  // (the lower edge: every extra candidate costs hit-filter and selection work)
  const double jd = lo < hi ? lo : (0.5 * (mu + cf) > lo ? lo : 0.5 * (mu + cf));
  if (jd >= (double)(nk - 1)) {
    if (threadIdx.x == 0) a.threshold[q] = 0ull;
    return;
  }
  const uint64_t* gkey = a.sample_key + (int64_t)q * a.sample_cap;
  const bool staged = nk <= kThrSmemKeys;
  if (staged)
    for (int i = threadIdx.x; i < nk; i += blockDim.x) s_key[i] = gkey[i];
  // radix select (8-bit digits, most significant first) of the key with exactly `jd`
  // larger keys: one histogram pass over the kept sample per digit. The rank half (low 32
  // bits) is resolved only when the jd-th key's score is shared by more than two smaller
  // sampled keys: otherwise T keeps that score with the rank half zeroed, T <= the jd-th
  // key, admitting only the few candidates tied on its score (exactness needs T <= the
  // true k-th key, never an exact T) -- four passes instead of eight
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_need;
  __shared__ uint32_t s_binc;  // sampled keys in the chosen digit's bin
  if (threadIdx.x == 0) {
    s_prefix = 0ull;
    s_need = (uint32_t)jd + 1u;
  }
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0u;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    for (int i = threadIdx.x; i < nk; i += blockDim.x) {
      const uint64_t k = staged ? s_key[i] : __ldcg(gkey + i);
      if (shift == 56 || ((k ^ prefix) >> (shift + 8)) == 0ull)
        atomicAdd(hist + ((k >> shift) & 0xFFu), 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // one warp: find the digit holding rank `need` (from the top)
      const uint32_t need = s_need;
      // lane l owns bins [255 - 8l, 255 - 8l - 7]
      uint32_t c[8], sum = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * threadIdx.x - j];
        sum += c[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if ((int)threadIdx.x >= d) incl += y;
      }
      const uint32_t excl = incl - sum;
      if (excl < need && need <= incl) {
        uint32_t cum = excl;
        for (int j = 0; j < 8; ++j) {
          if (cum + c[j] >= need) {
            s_prefix = prefix | ((uint64_t)(255 - 8 * threadIdx.x - j) << shift);
            s_need = need - cum;
            s_binc = c[j];
            break;
          }
          cum += c[j];
        }
      }
    }
    __syncthreads();
    if (shift == 32 && s_binc - s_need <= 2u) break;  // uniform: shared values
  }
  if (threadIdx.x == 0) a.threshold[q] = s_prefix;
}

// Flag queries whose emit pass over- or under-flowed (or all, when forced).
__global__ void k_check(int n_queries, int k, int cap, const uint32_t* __restrict__ cnt,
                        const uint64_t* __restrict__ thr, int force, Fallback* fb,
                        uint32_t* active, uint32_t* total_flagged) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n_queries) return;
  const uint32_t c = cnt[q];
  // exact when every key >= T was kept and either k of them exist or T admits all
  const bool ok = c <= (uint32_t)cap && (c >= (uint32_t)k || thr[q] == 0ull);

  Fallback f;
  f.lo = 0;
  f.shift = 52;
  f.above = 0;
  f.need = (uint64_t)k;
#ifdef FB_CHECK_PRINT
  printf("k_check: query %d count %u cap %d k %d flagged %d\n", q, c, cap, k, (int)(force || !ok));
#endif
  if (force || !ok) {
    f.state = Q_FLAGGED;
    atomicAdd(active, 1u);
    atomicAdd(total_flagged, 1u);
  } else {
    f.state = Q_OK;
  }
  fb[q] = f;
}

__global__ void k_zero_hist(int n_queries, const Fallback* fb, uint32_t* hist,
                            const uint32_t* active) {
  if (*active == 0) return;
  const int64_t total = (int64_t)n_queries * kHistBins;
  for (int64_t i = grid_tid(); i < total; i += grid_stride()) {
    const int q = (int)(i / kHistBins);
    if (fb[q].state == Q_FLAGGED) hist[i] = 0;
  }
}

// Narrow each flagged query's key window to the histogram bin holding rank `need`;
// resolve once the keys >= that bin's lower edge fit the candidate buffer.
__device__ void resolve_query(int q, int k, int cap, Fallback* fb, const uint32_t* hist,
                              uint64_t* threshold, uint32_t* cnt, uint32_t* elig,
                              uint32_t* active) {
  if (fb[q].state != Q_FLAGGED) return;
  Fallback f = fb[q];
  const uint32_t* h = hist + (int64_t)q * kHistBins;
  uint64_t cum = 0;
  bool found = false;
  uint64_t T = 0;
  for (int b = kHistBins - 1; b >= 0; --b) {
    const uint64_t c = h[b];
    if (cum + c >= f.need) {
      const uint64_t edge = f.lo + ((uint64_t)b << f.shift);
      if (f.above + cum + c <= (uint64_t)cap || f.shift == 0) {
        T = edge;
        found = true;
      } else {
        f.above += cum;
        f.need -= cum;
        f.lo = edge;
        f.shift = f.shift >= 12 ? f.shift - 12 : 0;
        fb[q] = f;
        return;
      }
      break;
    }
    cum += c;
  }
  // found: threshold at the bin edge; !found: fewer than k eligible keys -> take all
  threshold[q] = found ? T : 0ull;
  cnt[q] = 0;
  elig[q] = 0;
  f.state = Q_RESOLVED;
  fb[q] = f;
  atomicSub(active, 1u);
  atomicAdd(active + 1, 1u);
}

__global__ void k_resolve(int n_queries, int k, int cap, Fallback* fb, const uint32_t* hist,
                          uint64_t* threshold, uint32_t* cnt, uint32_t* elig, uint32_t* active) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n_queries) resolve_query(q, k, cap, fb, hist, threshold, cnt, elig, active);
}

// The whole exact fallback in ONE cooperative launch: nothing but a flag read when no
// query was flagged (the common case); otherwise up to 6 rounds of (zero histograms ->
// SIMT histogram scan of the flagged queries -> narrow/resolve), grid-synchronised, then
// the re-emit of the resolved queries.
__global__ void __launch_bounds__(256) k_fallback(FallbackArgs f) {
  extern __shared__ __align__(16) uint8_t smem_items[];
  if (__ldcg(f.active) == 0u) return;  // written by k_check: uniform across the grid
  cg::grid_group g = cg::this_grid();
  const int64_t n_hist = (int64_t)f.n_queries * kHistBins;
  for (int pass = 0; pass < 6; ++pass) {
    for (int64_t i = grid_tid(); i < n_hist; i += grid_stride())
      if (f.fb[i / kHistBins].state == Q_FLAGGED) f.hist_buf[i] = 0u;
    g.sync();
    scan_simt_body<SCAN_HIST>(f.hist, smem_items);
    g.sync();
    for (int64_t q = grid_tid(); q < f.n_queries; q += grid_stride())
      resolve_query((int)q, f.k, f.cap, f.fb, f.hist_buf, f.threshold, f.cnt, f.elig, f.active);
    g.sync();
    if (__ldcg(f.active) == 0u) break;  // read after the sync: uniform
  }
  scan_simt_body<SCAN_EMIT>(f.emit, smem_items);
}

// ------------------------------------------------------------------------------------
// Exact selection: sort each query's candidates (chunks of kSelectChunk in smem), then
// place every element at its global rank by binary search in the other chunks.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int count_greater(const uint64_t* a, int n, uint64_t x, bool or_equal) {
  // a sorted descending; number of elements > x (or >= x)
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool before = or_equal ? (a[mid] >= x) : (a[mid] > x);
    if (before) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void write_out(const SelectArgs& a, int q, int rank, uint64_t key,
                                          uint32_t slot, int32_t qsum) {
  const int64_t o = (int64_t)q * a.k + rank;
  const int32_t sc = key_score(key);
  a.out_ids[o] = a.item_ids[slot];
  a.out_scores[o] = sc;
  if (a.out_keys) a.out_keys[o] = key;
  if (a.out_fscores) {
    const int32_t rs = a.row_sum ? a.row_sum[slot] : 0;
    a.out_fscores[o] = dequant_dot(sc, rs, qsum, a.dim, a.gmin, a.gmax);
  }
}

__global__ void __launch_bounds__(kSelectThreads) k_select(SelectArgs a) {
  extern __shared__ __align__(16) uint8_t smem_sel[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem_sel);
  uint32_t* s_val = reinterpret_cast<uint32_t*>(smem_sel + sizeof(uint64_t) * kSelectChunk);
  __shared__ int32_t s_qsum;
  const int q = blockIdx.x;
  const int n = (int)min(a.cnt[q], (uint32_t)a.cap);
  const int kk = min(a.k, n);
  if (threadIdx.x == 0) {
    a.out_count[q] = kk;
    int32_t s = 0;
    if (a.out_fscores)
      for (int c = 0; c < a.dim; ++c) s += a.queries[(int64_t)q * a.dim_pad + c];
    s_qsum = s;
  }
  // padding rows of the output
  for (int r = kk + threadIdx.x; r < a.k; r += blockDim.x) {
    const int64_t o = (int64_t)q * a.k + r;
    a.out_ids[o] = ~0ull;
    a.out_scores[o] = INT32_MIN;
    if (a.out_keys) a.out_keys[o] = 0ull;
    if (a.out_fscores) a.out_fscores[o] = 0.0;
  }
  __syncthreads();
  const int32_t qsum = s_qsum;
  uint64_t* gk = const_cast<uint64_t*>(a.cand_key) + (int64_t)q * a.cap;
  uint32_t* gs = a.cand_slot + (int64_t)q * a.cap;
  const int n_chunks = (n + kSelectChunk - 1) / kSelectChunk;
  for (int c = 0; c < n_chunks; ++c) {
    const int base = c * kSelectChunk;
    const int len = min(kSelectChunk, n - base);
    const int np2 = pow2_ceil(len);
    __syncthreads();
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
      s_key[i] = i < len ? gk[base + i] : 0ull;
      s_val[i] = i < len ? gs[base + i] : 0u;
    }
    bitonic_desc<true>(s_key, s_val, np2);
    if (n_chunks == 1) {
      for (int i = threadIdx.x; i < kk; i += blockDim.x) write_out(a, q, i, s_key[i], s_val[i], qsum);
      return;
    }
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      gk[base + i] = s_key[i];
      gs[base + i] = s_val[i];
    }
  }
  __syncthreads();
  __threadfence_block();
  for (int c = 0; c < n_chunks; ++c) {
    const int base = c * kSelectChunk;
    const int len = min(kSelectChunk, n - base);
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const uint64_t x = gk[base + i];
      int rank = i;
      for (int d = 0; d < n_chunks && rank < kk; ++d) {
        if (d == c) continue;
        const int dbase = d * kSelectChunk;
        const int dlen = min(kSelectChunk, n - dbase);
        rank += count_greater(gk + dbase, dlen, x, d < c);
      }
      if (rank < kk) write_out(a, q, rank, x, gs[base + i], qsum);
    }
  }
}

// ------------------------------------------------------------------------------------
// Key-only exact selection (index with a rank -> slot table): per query CTA,
//   1. the candidate keys are staged in shared memory (<= kRsMaxK of them; larger sets
//      are re-read from L2 by each pass);
//   2. an MSD radix select (8-bit digits from the highest bit where the keys differ)
//      finds the lower edge K of the top min(k, n) keys -- it stops as soon as a digit
//      bin completes the count, so usually after 2-4 histogram passes;
//   3. the keys >= K are compacted (exactly min(k, n) of them, keys being unique);
//   4. a bucket sort orders them (4096 bins on the top bits of the compressed key, one
//      scatter through the dead candidate buffer, ranks within the bins); output rank =
//      kk - 1 - sorted position;
//   5. ids come from id_of_rank (one gather), scores from the key, dequantised scores
//      through slot_of_rank.
// Same output as k_select (the oracle's (score desc, item_id asc) order).
// ------------------------------------------------------------------------------------
constexpr int kRsThreads = 1024;
constexpr int kRsMaxK = kSelectMaxCand;            // 24576 selected keys sorted in smem
// shared memory: the compacted / sorted keys (kRsMaxK u64; also the staging area of the
// candidates when they fit), then the bucket-sort bin counters and starts
constexpr size_t kRsCntOff = (size_t)kRsMaxK * 8;
constexpr int kRsBins = 4096;
constexpr size_t kRsSmem = kRsCntOff + (size_t)2 * kRsBins * 4;

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
    v = o > v ? o : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
    v = o < v ? o : v;
  }
  return v;
}

__global__ void __launch_bounds__(kRsThreads, 1) k_select_radix(SelectArgs a) {
  extern __shared__ __align__(16) uint8_t smem_rs[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(smem_rs);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem_rs + kRsCntOff);
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_red[2][32];
  __shared__ uint64_t s_lo;       // lower edge of the selected keys
  __shared__ uint64_t s_prefix;
  __shared__ uint32_t s_need, s_done, s_pos;
  __shared__ uint32_t s_wsum[32];
  __shared__ int32_t s_qsum;
  const int q = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int n = (int)min(a.cnt[q], (uint32_t)a.cap);
  const int kk = min(a.k, n);
  if (t == 0) {
    a.out_count[q] = kk;
    int32_t sum = 0;
    if (a.out_fscores)
      for (int c = 0; c < a.dim; ++c) sum += a.queries[(int64_t)q * a.dim_pad + c];
    s_qsum = sum;
  }
  for (int r = kk + t; r < a.k; r += kRsThreads) {
    const int64_t o = (int64_t)q * a.k + r;
    a.out_ids[o] = ~0ull;
    a.out_scores[o] = INT32_MIN;
    if (a.out_keys) a.out_keys[o] = 0ull;
    if (a.out_fscores) a.out_fscores[o] = 0.0;
  }
  if (kk == 0) return;
  const uint64_t* gk = a.cand_key + (int64_t)q * a.cap;

  // 1. load (staged in smem when the candidates fit, else re-read from L2 per pass) +
  //    max / min
  const bool staged = n <= kRsMaxK;
  uint64_t mx = 0ull, mn = ~0ull;
  constexpr int kLdU = 8;  // candidate loads in flight per thread
  for (int i0 = 0; i0 < n; i0 += kRsThreads * kLdU) {
    uint64_t kv[kLdU];
#pragma unroll
    for (int u = 0; u < kLdU; ++u) {
      const int i = i0 + u * kRsThreads + t;
      kv[u] = i < n ? gk[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kLdU; ++u) {
      const int i = i0 + u * kRsThreads + t;
      if (i < n) {
        if (staged) s_key[i] = kv[u];
        mx = kv[u] > mx ? kv[u] : mx;
        mn = kv[u] < mn ? kv[u] : mn;
      }
    }
  }
  mx = warp_max_u64(mx);
  mn = warp_min_u64(mn);
  if (lane == 0) {
    s_red[0][wid] = mx;
    s_red[1][wid] = mn;
  }
  __syncthreads();
  if (wid == 0) {
    mx = warp_max_u64(s_red[0][lane]);
    mn = warp_min_u64(s_red[1][lane]);
    if (lane == 0) {
      s_red[0][0] = mx;
      s_red[1][0] = mn;
      s_lo = mn;  // n <= k: every key is selected
      s_need = (uint32_t)kk;
      s_done = n <= kk ? 1u : 0u;
      const int hb = 63 - __clzll((long long)(mx ^ mn));
      const int shift = (hb / 8) * 8;
      s_prefix = shift + 8 >= 64 ? 0ull : (mx >> (shift + 8)) << (shift + 8);
      s_pos = (uint32_t)shift;  // current digit position
    }
  }
  __syncthreads();
  mx = s_red[0][0];

  // 2. MSD radix select of the lower edge of the top kk keys
  while (!s_done) {
    const int shift = (int)s_pos;
    const uint64_t prefix = s_prefix;
    for (int b = t; b < 256; b += kRsThreads) hist[b] = 0u;
    __syncthreads();
    for (int i = t; i < n; i += kRsThreads) {
      const uint64_t k = staged ? s_key[i] : __ldcg(gk + i);
      if (shift + 8 >= 64 || ((k ^ prefix) >> (shift + 8)) == 0ull)
        atomicAdd(hist + ((k >> shift) & 0xFFu), 1u);
    }
    __syncthreads();
    if (wid == 0) {
      const uint32_t need = s_need;
      uint32_t c[8], sum = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[255 - 8 * lane - j];
        sum += c[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      const uint32_t excl = incl - sum;
      if (excl < need && need <= incl) {
        uint32_t cum = excl;
        for (int j = 0; j < 8; ++j) {
          if (cum + c[j] >= need) {
            const uint64_t edge = prefix | ((uint64_t)(255 - 8 * lane - j) << shift);
            if (cum + c[j] == need || shift == 0) {
              s_lo = edge;  // the whole bin completes the count
              s_done = 1u;
            } else {
              s_prefix = edge;
              s_need = need - cum;
              s_pos = (uint32_t)(shift - 8);
            }
            break;
          }
          cum += c[j];
        }
      }
    }
    __syncthreads();
  }
  const uint64_t lo = s_lo;

  // 3. compaction of the kk keys >= lo to s_key[0, kk) (re-read from global memory, so
  //    the shared copy can be overwritten). Keys are compressed order-preservingly to
  //    ((score_bits - score_lo) << id_bits) | (n_slots - 1 - id_rank): ranks are a
  //    permutation of [0, n_slots), so the id part needs only id_bits bits.
  const uint32_t sb_lo = (uint32_t)(lo >> 32);
  const uint32_t id_base = 0u - (uint32_t)a.n_slots;  // low word of the key at rank n-1
  const int id_bits = a.n_slots <= 1 ? 0 : 64 - __clzll((long long)(a.n_slots - 1));
  if (t == 0) s_pos = 0u;
  __syncthreads();
  // Staged candidates are compacted in place: all keys of a chunk are read before any
  // kept key of it is written (one barrier per chunk), and writes stay below the chunk's
  // end (kept <= read). Otherwise the keys are re-read from L2.
  constexpr int kCmU = 4;
  for (int i0 = 0; i0 < n; i0 += kRsThreads * kCmU) {
    uint64_t kv[kCmU];
#pragma unroll
    for (int u = 0; u < kCmU; ++u) {
      const int i = i0 + u * kRsThreads + t;
      kv[u] = i < n ? (staged ? s_key[i] : __ldcg(gk + i)) : 0ull;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kCmU; ++u) {
      const int i = i0 + u * kRsThreads + t;
      const bool keep = i < n && kv[u] >= lo;
      const uint32_t b = __ballot_sync(0xffffffffu, keep);
      uint32_t base = 0u;
      if (lane == 0 && b != 0u) base = atomicAdd(&s_pos, (uint32_t)__popc(b));
      base = __shfl_sync(0xffffffffu, base, 0);
      if (keep)
        s_key[base + __popc(b & ((1u << lane) - 1u))] =
            ((uint64_t)((uint32_t)(kv[u] >> 32) - sb_lo) << id_bits) |
            (uint64_t)((uint32_t)kv[u] - id_base);
    }
  }
  __syncthreads();

  // 4. bucket sort of the compressed keys s_key[0, kk) into ascending order: 4096 bins on
  //    the top bits (one histogram pass, one scan, one scatter), then each key's rank
  //    inside its bin by counting the bin's smaller keys (bins hold a few keys: the top
  //    bits are the score). Result in s_key[0, kk); s_key[kRsMaxK, ...) is the scratch.
  const uint64_t cmax = ((uint64_t)((uint32_t)(mx >> 32) - sb_lo) << id_bits) |
                        (uint64_t)((uint32_t)mx - id_base);
  const int nbits = cmax == 0ull ? 0 : 64 - __clzll((long long)cmax);
  constexpr int kBins = kRsBins;
  const int bshift = nbits > 12 ? nbits - 12 : 0;
  uint32_t* s_bcnt = s_cnt;           // [kBins] counts, then fill pointers = bin ends
  uint32_t* s_bstart = s_cnt + kBins; // [kBins] bin starts
  uint64_t* src = s_key;
  // scatter scratch: the upper half of the shared buffer when kk fits there, else the
  // query's candidate buffer (dead after the compaction; cap >= kk)
  const bool dst_smem = kk <= kRsMaxK / 2;
  uint64_t* dst = dst_smem ? s_key + kRsMaxK / 2 : const_cast<uint64_t*>(gk);
  for (int b = t; b < kBins; b += kRsThreads) s_bcnt[b] = 0u;
  __syncthreads();
  for (int i = t; i < kk; i += kRsThreads) atomicAdd(s_bcnt + (int)(src[i] >> bshift), 1u);
  __syncthreads();
  {  // exclusive scan of the bin counts: thread t owns bins 4t .. 4t + 3
    uint32_t v[4], run = 0u;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[i] = run;
      run += s_bcnt[4 * t + i];
    }
    uint32_t incl = run;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += y;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const uint32_t ws = s_wsum[lane];
      uint32_t wi = ws;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, wi, d);
        if (lane >= d) wi += y;
      }
      s_wsum[lane] = wi - ws;
    }
    __syncthreads();
    const uint32_t off = s_wsum[wid] + incl - run;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      s_bstart[4 * t + i] = v[i] + off;
      s_bcnt[4 * t + i] = v[i] + off;  // fill pointer
    }
  }
  __syncthreads();
  for (int i = t; i < kk; i += kRsThreads) {
    const uint64_t c = src[i];
    dst[atomicAdd(s_bcnt + (int)(c >> bshift), 1u)] = c;
  }
  __syncthreads();
  if (dst_smem) {
    for (int i = t; i < kk; i += kRsThreads) {
      const uint64_t c = dst[i];
      const int b = (int)(c >> bshift);
      const uint32_t lo_b = s_bstart[b], hi_b = s_bcnt[b];
      uint32_t r = lo_b;
      for (uint32_t j = lo_b; j < hi_b; ++j) r += dst[j] < c ? 1u : 0u;
      src[r] = c;
    }
  } else {
    // the bin-ordered keys come back into shared memory (src is dead after the scatter),
    // the in-bin ranks are counted there and the sorted keys go out to the global buffer
    // and back -- two coalesced copies instead of O(bin size) L2 reads per key
    for (int i = t; i < kk; i += kRsThreads) src[i] = __ldcg(dst + i);
    __syncthreads();
    for (int i = t; i < kk; i += kRsThreads) {
      const uint64_t c = src[i];
      const int b = (int)(c >> bshift);
      const uint32_t lo_b = s_bstart[b], hi_b = s_bcnt[b];
      uint32_t r = lo_b;
      for (uint32_t j = lo_b; j < hi_b; ++j) r += src[j] < c ? 1u : 0u;
      dst[r] = c;
    }
    __syncthreads();
    for (int i = t; i < kk; i += kRsThreads) src[i] = __ldcg(dst + i);
  }
  __syncthreads();

  // 5. outputs (ascending sorted position p -> rank kk - 1 - p); all gathers of a
  //    thread's outputs are issued before any is consumed
  const int32_t qsum = s_qsum;
  constexpr int kOutU = 5;  // gathers in flight per thread
  const uint64_t id_mask = id_bits >= 64 ? ~0ull : ((1ull << id_bits) - 1ull);
  // ids straight from the rank (one gather) unless the dequantised scores need the slot
  const bool by_id = a.id_of_rank != nullptr && a.out_fscores == nullptr;
  if (by_id && a.id_dense) {
    // dense ids (fb_index_t.id_dense): id = base + rank, computed, no gather
    for (int r = t; r < kk; r += kRsThreads) {
      const uint64_t c = src[kk - 1 - r];
      const uint32_t sb = (uint32_t)(c >> id_bits) + sb_lo;
      const uint32_t low = (uint32_t)(c & id_mask) + id_base;
      const uint64_t key = ((uint64_t)sb << 32) | low;
      const int64_t o = (int64_t)q * a.k + r;
      a.out_ids[o] = a.dense_id_base + (uint64_t)(0xFFFFFFFFu - low);
      a.out_scores[o] = key_score(key);
      if (a.out_keys) a.out_keys[o] = key;
    }
    return;
  }
  if (by_id) {
    // ids only: kIdU id gathers in flight per thread (one round at k = 10000); the keys
    // are re-read from shared memory. The random gathers are the kernel's largest cost
    // (~45 % at config 2, FB timing ablation in DESIGN §4.2).
    constexpr int kIdU = 12;
    for (int r0 = 0; r0 < kk; r0 += kRsThreads * kIdU) {
      uint64_t iid[kIdU];
#pragma unroll
      for (int u = 0; u < kIdU; ++u) {
        const int r = r0 + u * kRsThreads + t;
        iid[u] = 0ull;
        if (r < kk) {
          const uint32_t low = (uint32_t)(src[kk - 1 - r] & id_mask) + id_base;
          iid[u] = __ldg(a.id_of_rank + (0xFFFFFFFFu - low));
        }
      }
#pragma unroll
      for (int u = 0; u < kIdU; ++u) {
        const int r = r0 + u * kRsThreads + t;
        if (r < kk) {
          const uint64_t c = src[kk - 1 - r];
          const uint32_t sb = (uint32_t)(c >> id_bits) + sb_lo;
          const uint32_t low = (uint32_t)(c & id_mask) + id_base;
          const uint64_t key = ((uint64_t)sb << 32) | low;
          const int64_t o = (int64_t)q * a.k + r;
          a.out_ids[o] = iid[u];
          a.out_scores[o] = key_score(key);
          if (a.out_keys) a.out_keys[o] = key;
        }
      }
    }
    return;
  }
  for (int r0 = 0; r0 < kk; r0 += kRsThreads * kOutU) {
    uint64_t key[kOutU];
    uint32_t slot[kOutU];
#pragma unroll
    for (int u = 0; u < kOutU; ++u) {
      const int r = r0 + u * kRsThreads + t;
      key[u] = 0ull;
      slot[u] = 0u;
      if (r < kk) {
        const uint64_t c = src[kk - 1 - r];
        const uint32_t sb = (uint32_t)(c >> id_bits) + sb_lo;
        const uint32_t low = (uint32_t)(c & id_mask) + id_base;
        key[u] = ((uint64_t)sb << 32) | low;
        slot[u] = 0xFFFFFFFFu - low;  // the rank
        if (!by_id) slot[u] = __ldg(a.slot_of_rank + slot[u]);
      }
    }
    uint64_t iid[kOutU];
    int32_t rsum[kOutU];
#pragma unroll
    for (int u = 0; u < kOutU; ++u) {
      const int r = r0 + u * kRsThreads + t;
      iid[u] = r < kk ? __ldg((by_id ? a.id_of_rank : a.item_ids) + slot[u]) : 0ull;
      rsum[u] = (r < kk && a.out_fscores && a.row_sum) ? __ldg(a.row_sum + slot[u]) : 0;
    }
#pragma unroll
    for (int u = 0; u < kOutU; ++u) {
      const int r = r0 + u * kRsThreads + t;
      if (r < kk) {
        const int64_t o = (int64_t)q * a.k + r;
        const int32_t sc = key_score(key[u]);
        a.out_ids[o] = iid[u];
        a.out_scores[o] = sc;
        if (a.out_keys) a.out_keys[o] = key[u];
        if (a.out_fscores) a.out_fscores[o] = dequant_dot(sc, rsum[u], qsum, a.dim, a.gmin, a.gmax);
      }
    }
  }
}

// ------------------------------------------------------------------------------------
// Shard merge (serve._reduce_topk): n_lists lists per query, each sorted by
// (score desc, item_id asc) -> global top-k. Compares (score, id) pairs directly, so
// shards only need shard-local id ranks.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ bool pair_before(int32_t sa, uint64_t ia, int32_t sb, uint64_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// number of elements of list (s, ids)[0, n) ordered strictly before (x_s, x_i)
// (or_equal: before-or-equal)
__device__ __forceinline__ int count_before(const int32_t* s, const uint64_t* ids, int n,
                                            int32_t xs, uint64_t xi, bool or_equal) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const bool before = pair_before(s[mid], ids[mid], xs, xi) ||
                        (or_equal && s[mid] == xs && ids[mid] == xi);
    if (before) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_merge(const int32_t* __restrict__ in_scores, const uint64_t* __restrict__ in_ids,
                        const double* __restrict__ in_fs, const int32_t* __restrict__ in_count,
                        int n_lists, int n_queries, int k_in, int k_out,
                        uint64_t* out_ids, int32_t* out_scores, int32_t* out_count,
                        double* out_fs) {
  const int q = blockIdx.x;
  int total = 0;
  for (int l = 0; l < n_lists; ++l) total += min(in_count[l * n_queries + q], k_in);
  const int kk = min(total, k_out);
  if (threadIdx.x == 0) out_count[q] = kk;
  for (int r = kk + threadIdx.x; r < k_out; r += blockDim.x) {
    const int64_t o = (int64_t)q * k_out + r;
    out_ids[o] = ~0ull;
    out_scores[o] = INT32_MIN;
    if (out_fs) out_fs[o] = 0.0;
  }
  for (int l = 0; l < n_lists; ++l) {
    const int64_t lb = ((int64_t)l * n_queries + q) * k_in;
    const int len = min(in_count[l * n_queries + q], k_in);
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
      const int32_t xs = in_scores[lb + i];
      const uint64_t xi = in_ids[lb + i];
      int rank = i;
      for (int d = 0; d < n_lists && rank < kk; ++d) {
        if (d == l) continue;
        const int64_t db = ((int64_t)d * n_queries + q) * k_in;
        const int dlen = min(in_count[d * n_queries + q], k_in);
        rank += count_before(in_scores + db, in_ids + db, dlen, xs, xi, d < l);
      }
      if (rank < kk) {
        const int64_t o = (int64_t)q * k_out + rank;
        out_ids[o] = xi;
        out_scores[o] = xs;
        if (out_fs) out_fs[o] = in_fs ? in_fs[lb + i] : 0.0;
      }
    }
  }
}

__global__ void k_dequant(const int32_t* __restrict__ scores, const int32_t* __restrict__ rs,
                          const int32_t* __restrict__ qs, int n_queries, int k,
                          const int32_t* __restrict__ count, int dim, double gmin, double gmax,
                          double* out) {
  const int64_t total = (int64_t)n_queries * k;
  for (int64_t i = grid_tid(); i < total; i += grid_stride()) {
    const int q = (int)(i / k);
    const int r = (int)(i - (int64_t)q * k);
    out[i] = (count != nullptr && r >= count[q]) ? 0.0
                                                 : dequant_dot(scores[i], rs[i], qs[q], dim, gmin, gmax);
  }
}

int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

}  // namespace

// ------------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------------
int launch_bloom_build(const uint64_t* fid, const uint64_t* value, const int64_t* slot,
                       int64_t n_pairs, int64_t n_words, int m_bits, int k, uint64_t* planes,
                       cudaStream_t s) {
  if (n_pairs == 0) return FB_OK;
  k_bloom_build<<<grid_for(n_pairs, 256), 256, 0, s>>>(
      fid, value, slot, n_pairs, n_words, m_bits, k,
      reinterpret_cast<unsigned long long*>(planes));
  FB_LAUNCH_CHECK("k_bloom_build");
  return FB_OK;
}

int launch_filter_eval(const fb_index_t& idx, const fb_filter_prog_t& prog, int64_t w0, int64_t w1,
                       int apply_valid, uint64_t* out, cudaStream_t s) {
  const int64_t total = (w1 - w0) * prog.n_queries;
  if (total <= 0) return FB_OK;
  const size_t smem = (size_t)prog.n_leaves * kFeWords * sizeof(uint64_t);
  if (prog.n_leaves > 0 && smem <= 96 * 1024) {
    if (smem > 48 * 1024)
      FB_CUDA(cudaFuncSetAttribute(k_filter_eval_shared, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    const int64_t chunks = (w1 - w0 + kFeWords - 1) / kFeWords;
    const int grid = (int)std::min<int64_t>(chunks, 148LL * 16);
    k_filter_eval_shared<<<grid, 256, smem, s>>>(idx, prog, w0, w1, apply_valid, out);
    FB_LAUNCH_CHECK("k_filter_eval_shared");
    return FB_OK;
  }
  k_filter_eval<<<grid_for(total, 256), 256, 0, s>>>(idx, prog, w0, w1, apply_valid, out);
  FB_LAUNCH_CHECK("k_filter_eval");
  return FB_OK;
}

int launch_quantize(const float* x, int64_t rows, int cols, double gmin, double gmax, int8_t* out,
                    int out_stride, cudaStream_t s) {
  const int64_t total = rows * out_stride;
  if (total <= 0) return FB_OK;
  const double scale = 255.0 / (gmax - gmin);
  k_quantize<float><<<grid_for(total, 256), 256, 0, s>>>(x, rows, cols, gmin, scale, out, out_stride);
  FB_LAUNCH_CHECK("k_quantize");
  return FB_OK;
}

int launch_quantize_f64(const double* x, int64_t rows, int cols, double gmin, double gmax,
                        int8_t* out, int out_stride, cudaStream_t s) {
  const int64_t total = rows * out_stride;
  if (total <= 0) return FB_OK;
  const double scale = 255.0 / (gmax - gmin);
  k_quantize<double><<<grid_for(total, 256), 256, 0, s>>>(x, rows, cols, gmin, scale, out,
                                                          out_stride);
  FB_LAUNCH_CHECK("k_quantize_f64");
  return FB_OK;
}

int launch_dot_rows_i8(const int8_t* rows, int64_t n, int dim, int stride, const int8_t* vec,
                       int32_t* out, cudaStream_t s) {
  if (n <= 0) return FB_OK;
  k_dot_rows_i8<<<grid_for(n, 256), 256, 0, s>>>(rows, n, dim, stride, vec, out);
  FB_LAUNCH_CHECK("k_dot_rows_i8");
  return FB_OK;
}

int launch_dot_rows_f64(const float* rows, int64_t n, int dim, const float* vec, double* out,
                        cudaStream_t s) {
  if (n <= 0) return FB_OK;
  k_dot_rows_f64<<<grid_for(n, 128), 128, 0, s>>>(rows, n, dim, vec, out);
  FB_LAUNCH_CHECK("k_dot_rows_f64");
  return FB_OK;
}

int launch_task_dots_f64(const float* cache, int64_t n_rows, int dim, const int64_t* rows,
                         const int32_t* count, int64_t n_cand, const float* users, int n_req,
                         int n_tasks, double* out, cudaStream_t s) {
  const int64_t total = (int64_t)n_req * n_cand;
  if (total <= 0 || n_tasks <= 0) return FB_OK;
  const size_t smem = (size_t)kTdRows * (dim + 4) * sizeof(float) + (size_t)n_tasks * dim * sizeof(double);
  if (dim >= 8 && dim <= 128 && dim % 4 == 0 && (reinterpret_cast<uintptr_t>(cache) & 15) == 0 && smem <= 200 * 1024 && n_req <= 65535) {
    if (smem > 48 * 1024)
      FB_CUDA(cudaFuncSetAttribute(k_task_dots_f64_smem,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const dim3 grid((unsigned)((n_cand + kTdRows - 1) / kTdRows), (unsigned)n_req);
    k_task_dots_f64_smem<<<grid, kTdRows, smem, s>>>(cache, n_rows, dim, rows, count, n_cand,
                                                     users, n_tasks, out);
    FB_LAUNCH_CHECK("k_task_dots_f64_smem");
    return FB_OK;
  }
  k_task_dots_f64<<<grid_for(total, 128), 128, 0, s>>>(cache, n_rows, dim, rows, count, n_cand,
                                                       users, n_req, n_tasks, out);
  FB_LAUNCH_CHECK("k_task_dots_f64");
  return FB_OK;
}

int launch_row_sums(const int8_t* x, int64_t rows, int cols, int stride, int32_t* out,
                    cudaStream_t s) {
  if (rows <= 0) return FB_OK;
  k_row_sums<<<grid_for(rows, 256), 256, 0, s>>>(x, rows, cols, stride, out);
  FB_LAUNCH_CHECK("k_row_sums");
  return FB_OK;
}

int launch_scan_simt(const ScanArgs& a, cudaStream_t s) {
  if (a.total_words <= 0 || a.n_queries <= 0) return FB_OK;
  const int64_t n_work = (a.total_words + a.word_stride - 1) / a.word_stride;
  const size_t smem = simt_smem(a);
  int grid = (int)(n_work < 148 * 8 ? n_work : 148 * 8);
  if (a.mode == SCAN_EMIT) {
    if (smem > 48 * 1024)
      FB_CUDA(cudaFuncSetAttribute(k_scan_simt<SCAN_EMIT>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_scan_simt<SCAN_EMIT><<<grid, 256, smem, s>>>(a);
  } else {
    if (smem > 48 * 1024)
      FB_CUDA(cudaFuncSetAttribute(k_scan_simt<SCAN_HIST>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_scan_simt<SCAN_HIST><<<grid, 256, smem, s>>>(a);
  }
  FB_LAUNCH_CHECK("k_scan_simt");
  return FB_OK;
}

int launch_threshold(const ThresholdArgs& a, cudaStream_t s) {
  if (a.n_queries <= 0) return FB_OK;
  const size_t smem = (size_t)std::min(a.sample_cap, kThrSmemKeys) * sizeof(uint64_t);
  FB_CUDA(cudaFuncSetAttribute(k_threshold, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  k_threshold<<<a.n_queries, kSelectThreads, smem, s>>>(a);
  FB_LAUNCH_CHECK("k_threshold");
  return FB_OK;
}

int launch_check(int32_t n_queries, int32_t k, int32_t cap, const uint32_t* cnt,
                 const uint64_t* thr, int force, Fallback* fb, uint32_t* active,
                 uint32_t* total_flagged, cudaStream_t s) {
  if (n_queries <= 0) return FB_OK;
  k_check<<<(n_queries + 255) / 256, 256, 0, s>>>(n_queries, k, cap, cnt, thr, force, fb, active,
                                                  total_flagged);
  FB_LAUNCH_CHECK("k_check");
  return FB_OK;
}

int launch_zero_hist(int32_t n_queries, const Fallback* fb, uint32_t* hist,
                     const uint32_t* active, cudaStream_t s) {
  if (n_queries <= 0) return FB_OK;
  k_zero_hist<<<grid_for((int64_t)n_queries * kHistBins, 256), 256, 0, s>>>(n_queries, fb, hist,
                                                                             active);
  FB_LAUNCH_CHECK("k_zero_hist");
  return FB_OK;
}

int launch_resolve(int32_t n_queries, int32_t k, int32_t cap, Fallback* fb, uint32_t* hist,
                   uint64_t* threshold, uint32_t* cnt, uint32_t* elig, uint32_t* active,
                   int final_pass, cudaStream_t s) {
  (void)final_pass;
  if (n_queries <= 0) return FB_OK;
  k_resolve<<<(n_queries + 127) / 128, 128, 0, s>>>(n_queries, k, cap, fb, hist, threshold, cnt,
                                                    elig, active);
  FB_LAUNCH_CHECK("k_resolve");
  return FB_OK;
}

int launch_fallback(const FallbackArgs& f, cudaStream_t s) {
  if (f.n_queries <= 0) return FB_OK;
  const size_t smem = std::max(simt_smem(f.hist), simt_smem(f.emit));
  if (smem > 48 * 1024)
    FB_CUDA(cudaFuncSetAttribute(k_fallback, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  int per_sm = 0, n_sm = 148;
  FB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fallback, 256, smem));
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = std::max(1, std::min(per_sm, 4) * n_sm);
  FallbackArgs args = f;
  void* params[] = {&args};
  FB_CUDA(cudaLaunchCooperativeKernel((const void*)k_fallback, dim3(grid), dim3(256), params,
                                      smem, s));
  FB_LAUNCH_CHECK("k_fallback");
  return FB_OK;
}

bool select_by_rank(int32_t cap, int32_t k, const uint32_t* slot_of_rank) {
  (void)cap;  // any candidate count: beyond kRsMaxK the select reads them from L2
  return slot_of_rank != nullptr && k <= kRsMaxK;
}

int launch_select(const SelectArgs& a, cudaStream_t s) {
  if (a.n_queries <= 0) return FB_OK;
  if (select_by_rank(a.cap, a.k, a.slot_of_rank)) {
    FB_CUDA(cudaFuncSetAttribute(k_select_radix, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)kRsSmem));
    k_select_radix<<<a.n_queries, kRsThreads, kRsSmem, s>>>(a);
    FB_LAUNCH_CHECK("k_select_radix");
    return FB_OK;
  }
  const size_t smem = (size_t)kSelectChunk * (sizeof(uint64_t) + sizeof(uint32_t));
  FB_CUDA(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_select<<<a.n_queries, kSelectThreads, smem, s>>>(a);
  FB_LAUNCH_CHECK("k_select");
  return FB_OK;
}

int launch_ivf_scan(const IvfScanArgs& a, cudaStream_t s) {
  const int64_t pairs = (int64_t)a.n_queries * a.nprobe;
  if (pairs <= 0) return FB_OK;
  const int grid = (int)std::min<int64_t>(pairs, 148LL * 64);
  const int kmax = a.has_prog ? a.prog.k_max : 1;
  if (kmax <= 5) {
    k_ivf_scan<5><<<grid, kIvfThreads, 0, s>>>(a);
  } else {
    k_ivf_scan<8><<<grid, kIvfThreads, 0, s>>>(a);
  }
  FB_LAUNCH_CHECK("k_ivf_scan");
  return FB_OK;
}

int launch_union_merge(const uint64_t* keys, const int32_t* counts, int B, int T, int k,
                       int64_t n_words, uint64_t* bitmap, const uint64_t* id_of_rank,
                       uint64_t* merged, int64_t* merged_ranks, int32_t* mcount, cudaStream_t s) {
  if (B <= 0) return FB_OK;
  if (B > 65535) return fail(FB_ERR_INVALID, "too many requests");
  const int out_len = T * k;
  FB_CUDA(cudaMemsetAsync(merged, 0xFF, sizeof(uint64_t) * (size_t)B * out_len, s));
  if (merged_ranks)
    FB_CUDA(cudaMemsetAsync(merged_ranks, 0xFF, sizeof(int64_t) * (size_t)B * out_len, s));
  const int64_t total = (int64_t)B * T * k;
  auto* bm = reinterpret_cast<unsigned long long*>(bitmap);
  if (total > 0) {
    k_union_mark<<<grid_for(total, 256), 256, 0, s>>>(keys, counts, B, T, k, n_words, bm);
    FB_LAUNCH_CHECK("k_union_mark");
  }
  // per-segment counts: the caller's scratch past the bitmaps (B * kUnionSegs u32)
  uint32_t* seg_cnt = reinterpret_cast<uint32_t*>(bitmap + (size_t)B * n_words);
  const dim3 grid(kUnionSegs, B);
  k_union_count<<<grid, kUnionThreads, 0, s>>>(bm, n_words, seg_cnt);
  FB_LAUNCH_CHECK("k_union_count");
  k_union_extract<<<grid, kUnionThreads, 0, s>>>(bm, n_words, seg_cnt, id_of_rank, out_len, merged,
                                                 merged_ranks, mcount);
  FB_LAUNCH_CHECK("k_union_extract");
  return FB_OK;
}

int launch_merge(const int32_t* in_scores, const uint64_t* in_ids, const double* in_fscores,
                 const int32_t* in_count, int n_lists, int n_queries, int k_in, int k_out,
                 uint64_t* out_ids, int32_t* out_scores, int32_t* out_count, double* out_fscores,
                 cudaStream_t s) {
  if (n_queries <= 0) return FB_OK;
  k_merge<<<n_queries, 512, 0, s>>>(in_scores, in_ids, in_fscores, in_count, n_lists, n_queries,
                                    k_in, k_out, out_ids, out_scores, out_count, out_fscores);
  FB_LAUNCH_CHECK("k_merge");
  return FB_OK;
}

int launch_dequant(const int32_t* scores, const int32_t* item_row_sum, const int32_t* query_sum,
                   int n_queries, int k, const int32_t* count, int dim, double gmin, double gmax,
                   double* out, cudaStream_t s) {
  const int64_t total = (int64_t)n_queries * k;
  if (total <= 0) return FB_OK;
  k_dequant<<<grid_for(total, 256), 256, 0, s>>>(scores, item_row_sum, query_sum, n_queries, k,
                                                 count, dim, gmin, gmax, out);
  FB_LAUNCH_CHECK("k_dequant");
  return FB_OK;
}

// ------------------------------------------------------------------------------------
// Final ranking of multi-task retrieval (ref retrieval.retrieve, retrieval.py:190:
// order = np.lexsort((merged, -final))[:topk]): per request CTA, the first n = count[b]
// entries of final[b, :] (merged candidates in ascending id order, so position breaks ties
// as the id does) ordered by (final desc, position asc) with NumPy's float order: NaN after
// every number, -0.0 == +0.0. Keys u = orderable(-final) ascending:
//   1. keys staged in smem; an MSD radix select finds the boundary prefix of the kk-th key;
//   2. keys below the boundary are kept, keys on it in position order until kk are kept;
//   3. a bitonic sort of the kk (key, position) pairs; order[b, r] = position.
// ------------------------------------------------------------------------------------
constexpr int kFtThreads = 1024;
constexpr int kFtMaxN = 24576;   // staged keys per request
constexpr int kFtMaxK = 8192;    // sorted selection (power of two)
constexpr size_t kFtSmem = (size_t)kFtMaxN * 8 + (size_t)kFtMaxK * 4 + 256 * 4 + 64 * 4;

__device__ __forceinline__ uint64_t ft_key(double v) {
  const double u = -v;
  if (u != u) return ~0ull;  // NaN: after every number
  uint64_t b = (uint64_t)__double_as_longlong(u == 0.0 ? 0.0 : u);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void __launch_bounds__(kFtThreads, 1)
    k_final_topk(const double* __restrict__ final_, int64_t ld, const int32_t* __restrict__ count,
                 int32_t topk, int64_t* __restrict__ order, int32_t* __restrict__ out_count) {
  extern __shared__ __align__(16) uint8_t ft_smem[];
  uint64_t* s_key = reinterpret_cast<uint64_t*>(ft_smem);               // [kFtMaxN]
  uint32_t* s_pos = reinterpret_cast<uint32_t*>(s_key + kFtMaxN);       // [kFtMaxK]
  uint32_t* s_hist = s_pos + kFtMaxK;                                   // [256]
  uint32_t* s_misc = s_hist + 256;                                      // [64]
  const int b = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n = min(count[b], kFtMaxN);
  const int kk = min(topk, n);
  const double* f = final_ + (int64_t)b * ld;
  for (int i = t; i < n; i += kFtThreads) s_key[i] = ft_key(f[i]);
  // 1. radix select: prefix / mask of the kk-th smallest key, r = its rank inside the bin
  uint64_t prefix = 0ull, mask = 0ull;
  int r = kk;
  __syncthreads();
  for (int shift = 56; shift >= 0 && kk > 0; shift -= 8) {
    for (int i = t; i < 256; i += kFtThreads) s_hist[i] = 0u;
    __syncthreads();
    for (int i = t; i < n; i += kFtThreads) {
      const uint64_t u = s_key[i];
      if ((u & mask) == prefix) atomicAdd(s_hist + (int)((u >> shift) & 0xFF), 1u);
    }
    __syncthreads();
    if (warp == 0) {  // the digit whose cumulative count reaches r
      uint32_t c[8], sum = 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = s_hist[lane * 8 + j];
        sum += c[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      uint32_t run = incl - sum;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (run < (uint32_t)r && run + c[j] >= (uint32_t)r) {
          s_misc[0] = (uint32_t)(lane * 8 + j);
          s_misc[1] = run;
          s_misc[2] = c[j];
        }
        run += c[j];
      }
    }
    __syncthreads();
    const uint32_t d = s_misc[0];
    r -= (int)s_misc[1];
    const uint32_t bin = s_misc[2];
    prefix |= (uint64_t)d << shift;
    mask |= 0xFFull << shift;
    __syncthreads();
    if ((int)bin == r) break;  // the whole bin completes the count
  }
  // 2. selection: keys below the boundary (any order), then r keys on it in position order
  if (t == 0) s_misc[3] = 0u;
  __syncthreads();
  for (int i = t; i < n; i += kFtThreads) {
    const uint64_t u = s_key[i];
    if ((u & mask) < prefix) s_pos[atomicAdd(s_misc + 3, 1u)] = (uint32_t)i;
  }
  __syncthreads();
  const uint32_t n_lt = s_misc[3];
  uint32_t taken = 0u;
  for (int base = 0; base < n && (int)taken < r; base += kFtThreads) {
    const int i = base + t;
    const bool e = i < n && (s_key[i] & mask) == prefix;
    const uint32_t bal = __ballot_sync(0xffffffffu, e);
    if (lane == 0) s_misc[32 + warp] = (uint32_t)__popc(bal);
    __syncthreads();
    uint32_t before = 0u, total = 0u;
    for (int w = 0; w < kFtThreads / 32; ++w) {
      const uint32_t c = s_misc[32 + w];
      before += w < warp ? c : 0u;
      total += c;
    }
    const uint32_t pos = taken + before + (uint32_t)__popc(bal & ((1u << lane) - 1u));
    if (e && (int)pos < r) s_pos[n_lt + pos] = (uint32_t)i;
    taken += total;
    __syncthreads();
  }
  __syncthreads();
  // 3. bitonic sort of (key, position) over the next power of two >= kk; padding last
  int P = 1;
  while (P < kk) P <<= 1;
  // keys of the selected positions into registers, then over the (now free) key buffer
  constexpr int kPer = kFtMaxK / kFtThreads;
  uint64_t kv[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = t + j * kFtThreads;
    kv[j] = i < kk ? s_key[s_pos[i]] : ~0ull;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = t + j * kFtThreads;
    if (i < P) {
      s_key[i] = kv[j];
      if (i >= kk) s_pos[i] = 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int x = t; x < P / 2; x += kFtThreads) {
        const int lo = 2 * x - (x & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t ka = s_key[lo], kb = s_key[hi];
        const uint32_t pa = s_pos[lo], pb = s_pos[hi];
        const bool gt = ka > kb || (ka == kb && pa > pb);
        if (gt == up) {
          s_key[lo] = kb; s_key[hi] = ka;
          s_pos[lo] = pb; s_pos[hi] = pa;
        }
      }
      __syncthreads();
    }
  }
  int64_t* o = order + (int64_t)b * topk;
  for (int i = t; i < topk; i += kFtThreads) o[i] = i < kk ? (int64_t)s_pos[i] : 0;
  if (t == 0) out_count[b] = kk;
}

int launch_final_topk(const double* final_, int64_t ld, const int32_t* count, int n_requests,
                      int topk, int64_t* order, int32_t* out_count, cudaStream_t s) {
  if (n_requests <= 0 || topk <= 0) return FB_OK;
  if (topk > kFtMaxK) return fail(FB_ERR_UNSUPPORTED, "final top-k above 8192");
  if (ld > kFtMaxN) return fail(FB_ERR_UNSUPPORTED, "more than 24576 merged candidates");
  FB_CUDA(cudaFuncSetAttribute(k_final_topk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)kFtSmem));
  k_final_topk<<<n_requests, kFtThreads, kFtSmem, s>>>(final_, ld, count, topk, order, out_count);
  FB_LAUNCH_CHECK("k_final_topk");
  return FB_OK;
}

// ------------------------------------------------------------------------------------
// OverArch value model (ref value_model.py:31-91, evaluated by retrieval.retrieve): a
// formula over the task scores compiled on the host to postfix bytecode (overarch.py
// value_model_code) and run element-wise in float64, one thread per (request, candidate),
// with a register stack. Every operation rounds as NumPy does (no FMA contraction: the
// intrinsics pin each add / mul / div); min / max propagate NaN; clamp keeps NaN; `if`
// evaluates both branches. A zero divisor on a valid candidate (index < count[b]) sets
// *zero_flag (the caller raises DivByZero).
// ------------------------------------------------------------------------------------
enum : uint8_t {
  VM_CONST = 0, VM_TASK = 1, VM_ADD = 2, VM_SUB = 3, VM_MUL = 4, VM_DIV = 5, VM_MIN = 6,
  VM_MAX = 7, VM_CLAMP = 8, VM_IF_LT = 9, VM_IF_LE = 10, VM_IF_GT = 11, VM_IF_GE = 12,
  VM_IF_EQ = 13
};
constexpr int kVmStack = 16;

__global__ void k_value_model(const uint16_t* __restrict__ code, int n_code,
                              const double* __restrict__ consts, const double* __restrict__ ts,
                              int B, int T, int64_t C, const int32_t* __restrict__ count,
                              double* __restrict__ out, int32_t* __restrict__ zero_flag) {
  const int64_t total = (int64_t)B * C;
  for (int64_t g = grid_tid(); g < total; g += grid_stride()) {
    const int64_t b = g / C, i = g - b * C;
    const bool valid = i < (int64_t)count[b];
    double st[kVmStack];
    int sp = 0;
    for (int pc = 0; pc < n_code; ++pc) {
      const uint32_t w = code[pc];
      const uint32_t op = w & 0xFF, arg = w >> 8;
      if (op == VM_CONST) {
        st[sp++] = consts[arg];
      } else if (op == VM_TASK) {
        st[sp++] = ts[(b * T + arg) * C + i];
      } else if (op == VM_CLAMP) {  // np.clip: minimum(maximum(x, lo), hi)
        const double x = st[sp - 1], lo = consts[arg], hi = consts[arg + 1];
        const double t = (x != x || lo != lo) ? (x + lo) : (lo > x ? lo : x);
        st[sp - 1] = (t != t || hi != hi) ? (t + hi) : (hi < t ? hi : t);
      } else if (op >= VM_IF_LT) {  // left right then else -> cond ? then : else
        const double e = st[sp - 1], t = st[sp - 2], r = st[sp - 3], l = st[sp - 4];
        const bool c = op == VM_IF_LT ? l < r : op == VM_IF_LE ? l <= r : op == VM_IF_GT ? l > r
                       : op == VM_IF_GE ? l >= r : l == r;
        sp -= 3;
        st[sp - 1] = c ? t : e;
      } else {
        const double y = st[sp - 1], x = st[sp - 2];
        double z;
        switch (op) {
          case VM_ADD: z = __dadd_rn(x, y); break;
          case VM_SUB: z = __dsub_rn(x, y); break;
          case VM_MUL: z = __dmul_rn(x, y); break;
          case VM_DIV:
            if (y == 0.0 && valid) atomicOr(zero_flag, 1);
            z = __ddiv_rn(x, y);
            break;
          case VM_MIN: z = (x != x || y != y) ? (x + y) : (y < x ? y : x); break;
          default: z = (x != x || y != y) ? (x + y) : (y > x ? y : x); break;
        }
        sp -= 1;
        st[sp - 1] = z;
      }
    }
    out[g] = st[0];
  }
}

int launch_value_model(const uint16_t* code, int n_code, const double* consts, const double* ts,
                       int B, int T, int64_t C, const int32_t* count, double* out,
                       int32_t* zero_flag, cudaStream_t s) {
  const int64_t total = (int64_t)B * C;
  if (total <= 0) return FB_OK;
  k_value_model<<<grid_for(total, 256), 256, 0, s>>>(code, n_code, consts, ts, B, T, C, count,
                                                     out, zero_flag);
  FB_LAUNCH_CHECK("k_value_model");
  return FB_OK;
}

}  // namespace fb
