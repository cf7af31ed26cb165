// Publish-side k-means (reference ivf.py:68-145) on the GPU.
//
// The reference trains on float64 copies of the embeddings with numpy. Everything whose
// floating-point order numpy pins down is reproduced bit for bit here:
//   * D^2 seeding distances  np.sum((data - c) ** 2, axis=1)   (ivf.py:86, 97): numpy's
//     pairwise row sum (eight strided partial sums, fixed combine tree; recursive above 128);
//   * totals                 best.sum(), d2[...].sum()          (ivf.py:89, 135): pairwise
//     sum over n, evaluated as the same tree (leaves in parallel, then one combine pass);
//   * the D^2 draw           searchsorted(cumsum(best), r, 'right') (ivf.py:95): decided
//     from a parallel prefix with a rigorous error bound, falling back to the exact
//     sequential cumsum when the bound cannot separate the crossing;
//   * cluster means          data64[members].mean(axis=0)      (ivf.py:131-133): sequential
//     column sums in ascending member order, divided by the count.
// Lloyd assignment distances (ivf.py:68-73) go through a BLAS GEMM in the reference, whose
// summation order is not specified; here they are fused fp64 FMA tiles with the same
// (|x|^2 - 2 x.c) + |c|^2 form, clamp at zero and first-minimum argmin.
#include <algorithm>
#include <map>
#include <mutex>

#include "fb_internal.cuh"

namespace fb {
namespace {

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

int grid_of(int64_t work, int block) {
  int64_t g = (work + block - 1) / block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148LL * 32));
}

// numpy pairwise sum of f(i), i in [lo, lo + n) (numpy's pairwise_sum in loops_utils.h.src)
template <class F>
__device__ double pairwise_gen(const F& f, int64_t lo, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = f(lo + j);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(lo + i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, f(lo + i));
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_gen(f, lo, n2), pairwise_gen(f, lo + n2, n - n2));
}

// ---- D^2 seeding distances -----------------------------------------------------------
// 8 <= dim <= 128, dim % 8 == 0: a group of 8 lanes per point, lane j owning numpy's partial
// sum j (elements j, j + 8, ...); the combine tree is three xor-shuffles (IEEE addition
// commutes, so both partners compute the same pair sum).
__global__ void k_min_sqdist_g8(const double* __restrict__ x, int64_t n, int dim, int64_t crow,
                                double* __restrict__ best, int init) {
  const int lane8 = threadIdx.x & 7;
  const int m8 = dim >> 3;
  double cv[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) cv[m] = m < m8 ? x[crow * dim + lane8 + 8 * m] : 0.0;
  const int64_t warps = gstride() >> 5;
  for (int64_t base = (gtid() >> 5) * 4; base < n; base += warps * 4) {
    const int64_t i = base + ((threadIdx.x & 31) >> 3);
    const bool ok = i < n;
    const double* row = x + (ok ? i : 0) * dim + lane8;
    double r;
    {
      const double d = __dsub_rn(row[0], cv[0]);
      r = __dmul_rn(d, d);
    }
#pragma unroll
    for (int m = 1; m < 16; ++m) {
      if (m < m8) {
        const double d = __dsub_rn(row[8 * m], cv[m]);
        r = __dadd_rn(r, __dmul_rn(d, d));
      }
    }
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (ok && lane8 == 0) {
      const double s = __dadd_rn(0.0, r);
      best[i] = init ? s : (best[i] <= s ? best[i] : s);
    }
  }
}

__global__ void k_min_sqdist_any(const double* __restrict__ x, int64_t n, int dim, int64_t crow,
                                 double* __restrict__ best, int init) {
  const double* c = x + crow * dim;
  for (int64_t i = gtid(); i < n; i += gstride()) {
    const double* row = x + i * dim;
    const double s = __dadd_rn(0.0, pairwise_gen([&](int64_t j) {
      const double d = __dsub_rn(row[j], c[j]);
      return __dmul_rn(d, d);
    }, 0, dim));
    best[i] = init ? s : (best[i] <= s ? best[i] : s);
  }
}

// ---- exact pairwise sum of n doubles --------------------------------------------------
// The recursion tree depends on n only. Node t of the deepest level D is reached by the bit
// path of t (MSB first); a leaf met at depth l is owned by the path whose low D - l bits are
// zero and stored at index t, so every node (l, j) lives at j << (D - l).
__device__ __forceinline__ bool walk(int64_t n, int D, int l, int64_t j, int64_t& start,
                                     int64_t& len, int& leaf_depth) {
  start = 0;
  len = n;
  for (int d = 0; d < l; ++d) {
    if (len <= 128) {
      leaf_depth = d;
      return false;  // an ancestor is a leaf
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((j >> (l - 1 - d)) & 1) {
      start += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  leaf_depth = len <= 128 ? l : -1;
  return true;
}

__global__ void k_pairwise_leaves(const double* __restrict__ x, int64_t n, int D,
                                  double* __restrict__ node) {
  const int64_t leaves = 1LL << D;
  for (int64_t t = gtid(); t < leaves; t += gstride()) {
    // find the leaf on t's path
    int64_t start = 0, len = n;
    int l = 0;
    while (len > 128 && l < D) {
      int64_t n2 = len / 2;
      n2 -= n2 % 8;
      if ((t >> (D - 1 - l)) & 1) {
        start += n2;
        len -= n2;
      } else {
        len = n2;
      }
      ++l;
    }
    if ((t & ((1LL << (D - l)) - 1)) != 0) continue;  // not the leaf's owner
    const double* a = x + start;
    node[t] = pairwise_gen([&](int64_t i) { return a[i]; }, 0, len);
  }
}

__global__ void k_pairwise_combine(int64_t n, int D, double* __restrict__ node,
                                   double* __restrict__ out) {
  for (int l = D - 1; l >= 0; --l) {
    for (int64_t j = threadIdx.x; j < (1LL << l); j += blockDim.x) {
      int64_t start, len;
      int ld;
      if (!walk(n, D, l, j, start, len, ld) || len <= 128) continue;  // leaf or below a leaf
      const int sh = D - l;
      node[j << sh] = __dadd_rn(node[j << sh], node[((2 * j + 1) << (sh - 1))]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = __dadd_rn(0.0, node[0]);
}

int tree_depth(int64_t len, std::map<int64_t, int>& memo) {
  if (len <= 128) return 0;
  auto it = memo.find(len);
  if (it != memo.end()) return it->second;
  int64_t n2 = len / 2;
  n2 -= n2 % 8;
  const int d = 1 + std::max(tree_depth(n2, memo), tree_depth(len - n2, memo));
  memo[len] = d;
  return d;
}

int pairwise_depth(int64_t n) {
  std::map<int64_t, int> memo;
  return tree_depth(n, memo);
}

// ---- D^2 draw: first i with cumsum(x)[i] > u * total ----------------------------------
// approx[i] is any-order prefix sum of the non-negative x; the sequential prefix c_i and
// approx[i] both lie within (n u)/(1 - n u) * S of the exact prefix, so with
// delta = 2.5 n u max(total, approx[n-1]):  approx[i] <= r - delta  =>  c_i <= r, and
// approx[i] > r + delta  =>  c_i > r.
__global__ void k_draw_init(int64_t n, unsigned long long* lo) { *lo = (unsigned long long)n; }

__device__ __forceinline__ void draw_bounds(const double* total, const double* approx, int64_t n,
                                            double u, double& r, double& delta) {
  r = __dmul_rn(u, *total);
  const double s = fmax(*total, approx[n - 1]);
  delta = 2.5 * (double)n * 0x1p-53 * s;
}

__global__ void k_draw_first_above(const double* __restrict__ approx, int64_t n,
                                   const double* __restrict__ total, double u,
                                   unsigned long long* lo) {
  double r, delta;
  draw_bounds(total, approx, n, u, r, delta);
  const double lim = r - delta;
  for (int64_t i = gtid(); i < n; i += gstride())
    if (approx[i] > lim) {
      atomicMin(lo, (unsigned long long)i);
      break;  // later i of this thread are larger
    }
}

constexpr int kSeqChunk = 2048;
__global__ void __launch_bounds__(256) k_draw_resolve(const double* __restrict__ x,
                                                      const double* __restrict__ approx, int64_t n,
                                                      const double* __restrict__ total, double u,
                                                      const unsigned long long* lo,
                                                      int64_t* __restrict__ out,
                                                      int32_t* __restrict__ exact_walks) {
  __shared__ __align__(16) double buf[2][kSeqChunk];
  __shared__ int64_t s_idx;
  __shared__ int s_found;
  double r, delta;
  draw_bounds(total, approx, n, u, r, delta);
  const int64_t l = (int64_t)*lo;
  if (l >= n) {
    if (threadIdx.x == 0) *out = n - 1;
    return;
  }
  if (approx[l] > r + delta) {
    if (threadIdx.x == 0) *out = l;
    return;
  }
  // ambiguous: thread 0 walks the exact sequential cumsum (c_0 = x_0 since x_0 >= 0) while
  // warps 1.. stage the next chunk; chunks are zero-padded (adding +0 leaves c unchanged)
  if (threadIdx.x == 0) {
    s_idx = n - 1;
    s_found = 0;
    if (exact_walks) atomicAdd(exact_walks, 1);
  }
  auto stage = [&](int64_t c0, double* dst, int t0, int nt) {
    for (int i = t0; i < kSeqChunk; i += nt) dst[i] = c0 + i < n ? x[c0 + i] : 0.0;
  };
  stage(0, buf[0], threadIdx.x, blockDim.x);
  double c = 0.0;
  int cur = 0;
  for (int64_t c0 = 0;; c0 += kSeqChunk, cur ^= 1) {
    __syncthreads();
    if (s_found || c0 >= n) break;
    if (threadIdx.x >= 32) {
      if (c0 + kSeqChunk < n) stage(c0 + kSeqChunk, buf[cur ^ 1], threadIdx.x - 32, blockDim.x - 32);
    } else if (threadIdx.x == 0) {
      const double* b = buf[cur];
      for (int i = 0; i < kSeqChunk; i += 16) {
        double v[16];
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          const double2 t = *reinterpret_cast<const double2*>(b + i + j);
          v[j] = t.x;
          v[j + 1] = t.y;
        }
        double t = c;
#pragma unroll
        for (int j = 0; j < 16; ++j) t = __dadd_rn(t, v[j]);
        if (t > r) {  // the crossing is inside this block of 16: locate it
#pragma unroll 1
          for (int j = 0; j < 16; ++j) {
            c = __dadd_rn(c, v[j]);
            if (c > r) {
              s_idx = c0 + i + j;
              break;
            }
          }
          s_found = 1;
          break;
        }
        c = t;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *out = s_idx;
}

// ---- Lloyd assignment ---------------------------------------------------------------
// 64 points x 64 centres per tile pass, 256 threads with 4 x 4 fp64 accumulators; the block's
// 64 points stay in shared memory (widened layout [dim][64]) while all centre tiles stream
// past in 16-dim slabs. Running (min, argmin) per point with strict <, centres visited in
// increasing index per thread, then a 16-way reduction preferring the lower index.
constexpr int kAsBM = 64, kAsBN = 64, kAsBK = 16, kAsPad = 65;  // padded row stride
__global__ void __launch_bounds__(256) k_assign(const double* __restrict__ x, int64_t n, int dim,
                                                const double* __restrict__ cen, int k,
                                                const double* __restrict__ xx,
                                                const double* __restrict__ cc,
                                                int64_t* __restrict__ assign,
                                                double* __restrict__ mind2) {
  extern __shared__ double s_as[];
  double* Xs = s_as;                      // [dim][kAsPad]
  double* Cs = Xs + (size_t)dim * kAsPad;  // [kAsBK][kAsPad]
  double* Rv = Cs + kAsBK * kAsPad;        // [kAsBM][16]
  int* Ri = reinterpret_cast<int*>(Rv + kAsBM * 16);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t p0 = (int64_t)blockIdx.x * kAsBM;
  for (int e = tid; e < kAsBM * dim; e += 256) {
    const int p = e / dim, d = e - p * dim;
    Xs[d * kAsPad + p] = p0 + p < n ? x[(p0 + p) * dim + d] : 0.0;
  }
  double xv[4], bv[4];
  int bi[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t p = p0 + ty + 16 * i;
    xv[i] = p < n ? xx[p] : 0.0;
    bv[i] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    bi[i] = 0;
  }
  for (int c0 = 0; c0 < k; c0 += kAsBN) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < dim; k0 += kAsBK) {
      __syncthreads();
      for (int e = tid; e < kAsBK * kAsBN; e += 256) {
        const int c = e / kAsBK, d = e - c * kAsBK;
        Cs[d * kAsPad + c] = (c0 + c < k && k0 + d < dim) ? cen[(int64_t)(c0 + c) * dim + k0 + d] : 0.0;
      }
      __syncthreads();
      const int kk_end = min(kAsBK, dim - k0);
      for (int kk = 0; kk < kk_end; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = Xs[(k0 + kk) * kAsPad + ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Cs[kk * kAsPad + tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx + 16 * j;
      if (c < k) {
        const double cj = cc[c];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          double d2 = __dadd_rn(__dsub_rn(xv[i], __dmul_rn(2.0, acc[i][j])), cj);
          d2 = d2 > 0.0 ? d2 : 0.0;
          if (d2 < bv[i]) {
            bv[i] = d2;
            bi[i] = c;
          }
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    Rv[(ty + 16 * i) * 16 + tx] = bv[i];
    Ri[(ty + 16 * i) * 16 + tx] = bi[i];
  }
  __syncthreads();
  if (tid < kAsBM && p0 + tid < n) {
    double v = Rv[tid * 16];
    int b = Ri[tid * 16];
    for (int t = 1; t < 16; ++t) {
      const double w = Rv[tid * 16 + t];
      const int c = Ri[tid * 16 + t];
      if (w < v || (w == v && c < b)) {
        v = w;
        b = c;
      }
    }
    assign[p0 + tid] = b;
    mind2[p0 + tid] = v;
  }
}

// |row|^2 in numpy's pairwise order (stands in for einsum("ij,ij->i"), ivf.py:70-72)
__global__ void k_row_sqnorm(const double* __restrict__ x, int64_t n, int dim,
                             double* __restrict__ out) {
  for (int64_t i = gtid(); i < n; i += gstride()) {
    const double* row = x + i * dim;
    out[i] = __dadd_rn(0.0, pairwise_gen([&](int64_t j) { return __dmul_rn(row[j], row[j]); }, 0, dim));
  }
}

// ---- cluster means: thread per (cluster, column), members in ascending index ----------
__global__ void k_means(const double* __restrict__ x, int dim, const int64_t* __restrict__ order,
                        const int64_t* __restrict__ seg_start, const int64_t* __restrict__ seg_count,
                        int k, double* __restrict__ cen) {
  const int64_t total = (int64_t)k * dim;
  for (int64_t e = gtid(); e < total; e += gstride()) {
    const int c = (int)(e / dim), d = (int)(e - (int64_t)c * dim);
    const int64_t s = seg_start[c], m = seg_count[c];
    double acc = 0.0;
    int64_t i = 0;
    for (; i + 4 <= m; i += 4) {  // loads ahead of the dependent additions
      const double v0 = x[order[s + i] * dim + d], v1 = x[order[s + i + 1] * dim + d];
      const double v2 = x[order[s + i + 2] * dim + d], v3 = x[order[s + i + 3] * dim + d];
      acc = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(acc, v0), v1), v2), v3);
    }
    for (; i < m; ++i) acc = __dadd_rn(acc, x[order[s + i] * dim + d]);
    cen[(int64_t)c * dim + d] = __ddiv_rn(acc, (double)m);
  }
}

}  // namespace
}  // namespace fb

using namespace fb;

extern "C" {

int fb_kmeans_min_sqdist(const double* data, int64_t n, int32_t dim, int64_t center_row,
                         double* best, int32_t init, void* stream) {
  if (n < 0 || dim <= 0) return fail(FB_ERR_INVALID, "bad shape");
  if (center_row < 0 || center_row >= n) return fail(FB_ERR_INVALID, "center row out of range");
  if (n == 0) return FB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dim % 8 == 0 && dim <= 128) {
    k_min_sqdist_g8<<<grid_of((n + 3) / 4 * 32, 256), 256, 0, s>>>(data, n, dim, center_row, best,
                                                                   init);
    FB_LAUNCH_CHECK("k_min_sqdist_g8");
  } else {
    k_min_sqdist_any<<<grid_of(n, 128), 128, 0, s>>>(data, n, dim, center_row, best, init);
    FB_LAUNCH_CHECK("k_min_sqdist_any");
  }
  return FB_OK;
}

int64_t fb_pairwise_sum_scratch(int64_t n) { return n < 0 ? 0 : (1LL << pairwise_depth(n)); }

int fb_pairwise_sum_f64(const double* x, int64_t n, double* out, double* scratch,
                        int64_t scratch_len, void* stream) {
  if (n < 0) return fail(FB_ERR_INVALID, "n < 0");
  const int D = pairwise_depth(n);
  if (scratch_len < (1LL << D)) return fail(FB_ERR_INVALID, "scratch too small");
  if (D > 40) return fail(FB_ERR_INVALID, "n too large");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  k_pairwise_leaves<<<grid_of(1LL << D, 256), 256, 0, s>>>(x, n, D, scratch);
  FB_LAUNCH_CHECK("k_pairwise_leaves");
  k_pairwise_combine<<<1, 1024, 0, s>>>(n, D, scratch, out);
  FB_LAUNCH_CHECK("k_pairwise_combine");
  return FB_OK;
}

int fb_kmeans_draw(const double* best, const double* approx_prefix, int64_t n,
                   const double* total, double u, int64_t* out_idx, uint64_t* scratch,
                   int32_t* exact_walks, void* stream) {
  if (n <= 0) return fail(FB_ERR_INVALID, "n <= 0");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* lo = reinterpret_cast<unsigned long long*>(scratch);
  k_draw_init<<<1, 1, 0, s>>>(n, lo);
  FB_LAUNCH_CHECK("k_draw_init");
  k_draw_first_above<<<grid_of(n, 256), 256, 0, s>>>(approx_prefix, n, total, u, lo);
  FB_LAUNCH_CHECK("k_draw_first_above");
  k_draw_resolve<<<1, 256, 0, s>>>(best, approx_prefix, n, total, u, lo, out_idx, exact_walks);
  FB_LAUNCH_CHECK("k_draw_resolve");
  return FB_OK;
}

int fb_row_sqnorm_f64(const double* x, int64_t n, int32_t dim, double* out, void* stream) {
  if (n < 0 || dim <= 0) return fail(FB_ERR_INVALID, "bad shape");
  if (n == 0) return FB_OK;
  k_row_sqnorm<<<grid_of(n, 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(x, n, dim, out);
  FB_LAUNCH_CHECK("k_row_sqnorm");
  return FB_OK;
}

int fb_kmeans_assign(const double* data, int64_t n, int32_t dim, const double* centers, int32_t k,
                     const double* data_sq, const double* center_sq, int64_t* assign,
                     double* min_d2, void* stream) {
  if (n < 0 || dim <= 0 || k <= 0) return fail(FB_ERR_INVALID, "bad shape");
  if (n == 0) return FB_OK;
  const size_t smem = ((size_t)dim * kAsPad + kAsBK * kAsPad + kAsBM * 16) * sizeof(double) +
                      kAsBM * 16 * sizeof(int);
  if (smem > 227 * 1024) return fail(FB_ERR_UNSUPPORTED, "dim too large for the assignment tile");
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  const int64_t blocks = (n + kAsBM - 1) / kAsBM;
  if (blocks > 0x7fffffffLL) return fail(FB_ERR_INVALID, "n too large");
  k_assign<<<(unsigned)blocks, 256, smem, static_cast<cudaStream_t>(stream)>>>(
      data, n, dim, centers, k, data_sq, center_sq, assign, min_d2);
  FB_LAUNCH_CHECK("k_assign");
  return FB_OK;
}

int fb_kmeans_means(const double* data, int32_t dim, const int64_t* order,
                    const int64_t* seg_start, const int64_t* seg_count, int32_t k,
                    double* centers, void* stream) {
  if (dim <= 0 || k < 0) return fail(FB_ERR_INVALID, "bad shape");
  if (k == 0) return FB_OK;
  k_means<<<grid_of((int64_t)k * dim, 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(
      data, dim, order, seg_start, seg_count, k, centers);
  FB_LAUNCH_CHECK("k_means");
  return FB_OK;
}

}  // extern "C"
