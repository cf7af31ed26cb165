// Host half of the hot path in C++: filter text / postfix programs -> the batch device form
// (fb_filter_prog_t arrays) that fb_filter_eval and fb_topk_execute consume.
//
// Replaces, for a whole query batch, reference filter_query.parse_filter
// (filter_query.py:82-189, the text grammar), compile_filter (filter_query.py:280-311:
// post-order lowering, per-(fid, value) leaf de-duplication, hash_positions per leaf) and
// this package's FilterBatch.pack (the cross-query leaf table, register-machine lowering,
// CNF detection and feature-binned column windows). The output is byte-identical to the
// Python FilterBatch.pack of the same compiled filters (tests/test_pack_cpu.py).
//
// Errors: a text this parser does not accept (syntax, unknown names, non-ASCII input,
// integers beyond u64) is reported as FB_ERR_PARSE with the query index; the Python
// wrapper re-runs the reference-grammar parser on that one text to raise the reference's
// exception (FilterSyntaxError / UnknownFeature / UnknownValue) with its exact message.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <array>
#include <memory>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

#include <pthread.h>
#include <string>
#include <unordered_map>
#include <vector>

#include "fb_internal.cuh"

struct fb_vocab {
  std::unordered_map<std::string, uint64_t> feat, vals;
};

struct fb_pack {
  int64_t meta[FB_PACK_META_N];
  std::vector<int32_t> leaf_pos, op_offset, plane_list, rop_offset, qgroups;
  std::vector<uint16_t> ops, rops;
  std::vector<int16_t> leaf_slot, col_leaf;
  std::vector<uint32_t> qmask;
  std::vector<int64_t> push_bits;
  std::vector<uint64_t> leaf_fid, leaf_val;
};

namespace fb {
namespace {

// A small persistent worker pool for the per-query host work (parsing a batch of filter
// texts): threads are started once, a call splits [0, n) into one contiguous chunk per
// thread and the caller works on chunk 0. FB_PACK_THREADS caps the count (1 = serial).
class Pool {
 public:
  static Pool& get() {
    // never destroyed (no joins at process exit); a forked child has no workers, so it
    // runs every call serially
    static Pool* p = [] {
      pthread_atfork(nullptr, nullptr, [] { forked_child() = true; });
      return new Pool;
    }();
    return *p;
  }
  int size() const { return forked_child() ? 1 : (int)workers_.size() + 1; }
  void run(int n, const std::function<void(int, int)>& fn) {
    const int T = std::min(size(), std::max(1, n / 16));
    if (T <= 1) {
      fn(0, n);
      return;
    }
    std::unique_lock<std::mutex> lk(call_mu_);  // one parallel call at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      n_ = n;
      chunks_ = T;
      pending_ = T - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0, n / T);
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() {
    // four threads by default: the serving loop's other host threads (the Python driver,
    // the copy stream's callbacks) share the cores, and waking more workers per batch cost
    // more than it saved (fresh-filter e2e on the GPU box: 4 threads 179-190k q/s, 16: 170-173k)
    int t = std::min(4, (int)std::thread::hardware_concurrency());
    if (const char* e = getenv("FB_PACK_THREADS")) t = atoi(e);
    t = std::max(1, std::min(t, 16));
    for (int i = 1; i < t; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  static bool& forked_child() {
    static bool f = false;
    return f;
  }
  void loop(int id) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int, int)>* fn;
      int n, chunks;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        fn = fn_;
        n = n_;
        chunks = chunks_;
      }
      if (id < chunks) {
        (*fn)((int)((int64_t)n * id / chunks), (int)((int64_t)n * (id + 1) / chunks));
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int, int)>* fn_ = nullptr;
  int n_ = 0, chunks_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// ---- per-(fid, value, M, K) leaf position cache ------------------------------------------
struct PosKey {
  uint64_t fid, val;
  int32_t m, k;
  bool operator==(const PosKey& o) const {
    return fid == o.fid && val == o.val && m == o.m && k == o.k;
  }
};
struct PosKeyHash {
  size_t operator()(const PosKey& p) const {
    return (size_t)splitmix64(splitmix64(p.fid) ^ p.val ^
                              ((uint64_t)(uint32_t)p.m << 32 | (uint32_t)p.k) * 0x9E3779B97F4A7C15ull);
  }
};
struct Positions {
  int32_t n;
  int32_t p[FB_MAX_K_HASHES];
};
constexpr size_t kPosCacheMax = 1u << 20;
std::mutex g_pos_mu;
std::unordered_map<PosKey, Positions, PosKeyHash>* g_pos = nullptr;

// positions of many leaves under one lock (computed on a miss)
void lookup_positions(const uint64_t* fid, const uint64_t* val, size_t n, int m, int k,
                      std::vector<Positions>& out) {
  out.resize(n);
  std::lock_guard<std::mutex> g(g_pos_mu);
  if (g_pos == nullptr) g_pos = new std::unordered_map<PosKey, Positions, PosKeyHash>();
  if (g_pos->size() + n > kPosCacheMax) g_pos->clear();
  for (size_t i = 0; i < n; ++i) {
    const PosKey key{fid[i], val[i], m, k};
    auto it = g_pos->find(key);
    if (it == g_pos->end()) {
      Positions ps;
      ps.n = leaf_positions(fid[i], val[i], m, k, ps.p);
      it = g_pos->emplace(key, ps).first;
    }
    out[i] = it->second;
  }
}

// ---- one query's postfix program ---------------------------------------------------------
struct Op {
  uint8_t code;       // FB_OP_*
  uint64_t fid, val;  // PUSH_LEAF operand
  const int32_t* xpos = nullptr;  // explicit positions (CompiledFilter leaves); null: hash
  int32_t nxpos = 0;
};

// ---- text grammar (reference filter_query.py:82-189) --------------------------------------
enum Tok { T_LPAR, T_RPAR, T_EQ, T_STR, T_INT, T_IDENT, T_AND, T_OR, T_NOT, T_EOF };
struct Token {
  Tok kind;
  const char* s;
  size_t n;
};

bool is_ws(unsigned char c) {
  return c == ' ' || (c >= '\t' && c <= '\r') || (c >= 0x1c && c <= 0x1f);
}
bool is_ident0(unsigned char c) { return (c >= 'A' && c <= 'Z') || (c >= 'a' && c <= 'z') || c == '_'; }
bool is_digit(unsigned char c) { return c >= '0' && c <= '9'; }

bool kw_eq(const char* s, size_t n, const char* kw) {
  if (strlen(kw) != n) return false;
  for (size_t i = 0; i < n; ++i)
    if ((s[i] & ~0x20) != kw[i]) return false;
  return true;
}

// false on any input the reference tokenizer would reject or that needs Unicode semantics
bool tokenize(const char* t, std::vector<Token>& toks) {
  toks.clear();
  size_t i = 0;
  const size_t n = strlen(t);
  while (i < n) {
    const unsigned char c = (unsigned char)t[i];
    if (c >= 0x80) return false;  // Unicode \s / \d classes: the Python parser decides
    if (is_ws(c)) {
      ++i;
      continue;
    }
    if (c == '(') {
      toks.push_back({T_LPAR, t + i, 1});
      ++i;
    } else if (c == ')') {
      toks.push_back({T_RPAR, t + i, 1});
      ++i;
    } else if (c == '=') {
      toks.push_back({T_EQ, t + i, 1});
      ++i;
    } else if (c == '"') {
      size_t j = i + 1;
      while (j < n && t[j] != '"') {
        if ((unsigned char)t[j] >= 0x80) return false;
        ++j;
      }
      if (j >= n) return false;  // unterminated string
      toks.push_back({T_STR, t + i + 1, j - i - 1});
      i = j + 1;
    } else if (is_digit(c)) {
      size_t j = i;
      while (j < n && is_digit((unsigned char)t[j])) ++j;
      toks.push_back({T_INT, t + i, j - i});
      i = j;
    } else if (is_ident0(c)) {
      size_t j = i + 1;
      while (j < n && (is_ident0((unsigned char)t[j]) || is_digit((unsigned char)t[j]) || t[j] == '.'))
        ++j;
      Tok k = T_IDENT;
      if (kw_eq(t + i, j - i, "AND")) k = T_AND;
      else if (kw_eq(t + i, j - i, "OR")) k = T_OR;
      else if (kw_eq(t + i, j - i, "NOT")) k = T_NOT;
      toks.push_back({k, t + i, j - i});
      i = j;
    } else {
      return false;
    }
  }
  toks.push_back({T_EOF, t + n, 0});
  return true;
}

bool parse_u64(const char* s, size_t n, uint64_t& v) {
  v = 0;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t d = (uint64_t)(s[i] - '0');
    if (v > (UINT64_MAX - d) / 10) return false;  // beyond u64: to_bytes(8) would raise
    v = v * 10 + d;
  }
  return true;
}

// Recursive descent emitting postfix directly: And/Or children fold left exactly as
// compile_filter's emit (filter_query.py:292-300) lowers the parser's n-ary nodes.
struct Parser {
  const std::vector<Token>& tk;
  const fb_vocab* vocab;
  std::vector<Op>& out;
  size_t i = 0;
  int depth = 0;
  bool expr() {
    if (++depth > 2000) return false;
    if (!or_term()) return false;
    while (tk[i].kind == T_AND) {
      ++i;
      if (!or_term()) return false;
      out.push_back({FB_OP_AND, 0, 0});
    }
    --depth;
    return true;
  }
  bool or_term() {
    if (!factor()) return false;
    while (tk[i].kind == T_OR) {
      ++i;
      if (!factor()) return false;
      out.push_back({FB_OP_OR, 0, 0});
    }
    return true;
  }
  bool factor() {
    if (tk[i].kind == T_NOT) {
      ++i;
      if (++depth > 2000) return false;
      if (!factor()) return false;
      --depth;
      out.push_back({FB_OP_NOT, 0, 0});
      return true;
    }
    if (tk[i].kind == T_LPAR) {
      ++i;
      if (!expr()) return false;
      if (tk[i].kind != T_RPAR) return false;
      ++i;
      return true;
    }
    return leaf();
  }
  bool leaf() {
    const Token& f = tk[i++];
    uint64_t fid, val;
    if (f.kind == T_IDENT) {
      if (vocab == nullptr) return false;
      auto it = vocab->feat.find(std::string(f.s, f.n));
      if (it == vocab->feat.end()) return false;
      fid = it->second;
    } else if (f.kind == T_INT) {
      if (!parse_u64(f.s, f.n, fid)) return false;
    } else {
      return false;
    }
    if (tk[i++].kind != T_EQ) return false;
    const Token& v = tk[i++];
    if (v.kind == T_STR) {
      if (vocab == nullptr) return false;
      auto it = vocab->vals.find(std::string(v.s, v.n));
      if (it == vocab->vals.end()) return false;
      val = it->second;
    } else if (v.kind == T_INT) {
      if (!parse_u64(v.s, v.n, val)) return false;
    } else {
      return false;
    }
    out.push_back({FB_OP_PUSH_LEAF, fid, val});
    return true;
  }
};

bool parse_text(const char* text, const fb_vocab* vocab, std::vector<Op>& out) {
  thread_local std::vector<Token> toks;
  out.clear();
  if (!tokenize(text, toks)) return false;
  Parser p{toks, vocab, out};
  if (!p.expr()) return false;
  return toks[p.i].kind == T_EOF;
}

// ---- CNF of a postfix program over global leaves -----------------------------------------
// Same result as pushing NOTs to the literals (De Morgan), flattening same-operator chains
// and requiring an AND of ORs of literals, but on flat per-op arrays: every node's NOT
// parity is known top-down, so its effective operator is AND/OR swapped under odd parity;
// the groups are the maximal non-AND subtrees below the root's AND region, in DFS order
// (= order of their first push), each of which must contain no effective AND.
using Lit = std::pair<int32_t, bool>;  // (global leaf, negated)

struct CnfScratch {
  std::vector<int32_t> st, left, right, parity, eff, grp, gid;
};

// The batch's CNF, flat: query q's groups are [qstart[q], qstart[q+1]), group g's literals
// lits[gstart[g] .. gstart[g+1]) (a group's literals are contiguous in push order).
struct Cnf {
  std::vector<Lit> lits;
  std::vector<int32_t> gstart, qstart;
  int groups(int q) const { return qstart[q + 1] - qstart[q]; }
};

// appends query's groups to c (the caller closes the query with qstart.push_back)
bool cnf_groups(const std::vector<std::pair<uint8_t, int32_t>>& ops, Cnf& c, CnfScratch& w) {
  const int n = (int)ops.size();
  if (n == 0) return false;
  w.st.clear();
  w.left.assign(n, -1);
  w.right.assign(n, -1);
  for (int i = 0; i < n; ++i) {
    const uint8_t c = ops[i].first;
    if (c == FB_OP_NOT) {
      if (w.st.empty()) return false;
      w.left[i] = w.st.back();
      w.st.back() = i;
    } else if (c == FB_OP_AND || c == FB_OP_OR) {
      if (w.st.size() < 2) return false;
      w.right[i] = w.st.back();
      w.st.pop_back();
      w.left[i] = w.st.back();
      w.st.back() = i;
    } else {
      w.st.push_back(i);
    }
  }
  if (w.st.size() != 1) return false;
  const int root = w.st[0];
  // NOT parity, top-down (a parent follows its children in postfix order)
  w.parity.assign(n, 0);
  for (int i = n - 1; i >= 0; --i) {
    const int p = w.parity[i] ^ (ops[i].first == FB_OP_NOT ? 1 : 0);
    if (w.left[i] >= 0) w.parity[w.left[i]] = p;
    if (w.right[i] >= 0) w.parity[w.right[i]] = p;
  }
  // effective operator, bottom-up (0 literal, 2 AND, 3 OR; a NOT takes its operand's)
  w.eff.assign(n, 0);
  for (int i = 0; i < n; ++i) {
    const uint8_t c = ops[i].first;
    if (c == FB_OP_NOT) w.eff[i] = w.eff[w.left[i]];
    else if (c == FB_OP_AND || c == FB_OP_OR)
      w.eff[i] = ((c == FB_OP_AND) != (w.parity[i] != 0)) ? 2 : 3;
  }
  // region labels, top-down: -1 = root AND region, else the node index of the group root
  w.grp.assign(n, -2);
  w.grp[root] = w.eff[root] == 2 ? -1 : root;
  for (int i = n - 1; i >= 0; --i) {
    const int g = w.grp[i];
    for (const int c : {w.left[i], w.right[i]}) {
      if (c < 0) continue;
      if (g == -1) {
        w.grp[c] = w.eff[c] == 2 ? -1 : c;
      } else {
        if (w.eff[c] == 2) return false;  // an AND inside an OR clause
        w.grp[c] = g;
      }
    }
  }
  // groups in order of their first literal; literals in push order
  int last = -2;
  for (int i = 0; i < n; ++i) {
    if (ops[i].first != FB_OP_PUSH_LEAF) continue;
    if (w.grp[i] != last) {
      last = w.grp[i];
      c.gstart.push_back((int32_t)c.lits.size());
    }
    c.lits.push_back({ops[i].second, w.parity[i] != 0});
  }
  return true;
}

constexpr int kCnfMaxWords = 8;
constexpr int kCnfMaxGroups = 8;
constexpr int kRopMaxLeaves = 1 << 13;

// FilterBatch._pack_cnf: literal columns binned by feature into 64-column windows
bool pack_cnf(const Cnf& cnf, int nq, const std::vector<uint64_t>& leaf_fid, fb_pack& P) {
  std::vector<Lit> lits;
  std::vector<int> lit_idx(2 * leaf_fid.size() + 2, -1);  // (leaf, negated) -> literal
  auto slot = [](const Lit& l) { return 2 * (size_t)l.first + (l.second ? 1 : 0); };
  int gmax = 0;
  for (int q = 0; q < nq; ++q) gmax = std::max(gmax, cnf.groups(q));
  for (const Lit& l : cnf.lits)
    if (lit_idx[slot(l)] < 0) {
      lit_idx[slot(l)] = (int)lits.size();
      lits.push_back(l);
    }
  if (gmax > kCnfMaxGroups) return false;
  // features in first-seen order, each with its literals in literal order
  std::vector<uint64_t> fids;
  std::unordered_map<uint64_t, std::vector<int>> by_fid;
  for (int i = 0; i < (int)lits.size(); ++i) {
    const uint64_t f = leaf_fid[lits[i].first];
    auto it = by_fid.find(f);
    if (it == by_fid.end()) {
      fids.push_back(f);
      it = by_fid.emplace(f, std::vector<int>()).first;
    }
    it->second.push_back(i);
  }
  std::vector<std::vector<int>> bins;
  bool small = true;
  for (uint64_t f : fids) small &= by_fid[f].size() <= 64;
  if (small) {
    std::vector<uint64_t> order = fids;
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
      const size_t na = by_fid[a].size(), nb = by_fid[b].size();
      return na != nb ? na > nb : a < b;
    });
    for (uint64_t f : order) {
      const auto& v = by_fid[f];
      bool placed = false;
      for (auto& b : bins)
        if (b.size() + v.size() <= 64) {
          b.insert(b.end(), v.begin(), v.end());
          placed = true;
          break;
        }
      if (!placed) bins.push_back(v);
    }
  }
  std::vector<int> col(lits.size());
  int n_cols;
  if (!bins.empty() && 2 * (int)bins.size() <= kCnfMaxWords) {
    for (int bi = 0; bi < (int)bins.size(); ++bi)
      for (int i = 0; i < (int)bins[bi].size(); ++i) col[bins[bi][i]] = 64 * bi + i;
    n_cols = 64 * ((int)bins.size() - 1) + (int)bins.back().size();
  } else {
    for (int i = 0; i < (int)lits.size(); ++i) col[i] = i;
    n_cols = (int)lits.size();
  }
  const int words = (n_cols + 31) / 32;
  if (words > kCnfMaxWords) return false;
  P.qmask.assign((size_t)nq * gmax * words, 0u);
  for (int q = 0; q < nq; ++q)
    for (int gi = 0; gi < cnf.groups(q); ++gi) {
      const int g = cnf.qstart[q] + gi;
      for (int j = cnf.gstart[g]; j < cnf.gstart[g + 1]; ++j) {
        const int c = col[lit_idx[slot(cnf.lits[j])]];
        P.qmask[((size_t)q * gmax + gi) * words + (c >> 5)] |= 1u << (c & 31);
      }
    }
  P.col_leaf.assign(n_cols, 0);
  for (int i = 0; i < (int)lits.size(); ++i)
    P.col_leaf[col[i]] = (int16_t)(lits[i].second ? ~lits[i].first : lits[i].first);
  bool windowed = gmax <= 4;
  for (int q = 0; q < nq && windowed; ++q)
    for (int g = 0; g < gmax && windowed; ++g) {
      const uint32_t* m = &P.qmask[((size_t)q * gmax + g) * words];
      int first = -1, last = -1;
      for (int w = 0; w < words; ++w)
        if (m[w]) {
          if (first < 0) first = w;
          last = w;
        }
      if (first < 0) first = last = 0;
      windowed = (first >> 1) == (last >> 1);
    }
  P.qgroups.resize(nq);
  for (int q = 0; q < nq; ++q) P.qgroups[q] = (int32_t)cnf.groups(q);
  P.meta[FB_PACK_IS_CNF] = 1;
  P.meta[FB_PACK_N_COLS] = n_cols;
  P.meta[FB_PACK_CNF_WORDS] = words;
  P.meta[FB_PACK_CNF_GMAX] = gmax;
  P.meta[FB_PACK_CNF_WINDOWED] = windowed ? 1 : 0;
  return true;
}

// lower_to_register_ops: PUSH l; AND -> ANDL l, PUSH l; OR -> ORL l, PUSH l; NOT -> PUSHN l
int lower_rops(const std::vector<std::pair<uint8_t, int32_t>>& ops, std::vector<uint16_t>& out,
               std::vector<std::pair<int, int32_t>>& r) {
  r.clear();
  for (const auto& o : ops) {
    if (o.first == FB_OP_PUSH_LEAF) {
      r.push_back({FB_ROP_PUSH, o.second});
    } else if (o.first == FB_OP_NOT) {
      if (!r.empty() && r.back().first == FB_ROP_PUSH) r.back().first = FB_ROP_PUSHN;
      else r.push_back({FB_ROP_NOT, 0});
    } else {
      const bool a = o.first == FB_OP_AND;
      if (!r.empty() && r.back().first == FB_ROP_PUSH && r.size() >= 2)
        r.back().first = a ? FB_ROP_ANDL : FB_ROP_ORL;
      else
        r.push_back({a ? FB_ROP_ANDS : FB_ROP_ORS, 0});
    }
  }
  int depth = 0, peak = 0;
  for (const auto& x : r) {
    if (x.first == FB_ROP_PUSH || x.first == FB_ROP_PUSHN) ++depth;
    else if (x.first == FB_ROP_ANDS || x.first == FB_ROP_ORS) --depth;
    peak = std::max(peak, depth);
  }
  for (const auto& x : r) out.push_back((uint16_t)((x.first << 13) | (x.second & 0x1FFF)));
  while (out.size() % FB_ROP_ALIGN) out.push_back((uint16_t)(FB_ROP_NOP << 13));
  return peak;
}

// The batch form of programs[q] (empty = unfiltered).
int pack_programs(const std::vector<std::vector<Op>>& progs, const std::vector<char>& filtered,
                  int32_t m_bits, int32_t k_hashes, fb_pack& P) {
  auto TT0 = std::chrono::steady_clock::now();
  const int nq = (int)progs.size();
  memset(P.meta, 0, sizeof(P.meta));
  P.meta[FB_PACK_N_QUERIES] = nq;
  // global leaves in order of first push across the batch
  std::vector<std::pair<const int32_t*, int32_t>> leaf_x;  // first push's explicit positions
  // open-addressing (fid, value) -> global leaf table, grown at half load
  std::vector<int32_t> tab(1024, -1);
  size_t tmask = tab.size() - 1;
  auto slot_of = [&](uint64_t f, uint64_t v) -> int32_t& {
    size_t h = (size_t)splitmix64(splitmix64(f) ^ v) & tmask;
    while (tab[h] >= 0 && !(P.leaf_fid[tab[h]] == f && P.leaf_val[tab[h]] == v)) h = (h + 1) & tmask;
    return tab[h];
  };
  P.op_offset.assign(1, 0);
  P.rop_offset.assign(1, 0);
  P.push_bits.assign(nq, 0);
  std::vector<std::vector<std::pair<uint8_t, int32_t>>> gops(nq);
  int max_stack = 1;
  for (int q = 0; q < nq; ++q) {
    if (filtered[q]) {
      gops[q].reserve(progs[q].size());
      int depth = 0, peak = 0;
      for (const Op& o : progs[q]) {
        if (o.code == FB_OP_PUSH_LEAF) {
          int32_t& e = slot_of(o.fid, o.val);
          int32_t g = e;
          if (g < 0) {
            g = e = (int32_t)P.leaf_fid.size();
            P.leaf_fid.push_back(o.fid);
            P.leaf_val.push_back(o.val);
            leaf_x.push_back({o.xpos, o.nxpos});
            if (2 * P.leaf_fid.size() > tab.size()) {  // rehash
              tab.assign(tab.size() * 2, -1);
              tmask = tab.size() - 1;
              for (int32_t j = 0; j < (int32_t)P.leaf_fid.size(); ++j)
                slot_of(P.leaf_fid[j], P.leaf_val[j]) = j;
            }
          }
          gops[q].push_back({FB_OP_PUSH_LEAF, g});
          ++depth;
        } else if (o.code == FB_OP_AND || o.code == FB_OP_OR) {
          gops[q].push_back({o.code, 0});
          --depth;
        } else if (o.code == FB_OP_NOT) {
          gops[q].push_back({FB_OP_NOT, 0});
        } else {
          return fail(FB_ERR_INVALID, "unknown filter opcode");
        }
        if (depth < 1) return fail(FB_ERR_INVALID, "unbalanced operation array (stack underflow)");
        peak = std::max(peak, depth);
      }
      if (depth != 1)
        return fail(FB_ERR_INVALID,
                    "unbalanced operation array (net depth " + std::to_string(depth) + ")");
      max_stack = std::max(max_stack, peak);
    }
  }
  auto TT1 = std::chrono::steady_clock::now();
  const int n_leaves = (int)P.leaf_fid.size();
  if (n_leaves > FB_MAX_LEAVES)
    return fail(FB_ERR_UNSUPPORTED,
                "more than " + std::to_string(FB_MAX_LEAVES) + " distinct leaves in a batch");
  if (max_stack > FB_MAX_STACK)
    return fail(FB_ERR_UNSUPPORTED, "filter stack depth " + std::to_string(max_stack) + " > " +
                                        std::to_string(FB_MAX_STACK));
  // each leaf's positions, flat: the compiled filter's own (QueryBloom.set_bits) when given,
  // else hashed (cached per (fid, value, M, K))
  std::vector<Positions> hashed;
  lookup_positions(P.leaf_fid.data(), P.leaf_val.data(), (size_t)n_leaves, m_bits, k_hashes, hashed);
  std::vector<int32_t> lp_off(n_leaves + 1, 0), lp;
  lp.reserve((size_t)n_leaves * k_hashes);
  for (int i = 0; i < n_leaves; ++i) {
    if (leaf_x[i].first != nullptr) {
      for (int j = 0; j < leaf_x[i].second; ++j) {
        const int32_t v = leaf_x[i].first[j];
        if (v < 0 || v >= m_bits) return fail(FB_ERR_INVALID, "leaf position outside [0, m_bits)");
        lp.push_back(v);
      }
    } else {
      lp.insert(lp.end(), hashed[i].p, hashed[i].p + hashed[i].n);
    }
    lp_off[i + 1] = (int32_t)lp.size();
  }
  auto npos = [&](int i) { return lp_off[i + 1] - lp_off[i]; };
  auto TT2 = std::chrono::steady_clock::now();
  // postfix ops, register ops, push bits, CNF
  const bool reg = n_leaves <= kRopMaxLeaves;
  int rmax = 0;
  bool all_cnf = true;
  bool any_groups = false;
  Cnf cnf;
  cnf.qstart.push_back(0);
  CnfScratch scratch;
  std::vector<std::pair<int, int32_t>> rscratch;
  size_t total_ops = 0;
  for (int q = 0; q < nq; ++q) total_ops += gops[q].size();
  P.ops.reserve(total_ops + 1);
  P.rops.reserve(total_ops + 8 * (size_t)nq);
  // per query (in parallel on the pool): postfix ops, register ops, push bits, CNF groups;
  // then concatenated in query order (each query's register ops are padded to
  // FB_ROP_ALIGN on their own, as the serial lowering pads them in place)
  struct QOut {
    std::vector<uint16_t> ops, rops;
    int64_t bits = 0;
    int rpeak = 0;
    bool cnf_ok = false;
    Cnf cnf;
  };
  std::vector<QOut> qo(nq);
  Pool::get().run(nq, [&](int q0, int q1) {
    CnfScratch sc;
    std::vector<std::pair<int, int32_t>> rs;
    for (int q = q0; q < q1; ++q) {
      if (!filtered[q]) continue;
      QOut& o = qo[q];
      o.ops.reserve(gops[q].size());
      for (const auto& x : gops[q]) {
        if (x.first == FB_OP_PUSH_LEAF) {
          o.ops.push_back((uint16_t)x.second);
          o.bits += npos(x.second);
        } else {
          o.ops.push_back((uint16_t)(x.first << 14));
        }
      }
      o.rpeak = lower_rops(gops[q], o.rops, rs);
      o.cnf_ok = cnf_groups(gops[q], o.cnf, sc);
    }
  });
  (void)scratch;
  (void)rscratch;
  for (int q = 0; q < nq; ++q) {
    if (filtered[q]) {
      const QOut& o = qo[q];
      P.ops.insert(P.ops.end(), o.ops.begin(), o.ops.end());
      P.push_bits[q] = o.bits;
      rmax = std::max(rmax, o.rpeak);
      P.rops.insert(P.rops.end(), o.rops.begin(), o.rops.end());
      if (all_cnf) {
        if (!o.cnf_ok) {
          all_cnf = false;
        } else {
          const int32_t base = (int32_t)cnf.lits.size();
          for (const int32_t g : o.cnf.gstart) cnf.gstart.push_back(g + base);
          cnf.lits.insert(cnf.lits.end(), o.cnf.lits.begin(), o.cnf.lits.end());
        }
      }
    }
    if (all_cnf) {
      cnf.qstart.push_back((int32_t)cnf.gstart.size());
      any_groups |= cnf.groups(q) > 0;
    }
    P.op_offset.push_back((int32_t)P.ops.size());
    P.rop_offset.push_back((int32_t)P.rops.size());
  }
  auto TT3 = std::chrono::steady_clock::now();
  if (getenv("FB_PACK_TIMING"))
    fprintf(stderr, "  leaves %.3f positions %.3f lowering+cnf %.3f ms\n",
            std::chrono::duration<double, std::milli>(TT1 - TT0).count(),
            std::chrono::duration<double, std::milli>(TT2 - TT1).count(),
            std::chrono::duration<double, std::milli>(TT3 - TT2).count());
  int k_max = 1;
  for (int i = 0; i < n_leaves; ++i) k_max = std::max(k_max, npos(i));
  const int rows = std::max(1, n_leaves);
  P.leaf_pos.assign((size_t)rows * k_max, -1);
  std::vector<int32_t> planes;
  for (int i = 0; i < n_leaves; ++i)
    for (int j = 0; j < npos(i); ++j) {
      P.leaf_pos[(size_t)i * k_max + j] = lp[lp_off[i] + j];
      planes.push_back(lp[lp_off[i] + j]);
    }
  std::sort(planes.begin(), planes.end());
  planes.erase(std::unique(planes.begin(), planes.end()), planes.end());
  if (reg) {
    P.leaf_slot.assign((size_t)rows * k_max, -1);
    for (int i = 0; i < n_leaves; ++i)
      for (int j = 0; j < npos(i); ++j)
        P.leaf_slot[(size_t)i * k_max + j] = (int16_t)(
            std::lower_bound(planes.begin(), planes.end(), lp[lp_off[i] + j]) - planes.begin());
    P.plane_list = planes.empty() ? std::vector<int32_t>(1, 0) : planes;
    if (P.rops.empty())
      for (int i = 0; i < FB_ROP_ALIGN; ++i) P.rops.push_back((uint16_t)(FB_ROP_NOP << 13));
    if (all_cnf && any_groups) {
      cnf.gstart.push_back((int32_t)cnf.lits.size());
      pack_cnf(cnf, nq, P.leaf_fid, P);
    } else if (n_leaves == 0) {
      // no query is filtered: the zero-group CNF form (the scan's per-hit kernel)
      P.col_leaf.assign(1, 0);
      P.qmask.assign((size_t)nq, 0u);
      P.qgroups.assign((size_t)nq, 0);
      P.meta[FB_PACK_IS_CNF] = 1;
      P.meta[FB_PACK_N_COLS] = 1;
      P.meta[FB_PACK_CNF_WORDS] = 1;
      P.meta[FB_PACK_CNF_GMAX] = 1;
      P.meta[FB_PACK_CNF_WINDOWED] = 1;
    }
  } else {
    P.rops.clear();
    P.rop_offset.clear();
  }
  if (P.ops.empty()) P.ops.push_back(0);
  P.meta[FB_PACK_N_LEAVES] = rows;
  P.meta[FB_PACK_K_MAX] = k_max;
  P.meta[FB_PACK_MAX_STACK] = max_stack;
  P.meta[FB_PACK_HAS_ROPS] = reg ? 1 : 0;
  P.meta[FB_PACK_N_PLANES] = reg ? (int64_t)P.plane_list.size() : 0;
  P.meta[FB_PACK_RMAX_STACK] = reg ? rmax : 0;
  P.meta[FB_PACK_N_ROPS] = reg ? (int64_t)P.rops.size() : 0;
  P.meta[FB_PACK_DISTINCT_LEAVES] = n_leaves;
  P.meta[FB_PACK_DISTINCT_PLANES] = (int64_t)planes.size();
  return FB_OK;
}

}  // namespace
}  // namespace fb

extern "C" {

int fb_vocab_create(int32_t n_feat, const char* const* feat_names, const uint64_t* feat_ids,
                    int32_t n_vals, const char* const* val_names, const uint64_t* val_ids,
                    fb_vocab_t** out) {
  if (out == nullptr || n_feat < 0 || n_vals < 0) return fb::fail(FB_ERR_INVALID, "bad vocabulary");
  auto v = std::make_unique<fb_vocab>();
  for (int i = 0; i < n_feat; ++i) v->feat[feat_names[i]] = feat_ids[i];
  for (int i = 0; i < n_vals; ++i) v->vals[val_names[i]] = val_ids[i];
  *out = v.release();
  return FB_OK;
}

void fb_vocab_free(fb_vocab_t* v) { delete v; }

int fb_pack_text(int32_t n_queries, const char* const* texts, const fb_vocab_t* vocab,
                 int32_t m_bits, int32_t k_hashes, fb_pack_t** out, int32_t* bad_query) {
  if (out == nullptr || n_queries < 0) return fb::fail(FB_ERR_INVALID, "bad arguments");
  if (m_bits < 1 || k_hashes < 1) return fb::fail(FB_ERR_INVALID, "m_bits and k_hashes must be >= 1");
  if (k_hashes > FB_MAX_K_HASHES) return fb::fail(FB_ERR_UNSUPPORTED, "k_hashes > FB_MAX_K_HASHES");
  *out = nullptr;
  std::vector<std::vector<fb::Op>> progs(n_queries);
  std::vector<char> filtered(n_queries, 0);
  auto T0 = std::chrono::steady_clock::now();
  // texts parse independently: split over the pool; the first bad query is reported
  std::vector<char> bad(n_queries, 0);
  fb::Pool::get().run(n_queries, [&](int q0, int q1) {
    for (int q = q0; q < q1; ++q) {
      const char* t = texts[q];
      if (t == nullptr || t[0] == '\0') continue;
      if (!fb::parse_text(t, vocab, progs[q]))
        bad[q] = 1;
      else
        filtered[q] = 1;
    }
  });
  for (int q = 0; q < n_queries; ++q)
    if (bad[q]) {
      if (bad_query) *bad_query = q;
      return fb::fail(FB_ERR_PARSE, "filter text not accepted (query " + std::to_string(q) + ")");
    }
  auto T1 = std::chrono::steady_clock::now();
  auto P = std::make_unique<fb_pack>();
  const int rc = fb::pack_programs(progs, filtered, m_bits, k_hashes, *P);
  auto T2 = std::chrono::steady_clock::now();
  if (getenv("FB_PACK_TIMING"))
    fprintf(stderr, "parse %.3f ms pack %.3f ms\n",
            std::chrono::duration<double, std::milli>(T1 - T0).count(),
            std::chrono::duration<double, std::milli>(T2 - T1).count());
  if (rc) return rc;
  *out = P.release();
  return FB_OK;
}

int fb_pack_postfix(int32_t n_queries, const int64_t* op_offset, const uint8_t* opcode,
                    const uint64_t* fid, const uint64_t* value, const int64_t* pos_offset,
                    const int32_t* pos, int32_t m_bits, int32_t k_hashes, fb_pack_t** out) {
  if (out == nullptr || n_queries < 0 || op_offset == nullptr)
    return fb::fail(FB_ERR_INVALID, "bad arguments");
  if (m_bits < 1 || k_hashes < 1) return fb::fail(FB_ERR_INVALID, "m_bits and k_hashes must be >= 1");
  if (k_hashes > FB_MAX_K_HASHES) return fb::fail(FB_ERR_UNSUPPORTED, "k_hashes > FB_MAX_K_HASHES");
  *out = nullptr;
  std::vector<std::vector<fb::Op>> progs(n_queries);
  std::vector<char> filtered(n_queries, 0);
  auto T0 = std::chrono::steady_clock::now();
  for (int q = 0; q < n_queries; ++q) {
    const int64_t a = op_offset[q], b = op_offset[q + 1];
    if (b < a) return fb::fail(FB_ERR_INVALID, "op_offset not ascending");
    if (b == a) continue;  // unfiltered
    filtered[q] = 1;
    progs[q].reserve((size_t)(b - a));
    for (int64_t i = a; i < b; ++i) {
      fb::Op o{opcode[i], fid[i], value[i]};
      if (pos_offset != nullptr && opcode[i] == FB_OP_PUSH_LEAF) {
        o.xpos = pos + pos_offset[i];
        o.nxpos = (int32_t)(pos_offset[i + 1] - pos_offset[i]);
      }
      progs[q].push_back(o);
    }
  }
  auto P = std::make_unique<fb_pack>();
  const int rc = fb::pack_programs(progs, filtered, m_bits, k_hashes, *P);
  if (rc) return rc;
  *out = P.release();
  return FB_OK;
}

int fb_pack_meta(const fb_pack_t* p, int64_t* meta) {
  if (p == nullptr || meta == nullptr) return fb::fail(FB_ERR_INVALID, "null pack");
  memcpy(meta, p->meta, sizeof(p->meta));
  return FB_OK;
}

int fb_pack_array(const fb_pack_t* p, int32_t which, const void** data, int64_t* n_elems) {
  if (p == nullptr || data == nullptr || n_elems == nullptr)
    return fb::fail(FB_ERR_INVALID, "null pack");
  switch (which) {
#define FB_ARR(id, v)         \
  case id:                    \
    *data = p->v.data();      \
    *n_elems = (int64_t)p->v.size(); \
    return FB_OK;
    FB_ARR(FB_PACK_LEAF_POS, leaf_pos)
    FB_ARR(FB_PACK_OP_OFFSET, op_offset)
    FB_ARR(FB_PACK_OPS, ops)
    FB_ARR(FB_PACK_PLANE_LIST, plane_list)
    FB_ARR(FB_PACK_LEAF_SLOT, leaf_slot)
    FB_ARR(FB_PACK_ROP_OFFSET, rop_offset)
    FB_ARR(FB_PACK_ROPS, rops)
    FB_ARR(FB_PACK_COL_LEAF, col_leaf)
    FB_ARR(FB_PACK_QMASK, qmask)
    FB_ARR(FB_PACK_QGROUPS, qgroups)
    FB_ARR(FB_PACK_PUSH_BITS, push_bits)
    FB_ARR(FB_PACK_LEAF_FID, leaf_fid)
    FB_ARR(FB_PACK_LEAF_VAL, leaf_val)
#undef FB_ARR
    default:
      return fb::fail(FB_ERR_INVALID, "unknown pack array");
  }
}

void fb_pack_free(fb_pack_t* p) { delete p; }

}  // extern "C"
