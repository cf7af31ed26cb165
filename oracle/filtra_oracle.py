"""CPU oracle for the filtered int8 top-k hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package's hot-path
arithmetic (``/root/reference/pkg/src/filtra``; cited below as ``ref/<file>:<line>``).
It exists so that the CUDA path can be checked bit-for-bit on the GPU box, where
the reference itself is not present.

Who may import it: ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs -- and there only as the checker or
as the timed CPU baseline. The product package ``paper_2511_14881_b200`` never
imports it; it has no CPU fallback.

Parity pinning: every function here is checked against golden vectors produced
by running the real reference in the build container (``tests/golden/make_golden.py``
-> ``tests/golden/*.npz``; see ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

U64 = 0xFFFFFFFFFFFFFFFF
FNV_OFFSET = 0xCBF29CE484222325  # ref/bloom.py:21
FNV_PRIME = 0x100000001B3        # ref/bloom.py:22
GAMMA = 0x9E3779B97F4A7C15       # ref/bloom.py:62
WORD_BITS = 64                   # ref/bitset.py:10
TILE_ROWS = 4096                 # ref/ivf.py:24

OP_PUSH_LEAF, OP_AND, OP_OR, OP_NOT = 0, 1, 2, 3  # ref/filter_query.py:253-257


# --------------------------------------------------------------------------------------
# hashing (ref/bloom.py:48-88)
# --------------------------------------------------------------------------------------

def fnv1a64_pair(fid: int, value: int) -> int:
    """FNV-1a-64 over ``fid.to_bytes(8,'little') + value.to_bytes(8,'little')``
    (ref/bloom.py:48-53, 65-68)."""
    h = FNV_OFFSET
    for word in (fid, value):
        for i in range(8):
            h ^= (word >> (8 * i)) & 0xFF
            h = (h * FNV_PRIME) & U64
    return h


def splitmix64(z: int) -> int:
    """SplitMix64 finaliser (ref/bloom.py:56-59)."""
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & U64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & U64
    return (z ^ (z >> 31)) & U64


def hash_positions(fid: int, value: int, m_bits: int, k_hashes: int) -> tuple[int, ...]:
    """Sorted, de-duplicated ``splitmix64(seed ^ i*GAMMA) mod M`` (ref/bloom.py:71-88)."""
    seed = fnv1a64_pair(fid, value)
    return tuple(sorted({splitmix64(seed ^ ((i * GAMMA) & U64)) % m_bits
                         for i in range(k_hashes)}))


def _np_splitmix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def hash_positions_np(fids: np.ndarray, values: np.ndarray, m_bits: int,
                      k_hashes: int) -> np.ndarray:
    """Vectorised :func:`hash_positions`: int64 ``[n, K]``, sorted ascending per
    row, duplicates replaced by -1 and moved to the end (same set semantics as
    ref/bloom.py:82-83)."""
    fids = np.asarray(fids, dtype=np.uint64)
    values = np.asarray(values, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = np.full(fids.shape, FNV_OFFSET, dtype=np.uint64)
        for word in (fids, values):
            for i in range(8):
                h ^= (word >> np.uint64(8 * i)) & np.uint64(0xFF)
                h *= np.uint64(FNV_PRIME)
        pos = np.empty((fids.shape[0], k_hashes), dtype=np.int64)
        for i in range(k_hashes):
            z = h ^ np.uint64((i * GAMMA) & U64)
            pos[:, i] = (_np_splitmix64(z) % np.uint64(m_bits)).astype(np.int64)
    pos.sort(axis=1)
    dup = np.zeros_like(pos, dtype=bool)
    dup[:, 1:] = pos[:, 1:] == pos[:, :-1]
    pos[dup] = np.iinfo(np.int64).max
    pos.sort(axis=1)
    pos[pos == np.iinfo(np.int64).max] = -1
    return pos


# --------------------------------------------------------------------------------------
# bloom planes (ref/bloom.py:114-181)
# --------------------------------------------------------------------------------------

def n_words(n_slots: int) -> int:
    return (n_slots + WORD_BITS - 1) // WORD_BITS  # ref/bitset.py:15


def build_bloom_pairs(fids: np.ndarray, values: np.ndarray, slots: np.ndarray,
                      n_slots: int, m_bits: int, k_hashes: int) -> np.ndarray:
    """Planes ``uint64[M, ceil(n_slots/64)]``: for every (fid, value, slot) pair set
    bit ``(p, slot)`` for each hash position p (ref/bloom.py:126-143)."""
    planes = np.zeros((m_bits, n_words(n_slots)), dtype=np.uint64)
    if len(fids) == 0:
        return planes
    pos = hash_positions_np(fids, values, m_bits, k_hashes)
    slots = np.asarray(slots, dtype=np.int64)
    rows = np.repeat(slots[:, None], pos.shape[1], axis=1)
    keep = pos >= 0
    p = pos[keep]
    s = rows[keep]
    np.bitwise_or.at(planes, (p, s >> 6), np.uint64(1) << (s & 63).astype(np.uint64))
    return planes


def build_bloom(slot_features: list[list[tuple[int, int]]], m_bits: int, k_hashes: int,
                n_slots: int | None = None) -> np.ndarray:
    """List-of-pairs front end of :func:`build_bloom_pairs` (ref/bloom.py:114-125)."""
    if n_slots is None:
        n_slots = len(slot_features)
    f, v, s = [], [], []
    for slot, pairs in enumerate(slot_features):
        for fid, val in pairs:
            f.append(fid)
            v.append(val)
            s.append(slot)
    return build_bloom_pairs(np.array(f, dtype=np.uint64), np.array(v, dtype=np.uint64),
                             np.array(s, dtype=np.int64), n_slots, m_bits, k_hashes)


def bloom_eval_leaf(planes: np.ndarray, set_bits, w0: int, w1: int) -> np.ndarray:
    """AND of the selected plane rows over words [w0, w1); all-ones when the leaf
    has no positions (ref/bloom.py:170-181)."""
    if len(set_bits) == 0:
        return np.full(w1 - w0, U64, dtype=np.uint64)
    return np.bitwise_and.reduce(planes[list(set_bits), w0:w1], axis=0)


# --------------------------------------------------------------------------------------
# filter programs (ref/filter_query.py:280-356)
# --------------------------------------------------------------------------------------
# An expression is a nested tuple: ("leaf", fid, value) | ("and", [..]) | ("or", [..])
# | ("not", child). This is the JSON form the golden fixtures use.

def compile_expr(expr, m_bits: int, k_hashes: int):
    """Post-order lowering with per-(fid, value) leaf de-duplication and binary
    chaining of AND/OR children (ref/filter_query.py:280-311).

    Returns ``(ops, leaves)`` with ``ops = [(opcode, leaf_idx)]`` and
    ``leaves = [(fid, value, positions)]``.
    """
    leaf_index: dict[tuple[int, int], int] = {}
    leaves: list[tuple[int, int, tuple[int, ...]]] = []
    ops: list[tuple[int, int]] = []

    def emit(node):
        kind = node[0]
        if kind == "leaf":
            key = (int(node[1]), int(node[2]))
            idx = leaf_index.get(key)
            if idx is None:
                idx = len(leaves)
                leaf_index[key] = idx
                leaves.append((key[0], key[1], hash_positions(key[0], key[1], m_bits, k_hashes)))
            ops.append((OP_PUSH_LEAF, idx))
        elif kind == "not":
            emit(node[1])
            ops.append((OP_NOT, 0))
        elif kind in ("and", "or"):
            code = OP_AND if kind == "and" else OP_OR
            children = node[1]
            emit(children[0])
            for child in children[1:]:
                emit(child)
                ops.append((code, 0))
        else:
            raise TypeError(f"not a filter node: {node!r}")

    emit(expr)
    return ops, leaves


def eval_compiled(ops, leaves, planes: np.ndarray, valid: np.ndarray,
                  slot_range: tuple[int, int] | None = None) -> np.ndarray:
    """Stack machine over packed words: PUSH_LEAF = leaf AND, AND/OR word-wise,
    NOT = ``~x & valid``, result ``& valid``; range start must be 64-aligned
    (ref/filter_query.py:314-356)."""
    if slot_range is None:
        w0, w1 = 0, planes.shape[1]
    else:
        s0, s1 = slot_range
        if s0 % WORD_BITS:
            raise ValueError(f"slot range start {s0} not 64-aligned")
        w0, w1 = s0 >> 6, (s1 + WORD_BITS - 1) >> 6
    valid_slice = valid[w0:w1]
    stack: list[np.ndarray] = []
    for op, arg in ops:
        if op == OP_PUSH_LEAF:
            stack.append(bloom_eval_leaf(planes, leaves[arg][2], w0, w1).copy())
        elif op == OP_NOT:
            stack[-1] = ~stack[-1] & valid_slice
        else:
            rhs = stack.pop()
            stack[-1] = (stack[-1] & rhs) if op == OP_AND else (stack[-1] | rhs)
    if len(stack) != 1:
        raise ValueError("unbalanced operation array")
    return stack[0] & valid_slice


def to_bool(words: np.ndarray, n_slots: int) -> np.ndarray:
    """ref/bitset.py:60-63 (little-endian bit order)."""
    bits = np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")
    return bits[:n_slots].astype(bool)


def from_bool(flags: np.ndarray) -> np.ndarray:
    """ref/bitset.py:51-57."""
    flags = np.asarray(flags, dtype=bool)
    padded = n_words(len(flags)) * WORD_BITS
    if padded != len(flags):
        flags = np.concatenate([flags, np.zeros(padded - len(flags), dtype=bool)])
    return np.packbits(flags, bitorder="little").view(np.uint64)


# --------------------------------------------------------------------------------------
# quantization (ref/quantize.py:18-102)
# --------------------------------------------------------------------------------------

def quant_scale(gmin: float, gmax: float) -> float:
    return 255.0 / (gmax - gmin)  # ref/quantize.py:25-27


def quantize(x: np.ndarray, gmin: float, gmax: float) -> np.ndarray:
    """``clip(rint((x - min) * scale) - 128, -128, 127)`` in float64, rint = half to
    even (ref/quantize.py:64-76)."""
    v = np.asarray(x, dtype=np.float64)
    q = np.rint((v - gmin) * quant_scale(gmin, gmax)) - 128.0
    np.clip(q, -128.0, 127.0, out=q)
    return q.astype(np.int8)


def dequantize(q, gmin: float, gmax: float):
    """ref/quantize.py:79-81."""
    return (np.asarray(q, dtype=np.float64) + 128.0) / quant_scale(gmin, gmax) + gmin


# --------------------------------------------------------------------------------------
# scan + selection (ref/ivf.py:272-343, ref/serve.py:98-100)
# --------------------------------------------------------------------------------------

@dataclass
class OracleTopk:
    item_ids: np.ndarray  # uint64
    scores: np.ndarray    # int32


def select_topk(scores: np.ndarray, ids: np.ndarray, topk: int):
    """Exact (score desc, id asc) top-k via partition + lexsort (ref/ivf.py:272-282)."""
    m = len(scores)
    if m == 0 or topk <= 0:
        return ids[:0], scores[:0]
    if topk < m:
        kth = np.partition(scores, m - topk)[m - topk]
        cand = np.flatnonzero(scores >= kth)
        scores, ids = scores[cand], ids[cand]
    order = np.lexsort((ids, -scores.astype(np.int64)))[:topk]
    return ids[order], scores[order]


def search_clusters(items_q: np.ndarray, valid: np.ndarray, item_ids: np.ndarray,
                    cluster_offsets: np.ndarray, query_q: np.ndarray, clusters,
                    mask: np.ndarray | None, topk: int) -> OracleTopk:
    """Tile loop over each cluster's slot range: eligible = valid & mask; int32
    ``tile @ q``; keep eligible; exact top-k (ref/ivf.py:285-334)."""
    n_slots = items_q.shape[0]
    qi32 = np.asarray(query_q, dtype=np.int8).astype(np.int32)
    valid_bool = to_bool(valid, n_slots)
    mask_bool = to_bool(mask, n_slots) if mask is not None else None
    slot_parts, score_parts = [], []
    for c in clusters:
        start, end = (int(x) for x in cluster_offsets[int(c)])
        for t0 in range(start, end, TILE_ROWS):
            t1 = min(t0 + TILE_ROWS, end)
            eligible = valid_bool[t0:t1]
            if mask_bool is not None:
                eligible = eligible & mask_bool[t0:t1]
            if not eligible.any():
                continue
            scores = items_q[t0:t1].astype(np.int32) @ qi32
            keep = np.flatnonzero(eligible)
            slot_parts.append(keep + t0)
            score_parts.append(scores[keep])
    if slot_parts:
        slots = np.concatenate(slot_parts)
        scores = np.concatenate(score_parts).astype(np.int32)
        ids = item_ids[slots]
    else:
        ids = np.empty(0, dtype=np.uint64)
        scores = np.empty(0, dtype=np.int32)
    top_ids, top_scores = select_topk(scores, ids, topk)
    return OracleTopk(item_ids=top_ids, scores=top_scores)


def probe_centroids(centroids: np.ndarray, query: np.ndarray, nprobe: int) -> np.ndarray:
    """f64 dots, highest first, ties by ascending cluster id (ref/ivf.py:261-269,
    ref/vecmath.py:15-24)."""
    n_clusters = centroids.shape[0]
    nprobe = min(max(nprobe, 1), n_clusters)
    rows = np.asarray(centroids, dtype=np.float32).astype(np.float64)
    vec = np.asarray(query, dtype=np.float32).astype(np.float64)
    scores = np.sum(rows * vec, axis=1)
    order = np.lexsort((np.arange(n_clusters), -scores))
    return order[:nprobe].astype(np.int64)


def codesigned_search(items_q, valid, item_ids, cluster_offsets, planes, program,
                      query_q, clusters, k0) -> OracleTopk:
    """Filter only the given clusters' ranges into a zero mask, then scan
    (ref/retrieval.py:110-144). ``program`` is ``(ops, leaves)`` or None."""
    mask = None
    if program is not None:
        ops, leaves = program
        mask = np.zeros(n_words(items_q.shape[0]), dtype=np.uint64)
        for c in clusters:
            start, end = (int(x) for x in cluster_offsets[int(c)])
            if start == end:
                continue
            mask[start >> 6:(end + 63) >> 6] = eval_compiled(ops, leaves, planes, valid,
                                                             slot_range=(start, end))
    return search_clusters(items_q, valid, item_ids, cluster_offsets, query_q, clusters,
                           mask, k0)


def reduce_topk(ids: np.ndarray, scores: np.ndarray, k: int):
    """Global lexsort merge of concatenated shard results (ref/serve.py:98-100)."""
    order = np.lexsort((ids, -np.asarray(scores, dtype=np.int64)))[:k]
    return ids[order], scores[order]


def brute_force_int8(items_q: np.ndarray, item_ids: np.ndarray, query_q: np.ndarray,
                     topk: int, keep: np.ndarray | None = None) -> OracleTopk:
    """Full-scan int8 oracle (ref/evaluation.py:45-69, ``score="int8_dot"``)."""
    scores = items_q.astype(np.int32) @ np.asarray(query_q, dtype=np.int8).astype(np.int32)
    ids = item_ids
    if keep is not None:
        idx = np.flatnonzero(keep)
        ids, scores = ids[idx], scores[idx]
    order = np.lexsort((ids, -scores.astype(np.int64)))[:topk]
    return OracleTopk(item_ids=ids[order], scores=scores[order].astype(np.int32))


# --------------------------------------------------------------------------------------
# multi-task retrieval: merge, re-scoring, value model, final top-k (config 5;
# ref/retrieval.py:147-199, ref/scoring.py:61-130, ref/value_model.py:97-221)
# --------------------------------------------------------------------------------------
def merge_candidates(per_task: list, merge: str) -> np.ndarray:
    """Union keeps any task's ids, intersection the common ones; ascending unique
    (ref/retrieval.py:147-160)."""
    if merge == "union":
        out = per_task[0]
        for ids in per_task[1:]:
            out = np.union1d(out, ids)
        return out
    out = np.unique(per_task[0])
    for ids in per_task[1:]:
        out = np.intersect1d(out, ids, assume_unique=False)
    return out


def score_dot(user: np.ndarray, items: np.ndarray) -> np.ndarray:
    """Identity mixture-of-logits = the f64 dot product, pairwise-summed per row
    (ref/scoring.py:99-130 with identity projections; ref/vecmath.py:15-24)."""
    items64 = np.atleast_2d(np.asarray(items, dtype=np.float32)).astype(np.float64)
    return np.sum(items64 * np.asarray(user, dtype=np.float32).astype(np.float64), axis=1)


def score_mlp(hidden, heads, task, user, items) -> np.ndarray:
    """ReLU MLP on user||item, per-task linear head, f64 (ref/scoring.py:61-84)."""
    items = np.atleast_2d(np.asarray(items, dtype=np.float32))
    x = np.concatenate(
        [np.broadcast_to(np.asarray(user, dtype=np.float64), (items.shape[0], len(user))),
         items.astype(np.float64)], axis=1)
    for w, b in hidden:
        x = x @ w.astype(np.float64).T + b.astype(np.float64)
        np.maximum(x, 0.0, out=x)
    w, b = heads[task]
    return x @ w.astype(np.float64) + float(b)


def score_mol(components, gate_w, gate_b, user, items) -> np.ndarray:
    """Softmax-gated sum of projected dot products, f64 (ref/scoring.py:87-119)."""
    items64 = np.atleast_2d(np.asarray(items, dtype=np.float32)).astype(np.float64)
    user64 = np.asarray(user, dtype=np.float32).astype(np.float64)
    n = items64.shape[0]
    dots = np.empty((n, len(components)), dtype=np.float64)
    for j, (u_proj, i_proj) in enumerate(components):
        u_p = u_proj.astype(np.float64) @ user64
        i_p = items64 @ i_proj.astype(np.float64).T
        dots[:, j] = np.sum(i_p * u_p, axis=1)
    logits = (np.concatenate([np.broadcast_to(user64, (n, len(user64))), items64], axis=1)
              @ gate_w.astype(np.float64).T + gate_b.astype(np.float64))
    logits -= logits.max(axis=1, keepdims=True)
    gates = np.exp(logits)
    gates /= gates.sum(axis=1, keepdims=True)
    return np.sum(gates * dots, axis=1)


def value_model_eval(spec, task_scores: dict):
    """JSON formula over per-item f64 arrays, strict (both if-branches evaluated); a zero
    divisor in any lane raises ZeroDivisionError (ref/value_model.py:97-129, 164-213).
    ``spec=None`` is the per-request mean of the tasks (ref/value_model.py:216-221)."""
    if spec is None:
        names = list(task_scores)
        if len(names) == 1:
            spec = {"op": "task", "task": names[0]}
        else:
            spec = {"op": "mul", "args": [{"op": "const", "value": 1.0 / len(names)},
                                          {"op": "add", "args": [{"op": "task", "task": t}
                                                                 for t in names]}]}

    def walk(n):
        op = n["op"]
        if op == "const":
            return float(n["value"])
        if op == "task":
            return np.asarray(task_scores[n["task"]], dtype=np.float64)
        if op in ("add", "mul", "min", "max"):
            acc = walk(n["args"][0])
            for x in n["args"][1:]:
                v = walk(x)
                acc = (acc + v if op == "add" else acc * v if op == "mul"
                       else np.minimum(acc, v) if op == "min" else np.maximum(acc, v))
            return acc
        if op == "sub":
            return walk(n["args"][0]) - walk(n["args"][1])
        if op == "div":
            den = walk(n["args"][1])
            if np.any(np.asarray(den) == 0.0):
                raise ZeroDivisionError("division by zero in value model")
            return walk(n["args"][0]) / den
        if op == "clamp":
            return np.clip(walk(n["args"][0]), float(n["lo"]), float(n["hi"]))
        if op == "if":
            c = n["cond"]
            cmp = {"<": np.less, "<=": np.less_equal, ">": np.greater,
                   ">=": np.greater_equal, "==": np.equal}[c["cmp"]]
            return np.where(cmp(walk(c["left"]), walk(c["right"])), walk(n["then"]),
                            walk(n["else"]))
        raise ValueError(f"unknown formula op {op!r}")

    return walk(spec)


def retrieve(per_task_ids: list, merge: str, cache_ids: np.ndarray, cache_vectors: np.ndarray,
             score_fn, task_names: list, users: np.ndarray, vm_spec, topk: int):
    """Merge -> cache gather -> per-task scores -> value model -> (score desc, id asc)
    top-k (ref/retrieval.py:163-199). ``score_fn(task, user, vectors)`` re-scores."""
    merged = merge_candidates(per_task_ids, merge)
    if len(merged) == 0:
        return merged, np.empty(0), np.empty((0, len(task_names)))
    row_of = {int(i): r for r, i in enumerate(cache_ids)}
    vectors = cache_vectors[np.array([row_of[int(i)] for i in merged], dtype=np.int64)]
    ts = {t: score_fn(t, users[j], vectors) for j, t in enumerate(task_names)}
    final = np.asarray(value_model_eval(vm_spec, ts), dtype=np.float64)
    order = np.lexsort((merged, -final))[:topk]
    return (merged[order], final[order],
            np.stack([ts[t][order] for t in task_names], axis=1))


# --------------------------------------------------------------------------------------
# publish-side k-means and IVF layout (ref/ivf.py:68-258)
# --------------------------------------------------------------------------------------

def kmeans_pp_init(data: np.ndarray, k: int, seed: int) -> np.ndarray:
    """D^2 seeding (ref/ivf.py:76-101): row indices of the k chosen centres. The first is
    uniform; each next one is drawn with probability proportional to the squared distance
    to the nearest chosen centre (cumsum + searchsorted 'right' on u * total); with zero
    total mass, uniformly among the rows not yet chosen."""
    x = np.asarray(data, dtype=np.float64)
    n = x.shape[0]
    if k > n:
        raise ValueError(f"k={k} exceeds number of rows n={n}")
    gen = np.random.default_rng(seed)
    picks = [int(gen.integers(n))]
    dist = ((x - x[picks[0]]) ** 2).sum(axis=1)
    used = np.zeros(n, dtype=bool)
    used[picks[0]] = True
    while len(picks) < k:
        mass = dist.sum()
        if mass <= 0.0:
            free = np.nonzero(~used)[0]
            nxt = int(free[gen.integers(free.size)])
        else:
            target = gen.random() * mass
            nxt = min(int(np.searchsorted(np.cumsum(dist), target, side="right")), n - 1)
        picks.append(nxt)
        used[nxt] = True
        dist = np.minimum(dist, ((x - x[nxt]) ** 2).sum(axis=1))
    return np.array(picks, dtype=np.int64)


def sq_dists(x: np.ndarray, c: np.ndarray) -> np.ndarray:
    """(|x|^2 - 2 x.c) + |c|^2 clamped at 0 (ref/ivf.py:68-73)."""
    xx = np.einsum("ij,ij->i", x, x)
    cc = np.einsum("ij,ij->i", c, c)
    return np.maximum(xx[:, None] - 2.0 * (x @ c.T) + cc[None, :], 0.0)


def kmeans_train(data: np.ndarray, k: int, max_iters: int = 25, tol: float = 1e-4,
                 seed: int = 0):
    """Lloyd from D^2 seeding (ref/ivf.py:104-145) -> (centres float32 [k, d], assign i64).
    Empty clusters take the costliest point of the first largest cluster before the means;
    stop when the relative inertia gain is <= tol or after max_iters."""
    x = np.asarray(data, dtype=np.float64)
    n = x.shape[0]
    cen = x[kmeans_pp_init(x, k, seed)].astype(np.float32).astype(np.float64)
    last = None
    lab = np.zeros(n, dtype=np.int64)
    for _ in range(max_iters):
        d2 = sq_dists(x, cen)
        lab = d2.argmin(axis=1)
        size = np.bincount(lab, minlength=k)
        cost = d2[np.arange(n), lab]
        for c in np.nonzero(size == 0)[0]:
            big = int(size.argmax())
            mem = np.nonzero(lab == big)[0]
            j = mem[cost[mem].argmax()]
            lab[j] = c
            cost[j] = 0.0
            size[big] -= 1
            size[c] += 1
        for c in range(k):
            cen[c] = x[lab == c].mean(axis=0)
        d2 = sq_dists(x, cen)
        lab = d2.argmin(axis=1)
        cur = float(d2[np.arange(n), lab].sum())
        if last is not None and last - cur <= tol * last:
            break
        last = cur
    return cen.astype(np.float32), lab


def ivf_layout(assign: np.ndarray, item_ids: np.ndarray, k: int):
    """Cluster-major slot layout (ref/ivf.py:229-249) -> (perm i64 [n_slots], offsets u64
    [k, 2]): members of each cluster by ascending item id, ranges padded to 64."""
    parts, offs, pos = [], np.zeros((k, 2), dtype=np.uint64), 0
    for c in range(k):
        mem = np.nonzero(assign == c)[0]
        mem = mem[np.argsort(item_ids[mem], kind="stable")]
        width = -(-mem.size // WORD_BITS) * WORD_BITS
        block = np.full(width, -1, dtype=np.int64)
        block[: mem.size] = mem
        parts.append(block)
        offs[c] = (pos, pos + width)
        pos += width
    perm = np.concatenate(parts) if parts else np.zeros(0, dtype=np.int64)
    return perm, offs
