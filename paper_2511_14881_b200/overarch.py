"""Multi-task retrieval on the GPU (BASELINE config 5).

The reference serves a request of T task queries that share one filter as: one
co-designed filtered search per task, ``merge_candidates`` of the per-task id lists,
re-scoring of the merged candidates with cached float32 item embeddings per task, the
value-model formula over the per-task scores, and a final (score desc, id asc) top-k
(``retrieval.retrieve``, ref/retrieval.py:147-199; ``scoring``, ref/scoring.py:22-130;
``value_model``, ref/value_model.py:97-221).

Here the whole batch of requests runs on the device:

* the B x T task queries go through ONE batched filtered top-k (``TopkOp``; every task
  row carries its request's compiled filter);
* the merge is a per-request sort + unique over the T candidate lists (union, or
  ids present in all T lists for intersection);
* cache rows are found by binary search over the cache's sorted ids;
* the identity mixture-of-logits scorer (the reference default: the float64 dot product)
  runs in ``fb_task_dots_f64`` with numpy's pairwise summation order, so its scores are
  bit-identical to the reference; MLP / general MoL scorers run as float64 tensor
  algebra (agreement within the reference's 1e-5 float tolerance);
* the value model is evaluated element-wise in float64 with the reference's operation
  order (IEEE operations, hence bit-identical for identical inputs);
* the final order is a stable sort of the final scores over the ascending merged ids,
  i.e. the reference's ``lexsort((merged, -final))``.
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from ._device import IdentityCache, device, to_dev, to_dev_u64, u64_host
from .bloom import BloomParams, FilterStats
from .engine import DeviceIndex, TopkOp, _u64_order_key
from .errors import DivByZero, FiltraError, MissingItem, UnknownTask
from .filter_query import FilterBatch
from .ivf import ScanStats
from .quantize import quantize_device

MERGE_UNION = "union"
MERGE_INTERSECTION = "intersection"
_PAD = (1 << 63) - 1  # order key of "no candidate"


# ------------------------------------------------------------------------------------
# embedding cache
# ------------------------------------------------------------------------------------
class DeviceCache:
    """``EmbeddingCache`` in HBM: float32 vectors plus the ids sorted for lookup
    (ref/scoring.py:22-52)."""

    def __init__(self, item_ids, vectors):
        dev = device()
        self.vectors = to_dev(vectors, torch.float32, dev).contiguous()
        ids = to_dev_u64(item_ids, dev)
        if ids.numel() != self.vectors.shape[0]:
            raise ValueError("ids and vectors disagree on length")
        key = _u64_order_key(ids)
        self._sorted_key, self._row = torch.sort(key)

    @classmethod
    def from_reference(cls, cache) -> "DeviceCache":
        return cls(np.asarray(cache.item_ids, dtype=np.uint64), np.asarray(cache.vectors))

    @property
    def dim(self) -> int:
        return int(self.vectors.shape[1])

    def rows_for(self, ids: torch.Tensor, valid: torch.Tensor) -> torch.Tensor:
        """Cache row of each id (int64 u64 bits); entries with ``valid`` False give -1.
        Raises ``MissingItem`` for a valid id the cache does not hold."""
        rows, bad = self.rows_and_missing(ids, valid)
        if bool(bad.any()):
            missing = int(ids[bad][0].item()) & 0xFFFFFFFFFFFFFFFF
            raise MissingItem(missing)
        return rows

    def rows_and_missing(self, ids: torch.Tensor, valid: torch.Tensor):
        """``rows_for`` without the host check: (rows, bool mask of valid ids the cache
        lacks), for callers that test it after a CUDA-graph replay."""
        key = _u64_order_key(ids)
        pos = torch.searchsorted(self._sorted_key, key).clamp_(max=self._sorted_key.numel() - 1)
        hit = self._sorted_key[pos] == key
        return torch.where(valid, self._row[pos], torch.full_like(pos, -1)), valid & ~hit


# ------------------------------------------------------------------------------------
# scorers
# ------------------------------------------------------------------------------------
def _is_identity_mol(scorer) -> bool:
    comps = getattr(scorer, "components", None)
    if comps is None or len(comps) != 1:
        return False
    u, i = (np.asarray(x) for x in comps[0])
    if u.shape[0] != u.shape[1] or i.shape != u.shape:
        return False
    eye = np.eye(u.shape[0], dtype=np.float32)
    return (np.array_equal(u, eye) and np.array_equal(i, eye)
            and not np.any(np.asarray(scorer.gate_weight)) and not np.any(np.asarray(scorer.gate_bias)))


class DeviceScorer:
    """Re-ranking scorer on the device: ``dot`` (identity MoL, exact kernel), ``mlp`` or
    ``mol`` (float64 tensor algebra) -- ref/scoring.py:61-130."""

    def __init__(self, kind: str, params: dict | None = None):
        self.kind = kind
        self.p = params or {}

    @classmethod
    def dot(cls) -> "DeviceScorer":
        return cls("dot")

    @classmethod
    def from_reference(cls, scorer) -> "DeviceScorer":
        if scorer is None or _is_identity_mol(scorer):
            return cls.dot()
        dev = device()
        f64 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.float32), device=dev).double()  # noqa: E731
        if hasattr(scorer, "hidden"):
            heads = {name: (f64(h.weight), float(h.bias)) for name, h in scorer.heads.items()}
            shared = scorer.shared_head
            return cls("mlp", {"hidden": [(f64(w), f64(b)) for w, b in scorer.hidden],
                               "heads": heads,
                               "shared": (f64(shared.weight), float(shared.bias)) if shared else None})
        if hasattr(scorer, "components"):
            return cls("mol", {"comps": [(f64(u), f64(i)) for u, i in scorer.components],
                               "gw": f64(scorer.gate_weight), "gb": f64(scorer.gate_bias)})
        raise TypeError(f"unsupported scorer {type(scorer).__name__}")

    def score(self, cache: DeviceCache, rows: torch.Tensor, count: torch.Tensor,
              users: torch.Tensor, tasks: list[str]) -> torch.Tensor:
        """rows int64 [B, C] (cache rows, -1 padding), count int32 [B], users float32
        [B, T, d] -> float64 [B, T, C] (padding lanes 0)."""
        B, C = rows.shape
        T = users.shape[1]
        out = torch.zeros((B, T, C), dtype=torch.float64, device=rows.device)
        if B == 0 or C == 0:
            return out
        if self.kind == "dot":
            r = rows.contiguous()
            u = users.to(torch.float32).contiguous()
            _native.check(_native.lib().fb_task_dots_f64(
                cache.vectors.data_ptr(), cache.vectors.shape[0], cache.dim, r.data_ptr(),
                count.to(torch.int32).contiguous().data_ptr(), C, u.data_ptr(), B, T,
                out.data_ptr(), _native.stream_ptr()))
            return out
        valid = rows >= 0
        items = cache.vectors[rows.clamp(min=0)].double()          # [B, C, d]
        u64 = users.to(torch.float32).double()                      # [B, T, d]
        for t, name in enumerate(tasks):
            if self.kind == "mlp":
                x = torch.cat([u64[:, t, None, :].expand(B, C, u64.shape[2]), items], dim=2)
                for w, b in self.p["hidden"]:
                    x = torch.relu(x @ w.T + b)
                head = self.p["heads"].get(name, self.p["shared"])
                if head is None:
                    raise KeyError(f"no output head for task {name!r}")
                s = x @ head[0] + head[1]
            else:
                dots = []
                for up, ip in self.p["comps"]:
                    u_p = u64[:, t, :] @ up.T                       # [B, d_p]
                    i_p = items @ ip.T                              # [B, C, d_p]
                    dots.append((i_p * u_p[:, None, :]).sum(dim=2))
                dots = torch.stack(dots, dim=2)                     # [B, C, P]
                x = torch.cat([u64[:, t, None, :].expand(B, C, u64.shape[2]), items], dim=2)
                logits = x @ self.p["gw"].T + self.p["gb"]
                logits = logits - logits.max(dim=2, keepdim=True).values
                g = torch.exp(logits)
                g = g / g.sum(dim=2, keepdim=True)
                s = (g * dots).sum(dim=2)
            out[:, t, :] = torch.where(valid, s, torch.zeros_like(s))
        return out


# ------------------------------------------------------------------------------------
# value model
# ------------------------------------------------------------------------------------
def value_model_spec(vm) -> dict | None:
    """JSON spec of a reference formula tree (ref/value_model.py:31-91) or a JSON dict;
    None stays None (per-request mean)."""
    if vm is None or isinstance(vm, dict):
        return vm
    name = type(vm).__name__
    if name == "Const":
        return {"op": "const", "value": vm.value}
    if name == "TaskScore":
        return {"op": "task", "task": vm.task}
    if name in ("Add", "Mul", "Min", "Max"):
        return {"op": name.lower(), "args": [value_model_spec(a) for a in vm.args]}
    if name == "Sub":
        return {"op": "sub", "args": [value_model_spec(vm.left), value_model_spec(vm.right)]}
    if name == "Div":
        return {"op": "div", "args": [value_model_spec(vm.num), value_model_spec(vm.den)]}
    if name == "Clamp":
        return {"op": "clamp", "args": [value_model_spec(vm.arg)], "lo": vm.lo, "hi": vm.hi}
    if name == "If":
        return {"op": "if", "cond": {"left": value_model_spec(vm.cond.left), "cmp": vm.cond.op,
                                     "right": value_model_spec(vm.cond.right)},
                "then": value_model_spec(vm.then), "else": value_model_spec(vm.orelse)}
    raise TypeError(f"not a formula node: {vm!r}")


def mean_of_tasks_spec(task_names: list[str]) -> dict:
    """ref/value_model.py:216-221: (1/T) * (t_0 + ... + t_{T-1})."""
    total = {"op": "add", "args": [{"op": "task", "task": t} for t in task_names]}
    if len(task_names) == 1:
        return total["args"][0]
    return {"op": "mul", "args": [{"op": "const", "value": 1.0 / len(task_names)}, total]}


def value_model_device(spec: dict, task_scores: dict[str, torch.Tensor],
                       valid: torch.Tensor | None = None, zero_flags: list | None = None
                       ) -> torch.Tensor:
    """Element-wise float64 evaluation in the reference's operation order; both branches
    of an ``if`` are evaluated; a zero divisor in any valid lane raises ``DivByZero`` (or,
    with ``zero_flags``, appends the device flag tensor for the caller to test later)."""
    some = next(iter(task_scores.values()))

    def const(v):
        return torch.full_like(some, float(v))

    def walk(n):
        op = n["op"]
        if op == "const":
            return const(n["value"])
        if op == "task":
            if n["task"] not in task_scores:
                raise UnknownTask(n["task"])
            return task_scores[n["task"]]
        if op in ("add", "mul", "min", "max"):
            acc = walk(n["args"][0])
            for a in n["args"][1:]:
                v = walk(a)
                acc = (acc + v if op == "add" else acc * v if op == "mul"
                       else torch.minimum(acc, v) if op == "min" else torch.maximum(acc, v))
            return acc
        if op == "sub":
            return walk(n["args"][0]) - walk(n["args"][1])
        if op == "div":
            den = walk(n["args"][1])
            zero = den == 0.0
            if valid is not None:
                zero = zero & valid
            if zero_flags is not None:
                zero_flags.append(zero.any())
            elif bool(zero.any()):
                raise DivByZero("division by zero in value model")
            return walk(n["args"][0]) / den
        if op == "clamp":
            return torch.clamp(walk(n["args"][0]), float(n["lo"]), float(n["hi"]))
        if op == "if":
            c = n["cond"]
            left, right = walk(c["left"]), walk(c["right"])
            cmp = {"<": torch.lt, "<=": torch.le, ">": torch.gt, ">=": torch.ge,
                   "==": torch.eq}[c["cmp"]](left, right)
            return torch.where(cmp, walk(n["then"]), walk(n["else"]))
        raise ValueError(f"unknown formula op {op!r}")

    return walk(spec)


_VM_OPS = {"add": 2, "sub": 3, "mul": 4, "div": 5, "min": 6, "max": 7}
_VM_IF = {"<": 9, "<=": 10, ">": 11, ">=": 12, "==": 13}
_VM_STACK = 16
_VM_CODE: dict = {}


def value_model_code(spec: dict, names: list[str]):
    """Postfix bytecode of a value-model formula for ``fb_value_model`` (u16 words
    op | arg << 8, float64 constants), in the reference's evaluation order
    (ref value_model.py:75-124: n-ary ops fold left). Returns None when the formula is
    deeper than the kernel's stack."""
    code: list[int] = []
    consts: list[float] = []
    depth = [0, 0]  # current, max

    def push():
        depth[0] += 1
        depth[1] = max(depth[1], depth[0])

    def walk(n):
        op = n["op"]
        if op == "const":
            code.append(0 | (len(consts) << 8))
            consts.append(float(n["value"]))
            push()
        elif op == "task":
            if n["task"] not in names:
                raise UnknownTask(n["task"])
            code.append(1 | (names.index(n["task"]) << 8))
            push()
        elif op in ("add", "mul", "min", "max"):
            walk(n["args"][0])
            for a in n["args"][1:]:
                walk(a)
                code.append(_VM_OPS[op])
                depth[0] -= 1
        elif op in ("sub", "div"):
            walk(n["args"][0])
            walk(n["args"][1])
            code.append(_VM_OPS[op])
            depth[0] -= 1
        elif op == "clamp":
            walk(n["args"][0])
            code.append(8 | (len(consts) << 8))
            consts.extend([float(n["lo"]), float(n["hi"])])
        elif op == "if":
            c = n["cond"]
            walk(c["left"])
            walk(c["right"])
            walk(n["then"])
            walk(n["else"])
            code.append(_VM_IF[c["cmp"]])
            depth[0] -= 3
        else:
            raise ValueError(f"unknown formula op {op!r}")

    walk(spec)
    if depth[1] > _VM_STACK or len(consts) >= 256 or len(names) >= 256:
        return None
    return code, consts


def value_model_kernel(spec: dict, names: list[str], ts: torch.Tensor, mcount: torch.Tensor,
                       zero: torch.Tensor | None = None):
    """The value model on ``fb_value_model``: ts float64 [B, T, C] task scores (task order
    = ``names``), mcount [B] valid candidates -> (final float64 [B, C], zero int32 [1] set
    to 1 when a valid candidate divides by zero). None when the formula does not compile
    (deeper than the kernel's stack)."""
    key = (json.dumps(spec, sort_keys=True, default=str), tuple(names), ts.device.index)
    hit = _VM_CODE.get(key)
    if hit is None:
        cc = value_model_code(spec, names)
        if cc is None:
            return None
        code, consts = cc
        dev = ts.device
        hit = (torch.from_numpy(np.asarray(code, dtype=np.uint16).view(np.int16)).to(dev),
               torch.tensor(consts or [0.0], dtype=torch.float64, device=dev), len(code))
        _VM_CODE[key] = hit
    code_t, consts_t, n_code = hit
    B, T, C = ts.shape
    t = ts.contiguous()
    cnt = mcount.to(torch.int32).contiguous()
    out = torch.empty((B, C), dtype=torch.float64, device=ts.device)
    if zero is None:
        zero = torch.zeros(1, dtype=torch.int32, device=ts.device)
    else:
        zero.zero_()
    _native.check(_native.lib().fb_value_model(code_t.data_ptr(), n_code, consts_t.data_ptr(),
                                               t.data_ptr(), B, T, C, cnt.data_ptr(),
                                               out.data_ptr(), zero.data_ptr(),
                                               _native.stream_ptr()))
    return out, zero


# ------------------------------------------------------------------------------------
# final ranking
# ------------------------------------------------------------------------------------
FINAL_TOPK_MAX_CAND = 24576  # fb_final_topk's staging limit (merged candidates per request)
FINAL_TOPK_MAX_K = 8192


def final_topk_device(final: torch.Tensor, mcount: torch.Tensor, topk: int):
    """``np.lexsort((merged, -final))[:topk]`` per request (ref retrieval.py:190) on the
    device: final float64 [B, C] over merged candidates in ascending id order, mcount int32
    [B] valid entries -> (order int64 [B, topk], n int32 [B] = min(topk, mcount)).
    NumPy's float order (NaN last, -0.0 == +0.0) through ``fb_final_topk``; shapes past its
    limits take a stable device sort instead."""
    B, C = final.shape
    topk = int(topk)
    if C > FINAL_TOPK_MAX_CAND or topk > FINAL_TOPK_MAX_K:
        valid = torch.arange(C, device=final.device)[None, :] < mcount[:, None]
        f = torch.where(valid, final, torch.full_like(final, -float("inf")))
        order = torch.sort(f, dim=1, descending=True, stable=True).indices[:, :topk]
        n = torch.clamp(mcount, max=topk).to(torch.int32)
        return order, n
    f = final.contiguous()
    cnt = mcount.to(torch.int32).contiguous()
    order = torch.empty((B, topk), dtype=torch.int64, device=final.device)
    n = torch.empty(B, dtype=torch.int32, device=final.device)
    _native.check(_native.lib().fb_final_topk(f.data_ptr(), C, cnt.data_ptr(), B, topk,
                                              order.data_ptr(), n.data_ptr(),
                                              _native.stream_ptr()))
    return order, n


# ------------------------------------------------------------------------------------
# merge
# ------------------------------------------------------------------------------------
def merge_device(ids: torch.Tensor, counts: torch.Tensor, merge: str):
    """Per-request merge of T candidate lists (``merge_candidates``, ref/retrieval.py:
    147-160). ids int64 (u64 bits) [B, T, k], counts [B, T] -> (merged [B, T*k] ascending
    u64 ids padded with the max key, mcount int32 [B])."""
    if merge not in (MERGE_UNION, MERGE_INTERSECTION):
        raise FiltraError(f"unknown merge {merge!r}")
    B, T, k = ids.shape
    live = torch.arange(k, device=ids.device)[None, None, :] < counts[:, :, None]
    key = torch.where(live, _u64_order_key(ids), torch.full_like(ids, _PAD)).view(B, T * k)
    key, _ = torch.sort(key, dim=1)
    first = torch.ones_like(key, dtype=torch.bool)
    first[:, 1:] = key[:, 1:] != key[:, :-1]
    keep = first & (key != _PAD)
    if merge == MERGE_INTERSECTION:
        # lists hold unique ids, so an id in all T lists occupies T consecutive slots
        if T > 1:
            ahead = torch.full_like(key, _PAD)
            ahead[:, : T * k - (T - 1)] = key[:, T - 1:]
            keep &= ahead == key
    # the kept keys are ascending already: compact them to the front (dropped slots go to
    # a spill column past the end)
    pos = torch.cumsum(keep, dim=1)
    mcount = pos[:, -1].to(torch.int32)
    dst = torch.where(keep, pos - 1, torch.full_like(pos, T * k))
    merged = torch.full((B, T * k + 1), _PAD, dtype=key.dtype, device=key.device)
    merged.scatter_(1, dst, key)
    return _u64_order_key(merged[:, : T * k]), mcount


# ------------------------------------------------------------------------------------
# batched multi-task operator
# ------------------------------------------------------------------------------------
@dataclass
class MultiTaskOutput:
    ids: torch.Tensor          # int64 (u64 bits) [B, topk], (score desc, id asc)
    scores: torch.Tensor       # float64 [B, topk] value-model score
    task_scores: torch.Tensor  # float64 [B, T, topk]
    count: torch.Tensor        # int32 [B]
    n_merged: torch.Tensor     # int32 [B] merged candidates per request

    def host(self, b: int):
        n = int(self.count[b])
        return (u64_host(self.ids[b, :n].contiguous()), self.scores[b, :n].cpu().numpy(),
                self.task_scores[b, :, :n].cpu().numpy().T)


class MultiTaskOp:
    """Config-5 operator: B requests x T task towers sharing one filter per request."""

    def __init__(self, index: DeviceIndex, cache: DeviceCache, n_requests: int,
                 task_names: list[str], k0: int, topk: int, merge: str = MERGE_UNION,
                 scorer: DeviceScorer | None = None, value_model=None, ranges=None,
                 flags: int = 0):
        if not (1 <= topk <= k0):
            raise FiltraError(f"need 1 <= topk <= k0, got topk={topk}, k0={k0}")
        if merge not in (MERGE_UNION, MERGE_INTERSECTION):
            raise FiltraError(f"unknown merge {merge!r}")
        self.index, self.cache = index, cache
        self.B, self.tasks = int(n_requests), list(task_names)
        self.T, self.k0, self.topk, self.merge = len(self.tasks), int(k0), int(topk), merge
        self.scorer = scorer or DeviceScorer.dot()
        self.spec = value_model_spec(value_model) or mean_of_tasks_spec(self.tasks)
        if ranges is None:
            ranges = np.array([[0, index.n_slots]], dtype=np.int64)
        self.op = TopkOp(index, self.B * self.T, self.k0, ranges, flags)

    def _merge_union(self, res):
        """Union merge through the id-rank bitmap (``fb_merge_union``): same output as
        ``merge_device(..., "union")``, plus the merged ids' ranks."""
        B, T, k = self.B, self.T, self.k0
        dev = res.keys.device
        if getattr(self, "_bitmap", None) is None:
            # B rank bitmaps, then 8 u64 of per-request segment counters
            self._bitmap = torch.zeros(B * (self.index.n_words + 8), dtype=torch.int64, device=dev)
        merged = torch.empty((B, T * k), dtype=torch.int64, device=dev)
        ranks = torch.empty((B, T * k), dtype=torch.int64, device=dev)
        mcount = torch.empty(B, dtype=torch.int32, device=dev)
        _native.check(_native.lib().fb_merge_union(
            res.keys.data_ptr(), res.count.data_ptr(), B, T, k, self.index.n_slots_pad,
            self.index.id_of_rank.data_ptr(), self._bitmap.data_ptr(), merged.data_ptr(),
            ranks.data_ptr(), mcount.data_ptr(), _native.stream_ptr()))
        return merged, ranks, mcount

    def _rows_of_ranks(self, merged, ranks, valid):
        """Cache rows through a rank -> cache-row table built once per operator (-1 where
        the cache lacks the id); raises ``MissingItem`` like ``DeviceCache.rows_for``."""
        if getattr(self, "_row_of_rank", None) is None:
            key = _u64_order_key(self.index.id_of_rank)
            sk = self.cache._sorted_key
            pos = torch.searchsorted(sk, key).clamp_(max=sk.numel() - 1)
            self._row_of_rank = torch.where(sk[pos] == key, self.cache._row[pos],
                                            torch.full_like(pos, -1))
        rows = self._row_of_rank[ranks.clamp(min=0)]
        bad = valid & (rows < 0)
        if bool(bad.any()):
            raise MissingItem(int(merged[bad][0].item()) & 0xFFFFFFFFFFFFFFFF)
        return torch.where(valid, rows, torch.full_like(rows, -1))

    def pack_filters(self, filters, params: BloomParams | None = None) -> FilterBatch | None:
        """One compiled filter per request, repeated for each of its tasks."""
        if filters is None or all(f is None for f in filters):
            return None
        rows = [f for f in filters for _ in range(self.T)]
        return FilterBatch.pack(rows, params or BloomParams())

    def __call__(self, users: torch.Tensor, batch: FilterBatch | None,
                 queries_q: torch.Tensor | None = None) -> MultiTaskOutput:
        B, T = self.B, self.T
        if users.shape[:2] != (B, T):
            raise ValueError(f"users must be [{B}, {T}, dim]")
        users = users.to(torch.float32)
        if queries_q is None:
            queries_q = quantize_device(users.reshape(B * T, -1), self.index.qp,
                                        out_stride=self.index.dim_pad)
        if self.merge == MERGE_UNION and self.index.id_of_rank is not None:
            res = self.op(queries_q, batch, keys=True)
            merged, ranks, mcount = self._merge_union(res)
            valid = torch.arange(merged.shape[1], device=merged.device)[None, :] < mcount[:, None]
            rows = self._rows_of_ranks(merged, ranks, valid)
        else:
            res = self.op(queries_q, batch)
            merged, mcount = merge_device(res.ids.view(B, T, self.k0),
                                          res.count.view(B, T), self.merge)
            valid = torch.arange(merged.shape[1], device=merged.device)[None, :] < mcount[:, None]
            rows = self.cache.rows_for(merged, valid)
        ts = self.scorer.score(self.cache, rows, mcount, users, self.tasks)    # [B, T, C]
        vm = value_model_kernel(self.spec, self.tasks, ts, mcount)
        if vm is None:
            final = value_model_device(self.spec, {t: ts[:, j, :] for j, t in enumerate(self.tasks)},
                                       valid)
        else:
            final, zero = vm
            if bool(zero.item()):
                raise DivByZero("division by zero in value model")
        order, n = final_topk_device(final, mcount, self.topk)
        return MultiTaskOutput(ids=torch.gather(merged, 1, order),
                               scores=torch.gather(final, 1, order),
                               task_scores=torch.gather(ts, 2, order[:, None, :].expand(B, T, -1)),
                               count=n, n_merged=mcount)


# ------------------------------------------------------------------------------------
# drop-in for reference retrieval.retrieve
# ------------------------------------------------------------------------------------
@dataclass
class RetrievedItem:
    item_id: int
    score: float
    task_scores: dict[str, float]


@dataclass
class RetrieveResult:
    items: list[RetrievedItem]
    stats: object
    scan: ScanStats
    filter_stats: FilterStats


# device copies of the reference engine's embedding cache / scorer, keyed weakly on the
# host objects: a snapshot hot swap drops the old engine and with it its HBM copy
_DEVICE_CACHE = IdentityCache()
_DEVICE_SCORER = IdentityCache()


def _weak_cached(table: IdentityCache, obj, make):
    return table.get_or_make(obj, make)


def retrieve(engine, req) -> RetrieveResult:
    """``retrieval.retrieve(engine, req)`` (ref/retrieval.py:163-199) on the GPU: per-task
    co-designed search (probed clusters honoured), device merge, re-scoring, value
    model, final top-k. ``engine`` is the reference ``Engine`` (duck-typed)."""
    from .retrieval import StageTimings, codesigned_search
    start = time.perf_counter()
    timings, scan_stats, filter_stats = StageTimings(), ScanStats(), FilterStats()
    if not _native.env_flag("FB_EAGER_B1"):
        # one CUDA-graph replay for the whole request (fastpath.py)
        from . import fastpath
        names = [t.task_name for t in req.tasks]
        vm = req.value_model if req.value_model is not None else engine.default_value_model
        spec = value_model_spec(vm) or mean_of_tasks_spec(names)
        fast = fastpath.retrieve_fast(
            engine, req, lambda c: _weak_cached(_DEVICE_CACHE, c, DeviceCache.from_reference),
            lambda sc: _weak_cached(_DEVICE_SCORER, sc, DeviceScorer.from_reference), spec, names)
        if fast is not None:
            ids_h, fin_h, ts_h, clusters, push_bits, dix = fast
            for j in range(len(names)):
                fastpath.scan_stats_for(dix.cluster_offsets, clusters[j], scan_stats)
                if req.filter is not None:
                    fastpath.filter_stats_for(dix.cluster_offsets, clusters[j], push_bits,
                                              filter_stats)
            items = [RetrievedItem(item_id=int(ids_h[i]), score=float(fin_h[i]),
                                   task_scores={t: float(ts_h[j, i]) for j, t in enumerate(names)})
                     for i in range(len(ids_h))]
            timings.scan_us = timings.total_us = int((time.perf_counter() - start) * 1e6)
            return RetrieveResult(items=items, stats=timings, scan=scan_stats,
                                  filter_stats=filter_stats)
    cf = engine.compile(req.filter) if req.filter is not None else None
    per_task = []
    for task in req.tasks:
        r = codesigned_search(engine.ivf, engine.bloom, cf, task.user_embedding, req.nprobe,
                              req.k0, scan_stats=scan_stats, filter_stats=filter_stats,
                              timings=timings)
        per_task.append(np.asarray(r.item_ids, dtype=np.uint64))
    t0 = time.perf_counter()
    dev = device()
    T, k = len(per_task), max(1, max((len(x) for x in per_task), default=1))
    ids = torch.zeros((1, T, k), dtype=torch.int64, device=dev)
    counts = torch.zeros((1, T), dtype=torch.int32, device=dev)
    for j, x in enumerate(per_task):
        if len(x):
            ids[0, j, : len(x)] = to_dev_u64(x, dev)
        counts[0, j] = len(x)
    merged, mcount = merge_device(ids, counts, req.merge)
    items: list[RetrievedItem] = []
    n = int(mcount[0])
    if n:
        dcache = _weak_cached(_DEVICE_CACHE, engine.cache, DeviceCache.from_reference)
        valid = torch.arange(merged.shape[1], device=dev)[None, :] < mcount[:, None]
        rows = dcache.rows_for(merged, valid)
        names = [t.task_name for t in req.tasks]
        users = torch.as_tensor(np.stack([np.asarray(t.user_embedding, dtype=np.float32)
                                          for t in req.tasks]), device=dev)[None]
        scorer = _weak_cached(_DEVICE_SCORER, engine.scorer, DeviceScorer.from_reference)
        ts = scorer.score(dcache, rows, mcount, users, names)
        vm = req.value_model if req.value_model is not None else engine.default_value_model
        spec = value_model_spec(vm) or mean_of_tasks_spec(names)
        vmk = value_model_kernel(spec, names, ts, mcount)
        if vmk is None:
            final = value_model_device(spec, {t: ts[:, j, :] for j, t in enumerate(names)}, valid)
        else:
            final, zero = vmk
            if bool(zero.item()):
                raise DivByZero("division by zero in value model")
        order = final_topk_device(final, mcount, min(req.topk, n))[0][0]
        ids_h = u64_host(merged[0, order].contiguous())
        fin_h = final[0, order].cpu().numpy()
        ts_h = ts[0][:, order].cpu().numpy()
        for i in range(len(order)):
            items.append(RetrievedItem(item_id=int(ids_h[i]), score=float(fin_h[i]),
                                       task_scores={t: float(ts_h[j, i]) for j, t in enumerate(names)}))
    timings.overarch_us = int((time.perf_counter() - t0) * 1e6)
    timings.total_us = int((time.perf_counter() - start) * 1e6)
    return RetrieveResult(items=items, stats=timings, scan=scan_stats, filter_stats=filter_stats)


__all__ = ["DeviceCache", "DeviceScorer", "MultiTaskOp", "MultiTaskOutput", "merge_device",
           "retrieve", "value_model_device", "value_model_spec", "mean_of_tasks_spec",
           "MERGE_UNION", "MERGE_INTERSECTION", "MissingItem", "DivByZero", "UnknownTask"]
