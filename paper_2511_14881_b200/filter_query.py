"""Filter expressions: grammar, AST, postfix compiler, and the GPU evaluator.

Grammar and lowering follow the reference (filter_query.py:1-311): OR binds tighter
than AND, NOT tightest; AND/OR children are chained pairwise in post-order; leaves
are de-duplicated per filter. ``FilterBatch`` packs a batch of compiled filters
into the device bytecode consumed by the fused scan (leaves de-duplicated across
the whole batch, positions hashed in C). ``eval_compiled`` runs ``fb_filter_eval``.
"""

from __future__ import annotations

import copy
import re
import threading
from collections import OrderedDict
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np
import torch

from . import _native, bitset
from ._device import device, to_dev_u64, u64_host
from .bloom import BloomIndex, BloomParams, FilterStats, QueryBloom, hash_positions_batch
from .errors import FilterSyntaxError, UnknownFeature, UnknownValue


# --- AST ------------------------------------------------------------------------------

@dataclass(frozen=True)
class Leaf:
    feature_id: int
    value: int


@dataclass(frozen=True)
class And:
    children: tuple


@dataclass(frozen=True)
class Or:
    children: tuple


@dataclass(frozen=True)
class Not:
    child: object


FilterExpr = object  # Leaf | And | Or | Not


@dataclass(frozen=True)
class Vocabulary:
    """Feature-name and string-value dictionaries (reference filter_query.py:60-77)."""

    feature_ids: dict[str, int] = field(default_factory=dict)
    values: dict[str, int] = field(default_factory=dict)

    @classmethod
    def from_schema(cls, feature_schema: dict[int, str], values: dict[str, int] | None = None):
        return cls(feature_ids={name: fid for fid, name in feature_schema.items()},
                   values=dict(values or {}))

    def feature_name(self, fid: int) -> str | None:
        for name, v in self.feature_ids.items():
            if v == fid:
                return name
        return None


# --- parser ---------------------------------------------------------------------------

_TOKEN = re.compile(r'\s+|(?P<lpar>\()|(?P<rpar>\))|(?P<eq>=)|(?P<string>"[^"]*")|'
                    r'(?P<int>\d+)|(?P<ident>[A-Za-z_][A-Za-z0-9_.]*)')
_KEYWORDS = ("AND", "OR", "NOT")


def _tokens(text: str):
    out, pos = [], 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        if m is None:
            raise FilterSyntaxError(pos, f"unexpected character {text[pos]!r}")
        if m.lastgroup is not None:
            kind, val = m.lastgroup, m.group()
            if kind == "ident" and val.upper() in _KEYWORDS:
                kind = val.upper()
            out.append((kind, val, pos))
        pos = m.end()
    out.append(("eof", "", len(text)))
    return out


def parse_filter(text: str, vocab: Vocabulary | None = None) -> FilterExpr:
    """Recursive descent: expr := or_term (AND or_term)*; or_term := factor (OR factor)*;
    factor := [NOT] (leaf | '(' expr ')'); leaf := name '=' value."""
    vocab = vocab or Vocabulary()
    toks = _tokens(text)
    i = 0

    def peek():
        return toks[i][0]

    def take(kind=None):
        nonlocal i
        tok = toks[i]
        if kind is not None and tok[0] != kind:
            raise FilterSyntaxError(tok[2], f"expected {kind}, found {tok[1]!r}")
        i += 1
        return tok

    def expr():
        parts = [or_term()]
        while peek() == "AND":
            take()
            parts.append(or_term())
        return parts[0] if len(parts) == 1 else And(tuple(parts))

    def or_term():
        parts = [factor()]
        while peek() == "OR":
            take()
            parts.append(factor())
        return parts[0] if len(parts) == 1 else Or(tuple(parts))

    def factor():
        if peek() == "NOT":
            take()
            return Not(factor())
        if peek() == "lpar":
            take()
            inner = expr()
            take("rpar")
            return inner
        return leaf()

    def leaf():
        kind, text_, pos = take()
        if kind == "ident":
            if text_ not in vocab.feature_ids:
                raise UnknownFeature(text_)
            fid = vocab.feature_ids[text_]
        elif kind == "int":
            fid = int(text_)
        else:
            raise FilterSyntaxError(pos, f"expected feature name, found {text_!r}")
        take("eq")
        kind, text_, pos = take()
        if kind == "string":
            lit = text_[1:-1]
            if lit not in vocab.values:
                raise UnknownValue(lit)
            value = vocab.values[lit]
        elif kind == "int":
            value = int(text_)
        else:
            raise FilterSyntaxError(pos, f"expected value, found {text_!r}")
        return Leaf(feature_id=fid, value=value)

    result = expr()
    if peek() != "eof":
        raise FilterSyntaxError(toks[i][2], f"trailing input {toks[i][1]!r}")
    return result


def format_filter(expr: FilterExpr, vocab: Vocabulary | None = None) -> str:
    """Inverse of :func:`parse_filter`."""
    vocab = vocab or Vocabulary()
    rev = {v: s for s, v in vocab.values.items()}

    def fmt(node, parent):
        if isinstance(node, Leaf):
            name = vocab.feature_name(node.feature_id)
            lhs = name if name is not None else str(node.feature_id)
            rhs = f'"{rev[node.value]}"' if node.value in rev else str(node.value)
            return f"{lhs} = {rhs}"
        if isinstance(node, Not):
            inner = fmt(node.child, "not")
            return f"NOT {inner}" if isinstance(node.child, Leaf) else f"NOT ({inner})"
        if isinstance(node, Or):
            body = " OR ".join(fmt(c, "or") for c in node.children)
            return f"({body})" if parent in ("or", "not") else body
        if isinstance(node, And):
            body = " AND ".join(fmt(c, "and") for c in node.children)
            return body if parent == "top" else f"({body})"
        raise TypeError(f"not a filter node: {node!r}")

    return fmt(expr, "top")


def expr_has_not(expr: FilterExpr) -> bool:
    if isinstance(expr, Not):
        return True
    if isinstance(expr, (And, Or)):
        return any(expr_has_not(c) for c in expr.children)
    return False


# --- compiled form --------------------------------------------------------------------

class OpCode(IntEnum):
    PUSH_LEAF = 0
    AND = 1
    OR = 2
    NOT = 3


@dataclass(frozen=True)
class CompiledFilter:
    """Postfix ops + one pre-hashed Bloom query per distinct leaf
    (reference filter_query.py:260-277)."""

    ops: tuple
    leaves: tuple

    def max_stack_depth(self) -> int:
        depth = peak = 0
        for op, _ in self.ops:
            if op == OpCode.PUSH_LEAF:
                depth += 1
            elif op in (OpCode.AND, OpCode.OR):
                depth -= 1
            peak = max(peak, depth)
        if depth != 1:
            raise ValueError(f"unbalanced operation array (net depth {depth})")
        return peak


_COMPILED: "OrderedDict[tuple, CompiledFilter]" = OrderedDict()
_COMPILED_MAX = 8192
_COMPILED_LOCK = threading.Lock()


def compile_filter(expr: FilterExpr, params: BloomParams) -> CompiledFilter:
    """``_compile_filter`` behind an LRU cache keyed by the (immutable) expression and the
    Bloom parameters: serving traffic repeats filters, and a compiled filter is immutable.
    Unhashable expressions are compiled directly."""
    try:
        key = (expr, params)
        hash(key)
    except TypeError:
        return _compile_filter(expr, params)
    with _COMPILED_LOCK:  # the reference server compiles from several worker threads
        hit = _COMPILED.get(key)
        if hit is not None:
            _COMPILED.move_to_end(key)
            return hit
    cf = _compile_filter(expr, params)
    with _COMPILED_LOCK:
        _COMPILED[key] = cf
        while len(_COMPILED) > _COMPILED_MAX:
            _COMPILED.popitem(last=False)
    return cf


def _compile_filter(expr: FilterExpr, params: BloomParams) -> CompiledFilter:
    """Post-order lowering with per-(fid, value) de-duplication (reference
    filter_query.py:280-311); all leaf positions hashed in one ``fb_hash_leaves`` call."""
    leaf_index: dict[tuple[int, int], int] = {}
    keys: list[tuple[int, int]] = []
    ops: list[tuple[OpCode, int]] = []

    def emit(node):
        if isinstance(node, Leaf):
            key = (int(node.feature_id), int(node.value))
            idx = leaf_index.get(key)
            if idx is None:
                idx = leaf_index[key] = len(keys)
                keys.append(key)
            ops.append((OpCode.PUSH_LEAF, idx))
        elif isinstance(node, Not):
            emit(node.child)
            ops.append((OpCode.NOT, 0))
        elif isinstance(node, (And, Or)):
            code = OpCode.AND if isinstance(node, And) else OpCode.OR
            emit(node.children[0])
            for child in node.children[1:]:
                emit(child)
                ops.append((code, 0))
        else:
            raise TypeError(f"not a filter node: {node!r}")

    emit(expr)
    pos, cnt = hash_positions_batch([k[0] for k in keys], [k[1] for k in keys], params)
    leaves = tuple((f, v, QueryBloom(tuple(int(p) for p in pos[i, : cnt[i]])))
                   for i, (f, v) in enumerate(keys))
    cf = CompiledFilter(ops=tuple(ops), leaves=leaves)
    cf.max_stack_depth()
    return cf


# register-machine opcodes (include/filtra_b200.h fb_ropcode)
ROP_PUSH, ROP_PUSHN, ROP_ANDL, ROP_ORL, ROP_ANDS, ROP_ORS, ROP_NOT, ROP_NOP = range(8)
ROP_MAX_LEAVES = 1 << 13
ROP_ALIGN = 8


def lower_to_register_ops(ops: list[tuple[int, int]]) -> tuple[list[int], int]:
    """Peephole-lower postfix ``(opcode, global_leaf)`` ops to the register machine the
    tensor-core epilogue runs: ``PUSH l; AND`` -> ``ANDL l``, ``PUSH l; OR`` -> ``ORL l``,
    ``PUSH l; NOT`` -> ``PUSHN l``. Returns (encoded u16 ops, max stack depth)."""
    out: list[tuple[int, int]] = []
    for op, leaf in ops:
        if op == OpCode.PUSH_LEAF:
            out.append((ROP_PUSH, leaf))
        elif op == OpCode.NOT:
            if out and out[-1][0] == ROP_PUSH:
                out[-1] = (ROP_PUSHN, out[-1][1])
            else:
                out.append((ROP_NOT, 0))
        else:
            combine_leaf = ROP_ANDL if op == OpCode.AND else ROP_ORL
            if out and out[-1][0] == ROP_PUSH and len(out) >= 2:
                out[-1] = (combine_leaf, out[-1][1])
            else:
                out.append((ROP_ANDS if op == OpCode.AND else ROP_ORS, 0))
    depth = peak = 0
    for code, _ in out:
        if code in (ROP_PUSH, ROP_PUSHN):
            depth += 1
        elif code in (ROP_ANDS, ROP_ORS):
            depth -= 1
        peak = max(peak, depth)
    return [(c << 13) | l for c, l in out], peak


CNF_MAX_WORDS = 8    # leaf columns per batch <= 256
CNF_MAX_GROUPS = 8


def cnf_groups(ops: list[tuple[int, int]]):
    """Conjunctive normal form of a postfix program over (global) leaves, or None.

    NOTs are pushed down to literals (De Morgan; exact for bitwise masks because the
    result is ANDed with validity at the end), same-operator nodes are flattened, and the
    result must be an AND of ORs of literals. Returns a list of groups, each a list of
    ``(leaf, negated)`` literals."""
    stack: list = []
    for op, leaf in ops:
        if op == OpCode.PUSH_LEAF:
            stack.append(("lit", leaf, False))
        elif op == OpCode.NOT:
            stack.append(("not", stack.pop()))
        else:
            rhs = stack.pop()
            lhs = stack.pop()
            stack.append(("and" if op == OpCode.AND else "or", [lhs, rhs]))
    if len(stack) != 1:
        return None

    def nnf(node, neg):
        kind = node[0]
        if kind == "lit":
            return ("lit", node[1], node[2] != neg)
        if kind == "not":
            return nnf(node[1], not neg)
        flip = {"and": "or", "or": "and"}
        k = flip[kind] if neg else kind
        kids = []
        for child in node[1]:
            c = nnf(child, neg)
            kids.extend(c[1] if c[0] == k else [c])
        return (k, kids)

    root = nnf(stack[0], False)

    def clause(node):
        if node[0] == "lit":
            return [(node[1], node[2])]
        if node[0] == "or" and all(c[0] == "lit" for c in node[1]):
            return [(c[1], c[2]) for c in node[1]]
        return None

    if root[0] == "and":
        groups = [clause(c) for c in root[1]]
        return None if any(g is None for g in groups) else groups
    g = clause(root)
    return None if g is None else [g]


def _pack_cnf(cnf, leaf_fid):
    """CNF column layout of a batch. Literals (leaf, negated) become columns; columns are
    grouped by feature id and the features bin-packed (first fit, decreasing) into 64-column
    windows, so a group whose literals share a feature -- the usual ``f in S`` group --
    tests one aligned u32 pair of the item's column bits. Falls back to first-seen order when
    the windows would need more than CNF_MAX_WORDS words. Returns the FilterBatch kwargs, or
    {} when the batch does not fit the CNF limits."""
    lits: dict[tuple[int, bool], int] = {}
    for groups in cnf:
        for g in groups:
            for lit in g:
                lits.setdefault(lit, len(lits))
    gmax = max(len(groups) for groups in cnf)
    if gmax > CNF_MAX_GROUPS:
        return {}
    by_fid: dict[int, list] = {}
    for lit in lits:
        by_fid.setdefault(leaf_fid[lit[0]], []).append(lit)
    bins: list[list] = []
    if all(len(v) <= 64 for v in by_fid.values()):
        for fid in sorted(by_fid, key=lambda f: (-len(by_fid[f]), f)):
            for b in bins:
                if len(b) + len(by_fid[fid]) <= 64:
                    b.extend(by_fid[fid])
                    break
            else:
                bins.append(list(by_fid[fid]))
    if bins and 2 * len(bins) <= CNF_MAX_WORDS:
        cols = {lit: 64 * bi + i for bi, b in enumerate(bins) for i, lit in enumerate(b)}
        n_cols = 64 * (len(bins) - 1) + len(bins[-1])
    else:
        cols, n_cols = dict(lits), len(lits)
    words = (n_cols + 31) // 32
    if words > CNF_MAX_WORDS:
        return {}
    qmask = np.zeros((len(cnf), gmax, words), dtype=np.uint32)
    for q, groups in enumerate(cnf):
        for gi, g in enumerate(groups):
            for lit in g:
                c = cols[lit]
                qmask[q, gi, c >> 5] |= np.uint32(1 << (c & 31))
    col_leaf = np.zeros(n_cols, dtype=np.int16)  # padding columns: leaf 0, never referenced
    for (leaf, neg), c in cols.items():
        col_leaf[c] = ~leaf if neg else leaf
    nz = qmask != 0
    first = np.where(nz.any(axis=2), nz.argmax(axis=2), 0)
    last = np.where(nz.any(axis=2), words - 1 - nz[:, :, ::-1].argmax(axis=2), 0)
    windowed = int(gmax <= 4 and bool(np.all((first >> 1) == (last >> 1))))
    return dict(col_leaf=col_leaf, qmask=qmask,
                qgroups=np.array([len(g) for g in cnf], dtype=np.int32),
                cnf_words=words, cnf_gmax=gmax, cnf_windowed=windowed)


class FilterBatch:
    """Device bytecode for a batch of compiled filters (one per query, ``None`` =
    unfiltered), mirroring ``fb_filter_prog_t`` (include/filtra_b200.h):

    * postfix ops ``(opcode << 14) | leaf`` with leaves de-duplicated across the batch
      (SIMT scan / ``fb_filter_eval``);
    * the register-machine form for the tensor-core scan: the batch's distinct planes
      (staged per tile in ``plane_list`` order), each leaf's positions as indices into
      that list, and peephole-lowered ``rops``.
    """

    def __init__(self, leaf_pos, op_offset, ops, max_stack, push_leaf_bits, *,
                 plane_list=None, leaf_slot=None, rop_offset=None, rops=None, rmax_stack=0,
                 col_leaf=None, qmask=None, qgroups=None, cnf_words=0, cnf_gmax=0,
                 cnf_windowed=0):
        self.n_queries = len(op_offset) - 1
        self.n_leaves = leaf_pos.shape[0]
        self.k_max = leaf_pos.shape[1]
        self.max_stack = max_stack
        self.host_leaf_pos = np.ascontiguousarray(leaf_pos, dtype=np.int16)
        self.host_op_offset = np.ascontiguousarray(op_offset, dtype=np.int32)
        self.host_ops = np.ascontiguousarray(ops, dtype=np.uint16)
        self.host_plane_list = (np.ascontiguousarray(plane_list, dtype=np.int16)
                                if plane_list is not None else None)
        self.host_leaf_slot = (np.ascontiguousarray(leaf_slot, dtype=np.int16)
                               if leaf_slot is not None else None)
        self.host_rop_offset = (np.ascontiguousarray(rop_offset, dtype=np.int32)
                                if rop_offset is not None else None)
        self.host_rops = np.ascontiguousarray(rops, dtype=np.uint16) if rops is not None else None
        self.rmax_stack = rmax_stack
        # CNF form (all queries AND-of-OR-of-literals): literal columns (leaf, or ~leaf when
        # negated), per query per group a column bitmask, and the group count per query
        self.host_col_leaf = (np.ascontiguousarray(col_leaf, dtype=np.int16)
                              if col_leaf is not None else None)
        self.host_qmask = np.ascontiguousarray(qmask, dtype=np.uint32) if qmask is not None else None
        self.host_qgroups = (np.ascontiguousarray(qgroups, dtype=np.int32)
                             if qgroups is not None else None)
        self.cnf_words = cnf_words
        self.cnf_gmax = cnf_gmax
        # 1 when every group's columns lie in one 64-column window (u32 words 2j, 2j+1) and
        # no query has more than 4 groups: the scan's register-resident filter test
        self.cnf_windowed = cnf_windowed
        # per query: sum over PUSH_LEAF ops of |set_bits| (FilterStats.words_read per word)
        self.push_leaf_bits = push_leaf_bits
        self._dev = None

    @property
    def n_planes(self) -> int:
        return 0 if self.host_plane_list is None else int(self.host_plane_list.size)

    @property
    def is_cnf(self) -> bool:
        return self.host_col_leaf is not None

    def host_arrays(self) -> list[np.ndarray]:
        arrs = [self.host_leaf_pos, self.host_op_offset, self.host_ops.view(np.int16)]
        if self.host_rops is not None:
            arrs += [self.host_plane_list, self.host_leaf_slot, self.host_rop_offset,
                     self.host_rops.view(np.int16)]
            if self.host_col_leaf is not None:
                arrs += [self.host_col_leaf, self.host_qmask.view(np.int32), self.host_qgroups]
        return arrs

    def clone_host(self) -> "FilterBatch":
        """A copy sharing the (read-only) host arrays, with no device arrays of its own yet."""
        c = copy.copy(self)
        c._dev = None
        return c

    def pin(self) -> "FilterBatch":
        """Stage the host arrays in pinned memory (asynchronous H2D copies); idempotent."""
        if getattr(self, "_pinned", None) is None:
            self._pinned = [torch.from_numpy(a).pin_memory() for a in self.host_arrays()]
        return self

    def pinned_arrays(self) -> list[torch.Tensor]:
        """Host arrays as tensors (pinned after ``pin()``; pageable otherwise)."""
        p = getattr(self, "_pinned", None)
        return p if p is not None else [torch.from_numpy(a) for a in self.host_arrays()]

    def to_device(self) -> "FilterBatch":
        """Upload the bytecode (one H2D copy per array); idempotent."""
        if self._dev is None:
            dev = device()
            self._dev = tuple(torch.from_numpy(a).to(dev) for a in self.host_arrays())
        return self

    @property
    def leaf_pos(self) -> torch.Tensor:
        return self.to_device()._dev[0]

    @property
    def op_offset(self) -> torch.Tensor:
        return self.to_device()._dev[1]

    @property
    def ops(self) -> torch.Tensor:
        return self.to_device()._dev[2]

    @classmethod
    def pack(cls, filters, params: BloomParams) -> "FilterBatch":
        if params.m_bits > 32767:
            raise NotImplementedError("device filter evaluation supports m_bits <= 32767")
        glob: dict[tuple[int, int], int] = {}
        leaf_rows: list[tuple[int, ...]] = []
        leaf_fid: list[int] = []
        ops: list[int] = []
        offsets = [0]
        rops: list[int] = []
        rop_offsets = [0]
        push_bits = []
        max_stack = 1
        rmax = 0
        cnf: list | None = []
        for cf in filters:
            nbits = 0
            if cf is not None:
                local = []
                for fid, val, qb in cf.leaves:
                    key = (int(fid), int(val))
                    g = glob.get(key)
                    if g is None:
                        g = glob[key] = len(leaf_rows)
                        leaf_rows.append(tuple(qb.set_bits))
                        leaf_fid.append(int(fid))
                    local.append(g)
                gops = []
                for op, arg in cf.ops:
                    if op == OpCode.PUSH_LEAF:
                        ops.append(local[arg])
                        gops.append((int(op), local[arg]))
                        nbits += len(cf.leaves[arg][2].set_bits)
                    else:
                        ops.append(int(op) << 14)
                        gops.append((int(op), 0))
                max_stack = max(max_stack, cf.max_stack_depth())
                enc, depth = lower_to_register_ops(gops)
                enc += [ROP_NOP << 13] * (-len(enc) % ROP_ALIGN)
                rops.extend(enc)
                rmax = max(rmax, depth)
                if cnf is not None:
                    groups = cnf_groups(gops)
                    cnf = None if groups is None else cnf + [groups]
            elif cnf is not None:
                cnf.append([])
            offsets.append(len(ops))
            rop_offsets.append(len(rops))
            push_bits.append(nbits)
        if len(leaf_rows) > _native.FB_MAX_LEAVES:
            raise NotImplementedError(f"more than {_native.FB_MAX_LEAVES} distinct leaves in a batch")
        if max_stack > _native.FB_MAX_STACK:
            raise NotImplementedError(f"filter stack depth {max_stack} > {_native.FB_MAX_STACK}")
        k_max = max([1] + [len(r) for r in leaf_rows])
        leaf_pos = np.full((max(1, len(leaf_rows)), k_max), -1, dtype=np.int16)
        for i, r in enumerate(leaf_rows):
            leaf_pos[i, : len(r)] = r
        planes = np.unique(leaf_pos[leaf_pos >= 0]).astype(np.int16)
        slot_of = {int(p): i for i, p in enumerate(planes)}
        leaf_slot = np.full_like(leaf_pos, -1)
        for i, r in enumerate(leaf_rows):
            leaf_slot[i, : len(r)] = [slot_of[p] for p in r]
        reg = len(leaf_rows) <= ROP_MAX_LEAVES
        cnf_kw = {}
        if reg and cnf is not None and any(cnf):
            cnf_kw = _pack_cnf(cnf, leaf_fid)
        elif reg and not leaf_rows:
            # no query is filtered: the CNF form with zero groups per query (one unused
            # column) lets the tensor-core scan take its per-hit kernel, where every gated
            # pair survives
            cnf_kw = dict(col_leaf=np.zeros(1, dtype=np.int16),
                          qmask=np.zeros((len(cnf), 1, 1), dtype=np.uint32),
                          qgroups=np.zeros(len(cnf), dtype=np.int32),
                          cnf_words=1, cnf_gmax=1, cnf_windowed=1)
        return cls(leaf_pos, np.array(offsets, dtype=np.int32),
                   np.array(ops if ops else [0], dtype=np.uint16), max_stack,
                   np.array(push_bits, dtype=np.int64),
                   plane_list=planes if (reg and planes.size) else (np.zeros(1, np.int16) if reg else None),
                   leaf_slot=leaf_slot if reg else None,
                   rop_offset=np.array(rop_offsets, dtype=np.int32) if reg else None,
                   rops=(np.array(rops if rops else [ROP_NOP << 13] * ROP_ALIGN, dtype=np.uint16)
                         if reg else None),
                   rmax_stack=rmax, **cnf_kw)

    @classmethod
    def from_leaf(cls, qb: QueryBloom, params: BloomParams) -> "FilterBatch":
        cf = CompiledFilter(ops=((OpCode.PUSH_LEAF, 0),), leaves=((0, 0, qb),))
        return cls.pack([cf], params)

    # scalar metadata of the device form, in the order ``struct_from`` reads it
    META_FIELDS = ("n_queries", "n_leaves", "k_max", "max_stack", "has_rops", "n_planes",
                   "rmax_stack", "n_rops", "is_cnf", "n_cols", "cnf_words", "cnf_gmax",
                   "cnf_windowed")

    def meta(self) -> list[int]:
        has_rops = self.host_rops is not None
        return [self.n_queries, self.n_leaves, self.k_max, self.max_stack, int(has_rops),
                self.n_planes if has_rops else 0, self.rmax_stack if has_rops else 0,
                int(self.host_rops.size) if has_rops else 0, int(self.is_cnf),
                int(self.host_col_leaf.size) if self.is_cnf else 0, int(self.cnf_words),
                int(self.cnf_gmax), int(self.cnf_windowed)]

    def device_arrays(self) -> list[torch.Tensor]:
        return list(self.to_device()._dev)

    @staticmethod
    def struct_from(d, meta) -> _native.FbFilterProg:
        """``fb_filter_prog_t`` from device arrays (``host_arrays()`` order) and ``meta()``
        (the custom-op boundary passes exactly these two)."""
        (nq, n_leaves, k_max, max_stack, has_rops, n_planes, rmax, n_rops, is_cnf, n_cols,
         cnf_words, cnf_gmax, cnf_windowed) = (int(x) for x in meta)
        need = 3 + (4 if has_rops else 0) + (3 if is_cnf else 0)
        if len(d) != need:
            raise ValueError(f"filter batch: {len(d)} device arrays, expected {need}")
        if has_rops:
            extra = (n_planes, rmax, n_rops, 0, d[3].data_ptr(), d[4].data_ptr(),
                     d[5].data_ptr(), d[6].data_ptr())
        else:
            extra = (0, 0, 0, 0, None, None, None, None)
        if is_cnf:
            cnf = (n_cols, cnf_words, cnf_gmax, cnf_windowed, d[7].data_ptr(), d[8].data_ptr(),
                   d[9].data_ptr())
        else:
            cnf = (0, 0, 0, 0, None, None, None)
        return _native.FbFilterProg(nq, n_leaves, k_max, max_stack, d[0].data_ptr(),
                                    d[1].data_ptr(), d[2].data_ptr(), *extra, *cnf)

    def struct(self) -> _native.FbFilterProg:
        return FilterBatch.struct_from(self.to_device()._dev, self.meta())

    def evaluate(self, bloom: BloomIndex, valid, w0: int, w1: int,
                 apply_valid: bool = True) -> np.ndarray:
        """``fb_filter_eval`` over words [w0, w1) for every query -> numpy u64 [B, w1-w0]."""
        lib = _native.lib()
        dev = device()
        nw = bloom.n_words
        if valid is None:
            valid_t = torch.full((nw,), -1, dtype=torch.int64, device=dev)
        else:
            valid_t = to_dev_u64(valid, dev)
        idx = _native.FbIndex(None, bloom.planes_dev.data_ptr(), valid_t.data_ptr(), None, None,
                              None, nw * 64, nw, 32, 32, bloom.params.m_bits, bloom.params.k_hashes)
        out = torch.empty((self.n_queries, max(0, w1 - w0)), dtype=torch.int64, device=dev)
        prog = self.struct()
        _native.check(lib.fb_filter_eval(idx, prog, int(w0), int(w1), 1 if apply_valid else 0,
                                         out.data_ptr(), _native.stream_ptr()))
        return u64_host(out)


def eval_compiled(cf: CompiledFilter, index: BloomIndex, valid: np.ndarray,
                  slot_range: tuple[int, int] | None = None,
                  stats: FilterStats | None = None) -> np.ndarray:
    """Stack-machine evaluation on the GPU (reference filter_query.py:314-356): NOT is
    ``~x & valid``, the result is ANDed with ``valid``; ``slot_range`` must start on a
    64-slot boundary; a ranged result equals the slice of the full one."""
    if slot_range is None:
        w0, w1 = 0, index.n_words
    else:
        s0, s1 = slot_range
        if s0 % bitset.WORD_BITS:
            raise ValueError(f"slot range start {s0} not 64-aligned")
        w0, w1 = s0 >> 6, (s1 + bitset.WORD_BITS - 1) >> 6
    if stats is not None:
        stats.slots_evaluated += (w1 - w0) * bitset.WORD_BITS
        stats.words_read += sum(len(cf.leaves[a][2].set_bits) for o, a in cf.ops
                                if o == OpCode.PUSH_LEAF and cf.leaves[a][2].set_bits) * (w1 - w0)
    if w1 <= w0:
        return np.empty(0, dtype=np.uint64)
    batch = FilterBatch.pack([cf], index.params)
    return batch.evaluate(index, valid, w0, w1, apply_valid=True)[0].copy()
