"""Filter expressions: grammar, AST, postfix compiler, and the GPU evaluator.

Grammar and lowering follow the reference (filter_query.py:1-311): OR binds tighter
than AND, NOT tightest; AND/OR children are chained pairwise in post-order; leaves
are de-duplicated per filter. ``FilterBatch`` packs a batch of compiled filters
into the device bytecode consumed by the fused scan (leaves de-duplicated across
the whole batch); the packing -- and, for request texts, parsing and compilation -- runs in
C++ (csrc/fb_pack.cpp). ``eval_compiled`` runs ``fb_filter_eval``.
"""

from __future__ import annotations

import copy
import ctypes
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


# --- batch device form (built by the C++ packer, csrc/fb_pack.cpp) ----------------------

def _flat_program(cf: CompiledFilter):
    """``cf`` as postfix arrays: opcode u8, leaf fid / value u64 per op, and the pushed
    leaf's positions (its QueryBloom.set_bits, so a compiled filter carrying its own
    positions -- e.g. ``bloom_eval_leaf``'s single leaf -- keeps them) as per-op counts +
    a flat int32 array; cached on the (immutable) compiled filter."""
    flat = cf.__dict__.get("_flat")
    if flat is None:
        n = len(cf.ops)
        codes = np.fromiter((int(o) for o, _ in cf.ops), dtype=np.uint8, count=n)
        args = np.fromiter((int(a) for _, a in cf.ops), dtype=np.int64, count=n)
        lf = np.array([int(l[0]) for l in cf.leaves] or [0], dtype=np.uint64)
        lv = np.array([int(l[1]) for l in cf.leaves] or [0], dtype=np.uint64)
        lpos = [np.asarray(l[2].set_bits, dtype=np.int64) for l in cf.leaves]
        push = codes == OpCode.PUSH_LEAF
        a = np.where(push, args, 0)
        cnt = np.array([len(lpos[int(x)]) if p else 0 for x, p in zip(a, push)], dtype=np.int64)
        pos = (np.concatenate([lpos[int(x)] for x, p in zip(a, push) if p])
               if cnt.sum() else np.zeros(0, np.int64))
        if pos.size and (pos.min() < 0 or pos.max() >= 1 << 31):
            raise ValueError("leaf position outside the int32 range")
        flat = (codes, np.where(push, lf[a], 0).astype(np.uint64),
                np.where(push, lv[a], 0).astype(np.uint64), cnt, pos.astype(np.int32))
        object.__setattr__(cf, "_flat", flat)
    return flat


_PACK_ARRAYS = ("leaf_pos", "op_offset", "ops", "plane_list", "leaf_slot", "rop_offset", "rops",
                "col_leaf", "qmask", "qgroups", "push_leaf_bits")
_PACK_DTYPES = (np.int32, np.int32, np.uint16, np.int32, np.int16, np.int32, np.uint16, np.int16,
                np.uint32, np.int32, np.int64)


def _take_pack(handle) -> dict:
    """FilterBatch kwargs from a ``fb_pack_t`` (arrays copied out, handle freed)."""
    lib = _native.load_library()
    try:
        meta = (ctypes.c_int64 * 16)()
        _native.check(lib.fb_pack_meta(handle, meta))
        meta = list(meta)
        arrs = {}
        for which, (name, dt) in enumerate(zip(_PACK_ARRAYS, _PACK_DTYPES)):
            data, n = ctypes.c_void_p(), ctypes.c_int64()
            _native.check(lib.fb_pack_array(handle, which, ctypes.byref(data), ctypes.byref(n)))
            if n.value == 0 or not data.value:
                arrs[name] = np.zeros(0, dtype=dt)
                continue
            buf = (ctypes.c_char * (n.value * np.dtype(dt).itemsize)).from_address(data.value)
            arrs[name] = np.frombuffer(buf, dtype=dt).copy()
    finally:
        lib.fb_pack_free(handle)
    nq, rows, k_max, max_stack, has_rops = meta[0:5]
    rmax, is_cnf, words, gmax, windowed = meta[6], meta[8], meta[10], meta[11], meta[12]
    kw = dict(leaf_pos=arrs["leaf_pos"].reshape(rows, k_max), op_offset=arrs["op_offset"],
              ops=arrs["ops"], max_stack=max_stack, push_leaf_bits=arrs["push_leaf_bits"])
    if has_rops:
        kw.update(plane_list=arrs["plane_list"], leaf_slot=arrs["leaf_slot"].reshape(rows, k_max),
                  rop_offset=arrs["rop_offset"], rops=arrs["rops"], rmax_stack=rmax)
    if is_cnf:
        kw.update(col_leaf=arrs["col_leaf"], qmask=arrs["qmask"].reshape(nq, gmax, words),
                  qgroups=arrs["qgroups"], cnf_words=words, cnf_gmax=gmax,
                  cnf_windowed=windowed)
    return kw


_VOCAB_LOCK = threading.Lock()


class _NativeVocab:
    def __init__(self, vocab):
        lib = _native.load_library()
        feats = [(k, v) for k, v in vocab.feature_ids.items() if 0 <= int(v) < 1 << 64]
        vals = [(k, v) for k, v in vocab.values.items() if 0 <= int(v) < 1 << 64]
        fn = (ctypes.c_char_p * max(1, len(feats)))(*[k.encode() for k, _ in feats])
        fi = np.array([int(v) for _, v in feats] or [0], dtype=np.uint64)
        vn = (ctypes.c_char_p * max(1, len(vals)))(*[k.encode() for k, _ in vals])
        vi = np.array([int(v) for _, v in vals] or [0], dtype=np.uint64)
        h = ctypes.c_void_p()
        _native.check(lib.fb_vocab_create(len(feats), fn, fi.ctypes.data, len(vals), vn,
                                          vi.ctypes.data, ctypes.byref(h)))
        self.handle = h
        self.sizes = (len(vocab.feature_ids), len(vocab.values))

    def __del__(self):
        try:
            _native.load_library().fb_vocab_free(self.handle)
        except Exception:
            pass


def _native_vocab(vocab):
    if vocab is None:
        return None
    # cached on the (frozen, unhashable) vocabulary object itself; rebuilt if its dicts grew
    with _VOCAB_LOCK:
        nv = vocab.__dict__.get("_fb_native")
        if nv is None or nv.sizes != (len(vocab.feature_ids), len(vocab.values)):
            nv = _NativeVocab(vocab)
            object.__setattr__(vocab, "_fb_native", nv)
        return nv



class FilterBatch:
    """Device bytecode for a batch of compiled filters (one per query, ``None`` =
    unfiltered), mirroring ``fb_filter_prog_t`` (include/filtra_b200.h):

    * postfix ops ``(opcode << 14) | leaf`` with leaves de-duplicated across the batch
      (SIMT scan / ``fb_filter_eval``);
    * the register-machine form for the tensor-core scan: the batch's distinct planes
      (staged per tile in ``plane_list`` order), each leaf's positions as indices into
      that list, and peephole-lowered ``rops``.
    """

    def __init__(self, leaf_pos, op_offset, ops, max_stack, push_leaf_bits=None, *,
                 plane_list=None, leaf_slot=None, rop_offset=None, rops=None, rmax_stack=0,
                 col_leaf=None, qmask=None, qgroups=None, cnf_words=0, cnf_gmax=0,
                 cnf_windowed=0):
        self.n_queries = len(op_offset) - 1
        self.n_leaves = leaf_pos.shape[0]
        self.k_max = leaf_pos.shape[1]
        self.max_stack = max_stack
        self.host_leaf_pos = np.ascontiguousarray(leaf_pos, dtype=np.int32)
        self.host_op_offset = np.ascontiguousarray(op_offset, dtype=np.int32)
        self.host_ops = np.ascontiguousarray(ops, dtype=np.uint16)
        self.host_plane_list = (np.ascontiguousarray(plane_list, dtype=np.int32)
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
        """Batch device form of compiled filters (``None`` = unfiltered), packed in C++
        (``fb_pack_postfix``): leaves de-duplicated across the batch, postfix and register
        ops, the CNF column windows."""
        flats = [None if cf is None else _flat_program(cf) for cf in filters]
        nq = len(flats)
        off = np.zeros(nq + 1, dtype=np.int64)
        for q, f in enumerate(flats):
            off[q + 1] = off[q] + (0 if f is None else len(f[0]))
        live = [f for f in flats if f is not None]
        codes = np.concatenate([f[0] for f in live]) if live else np.zeros(1, np.uint8)
        fid = np.concatenate([f[1] for f in live]) if live else np.zeros(1, np.uint64)
        val = np.concatenate([f[2] for f in live]) if live else np.zeros(1, np.uint64)
        cnt = np.concatenate([f[3] for f in live]) if live else np.zeros(1, np.int64)
        pos_off = np.zeros(cnt.size + 1, dtype=np.int64)
        np.cumsum(cnt, out=pos_off[1:])
        pos = np.concatenate([f[4] for f in live] + [np.zeros(1, np.int32)])
        h = ctypes.c_void_p()
        _native.check(_native.load_library().fb_pack_postfix(
            nq, off.ctypes.data, codes.ctypes.data, fid.ctypes.data, val.ctypes.data,
            pos_off.ctypes.data, pos.ctypes.data, params.m_bits, params.k_hashes,
            ctypes.byref(h)))
        return cls(**_take_pack(h))

    @classmethod
    def from_text(cls, texts, vocab: Vocabulary | None, params: BloomParams) -> "FilterBatch":
        """Parse + compile + pack one filter text per query (``None`` / ``""`` = unfiltered)
        in C++ (``fb_pack_text``): the serving path for request filters (reference
        serve.py:204-205 -> parse_filter -> compile_filter, for a whole batch). A text the
        native parser does not accept is re-parsed by ``parse_filter`` (the reference
        grammar), which raises the reference's exception; text that only the Unicode-aware
        Python tokenizer accepts is compiled in Python and packed through the same C++
        packer."""
        texts = list(texts)
        enc = [t.encode("utf-8") if t else None for t in texts]
        arr = (ctypes.c_char_p * max(1, len(enc)))(*enc)
        nv = _native_vocab(vocab)
        h, bad = ctypes.c_void_p(), ctypes.c_int32(-1)
        lib = _native.load_library()
        rc = lib.fb_pack_text(len(enc), arr, nv.handle if nv is not None else None,
                              params.m_bits, params.k_hashes, ctypes.byref(h), ctypes.byref(bad))
        if rc == _native.FB_ERR_PARSE:
            parse_filter(texts[bad.value], vocab)  # raises the reference's exception
            exprs = [parse_filter(t, vocab) if t else None for t in texts]
            return cls.pack([compile_filter(e, params) if e is not None else None for e in exprs],
                            params)
        _native.check(rc)
        return cls(**_take_pack(h))

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
