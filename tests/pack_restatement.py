"""Test infrastructure: the round-1 Python restatement of ``FilterBatch.pack`` (the batch
device form of compiled filters), kept as the cross-check for the C++ packer
(``fb_pack_postfix`` / ``fb_pack_text``, csrc/fb_pack.cpp). ``pack_py`` returns the same
arrays and scalars the C++ packer produces; tests/test_pack_cpu.py compares them byte for
byte. Not imported by the product package."""

from __future__ import annotations

import numpy as np

from paper_2511_14881_b200.filter_query import OpCode

FB_MAX_LEAVES = 16384
FB_MAX_STACK = 64

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



def pack_py(filters, params):
    """FilterBatch kwargs for ``filters`` (list of CompiledFilter or None)."""
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
    if len(leaf_rows) > FB_MAX_LEAVES:
        raise NotImplementedError(f"more than {FB_MAX_LEAVES} distinct leaves in a batch")
    if max_stack > FB_MAX_STACK:
        raise NotImplementedError(f"filter stack depth {max_stack} > {FB_MAX_STACK}")
    k_max = max([1] + [len(r) for r in leaf_rows])
    leaf_pos = np.full((max(1, len(leaf_rows)), k_max), -1, dtype=np.int32)
    for i, r in enumerate(leaf_rows):
        leaf_pos[i, : len(r)] = r
    planes = np.unique(leaf_pos[leaf_pos >= 0]).astype(np.int32)
    slot_of = {int(p): i for i, p in enumerate(planes)}
    leaf_slot = np.full(leaf_pos.shape, -1, dtype=np.int16)
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
    return dict(leaf_pos=leaf_pos, op_offset=np.array(offsets, dtype=np.int32),
                ops=np.array(ops if ops else [0], dtype=np.uint16), max_stack=max_stack,
                push_leaf_bits=np.array(push_bits, dtype=np.int64),
                plane_list=planes if (reg and planes.size) else (np.zeros(1, np.int32) if reg else None),
               leaf_slot=leaf_slot if reg else None,
               rop_offset=np.array(rop_offsets, dtype=np.int32) if reg else None,
               rops=(np.array(rops if rops else [ROP_NOP << 13] * ROP_ALIGN, dtype=np.uint16)
                     if reg else None),
               rmax_stack=rmax, **cnf_kw)

