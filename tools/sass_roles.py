"""Per-role instruction and stall breakdown of a warp-specialised kernel: joins an ncu SASS
source page (CSV) with nvdisasm -gi line info and buckets instructions by the kernel-body
line range their outermost call site falls in.

    python tools/sass_roles.py ncu_sass.csv disasm.sass <kernel-substring> name:lo-hi ...
"""
import collections
import csv
import re
import sys


def main():
    ncu_csv, sass, kernel = sys.argv[1:4]
    ranges = []
    for spec in sys.argv[4:]:
        name, rng = spec.split(":")
        lo, hi = rng.split("-")
        ranges.append((name, int(lo), int(hi)))
    chain, inside, run, cur = {}, False, False, None
    for raw in open(sass):
        if raw.startswith("//-----") and ".text." in raw:
            inside = kernel in raw
            continue
        if not inside:
            continue
        if raw.lstrip().startswith("//## File"):
            pairs = re.findall(r'"[^"]*?([^/"]+)", line (\d+)', raw)
            if not run:
                cur = [int(p[1]) for p in pairs if p[0].endswith(".cu")]
            run = True
            continue
        run = False
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", raw)
        if m:
            chain[int(m.group(1), 16)] = (cur, m.group(2))
    rows = list(csv.reader(open(ncu_csv)))
    h = rows[1]
    ia, iex = h.index("Address"), h.index("Instructions Executed")
    ism = h.index("Warp Stall Sampling (All Samples)")
    stall = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    base = int(rows[2][ia], 16)
    agg = collections.defaultdict(lambda: {"ex": 0.0, "sm": 0.0, "st": collections.Counter(),
                                           "op": collections.Counter()})
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        off = int(r[ia], 16) - base
        ch, txt = chain.get(off, (None, ""))
        role = "other"
        if ch:
            o = ch[-1]
            for name, lo, hi in ranges:
                if lo <= o <= hi:
                    role = name
        d = agg[role]
        ex = float(r[iex] or 0)
        d["ex"] += ex
        d["sm"] += float(r[ism] or 0)
        for i in stall:
            d["st"][h[i][6:]] += float(r[i] or 0)
        op = txt.split()
        if op:
            o = op[1] if op[0].startswith("@") else op[0]
            d["op"][o.split(".")[0]] += ex
    te = sum(d["ex"] for d in agg.values())
    ts = sum(d["sm"] for d in agg.values())
    for k, d in sorted(agg.items(), key=lambda x: -x[1]["ex"]):
        st = " ".join(f"{a}={100 * b / max(1, d['sm']):.0f}%" for a, b in d["st"].most_common(3))
        ops = " ".join(f"{a}:{100 * b / max(1, d['ex']):.0f}%" for a, b in d["op"].most_common(6))
        print(f"{k:9s} inst {100 * d['ex'] / te:5.1f}%  samples {100 * d['sm'] / ts:5.1f}%  | {st}\n"
              f"          ops: {ops}")
    return agg


if __name__ == "__main__":
    main()
