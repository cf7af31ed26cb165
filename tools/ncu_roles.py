"""Per-role instruction counts and stall reasons of a warp-specialised kernel from an ncu
capture: joins the SASS source page with ``nvdisasm -gi`` line info (innermost source line)
and buckets by source-line ranges.

    python tools/ncu_roles.py rep.ncu-rep kernel-regex cubin-sass src.cu tiles name:lo-hi ...
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


OUTER = "--outer" in sys.argv


def line_map(path, kernel):
    out, inside, line, in_run = {}, False, None, False
    for raw in open(path):
        if raw.startswith("//-----") and ".text." in raw:
            inside = kernel in raw
            continue
        if not inside:
            continue
        if raw.lstrip().startswith("//## File"):
            pairs = re.findall(r'"[^"]*?([^/"]+)", line (\d+)', raw)
            own = [ln for f, ln in pairs if f.endswith(".cu")]
            if not in_run:
                line = int(own[-1] if OUTER else own[0]) if own else None
            in_run = True
            continue
        in_run = False
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", raw)
        if m:
            out[int(m.group(1), 16)] = line
    return out


def main():
    rep, kre, sass, src, tiles = sys.argv[1:6]
    ranges = []
    for spec in [x for x in sys.argv[6:] if x != "--outer"]:
        name, rng = spec.split(":")
        lo, hi = rng.split("-")
        ranges.append((name, int(lo), int(hi)))
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "sass", "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[1]
    ia, iex = h.index("Address"), h.index("Instructions Executed")
    stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    import os
    lm = line_map(sass, os.environ.get("SASS_KERNEL", kre.split("|")[0]))
    ex, st = defaultdict(float), defaultdict(lambda: defaultdict(float))
    base = None
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        a = int(r[ia], 16)
        base = a if base is None else base
        ln = lm.get(a - base)
        name = "other"
        if ln is not None:
            for n, lo, hi in ranges:
                if lo <= ln <= hi:
                    name = n
                    break
        ex[name] += float(r[iex] or 0)
        for i in stall_cols:
            st[name][h[i][6:]] += float(r[i] or 0)
    t = float(tiles)
    total = sum(ex.values())
    print(f"total {total / t:.0f} warp-instructions per tile")
    for name in [n for n, _, _ in ranges] + ["other"]:
        tot = sum(st[name].values())
        top = sorted(st[name].items(), key=lambda x: -x[1])[:6]
        print(f"{name:9s} {ex[name] / t:7.0f} inst/tile  {tot:8.0f} samples :: " +
              ", ".join(f"{n} {100 * v / tot:.0f}%" for n, v in top if tot))


if __name__ == "__main__":
    main()
