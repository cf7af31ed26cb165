"""Join an ncu SASS source page (CSV) with ``nvdisasm -g`` line info and sum executed
instructions / stall samples per CUDA source line (the ncu CUDA view of our captures
carries no metrics).

    python tools/sass_lines.py ncu_sass.csv disasm.sass <mangled-kernel-substring> [--top N]
                               [--inner] [--src paper_2511_14881_b200/csrc/<file>.cu]
"""
import csv
import re
import sys
from collections import defaultdict


def line_map(sass_path, kernel, inner=False):
    out, cur, inside, line, in_run = {}, None, False, None, False
    for raw in open(sass_path):
        if raw.startswith("//-----") and ".text." in raw:
            inside = kernel in raw
            continue
        if not inside:
            continue
        if raw.lstrip().startswith("//## File"):
            pairs = re.findall(r'"[^"]*?([^/"]+)", line (\d+)', raw)
            own = [ln for f, ln in pairs if f.endswith(".cu")]
            # outermost caller (the kernel body), or with --inner the innermost .cu line
            # (nvdisasm repeats the location as a run of comments, innermost first)
            if not (inner and in_run):
                line = (own[0] if inner else own[-1]) if own else (pairs[-1][1] if pairs else None)
            in_run = True
            continue
        in_run = False
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", raw)
        if m:
            out[int(m.group(1), 16)] = line
    return out


def main():
    ncu_csv, sass, kernel = sys.argv[1:4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 50
    lm = line_map(sass, kernel, "--inner" in sys.argv)
    rows = list(csv.reader(open(ncu_csv)))
    h = rows[1]
    ia, iex = h.index("Address"), h.index("Instructions Executed")
    ism = h.index("Warp Stall Sampling (All Samples)")
    base = None
    ex, sm = defaultdict(float), defaultdict(float)
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        a = int(r[ia], 16)
        base = a if base is None else base
        ln = lm.get(a - base, "?")
        ex[ln] += float(r[iex] or 0)
        sm[ln] += float(r[ism] or 0)
    te, ts = sum(ex.values()), sum(sm.values())
    path = (sys.argv[sys.argv.index("--src") + 1] if "--src" in sys.argv
            else "paper_2511_14881_b200/csrc/fb_tc_kernel.cu")
    src = open(path).read().split("\n")
    keys = sorted(ex, key=lambda k: -(ex[k] / te + sm[k] / ts))[:top]
    for k in keys:
        n = int(k.split("<")[0]) if k not in ("?", None) else 0
        print(f"{str(k):>10} {100*ex[k]/te:6.2f}% ex {100*sm[k]/ts:6.2f}% smp | {src[n-1].strip()[:80] if n else ''}")


if __name__ == "__main__":
    main()
