"""Hot SASS regions of an ncu source-page CSV (``ncu -i X --page source --csv --print-source
sass``): instructions executed and stall samples per instruction, summed over windows.

    python tools/sass_hot.py sass.csv [--top N] [--window W]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ia, isrc = h.index("Address"), h.index("Source")
    iex = h.index("Instructions Executed")
    ism = h.index("Warp Stall Sampling (All Samples)")
    stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    data = []
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        ex = float(r[iex] or 0)
        sm = float(r[ism] or 0)
        st = {h[i][6:]: float(r[i] or 0) for i in stall_cols}
        data.append((r[ia], r[isrc], ex, sm, st))
    tot_ex = sum(d[2] for d in data)
    tot_sm = sum(d[3] for d in data)
    print(f"total inst {tot_ex:.0f}  samples {tot_sm:.0f}")
    for i, d in enumerate(data):
        if d[3] >= tot_sm * 0.004 or d[2] >= tot_ex * 0.004:
            top_st = sorted(d[4].items(), key=lambda x: -x[1])[:2]
            ts = " ".join(f"{k}={v:.0f}" for k, v in top_st if v > 0)
            print(f"{i:5d} {d[0]:>6} {100*d[2]/tot_ex:5.2f}% ex {100*d[3]/tot_sm:5.2f}% smp  {d[1][:60]:60s} {ts}")


if __name__ == "__main__":
    main()


def stall_totals(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    tot = {h[i][6:]: 0.0 for i in cols}
    for r in rows[2:]:
        for i in cols:
            if len(r) > i and r[i]:
                tot[h[i][6:]] += float(r[i])
    s = sum(tot.values())
    return {k: round(100 * v / s, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v}
