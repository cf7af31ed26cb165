"""Summarise ncu captures into profiles/ (run in the build container on files gpurun
brought back).

    python tools/ncu_summary.py report <file.ncu-rep> <out.md> [--traffic-json out.json]
    python tools/ncu_summary.py launches <launches.csv> <out.md>
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM bytes read"),
    ("dram__bytes_write.sum", "DRAM bytes written"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
     "tensor pipe (IMMA) active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v.replace(",", "")) * scale.get(unit, 1)


def report(path, out_md, traffic_json=None):
    head, units, rows = _raw(path)
    lines = [f"# ncu summary: `{path.split('/')[-1]}`", ""]
    for row in rows:
        name = row[head.index("Kernel Name")] if "Kernel Name" in head else "?"
        lines += [f"## {name[:120]}", "", "| metric | value |", "|---|---|"]
        vals = {}
        for key, label in METRICS:
            if key in head:
                i = head.index(key)
                vals[key] = (row[i], units[i])
                lines.append(f"| {label} (`{key}`) | {row[i]} {units[i]} |")
        lines.append("")
        if traffic_json and "dram__bytes_read.sum" in vals:
            rd = to_bytes(*vals["dram__bytes_read.sum"])
            wr = to_bytes(*vals["dram__bytes_write.sum"])
            with open(traffic_json, "w") as f:
                json.dump({"kernel": name, "source": path.split("/")[-1],
                           "dram_bytes_per_launch": int(rd + wr),
                           "dram_bytes_read": int(rd), "dram_bytes_write": int(wr)}, f, indent=1)
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")


def launches(path, out_md):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3, "second": 1e6, "s": 1e6}
        seq.append((r[ki].split("(")[0].replace("fb::<unnamed>::", ""), v * scale.get(r[ui], 1.0)))
    sel = [i for i, s in enumerate(seq) if s[0].endswith(("k_select", "k_select_radix"))]
    lines = [f"# Launch list: `{path.split('/')[-1]}`", "",
             "ncu `gpu__time_duration.sum`, `--clock-control none`, kernels serialised and "
             "cold-cache: compare shares, not absolutes.", ""]
    if len(sel) >= 2:
        step = seq[sel[-2] + 1: sel[-1] + 1]
        total = sum(t for _, t in step)
        agg = OrderedDict()
        for n, t in step:
            a = agg.setdefault(n, [0, 0.0])
            a[0] += 1
            a[1] += t
        lines += ["## One execute (last full step in the capture)", "",
                  "| kernel | launches | time (us) | share |", "|---|---|---|---|"]
        for n, (c, t) in agg.items():
            lines.append(f"| `{n}` | {c} | {t:.1f} | {100 * t / total:.1f}% |")
        lines += [f"| **total** | {len(step)} | {total:.1f} | 100% |", ""]
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        report(sys.argv[2], sys.argv[3], tj)
    else:
        launches(sys.argv[2], sys.argv[3])
