"""Summarise ncu artefacts into small committed files under profiles/.

    python scripts/ncu_summary.py report <file.ncu-rep> <out.json> [algorithmic_bytes]
    python scripts/ncu_summary.py launches <launches.csv> <out.txt>
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def report(path, out, alg=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")], "source": path}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = vals[i]
            d[k + "__unit"] = units[i]
    rb = float(d["dram__bytes_read.sum"]) * SCALE.get(d["dram__bytes_read.sum__unit"], 1)
    wb = float(d["dram__bytes_write.sum"]) * SCALE.get(d["dram__bytes_write.sum__unit"], 1)
    d["dram_bytes_per_launch"] = rb + wb
    if alg:
        d["algorithmic_bytes_per_launch"] = float(alg)
        d["traffic_over_algorithmic"] = (rb + wb) / float(alg)
    # stall summary from the source page
    src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if len(srows) > 2:
        h = srows[1]
        st = h.index("Warp Stall Sampling (All Samples)")
        sc = h.index("Source")
        data = [r for r in srows[2:] if r[st].isdigit()]
        tot = sum(int(r[st]) for r in data) or 1
        top = sorted(data, key=lambda r: -int(r[st]))[:8]
        d["top_stall_sass"] = [{"share": round(int(r[st]) / tot, 3), "sass": r[sc].strip()[:80]}
                               for r in top]
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps({k: d[k] for k in ("kernel", "dram_bytes_per_launch")}, indent=1))


def launches(path, out, cmd="python bench.py --steps 2 --warmup 1"):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        agg[r[ki][:80]][0] += 1
        agg[r[ki][:80]][1] += v
    tot = sum(v[1] for v in agg.values())
    outl = ["ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised:",
            f"compare SHARES, not absolutes) on: {cmd}",
            "", f"{'kernel':80s} {'n':>4s} {'ms':>9s} {'share':>6s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        outl.append(f"{k:80s} {c:4d} {t / 1e6:9.3f} {100 * t / tot:5.1f}%")
    open(out, "w").write("\n".join(outl) + "\n")
    print("\n".join(outl[:12]))


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
    else:
        launches(sys.argv[2], sys.argv[3], *sys.argv[4:5])
