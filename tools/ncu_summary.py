"""Summarise ncu output brought back in gpurun_out/ into committed profiles/.

    python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/rNN_launches.txt
    python tools/ncu_summary.py full gpurun_out/full_ew.ncu-rep      > profiles/rNN_ncu_ew.txt
    python tools/ncu_summary.py traffic ew_fused gpurun_out/full_ew.ncu-rep   (updates profiles/traffic.json)

The launch list is cold-cache and serialised (compare shares, not absolutes);
the full-set capture gives DRAM bytes per launch (the bench's roofline
``traffic``) and pipe utilisations.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def _raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def full(rep):
    h, units, rows = _raw(rep)
    for r in rows:
        name = r[h.index("Kernel Name")]
        print(f"kernel: {name}")
        for m in FULL_METRICS:
            if m in h:
                i = h.index(m)
                print(f"  {m:<70} {r[i]:>16} {units[i]}")
        if "dram__bytes_read.sum" in h:
            rd = _bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
            wr = _bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
            print(f"  {'traffic (read+write) bytes':<70} {rd + wr:>16.0f} byte")


def _bytes(v, unit):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def traffic(key, rep):
    h, units, rows = _raw(rep)
    r = rows[0]
    rd = _bytes(r[h.index("dram__bytes_read.sum")], units[h.index("dram__bytes_read.sum")])
    wr = _bytes(r[h.index("dram__bytes_write.sum")], units[h.index("dram__bytes_write.sum")])
    p = os.path.join(ROOT, "profiles", "traffic.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[key] = int(rd + wr)
    json.dump(d, open(p, "w"), indent=1, sort_keys=True)
    print(key, int(rd + wr))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    print(f"{'#':>4} {'ns':>12}  kernel")
    agg = collections.OrderedDict()
    for n, r in enumerate(rows[hi + 1:]):
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
        name = r[ki]
        print(f"{n:>4} {v:>12.0f}  {name[:110]}")
        agg.setdefault(name[:80], []).append(v)
    print("\nper kernel (count, mean us, total us):")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{len(v):>5} {sum(v) / len(v) / 1e3:>10.2f} {sum(v) / 1e3:>10.1f}  {k}")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "full":
        full(sys.argv[2])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    elif cmd == "launches":
        launches(sys.argv[2])
