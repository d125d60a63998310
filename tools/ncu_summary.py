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
    """Per-launch duration (and DRAM bytes when the capture had
    dram__bytes_read/write.sum), then per-kernel totals."""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    idi = h.index("ID") if "ID" in h else None
    launches_ = collections.OrderedDict()  # launch id -> [name, ns, bytes]
    for n, r in enumerate(rows[hi + 1:]):
        if len(r) <= vi:
            continue
        key = r[idi] if idi is not None else n
        metric = r[mi] if mi is not None else "gpu__time_duration.sum"
        ent = launches_.setdefault(key, [r[ki], 0.0, None])
        if metric.startswith("gpu__time_duration"):
            ent[1] = float(r[vi].replace(",", "")) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
        elif metric.startswith("dram__bytes"):
            ent[2] = (ent[2] or 0.0) + _bytes(r[vi], r[ui])
    has_bytes = any(e[2] is not None for e in launches_.values())
    print(f"{'#':>4} {'ns':>12} " + (f"{'DRAM MB':>9} {'GB/s':>7} " if has_bytes else "") + " kernel")
    agg = collections.OrderedDict()
    for n, (name, ns, nb) in enumerate(launches_.values()):
        extra = f"{nb / 1e6:>9.1f} {nb / ns if ns else 0:>7.0f} " if has_bytes else ""
        print(f"{n:>4} {ns:>12.0f} {extra} {name[:100]}")
        a = agg.setdefault(name[:80], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += ns
        a[2] += nb or 0.0
    print("\nper kernel (count, mean us, total us" + (", DRAM MB per launch, GB/s" if has_bytes else "") + "):")
    for k, (c, ns, nb) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        extra = f" {nb / c / 1e6:>9.1f} {nb / ns if ns else 0:>7.0f}" if has_bytes else ""
        print(f"{c:>5} {ns / c / 1e3:>10.2f} {ns / 1e3:>10.1f}{extra}  {k}")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "full":
        full(sys.argv[2])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    elif cmd == "launches":
        launches(sys.argv[2])
