"""Summarise ncu captures for profiles/: one block per kernel launch in a
`.ncu-rep` (duration, DRAM bytes, throughputs, occupancy, pipes), or the
per-kernel totals of a `--metrics gpu__time_duration.sum` launch list.

    python tools/ncu_summary.py rep  gpurun_out/g_ozgemm.ncu-rep [...]
    python tools/ncu_summary.py list gpurun_out/g_launches_n1024.csv
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "tensor INT pipe % (active)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def rep(path):
    head, units, rows = raw(path)
    col = {k: i for i, k in enumerate(head)}
    print(f"== {path}")
    for r in rows:
        print(f"kernel: {r[col['Kernel Name']]}")
        for key, label in KEYS:
            if key in col and r[col[key]] != "":
                print(f"  {label:28s} {r[col[key]]} {units[col[key]]}  [{key}]")
        # stall reasons with > 5 % of samples
        stalls = [(k, r[i]) for k, i in col.items()
                  if k.startswith("smsp__average_warp_latency_issue_stalled") and k.endswith(".ratio")]
        top = sorted(((float(v), k) for k, v in stalls if v not in ("", "n/a")), reverse=True)[:5]
        for v, k in top:
            print(f"  stall {k.split('stalled_')[1].split('.')[0]:22s} {v:.2f} cycles/issue")


def launch_list(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    tot = collections.defaultdict(lambda: [0, 0.0])
    unit = rows[0]["Metric Unit"] if rows else ""
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        t = float(r["Metric Value"].replace(",", ""))
        tot[name][0] += 1
        tot[name][1] += t
    all_t = sum(v[1] for v in tot.values())
    print(f"== {path}: {sum(v[0] for v in tot.values())} launches, {all_t:.1f} {unit} total (serialised, cold)")
    for name, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"  {name:40s} {c:6d} launches {t:12.1f} {unit} {100 * t / all_t:6.2f} %  avg {t / c:9.2f}")


if __name__ == "__main__":
    mode, paths = sys.argv[1], sys.argv[2:]
    for p in paths:
        (rep if mode == "rep" else launch_list)(p)
