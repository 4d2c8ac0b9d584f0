#!/usr/bin/env python
"""Summarise ncu output for profiles/: the launch list (gpu__time_duration per launch, shares per
kernel) and, from a --set full report, the counters the roofline and DESIGN.md cite.

    python tools/ncu_summary.py launches gpurun_out/launches_r1a.csv
    python tools/ncu_summary.py full gpurun_out/prof_r1a.ncu-rep
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum", "smsp__inst_executed.sum",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
]


def launches(path: str) -> None:
    with open(path) as f:
        txt = f.read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    per = collections.OrderedDict()
    tot = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)  # -> us
        e = per.setdefault(name, [0, 0.0])
        e[0] += 1
        e[1] += v
        tot += v
    print(f"launches: {sum(e[0] for e in per.values())}, total device time {tot / 1e3:.3f} ms")
    print("| kernel | launches | total ms | mean ms | share |")
    print("|---|---|---|---|---|")
    for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {n} | {t / 1e3:.3f} | {t / n / 1e3:.3f} | {100 * t / tot:.1f} % |")


def full(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    for d in data:
        name = d[col["Kernel Name"]]
        print(f"### {name[:140]}")
        print(f"grid {d[col.get('Grid Size', 0)]} block {d[col.get('Block Size', 0)]}")
        for m in FULL_METRICS:
            if m in col:
                print(f"- `{m}` = {d[col[m]]} {units[col[m]]}")
        print()


def traffic(path: str, workload: str, kernel: str, out: str = "profiles/traffic.json") -> None:
    """Record dram__bytes_read.sum + dram__bytes_write.sum of the (single) kernel in `path` as the
    per-launch traffic of `kernel` ("forward" / "adjoint") on `workload` (read by bench.py)."""
    import json
    import os
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    d = data[0]
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        tot += float(d[col[m]].replace(",", "")) * scale[units[col[m]]]
    t = {}
    if os.path.exists(out):
        with open(out) as f:
            t = json.load(f)
    t.setdefault(workload, {})[kernel] = {
        "dram_bytes": int(tot), "kernel": d[col["Kernel Name"]][:120],
        "duration_ms": float(d[col["gpu__time_duration.sum"]].replace(",", "")) *
        {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[units[col["gpu__time_duration.sum"]]],
        "source": os.path.basename(path)}
    with open(out, "w") as f:
        json.dump(t, f, indent=1)
    print(workload, kernel, t[workload][kernel])


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](*sys.argv[2:])
