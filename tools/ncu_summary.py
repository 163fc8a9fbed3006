#!/usr/bin/env python
"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into profiles/.

    python tools/ncu_summary.py --tag r01 --rep gpurun_out/prof_apply_c3.ncu-rep:C3:k_apply ...
                                --launches gpurun_out/launches_c3.csv:C3

Writes profiles/<tag>_<config>_<kernel>.txt (key metrics), profiles/<tag>_launches_<config>.txt
(per-kernel launch times and shares) and merges DRAM bytes per launch into
profiles/ncu_traffic.json (read by bench.py for the roofline "traffic" field).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "l1tex__m_l1tex2xbar_write_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
]


def raw(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def num(x: str) -> float:
    return float(x.replace(",", ""))


def to_bytes(v: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return num(v) * scale


def summarise_rep(tag, spec):
    rep, cfg, kern = spec.split(":")
    d = raw(rep)
    if not d:
        print("no data in", rep)
        return None
    name = f"{tag}_{cfg}_{kern}.txt"
    with open(os.path.join(PROF, name), "w") as f:
        f.write(f"# ncu --set full --clock-control none capture of {kern} ({cfg}); source {os.path.basename(rep)}\n")
        kname = d.get("Kernel Name", ("?", ""))[0]
        f.write(f"# kernel: {kname}\n")
        for k in KEYS:
            if k in d:
                f.write(f"{k:70s} {d[k][0]:>20s} {d[k][1]}\n")
    rd = d.get("dram__bytes_read.sum")
    wr = d.get("dram__bytes_write.sum")
    traffic = None
    if rd and wr:
        traffic = to_bytes(*rd) + to_bytes(*wr)
    print("wrote", name, "traffic", traffic)
    return cfg, kern, traffic


def summarise_launches(tag, spec):
    path, cfg = spec.split(":")
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, ui, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    us_scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
    times, dram = defaultdict(list), defaultdict(float)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki]
        for short in ("k_hist", "k_solve", "k_apply", "k_remap", "k_match", "k_idx1_table"):
            if short in k:
                k = short
                break
        if r[mi] == "gpu__time_duration.sum":
            times[k].append(num(r[vi]) * us_scale.get(r[ui], 1e-3))
        elif r[mi] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            dram[k] += to_bytes(r[vi], r[ui])
    tot = sum(sum(v) for v in times.values())
    name = f"{tag}_launches_{cfg}.txt"
    with open(os.path.join(PROF, name), "w") as f:
        f.write(f"# ncu --metrics gpu__time_duration.sum,dram__bytes_{{read,write}}.sum --clock-control none launch "
                f"list ({cfg}); cold-cache, serialised: compare shares, not absolutes\n")
        f.write(f"{'kernel':14s} {'launches':>8s} {'mean_us':>10s} {'min_us':>10s} {'share':>7s} {'dram_MB/launch':>15s}\n")
        for k, v in sorted(times.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"{k:14s} {len(v):8d} {sum(v)/len(v):10.2f} {min(v):10.2f} {sum(v)/tot:7.3f} "
                    f"{dram[k] / len(v) / 1e6:15.1f}\n")
    print("wrote", name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--rep", action="extend", nargs="+", default=[])
    ap.add_argument("--launches", action="extend", nargs="+", default=[])
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    tj = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for spec in a.rep:
        r = summarise_rep(a.tag, spec)
        if r and r[2] is not None:
            traffic.setdefault(r[0], {})[r[1]] = r[2]
    for spec in a.launches:
        summarise_launches(a.tag, spec)
    json.dump(traffic, open(tj, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
