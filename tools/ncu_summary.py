#!/usr/bin/env python
"""Summarise an ncu capture (--set full .ncu-rep) and a launch list (csv) into
profiles/: a JSON with the evidence counters bench.py cites (dram bytes per
launch of the dominant kernel) and a markdown table.

  python tools/ncu_summary.py --rep gpurun_out/prof_r01.ncu-rep \
      --launches gpurun_out/launches.csv --tag r01
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "LDS instructions"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "LDS wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "LDS bank conflicts"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "global-load requests (L1 tag stage)"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global-load sectors"),
    ("l1tex__t_sector_pipe_lsu_mem_global_op_ld_hit_rate.pct", "global-load L1 hit rate"),
    ("l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum", "global-load L1 output wavefronts"),
    ("idc__requests.sum", "constant-cache (IDC) requests"),
    ("idc__request_hit_rate.pct", "constant-cache hit rate"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__grid_size", "grid"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def to_bytes(v, unit):
    m = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * m.get(unit, 1)


def read_rep(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "?")}
        for key, _ in KEYS:
            if key in d:
                k[key] = {"value": d[key], "unit": units[hdr.index(key)]}
        rb = to_bytes(d["dram__bytes_read.sum"], units[hdr.index("dram__bytes_read.sum")])
        wb = to_bytes(d["dram__bytes_write.sum"], units[hdr.index("dram__bytes_write.sum")])
        k["dram_bytes"] = rb + wb
        stalls = []
        for key, v in d.items():
            if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v)))
                except ValueError:
                    pass
        k["stalls_per_issue"] = dict(sorted(stalls, key=lambda x: -x[1])[:6])
        lds_i = float(d.get("smsp__sass_inst_executed_op_shared_ld.sum", "0") or 0)
        lds_w = float(d.get("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "0") or 0)
        k["wavefronts_per_lds"] = lds_w / lds_i if lds_i else None
        kernels.append(k)
    return kernels


def read_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        agg[d["Kernel Name"]][0] += 1
        agg[d["Kernel Name"]][1] += float(d["Metric Value"])
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("--alg-bytes", type=float, default=None,
                    help="algorithmic HBM bytes per launch of the captured kernels (32 B x blocks)")
    ap.add_argument("--primary", action="store_true", help="also write profiles/ncu_summary.json (read by bench.py)")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    md = [f"# ncu summary {a.tag}", ""]
    if a.note:
        md += [a.note, ""]
    summary = {"tag": a.tag}
    if a.rep:
        ks = read_rep(a.rep)
        summary["kernels"] = ks
        dom = max(ks, key=lambda k: float(k["gpu__time_duration.sum"]["value"]))
        summary["dominant_kernel"] = dom["kernel"]
        summary["dominant_kernel_dram_bytes_per_launch"] = dom["dram_bytes"]
        summary["source"] = f"ncu --set full, {os.path.basename(a.rep)} ({a.tag})"
        summary["algorithmic_bytes_per_launch"] = a.alg_bytes
        md += ["## `ncu --set full` (one launch each)", "", "| metric | " + " | ".join(k["kernel"][:48] for k in ks) + " |",
               "|---|" + "---|" * len(ks)]
        for key, name in KEYS:
            md.append(f"| {name} (`{key}`) | " + " | ".join(
                f'{k[key]["value"]} {k[key]["unit"]}' if key in k else "-" for k in ks) + " |")
        md.append("| DRAM bytes (read+write) | " + " | ".join(f'{k["dram_bytes"]:.4g}' for k in ks) + " |")
        md.append("| LDS wavefronts per LDS instruction | " + " | ".join(
            f'{k["wavefronts_per_lds"]:.4f}' if k["wavefronts_per_lds"] else "-" for k in ks) + " |")
        md.append("| top warp stall reasons (warps per issue) | " + " | ".join(
            ", ".join(f"{n} {v:.2f}" for n, v in list(k["stalls_per_issue"].items())[:4]) for k in ks) + " |")
        md.append("")
    if a.launches:
        agg = read_launches(a.launches)
        tot = sum(t for _, t in agg.values())
        md += ["## launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, whole bench process)", "",
               "| launches | total ms | share | kernel |", "|---|---|---|---|"]
        for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append(f"| {c} | {t / 1e6:.3f} | {t / tot:.1%} | `{k[:90]}` |")
        md.append("")
        summary["launches"] = {k: {"count": c, "total_ns": t} for k, (c, t) in agg.items()}
        shutil.copy(a.launches, os.path.join(prof, f"{a.tag}_launches.csv"))
    json.dump(summary, open(os.path.join(prof, f"{a.tag}_ncu_summary.json"), "w"), indent=1)
    if a.primary:
        json.dump(summary, open(os.path.join(prof, "ncu_summary.json"), "w"), indent=1)
    open(os.path.join(prof, f"{a.tag}_ncu_summary.md"), "w").write("\n".join(md))
    print("\n".join(md))


if __name__ == "__main__":
    main()
