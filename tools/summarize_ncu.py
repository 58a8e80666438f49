#!/usr/bin/env python
"""Summarise ncu captures (run here, no GPU) into profiles/.

    python tools/summarize_ncu.py TAG

Reads gpurun_out/launches_TAG.csv (per-launch gpu__time_duration + dram bytes of one
bench step, cold-cache / serialised) and gpurun_out/prof_k2_TAG.ncu-rep (ncu --set
full on K2 launches), writes profiles/TAG_launches.json, profiles/TAG_k2_full.json
and refreshes profiles/k2_traffic.json (measured DRAM bytes per K2 launch, the
`traffic` field bench.py reports).
"""

from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "nsecond": 1e-3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(tag):
    rows = list(csv.reader(open(OUT / f"launches_{tag}.csv")))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, mi, ui, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").strip()
    agg = collections.defaultdict(lambda: {"launches": 0, "time_us": 0.0, "dram_bytes": 0.0})
    for i, m in per.items():
        a = agg[names[i]]
        a["launches"] += 1
        a["time_us"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(a["time_us"] for a in agg.values())
    for a in agg.values():
        a["share"] = a["time_us"] / total if total else 0.0
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]["time_us"])), total


def full(tag):
    rep = OUT / f"prof_k2_{tag}.ncu-rep"
    if not rep.exists():
        return None
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    keep = ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "launch__grid_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
            "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_selected")
    out = []
    for r in data:
        d = {}
        for k in keep:
            if k in hdr:
                i = hdr.index(k)
                d[k + (f" [{units[i]}]" if units[i] else "")] = r[i]
        out.append(d)
    return out


def main():
    tag = sys.argv[1]
    PROF.mkdir(exist_ok=True)
    agg, total = launches(tag)
    (PROF / f"{tag}_launches.json").write_text(json.dumps({"total_us": total, "kernels": agg}, indent=1))
    k2 = {k: v for k, v in agg.items() if "k_dp_" in k}
    n = sum(v["launches"] for v in k2.values())
    b = sum(v["dram_bytes"] for v in k2.values())
    if n:
        (PROF / "k2_traffic.json").write_text(json.dumps({
            "bytes_per_launch": b / n, "launches": n, "k2_dram_bytes_per_step": b,
            "source": f"gpurun_out/launches_{tag}.csv (ncu dram__bytes_read+write, all K2 launches of one step)"},
            indent=1))
    f = full(tag)
    if f is not None:
        (PROF / f"{tag}_k2_full.json").write_text(json.dumps(f, indent=1))
    for name, v in agg.items():
        print(f"{name:45s} {v['launches']:5d} {v['time_us'] / 1e3:9.3f} ms {100 * v['share']:6.2f}%  "
              f"dram {v['dram_bytes'] / 1e9:8.3f} GB")


if __name__ == "__main__":
    main()
