#!/usr/bin/env python
"""Summarise ncu output into the JSON/markdown committed under profiles/.

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep \
        --launches gpurun_out/launches.csv --out profiles/ncu_summary_r01.json

--rep       a `ncu --set full` report: per kernel, duration, DRAM bytes read /
            written, DRAM and L2 throughput, achieved occupancy, registers,
            dominant stall.  The K2 launches are labelled by site group
            (lora_qkv, lora_o, lora_gate_up, lora_down) from the template
            arguments (NS = fused sites; the 1-site groups by their order).
--launches  a `ncu --metrics gpu__time_duration.sum` CSV: per kernel name,
            launches, total time and share of the captured time.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import re
import subprocess
from collections import defaultdict
from pathlib import Path

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),  # ns? normalised below by unit
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "dram_pct_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_pct_peak": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "stall_long_scoreboard": ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", 1.0),
    "stall_barrier": ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", 1.0),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1.0),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1.0),
}

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def label(name: str, order: int, singles: list[str]) -> str:
    if "meta_sort" in name:
        return "meta_sort"
    if "meta_scatter" in name:
        return "meta_scatter"
    if "reft" in name:
        return "reft"
    if "lora" in name:
        ns = None
        mm = re.search(r"lora_team_kernel<[^,]+, (\d+), (\d+),", name)
        if mm:
            ns = int(mm.group(2))
        else:
            mm = re.search(r"lora_kernel<[^,]+, (?:true|false|1|0), (\d+), (\d+),", name)
            if mm:
                ns = int(mm.group(2))
        if ns == 3:
            return "lora_qkv"
        if ns == 2:
            return "lora_gate_up"
        return singles[order % len(singles)]
    return name.split("(")[0][:60]


def from_rep(rep: Path, singles: list[str]) -> dict:
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    single_order = 0
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        k = label(name, single_order, singles)
        if k in singles:
            single_order += 1
        rec = {"kernel": name}
        for key, (metric, _) in METRICS.items():
            if metric in hdr:
                i = hdr.index(metric)
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                v *= SCALE.get(units[i], 1.0)
                rec[key] = v
        if "dram_read_bytes" in rec:
            rec["dram_bytes_per_launch"] = rec["dram_read_bytes"] + rec.get("dram_write_bytes", 0.0)
        out.setdefault(k, rec)
    return out


def from_launches(path: Path) -> dict:
    text = path.read_text()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    iname, ival, iunit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= ival:
            continue
        try:
            us = float(r[ival].replace(",", "")) * SCALE.get(r[iunit], 1e-3)
        except ValueError:
            continue
        short = re.sub(r"\(.*", "", r[iname])
        agg[short][0] += 1
        agg[short][1] += us
    total = sum(v[1] for v in agg.values()) or 1.0
    return {k: {"launches": n, "total_us": round(t, 2), "share": round(t / total, 4)}
            for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rep")
    p.add_argument("--launches")
    p.add_argument("--out", required=True)
    p.add_argument("--note", default="")
    p.add_argument("--singles", default="lora_down,lora_o",
                   help="labels of the 1-site K2 launches in capture order (default: -s 2 -c 4 of a step)")
    a = p.parse_args()
    res = {"note": a.note}
    if a.rep:
        res["kernels"] = from_rep(Path(a.rep), a.singles.split(","))
    if a.launches:
        res["launches"] = from_launches(Path(a.launches))
    Path(a.out).write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main()
