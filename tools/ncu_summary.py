#!/usr/bin/env python
"""Summarise an ncu report (--set full) and a launch-list CSV into profiles/.

usage: python tools/ncu_summary.py gpurun_out/prof_TAG.ncu-rep [launches.csv] > profiles/TAG.md
Also writes profiles/pass2_traffic.json (dram bytes per pass-2 launch), which
bench.py reports as roofline.traffic.
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "regs",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__grid_size": "grid",
    "smsp__inst_executed.sum": "inst",
}


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m, k in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if k in ("dram_read", "dram_write"):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if k == "duration":
                    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3,
                          "ms": 1e3}.get(u, 1)
                d[k] = v
        res.append(d)
    return res


def launches(csv_path):
    rows = list(csv.reader(open(csv_path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr_i]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hdr_i + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3,
                  "ms": 1e3}.get(r[ui], 1)
            agg[r[ki].split("(")[0]].append(v)
    return agg


def main():
    rep = sys.argv[1]
    print(f"# ncu summary: {Path(rep).name}\n")
    print("`ncu --set full --clock-control none` (caches flushed between replays, "
          "serialised): per-launch durations are cold-cache.\n")
    print("| kernel | µs | DRAM read MB | DRAM write MB | DRAM % peak | GB/s | regs | warps active % | L2 hit % |")
    print("|---|---|---|---|---|---|---|---|---|")
    traffic = {}
    for d in ncu_raw(rep):
        mb_r = d.get("dram_read", 0) / 1e6
        mb_w = d.get("dram_write", 0) / 1e6
        gbs = (d.get("dram_read", 0) + d.get("dram_write", 0)) / (d["duration"] * 1e-6) / 1e9
        print(f"| {d['kernel'][-60:]} | {d['duration']:.2f} | {mb_r:.1f} | {mb_w:.1f} | "
              f"{d.get('dram_pct', 0):.1f} | {gbs:.0f} | {d.get('regs', 0):.0f} | "
              f"{d.get('warps_active_pct', 0):.1f} | {d.get('l2_hit_pct', 0):.1f} |")
        if "lars_pass2" in d["kernel"]:
            traffic["resnet50"] = int(d.get("dram_read", 0) + d.get("dram_write", 0))
    if len(sys.argv) > 2:
        print("\n## launch list (gpu__time_duration, µs)\n")
        print("| kernel | launches | mean µs | share of listed time |")
        print("|---|---|---|---|")
        agg = launches(sys.argv[2])
        tot = sum(sum(v) for v in agg.values())
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            print(f"| {k[-70:]} | {len(v)} | {sum(v) / len(v):.2f} | {100 * sum(v) / tot:.1f} % |")
    if traffic:
        (ROOT / "profiles" / "pass2_traffic.json").write_text(json.dumps(traffic))


if __name__ == "__main__":
    main()
