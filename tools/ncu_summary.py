#!/usr/bin/env python
"""Summarise ncu output into profiles/ (run in the build container, no GPU).

    python tools/ncu_summary.py full  <report.ncu-rep> <out.json> [--config cfg2]
    python tools/ncu_summary.py launches <launches.csv> <out.json>

`full`: the metrics the roofline story needs (duration, DRAM bytes, L2 hit
rate, occupancy, issue activity, stall mix, instructions per launch) plus
`traffic_bytes_per_launch` = dram read + write, which bench.py reports as
roofline.traffic when profiles/ncu_traffic.json matches its config.
`launches`: per-kernel launch counts and device-time shares from an
`ncu --metrics gpu__time_duration.sum` launch list.
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def _num(v, unit=""):
    try:
        x = float(str(v).replace(",", ""))
    except ValueError:
        return None
    return x * UNIT.get(unit, 1.0)


def full(rep, out, config=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

        def g(k):
            v, u = d.get(k, (None, ""))
            return None if v is None else _num(v, u)

        rec = {
            "kernel": d.get("Kernel Name", ("?", ""))[0],
            "duration_s": g("gpu__time_duration.sum"),
            "dram_read_bytes": g("dram__bytes_read.sum"),
            "dram_write_bytes": g("dram__bytes_write.sum"),
            "dram_throughput_pct_of_peak": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_hit_rate_pct": g("lts__t_sector_hit_rate.pct"),
            "l2_throughput_pct": g("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "registers_per_thread": g("launch__registers_per_thread"),
            "grid_size": g("launch__grid_size"),
            "stall_long_scoreboard_per_issue": g("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
            "inst_executed": g("smsp__inst_executed.sum") or g("sm__inst_executed.sum"),
            "l1_hit_rate_pct": g("l1tex__t_sector_hit_rate.pct"),
            "shared_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        }
        if rec["dram_read_bytes"] is not None and rec["dram_write_bytes"] is not None:
            rec["traffic_bytes_per_launch"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
            rec["dram_gbs"] = rec["traffic_bytes_per_launch"] / rec["duration_s"] / 1e9
        res.append(rec)
    summary = {"report": rep, "config": config, "launches": res}
    if res and config:
        summary["traffic_bytes_per_launch"] = res[0].get("traffic_bytes_per_launch")
    with open(out, "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1)[:2000])


def launches(csv_path, out):
    text = open(csv_path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(lambda: {"launches": 0, "time_s": 0.0})
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        t = _num(r["Metric Value"], r.get("Metric Unit", ""))
        per[name]["launches"] += 1
        per[name]["time_s"] += t or 0.0
    total = sum(v["time_s"] for v in per.values())
    table = sorted(({"kernel": k, **v, "share": v["time_s"] / total if total else 0} for k, v in per.items()),
                   key=lambda x: -x["time_s"])
    with open(out, "w") as fh:
        json.dump({"source": csv_path, "total_device_s": total, "kernels": table}, fh, indent=1)
    for t in table[:15]:
        print(f"{t['share'] * 100:6.2f}%  {t['launches']:5d}  {t['time_s'] * 1e3:10.3f} ms  {t['kernel'][:90]}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None
        full(sys.argv[2], sys.argv[3], cfg)
    else:
        launches(sys.argv[2], sys.argv[3])
