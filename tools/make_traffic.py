#!/usr/bin/env python
"""Build profiles/ncu_traffic.json from ncu --set full summaries
(tools/ncu_summary.py full): one entry per (config, mode, exact kernel).

    python tools/make_traffic.py SUMMARY.json[:mode0,mode1,...] ...

The launches of a summary are mapped to modes in order (the captures profile
the first warm-up step, modes 0..N-1); bench.py reports an entry only when the
kernel it launched has exactly this name (launch log, skrp_launch_log).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    entries = []
    for arg in sys.argv[1:]:
        path, _, modes = arg.partition(":")
        s = json.load(open(path))
        launches = s["launches"]
        ms = [int(x) for x in modes.split(",")] if modes else list(range(len(launches)))
        for m, l in zip(ms, launches):
            entries.append({"config": s["config"], "mode": m, "kernel": l["kernel"],
                            "traffic_bytes_per_launch": l["traffic_bytes_per_launch"],
                            "dram_read_bytes": l["dram_read_bytes"], "dram_write_bytes": l["dram_write_bytes"],
                            "duration_s_under_ncu": l["duration_s"], "l2_hit_rate_pct": l["l2_hit_rate_pct"],
                            "inst_executed": l.get("inst_executed"),
                            "source": os.path.relpath(os.path.abspath(path), ROOT)})
    out = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    with open(out, "w") as fh:
        json.dump({"note": "DRAM bytes per launch from ncu --set full --clock-control none captures of the "
                           "current kernels (first warm-up step, one launch per mode); bench.py matches config, "
                           "mode and the exact kernel instantiation", "entries": entries}, fh, indent=1)
    print(f"{len(entries)} entries -> {out}")


if __name__ == "__main__":
    main()
