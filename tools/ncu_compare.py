"""Summarise ncu reports (raw page) as JSON: duration, clocks, DRAM bytes,
L2 hit rate and throughput, instructions and L1 data-pipe wavefronts per
nonzero, issue activity, top stall reasons (source page samples).

  python tools/ncu_compare.py --nnz 1.7e9 --label v1=a.ncu-rep --label v3=b.ncu-rep > out.json
"""
import argparse
import csv
import io
import json
import subprocess

SCALE = {"": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "nsecond": 1e-9, "hz": 1.0,
         "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "%": 1.0, "inst": 1.0, "cycle": 1.0, "sector": 1.0, "warp": 1.0}


def raw_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    out = {}
    for h, u, v in zip(rows[0], rows[1], rows[2]):
        try:
            out[h] = float(v.replace(",", "")) * SCALE.get(u, 1.0)
        except ValueError:
            out[h] = v
    return out


def stall_mix(rep):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    if len(rows) < 3:
        return {}
    hdr = rows[1]
    cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    tot = {hdr[i][6:]: 0.0 for i in cols}
    for r in rows[2:]:
        for i in cols:
            try:
                tot[hdr[i][6:]] += float(r[i])
            except (ValueError, IndexError):
                pass
    s = sum(tot.values()) or 1.0
    return {k: round(100 * v / s, 1) for k, v in sorted(tot.items(), key=lambda x: -x[1])[:6]}


def summary(rep, nnz):
    m = raw_metrics(rep)
    dur = m.get("gpu__time_duration.sum", float("nan"))
    dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    wf = m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0.0)
    return {
        "report": rep,
        "kernel": m.get("Kernel Name"),
        "duration_ms": dur * 1e3,
        "sm_ghz": m.get("smsp__cycles_elapsed.avg.per_second", float("nan")) / 1e9,
        "dram_gb": dram / 1e9,
        "dram_gbs": dram / dur / 1e9,
        "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct"),
        "l2_throughput_pct": m.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "l2_to_sm_gb": m.get("l1tex__m_xbar2l1tex_read_bytes.sum", 0.0) / 1e9,
        "inst_per_nnz": m.get("smsp__inst_executed.sum", 0.0) / nnz,
        "issue_active_pct": m.get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "l1_data_pipe_pct": m.get("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "smem_wavefronts_per_nnz": wf / nnz,
        "stalls_pct": stall_mix(rep),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nnz", type=float, default=1.7e9)
    ap.add_argument("--label", action="append", default=[], help="name=report.ncu-rep")
    args = ap.parse_args()
    out = {}
    for lab in args.label:
        k, rep = lab.split("=", 1)
        out[k] = summary(rep, args.nnz)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
