#!/usr/bin/env python
"""bench.py -- all-mode sparse MTTKRP on B200 (BASELINE.json's metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (one process per GPU, NCCL)

Workload (default cfg2, the north-star config): Amazon-shaped synthetic
4.8M x 1.8M x 1.8M, 1.7e9 nonzeros (uniform coordinates, uniform(0,1)
values, generated on the GPU with the reference law), rank 32, fp32 factors
from the reference's random_factors(seed=0), equal-index partition with
devices = N (reference defaults: oversubscription 4, ISP capacity 8192),
deterministic-reduce.  A STEP is one all-mode MTTKRP (3 modes, chained:
each mode's all-gathered output is the next modes' factor) including the
inter-mode all-gather.  Inputs stay resident in HBM (27 GB per mode copy per
GPU >> 126 MB L2, so no L2 flush is needed between steps).

One JSON line on rank 0: value = N_modes * nnz / step time (nnz/s, whole
job), roofline of the tile kernel vs measured HBM copy bandwidth, e2e
through the public runner with pinned host buffers, the CPU oracle port on a
bounded sample, clocks sampled during the timed region.

--impl reference: the reference algorithm's CPU implementation (oracle/ C
port of the deterministic-reduce engine, all host threads) on a bounded
sample of the same workload; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "all-mode MTTKRP time & nnz/s at 1/2/4/8 B200; % of HBM roofline; vs host CPU"

CONFIGS = {
    "cfg1": dict(shape=(1000, 1000, 1000), nnz=1_000_000, rank=32, dist="uniform",
                 strategy="equal-index", modes=[0], host_gen=True,
                 desc="cfg1: synthetic 1000^3, 1M nnz uniform, R=32, single mode-0 MTTKRP"),
    "cfg2": dict(shape=(4_800_000, 1_800_000, 1_800_000), nnz=1_700_000_000, rank=32, dist="uniform",
                 strategy="equal-index", modes=None, host_gen=False,
                 desc="cfg2: Amazon-shaped 4.8Mx1.8Mx1.8M, 1.7B nnz uniform, R=32, all-mode MTTKRP"),
    # smaller same-law config for quick runs / profiling
    "cfg2s": dict(shape=(4_800_000, 1_800_000, 1_800_000), nnz=200_000_000, rank=32, dist="uniform",
                  strategy="equal-index", modes=None, host_gen=False,
                  desc="cfg2 shape at 200M nnz (quick profiling variant)"),
    # single-GPU (downscaled nnz) runs of the multi-GPU configs, same shapes and laws
    "cfg3s": dict(shape=(46, 240_000, 240_000), nnz=1_000_000_000, rank=32, dist="uniform",
                  strategy="equal-index", modes=None, host_gen=False,
                  desc="cfg3 Patents-shaped 46x240Kx240K uniform, R=32, all modes, 1.0B nnz (of 3.6B)"),
    "cfg4s": dict(acc="deterministic-reduce", shape=(8_200_000, 177_000, 8_100_000), nnz=500_000_000, rank=32, dist="zipf",
                  strategy="nnz-balanced", modes=None, host_gen=False,
                  desc="cfg4 Reddit-shaped 8.2Mx177Kx8.1M Zipf(1.2), R=32, all modes, 0.5B nnz (of 4.7B)"),
    # full multi-GPU configs (distributed plan build; one GPU cannot hold them)
    "cfg3": dict(shape=(46, 240_000, 240_000), nnz=3_600_000_000, rank=32, dist="uniform",
                 strategy="equal-index", modes=None, host_gen=False, dist_build=True, park_plans=True,
                 desc="cfg3 Patents-shaped 46x240Kx240K, 3.6B nnz uniform, R=32, all modes"),
    "cfg4": dict(acc="deterministic-reduce", shape=(8_200_000, 177_000, 8_100_000), nnz=4_700_000_000, rank=32, dist="zipf",
                 strategy="nnz-balanced", modes=None, host_gen=False, dist_build=True,
                 desc="cfg4 Reddit-shaped 8.2Mx177Kx8.1M, 4.7B nnz Zipf(1.2), R=32, all modes"),
    "cfg5": dict(acc="deterministic-reduce", shape=(10_000_000, 1_000_000, 100_000, 1_000), nnz=2_000_000_000, rank=64, dist="zipf",
                 strategy="nnz-balanced", modes=None, host_gen=False, kind="cpd", dist_build=True, park_plans=True,
                 desc="cfg5 4-mode 10Mx1Mx100Kx1K, 2B nnz Zipf(1.2), R=64, one full CPD-ALS iteration"),
    "cfg5s": dict(acc="deterministic-reduce", shape=(10_000_000, 1_000_000, 100_000, 1_000), nnz=200_000_000, rank=64, dist="zipf",
                  strategy="nnz-balanced", modes=None, host_gen=False, kind="cpd",
                  desc="cfg5 4-mode 10Mx1Mx100Kx1K Zipf(1.2), R=64, one full CPD-ALS iteration, 0.2B nnz (of 2B)"),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def pcie_h2d_gbs(dev, nbytes=1 << 31):
    """Measured pinned host -> device copy bandwidth (the out-of-core bound)."""
    import torch

    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return best


def plan_balance(plans):
    """Max shard share and max row share of the nonzeros per mode (SURVEY.md
    §8(d): the load-balance bound a single row / shard puts on N GPUs)."""
    import torch

    from paper_2507_15121_b200 import _lib

    out = {"max_shard_share": [], "max_row_share": []}
    for p in plans:
        sizes = getattr(p, "global_shard_nnz", None)
        sizes = np.asarray(sizes if sizes is not None else [s.nnz for s in p.shards], dtype=np.float64)
        out["max_shard_share"].append(float(sizes.max() / max(sizes.sum(), 1)))
        rows = p.coords[p.mode] if p.coords is not None else None
        if rows is None or not rows.is_cuda:
            out["max_row_share"].append(None)
            continue
        cnt = torch.empty(p.shape[p.mode], dtype=torch.int64, device=rows.device)
        _lib.call("skrp_histogram", rows.data_ptr(), rows.numel(), cnt.numel(), cnt.data_ptr(),
                  torch.cuda.current_stream(rows.device).cuda_stream)
        out["max_row_share"].append(float(cnt.max().item()) / max(rows.numel(), 1))
    return out


def kernel_key(name):
    """Kernel name without return type, namespaces and spaces: the form an
    ncu 'Kernel Name' and the library's demangled launch log share."""
    n = name.strip()
    if n.startswith("void "):
        n = n[5:]
    for ns in ("skrp::", "(anonymous namespace)::", "::"):
        n = n.replace(ns, "")
    return n.replace("(int)", "").replace(" ", "").replace("const", "")


def lookup_traffic(config, mode, kernel):
    """DRAM read+write bytes per launch of EXACTLY `kernel` (demangled name
    from the library's launch log) on `config`, mode `mode`, from one ncu
    --set full capture (profiles/ncu_traffic.json), or (None, reason): an
    entry for another template instantiation is never reused."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            pj = json.load(fh)
    except Exception:
        return None, "profiles/ncu_traffic.json unreadable"
    want = kernel_key(kernel)
    for e in pj.get("entries", []):
        if e.get("config") == config and e.get("mode") == mode and kernel_key(e.get("kernel", "")) == want:
            return e, None
    return None, f"no ncu capture of {want} on {config} mode {mode}"


def load_gather_ceiling():
    """Random 128-B row gathers from a 2-GB table (all DRAM misses), GB/s of
    row bytes, measured on a B200 by tools/pattern_ceiling.cu (r02r), or None."""
    path = os.path.join(ROOT, "profiles", "r02", "r02r_pattern_ceiling.jsonl")
    try:
        with open(path) as fh:
            for line in fh:
                d = json.loads(line)
                if d.get("part") == "gather_curve":
                    return max((p["row_gbs"] for p in d["points"] if p["table_mb"] == 2048), default=None)
    except Exception:
        return None
    return None


def roofline_block(config, modes, runner, dev_f, kern, alg, comp, peak, peak_src, world, seq=None):
    """Roofline of the dominant (MTTKRP) kernel per mode.  `frac` uses the
    bytes the kernel really moves: DRAM read + write per launch from the ncu
    --set full capture of EXACTLY the launched template instantiation
    (profiles/ncu_traffic.json, matched through the library's launch log),
    over the live per-launch time measured here with CUDA events.  The
    SURVEY.md §8(d) algorithmic figure (every gather charged to HBM; > 1 when
    L2 serves gathers) is `frac_algorithmic`; the compulsory lower bound
    (stream once, each factor once, output once) is `frac_compulsory`.
    `frac_miss_pattern` (needs `seq` = the sequential metadata bytes per
    mode): the DRAM floor of the kernel's own traffic -- metadata at the copy
    peak, every other DRAM byte at the measured random 128-B gather rate --
    over the live kernel time."""
    import torch

    from paper_2507_15121_b200 import _lib

    _lib.launch_log(clear=True)
    runner.run(dev_f)  # one eager pass, untimed: which kernels run per mode
    torch.cuda.synchronize()
    log = _lib.launch_log()
    names = [sorted({n for m, n in log if m == d}) for d in modes]
    per_mode, traffic, missing, floors = [], [], [], []
    gceil = load_gather_ceiling()
    for i, d in enumerate(modes):
        ent, why = (None, "N > 1: ncu captures are single-GPU") if world > 1 else (
            lookup_traffic(config, d, names[i][0]) if len(names[i]) == 1 else (None, "several kernels per mode"))
        t = ent["traffic_bytes_per_launch"] if ent else None
        traffic.append(t)
        if ent is None:
            missing.append(why)
        per_mode.append({"mode": d, "kernel": names[i], "ms": kern[i] * 1e3,
                         "dram_bytes_ncu": t, "ncu_source": ent.get("source") if ent else None,
                         "dram_gbs": t / kern[i] / 1e9 if t else None,
                         "frac_dram": t / kern[i] / 1e9 / peak if t else None,
                         "frac_algorithmic": alg[i] / kern[i] / 1e9 / peak,
                         "frac_compulsory": comp[i] / kern[i] / 1e9 / peak})
        if t and gceil and seq is not None:
            fl = seq[i] / peak / 1e9 + max(0.0, t - seq[i]) / gceil / 1e9
            floors.append(fl)
            per_mode[-1].update({"miss_pattern_floor_ms": fl * 1e3, "frac_miss_pattern": fl / kern[i]})
    ach_alg = sum(alg) / sum(kern) / 1e9
    if all(t is not None for t in traffic):
        achieved, basis = sum(traffic) / sum(kern) / 1e9, "measured DRAM bytes (ncu, same kernel) / live kernel time"
        tr = sum(traffic) / len(traffic)
    else:
        achieved, basis, tr = ach_alg, "algorithmic bytes (SURVEY.md §8(d)): " + "; ".join(missing), None
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": tr, "achieved_basis": basis, "peak_source": peak_src,
            "kernel": names[0][0] if names and names[0] else None,
            "kernel_ms_per_mode": [k * 1e3 for k in kern], "algorithmic_bytes_per_mode": alg,
            "compulsory_bytes_per_mode": comp, "achieved_algorithmic": ach_alg,
            "frac_algorithmic": ach_alg / peak, "frac_compulsory": sum(comp) / sum(kern) / 1e9 / peak,
            "per_mode": per_mode,
            "frac_miss_pattern": sum(floors) / sum(kern) if floors and len(floors) == len(modes) else None,
            "random_gather_gbs": gceil,
            "miss_pattern_basis": "metadata bytes at the copy peak + all other ncu DRAM bytes at the measured "
                                  "random 128-B gather rate (profiles/r02/r02r_pattern_ceiling.jsonl), / live time"}


def algorithmic_bytes(shape, nnz, rank, mode):
    n = len(shape)
    return nnz * (4 * n + 4) + nnz * (n - 1) * rank * 4 + shape[mode] * rank * 4


# --------------------------------------------------------------- clocks


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu_index = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# -------------------------------------------------------------- inputs


def host_sample(shape, nnz, seed, dist="uniform"):
    """The reference law on the host (uniform per-mode integers, uniform(0,1)
    values) without the dedup rounds: for the uniform configs the expected
    duplicate count of a sample is nnz^2 / (2 prod(shape)) < 1e-3."""
    rng = np.random.default_rng(seed)
    idx = np.empty((nnz, len(shape)), dtype=np.uint64)
    for w, s in enumerate(shape):
        idx[:, w] = rng.integers(0, s, nnz, dtype=np.int64)
    vals = rng.random(nnz)
    return idx, vals


def cpu_engine_run(shape, nnz, rank, threads, seed=1, steps=1, warmup=0):
    """The reference's deterministic-reduce engine restated in C (oracle/),
    best-tuned CPU configuration (devices = cores, one worker,
    ISP 8192).  Returns (nnz/s over all modes, seconds per all-mode pass)."""
    import oracle

    idx, vals = host_sample(shape, nnz, seed)
    fac0 = [np.random.default_rng(0).random((s, rank)) for s in shape]
    plans = []
    for d in range(len(shape)):
        order, counts = oracle.stable_order_c(idx, d, shape[d])
        bounds = oracle.equal_index_bounds(shape[d], min(4 * threads, shape[d]))
        prefix = np.concatenate([[0], np.cumsum(counts)])
        plans.append((np.ascontiguousarray(idx[order]), np.ascontiguousarray(vals[order]), prefix[bounds]))
    times = []
    for it in range(warmup + steps):
        facs = list(fac0)
        t0 = time.perf_counter()
        for d, (sidx, svals, offs) in enumerate(plans):
            facs[d] = oracle.engine_mode(sidx, svals, d, offs, 8192, facs, threads)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    t = min(times)
    return len(shape) * nnz / t, t


# ----------------------------------------------------------- reference arm

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def ref_package_legs(cfg, threads):
    """The UNMODIFIED reference package (`shardkrp` from baseline/_ref: numba
    `ec_accumulate` kernels.py:54-71 driven by engine.py:225-400) on a bounded
    sample of the config, in BASELINE.md §2's two configurations: the CLI
    defaults (1 simulated device, 1 worker, column_width 32) and the best-tuned
    one (8 simulated devices, 1 worker each, column_width 8192; more devices
    only add fp64 ring all-gather copies of the whole factor set per device).
    One warm-up pass (numba JIT), then the best of two timed passes.  Reports
    wall time of mttkrp_all_modes and the critical-path compute (max over the
    simulated devices of their compute seconds, summed over modes)."""
    if not os.path.isdir(os.path.join(REF_DIR, "shardkrp")):
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref /root/reference/pkg)"}
    if cfg["desc"].split(":")[0] not in ("cfg1", "cfg2") or cfg["dist"] != "uniform":
        return {"unavailable": "run on the cfg1 / cfg2 headline configs only (bounded CPU time)"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/skrp_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import shardkrp as ref

    shape = cfg["shape"]
    modes = list(range(len(shape))) if cfg["modes"] is None else cfg["modes"]
    sample = min(cfg["nnz"], 1_000_000 if len(modes) == 1 else 2_000_000)
    idx, vals = host_sample(shape, sample, 1)
    tensor = ref.SparseTensorCOO(shape, idx, vals)
    legs = []
    for name, m, cw in (("cli-default", 1, 32), ("best-tuned", min(8, threads), 8192)):
        pcfg = ref.PartitionConfig(devices=m)
        plans = [ref.build_mode_plan(tensor, d, pcfg) for d in modes]
        fs = ref.random_factors(shape, cfg["rank"], seed=0)
        pl = ref.PlatformConfig(devices=m, workers_per_device=1, rank=cfg["rank"], column_width=cw)
        best = None
        for it in range(3):
            devs = ref.make_devices(fs, pl)
            t0 = time.perf_counter()
            _, met = ref.mttkrp_all_modes(plans, devs, pl)
            wall = time.perf_counter() - t0
            crit = sum(max(mm.device_compute_seconds) for mm in met.modes)
            if it >= 1 and (best is None or wall < best[0]):
                best = (wall, crit)
        legs.append({"config": name, "devices": m, "workers_per_device": 1, "column_width": cw,
                     "isp_capacity": pcfg.isp_capacity, "sample_nnz": sample, "modes": modes,
                     "wall_s": best[0], "nnz_per_s_wall": len(modes) * sample / best[0],
                     "critical_path_compute_s": best[1], "nnz_per_s_compute": len(modes) * sample / best[1]})
    return {"kind": "reference", "package": "shardkrp " + getattr(ref, "__version__", "?") + " (baseline/_ref, numba)",
            "legs": legs}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle

    threads = os.cpu_count() or 1
    shape = cfg["shape"]
    nmodes = len(shape) if cfg["modes"] is None else len(cfg["modes"])
    sample = cfg["nnz"] if cfg["nnz"] <= 5_000_000 else cfg["nnz"] // 64
    modes_shape = shape
    t_all = []

    idx, vals = host_sample(shape, sample, 1)
    fac0 = [np.random.default_rng(0).random((s, cfg["rank"])) for s in shape]
    plans = []
    modes = list(range(len(shape))) if cfg["modes"] is None else cfg["modes"]
    for d in modes:
        order, counts = oracle.stable_order_c(idx, d, shape[d])
        bounds = oracle.equal_index_bounds(shape[d], min(4 * threads, shape[d]))
        prefix = np.concatenate([[0], np.cumsum(counts)])
        plans.append((d, np.ascontiguousarray(idx[order]), np.ascontiguousarray(vals[order]), prefix[bounds]))
    for it in range(args.warmup + args.steps):
        facs = list(fac0)
        t0 = time.perf_counter()
        for d, sidx, svals, offs in plans:
            facs[d] = oracle.engine_mode(sidx, svals, d, offs, 8192, facs, threads)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            t_all.append(dt)
    t = sum(t_all) / len(t_all)
    value = nmodes * sample / t
    kind, ms = "port", t * 1e3
    pkg = ref_package_legs(cfg, threads)
    # the arm reports the FASTER of the reference package (wall time of its own
    # public mttkrp_all_modes, best-tuned) and the C port: the conservative baseline
    for leg in pkg.get("legs", []):
        if leg["nnz_per_s_wall"] > value:
            value, kind, ms = leg["nnz_per_s_wall"], "reference", leg["wall_s"] * 1e3
            samp_ref = (f"{leg['sample_nnz']} nnz on the {cfg['desc'].split(':')[0]} shape/law, {nmodes} mode(s); "
                        f"shardkrp package ({leg['config']}: {leg['devices']} devices, column_width "
                        f"{leg['column_width']})")
    samp = f"{sample} nnz on the {cfg['desc'].split(':')[0]} shape/law ({'full' if sample == cfg['nnz'] else '1/64'}), {nmodes} mode(s) per step"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "shape": list(modes_shape), "nnz": cfg["nnz"], "rank": cfg["rank"],
                   "sample_nnz": sample, "partition": "equal-index, devices=cores, oversub 4, ISP 8192"},
        "cpu_baseline": {"value": value, "unit": "nnz/s", "cores": threads if kind == "port" else None,
                         "kind": kind, "sample": samp if kind == "port" else samp_ref, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "nnz/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "port": {"value": nmodes * sample / t, "ms_per_step": t * 1e3, "threads": threads, "sample": samp},
        "reference_package": pkg,
    }
    if kind == "reference":
        line["cpu_baseline"]["cores"] = min(8, threads)
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- our arm


def self_launch(args):
    """`python bench.py --gpus N` (N > 1) without torchrun's environment: re-run
    this script under torch.distributed.run with N ranks on this node (one
    process per GPU) and return its exit code; None when already a rank."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.emulate_world:
        return None
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ)
    # NCCL prints the communicator size at init (nRanks) so the driver can
    # check the collective really spanned N GPUs
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env["BENCH_SELF_LAUNCHED"] = "1"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def init_dist(args, dev=None):
    """Process group for N > 1 ranks: NCCL (one GPU per rank) unless
    BENCH_DIST_BACKEND says otherwise (gloo: CPU tests of the launch path).
    Fails loudly when the world does not match --gpus or the GPUs are short."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks were launched")
    if world == 1:
        return None
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
        if torch.cuda.device_count() < local_world:
            raise SystemExit(f"bench.py: {local_world} NCCL ranks on this node need as many GPUs, "
                             f"{torch.cuda.device_count()} visible")
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    if dist.get_world_size() != args.gpus:
        raise SystemExit(f"bench.py: process group has {dist.get_world_size()} ranks, --gpus {args.gpus}")
    return dist.get_backend()


def launch_check(args):
    """CPU-testable launch path: every rank joins the group and contributes 1
    to an all-reduce; rank 0 prints the world it saw (no GPU work)."""
    import torch
    import torch.distributed as dist

    backend = init_dist(args) or "none"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    seen = world
    if world > 1:
        t = torch.ones(1, dtype=torch.int64)
        dist.all_reduce(t)
        seen = int(t.item())
    if int(os.environ.get("RANK", "0")) == 0:
        print(json.dumps({"launch_check": True, "n_gpus": seen, "world_size": world, "backend": backend,
                          "self_launched": os.environ.get("BENCH_SELF_LAUNCHED") == "1"}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    import paper_2507_15121_b200 as sk
    from paper_2507_15121_b200.distributed import DistributedMttkrp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = torch.cuda.device_count()
    if ngpu == 0:
        raise SystemExit("bench.py: no CUDA device visible (the product path has no CPU fallback)")
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend == "nccl" and local >= ngpu:
        raise SystemExit(f"bench.py: local rank {local} has no GPU ({ngpu} visible)")
    local_gpu = local % ngpu  # > 1 rank per GPU only for the gloo smoke of the N>1 path
    torch.cuda.set_device(local_gpu)
    dev = torch.device("cuda", local_gpu)
    backend = init_dist(args, dev) or "none"

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    shape, nnz, R = cfg["shape"], cfg["nnz"], cfg["rank"]
    modes = list(range(len(shape))) if cfg["modes"] is None else cfg["modes"]
    pcfg = sk.PartitionConfig(devices=max(world, args.emulate_world), strategy=cfg["strategy"])
    pl = sk.PlatformConfig(devices=world, rank=R, accumulation=args.accumulation, tile_nnz=args.tile,
                           scheduling=args.scheduling,
                           kernel_variant=args.variant,
                           layout="panel" if args.fused_allgather else args.layout, l2_budget_mb=args.l2_mb,
                           max_blocks=args.max_blocks, fused_allgather=args.fused_allgather,
                           cell_lag=args.cell_lag, cell_variant=args.cell_variant, cell_outer_mb=args.cell_outer_mb,
                           cell_inner_mb=args.cell_inner_mb, cell_keep_arrays=False,
                           panel_smem_kb=args.panel_smem_kb)

    from paper_2507_15121_b200.engine import apply_layout

    t_setup = time.perf_counter()
    dist_build = world > 1 and (args.dist_build or cfg.get("dist_build", False))
    verify = rank == 0 and not dist_build and not args.no_parity and not args.stream_modes and not args.emulate_world
    plan_checks = []
    samples = None
    if verify:
        from oracle.scale import extract_row_samples, sample_parity_extracted, verify_plan_full
    if world == 1 and cfg.get("dist_build", False) and not cfg.get("park_plans", False):
        raise SystemExit(f"{args.config} does not fit one B200 ({nnz} nnz); run it with torchrun --nproc-per-node >= 2 "
                         f"or use the single-GPU '{args.config}s' variant")
    if dist_build:
        # each rank draws only its contiguous chunk of the global stream and
        # receives its shards' nonzeros (distplan.py); no rank holds the tensor
        from paper_2507_15121_b200.distplan import build_mode_plan_distributed
        from paper_2507_15121_b200.synth import synth_tensor_chunk

        tensor = synth_tensor_chunk(shape, nnz, rank, world, distribution=cfg["dist"], seed=0)
        plans = [build_mode_plan_distributed(tensor, d, pcfg, scheduling=args.scheduling) for d in modes]
    else:
        if cfg["host_gen"]:
            tensor = sk.synth_tensor(shape, nnz, distribution=cfg["dist"], seed=0)
        else:
            tensor = sk.synth_tensor_device(shape, nnz, distribution=cfg["dist"], seed=0)
        # full-size cfg3 on one GPU: 3 plans x 57.6 GB fit HBM only without the
        # source tensor and the sort workspace, so finished plans wait in host
        # memory while the next mode sorts, and come back once the source is gone
        park = world == 1 and cfg.get("park_plans", False)
        plans = []
        for d in modes:
            p_ = sk.build_mode_plan(tensor, d, pcfg, keep_permutation=verify)
            if verify:
                # full-scale plan properties against the SOURCE arrays (oracle/scale.py),
                # before any execution-layout reordering; then the permutation goes
                src_c, src_v = tensor.device_arrays()
                plan_checks.append(verify_plan_full(src_c, src_v, p_, cfg["strategy"], devices=pcfg.devices,
                                                    isp_capacity=pcfg.isp_capacity))
                del src_c, src_v
                p_.perm = None
            if park:
                # the execution layout now, beside the source: with every plan
                # back in HBM there is no room for its sort temporaries
                apply_layout(p_, pl, R, list(range(p_.shard_count)))
                torch.cuda.empty_cache()
            if park and d != modes[-1]:
                p_.to_host(pinned=False)
            torch.cuda.empty_cache()
            plans.append(p_)
        if verify:
            # the sampled rows' source nonzeros go to the host now, so the source
            # can leave HBM before the run (phase 2 after the run)
            src_c, src_v = tensor.device_arrays()
            samples = extract_row_samples(src_c, src_v, shape, modes,
                                          rows_per_mode=args.parity_rows // (4 if cfg.get("kind") == "cpd" else 1))
            del src_c, src_v
        if cfg.get("kind") != "cpd" or not verify or park:
            # (CP-ALS parity reads the source during its checked iteration,
            # unless the plans need its HBM: then the extracted rows serve)
            tensor.drop_device()
        torch.cuda.empty_cache()
        for p_ in plans:
            if p_.layout == "host":
                p_.to_device()
    build_s = [p.build_time for p in plans]
    torch.cuda.empty_cache()
    init = sk.random_factors(shape, R, seed=0)
    host_f = [torch.from_numpy(f.data.astype(np.float32)).pin_memory() for f in init]
    dev_f = [h.to(dev) for h in host_f]
    if args.shifts:
        for p_, sh in zip(plans, args.shifts.split(";")):
            p_.to_blocked([int(x) for x in sh.split(",")])
    streamed = []
    if args.stream_modes:
        # out-of-core execution: these modes' plans live
        # in pinned host memory and are streamed to HBM chunk by chunk each step
        streamed = list(range(len(plans))) if args.stream_modes == "all" else [int(x) for x in args.stream_modes.split(",")]
        for i in streamed:
            plans[i].to_host()
        torch.cuda.empty_cache()
    if args.emulate_world > 1:
        return emulate_world(args, cfg, plans, pl, dev_f, dev, build_s)
    runner = DistributedMttkrp(plans, pl, rank=rank, world=world, device=dev)
    runner.prepare(R)
    setup_s = time.perf_counter() - t_setup
    if cfg.get("kind") == "cpd":
        park_cpd = world == 1 and cfg.get("park_plans", False)
        return run_cpd(args, cfg, plans, runner, dev_f, dev, world, rank, local_gpu, setup_s, build_s,
                       tensor=tensor if verify and not park_cpd else None, plan_checks=plan_checks,
                       samples=samples if verify and park_cpd else None)

    for _ in range(args.warmup):
        runner.run(dev_f)
    rebalanced = []
    if args.rebalance and world > 1:
        for _ in range(args.rebalance_rounds):
            rebalanced = sorted(set(rebalanced) | set(runner.rebalance(dev_f)))
    barrier()

    # ---- timed region: K all-mode steps, inputs resident in HBM
    gpu_index = local_gpu
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gpu_index = int(vis.split(",")[local_gpu])
        except ValueError:
            pass
    clocks = ClockSampler(gpu_index)
    clocks.start()
    time.sleep(0.3)
    graph = None
    if world == 1 and not args.no_graph and not streamed:
        graph = runner.capture(dev_f)  # whole all-mode step as one CUDA graph
        graph.replay()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record()
    for k in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            runner.run(dev_f)
    e1.record()
    barrier()
    clk = clocks.stop()
    elapsed = e0.elapsed_time(e1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    step_s = elapsed / args.steps
    total_nnz = len(modes) * nnz
    value = total_nnz / step_s
    launches = args.steps * sum(runner.launches_per_mode(i) for i in range(len(modes)))

    # ---- per-kernel device time (eager pass, events on the launching stream)
    kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in modes]
           for _ in range(args.steps)]
    for k in range(args.steps):
        runner.run(dev_f, kernel_events=kev[k])
    torch.cuda.synchronize()
    kern = [sum(kev[k][i][0].elapsed_time(kev[k][i][1]) for k in range(args.steps)) / 1e3 / args.steps
            for i in range(len(modes))]

    # ---- roofline of the tile kernel on this rank
    peak, peak_src = load_peaks()
    alg = [runner.algorithmic_bytes(i) for i in range(len(modes))]
    achieved = sum(alg) / sum(kern) / 1e9
    # secondary roofline: compulsory bytes -- stream once,
    # every factor read once, output written once
    comp = [runner.local_nnz(i) * (4 * len(shape) + 4)
            + sum(shape[w] * R * 4 for w in range(len(shape)) if w != plans[i].mode)
            + runner.owned_rows(i) * R * 4 for i in range(len(modes))]
    balance = plan_balance(plans)
    seq = [runner.local_nnz(i) * (4 * len(shape) + 4) for i in range(len(modes))]
    roof = roofline_block(args.config, modes, runner, dev_f, kern, alg, comp, peak, peak_src, world, seq)

    # ---- end to end through the public runner with pinned host buffers:
    # every step uploads the factors it reads and downloads all outputs;
    # uploads/downloads are double-buffered against the neighbouring steps
    host_out = [[torch.empty((shape[d], R), dtype=torch.float32).pin_memory() for d in modes] for _ in range(2)]
    runner.run_host_pipelined(host_f, host_out, 2)
    barrier()
    x0 = torch.cuda.Event(enable_timing=True)
    x1 = torch.cuda.Event(enable_timing=True)
    x0.record()
    h2d, d2h = runner.run_host_pipelined(host_f, host_out, args.steps)
    h2d += sum(runner._exec(i, R).h2d_bytes for i in streamed)  # streamed plans cross the link every step
    x1.record()
    barrier()
    e2e_s = x0.elapsed_time(x1) / 1e3 / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- end to end through the DROP-IN API (reference engine.py:369-400):
    # float64 numpy factors in, make_devices + mttkrp_all_modes, float64 numpy
    # outputs back -- host wall clock around the whole call (it returns host
    # arrays), pinned staging and on-GPU conversions inside (hostio.py)
    e2e_api = None
    if world == 1 and not streamed and not args.no_e2e_api:
        api_cfg = sk.PlatformConfig(devices=1, rank=R, accumulation=args.accumulation, tile_nnz=args.tile,
                                    layout=args.layout, l2_budget_mb=args.l2_mb, max_blocks=args.max_blocks)
        np_f = [f.data for f in init]
        api_times = []
        for k in range(1 + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            outs_api, _ = sk.mttkrp_all_modes(plans, sk.make_devices(np_f, api_cfg), api_cfg)
            dt = time.perf_counter() - t0
            if k:
                api_times.append(dt)
        api_s = sum(api_times) / len(api_times)
        same = all(np.array_equal(a_, b_.double().cpu().numpy()) for a_, b_ in zip(outs_api, runner.outputs)) \
            if args.accumulation == "deterministic-reduce" else None
        del outs_api
        e2e_api = {"value": total_nnz / api_s, "unit": "nnz/s", "ms_per_step": api_s * 1e3,
                   "h2d_bytes_per_step": sum(f.nbytes for f in np_f),
                   "d2h_bytes_per_step": sum(shape[d] * R * 8 for d in modes),
                   "call": "make_devices(float64 numpy factors) + mttkrp_all_modes(plans, devices, cfg) -> "
                           "float64 numpy outputs (host wall clock)",
                   "bit_identical_to_runner": same}

    stream_info = None
    if streamed:
        ex_bytes = sum(runner._exec(i, R).h2d_bytes for i in streamed)
        stream_info = {"modes": streamed, "h2d_plan_bytes_per_step": ex_bytes,
                       "streamed_modes_ms": [kern[i] * 1e3 for i in streamed],
                       "h2d_plan_gbs": ex_bytes / sum(kern[i] for i in streamed) / 1e9,
                       "pcie_h2d_copy_gbs": pcie_h2d_gbs(dev),
                       "chunk_nnz": pl.stream_chunk_nnz}

    # ---- parity on a seeded sample of output rows (chained replay, fp64)
    parity = None
    if verify:
        parity = sample_parity_extracted(samples, [f.data for f in init], runner.outputs)
        parity["plans"] = plan_checks
        parity["plans_ok"] = all(c["ok"] for c in plan_checks)
    elif rank == 0 and not args.no_parity and not streamed:
        # distributed build: no rank holds the source tensor; rows owned here are
        # recomputed from this rank's plan arrays
        parity = sample_parity(plans, init, runner.outputs, modes, rows_per_mode=args.parity_rows,
                               owned=[runner.ownership[i][rank] for i in range(len(modes))] if dist_build else None)

    # ---- CPU baseline (rank 0, N=1 only): the C oracle port on a sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        sample = nnz if nnz <= 5_000_000 else nnz // 64
        if cfg["modes"] is not None:
            cpu_v, cpu_t = cpu_mode0(shape, sample, R, threads) if len(modes) == 1 else (None, None)
        else:
            cpu_v, cpu_t = cpu_engine_run(shape, sample, R, threads, steps=2, warmup=1)
        cpu = {"value": cpu_v, "unit": "nnz/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"{sample} nnz, same shape and law, {len(modes)} mode(s), C port of the reference "
                         f"deterministic-reduce engine (fp64), devices=cores, ISP 8192, 1 warm-up + best of 2; "
                         f"{cpu_t:.2f} s/pass"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nnz/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "shape": list(shape), "nnz": nnz, "rank": R,
                       "modes": modes, "partition": f"{cfg['strategy']}, devices={world}, oversub 4, ISP 8192",
                       "accumulation": args.accumulation, "tile_nnz": runner._exec(0, R).tile_nnz,
                       "layout": [p.layout for p in plans],
                       "block_shifts": [p.block_shifts for p in plans],
                       "parallelism": f"output-row shards x{world}", "scheduling": args.scheduling,
                       "rebalanced_modes": rebalanced,
                       "allgather": ("none (1 GPU)" if world == 1 else
                                     f"fused: panel write-back P2P-stores rows into every rank (CUDA IPC), "
                                     f"completion barrier over {backend}"
                                     if any(runner._fused(i) for i in range(len(modes))) else
                                     f"{backend} broadcasts of owned row ranges"),
                       "dist_backend": backend, "world_size": world,
                       "launch": "one CUDA graph per all-mode step" if graph is not None else "eager",
                       "l2": "no flush needed: per-mode inputs (nnz*16 B) >> 126 MB L2"},
            "roofline": roof,
            "balance": balance,
            "e2e": {"value": total_nnz / e2e_s, "unit": "nnz/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3},
            "e2e_api": e2e_api,
            "gpu_launches": launches,
            "stream": stream_info,
            "clocks": clk,
            "cpu_baseline": cpu,
            "parity": parity,
            "setup_seconds": setup_s, "plan_build_seconds": build_s,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def emulate_world(args, cfg, plans, pl, dev_f, dev, build_s, link_gbs=775.0):
    """Projected N-GPU step on ONE GPU (no multi-GPU box here): the plans are
    built for N devices; every rank's share (its shards, placement as the real
    N-rank run) is timed alone on this GPU, compute only; the per-mode
    all-gather is modelled as (N-1)/N of the output bytes entering each GPU at
    `link_gbs` (775 GB/s: measured kernel P2P rate on NVLink5 in
    B300_MICROARCH.md).  Prints one JSON line, kind "emulated"."""
    import torch

    from paper_2507_15121_b200.distributed import DistributedMttkrp

    n = args.emulate_world
    shape, R = cfg["shape"], cfg["rank"]
    modes = list(range(len(shape))) if cfg["modes"] is None else cfg["modes"]
    import dataclasses

    plcfg = dataclasses.replace(pl, devices=n)

    def time_ranks(history=None):
        per_rank = []
        for r in range(n):
            runner = DistributedMttkrp(plans, plcfg, rank=r, world=n, device=dev)
            runner.prepare(R)
            for rank_seconds in history or []:  # replay the rebalancing rounds
                runner.rebalance(rank_seconds=rank_seconds)
            for _ in range(args.warmup):
                runner.run(dev_f, exchange=False)
            kev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in modes]
                   for _ in range(args.steps)]
            for k in range(args.steps):
                runner.run(dev_f, kernel_events=kev[k], exchange=False)
            torch.cuda.synchronize()
            per_rank.append([sum(kev[k][i][0].elapsed_time(kev[k][i][1]) for k in range(args.steps)) / args.steps
                             for i in range(len(modes))])
            del runner
        return per_rank

    per_rank = time_ranks()
    before = None
    if args.rebalance:  # re-place from the measured per-rank times, then time again (rounds)
        before = per_rank
        history = []
        for _ in range(args.rebalance_rounds):
            history.append([[t / 1e3 for t in pr] for pr in per_rank])
            per_rank = time_ranks(history)
    gather_ms = [(n - 1) / n * shape[d] * R * 4 / (link_gbs * 1e9) * 1e3 for d in modes]
    step_ms = sum(max(pr[i] for pr in per_rank) + gather_ms[i] for i in range(len(modes)))
    line = {"kind": "emulated", "metric": METRIC, "n_gpus_emulated": n, "unit": "nnz/s",
            "value_projected": len(modes) * cfg["nnz"] / (step_ms / 1e3), "ms_per_step_projected": step_ms,
            "per_rank_kernel_ms_per_mode": per_rank, "allgather_ms_per_mode_modelled": gather_ms,
            "per_rank_kernel_ms_before_rebalance": before,
            "link_gbs_assumed": link_gbs,
            "config": {"workload": cfg["desc"], "partition": f"{cfg['strategy']}, devices={n}, oversub 4",
                       "scheduling": args.scheduling, "accumulation": args.accumulation,
                       "layout": [p.layout for p in plans]},
            "method": "each rank's shards timed alone on one B200 (compute only, CUDA events), max over ranks "
                      "per mode + modelled all-gather; not a multi-GPU measurement",
            "plan_build_seconds": build_s}
    print(json.dumps(line), flush=True)
    return 0


def run_cpd(args, cfg, plans, runner, dev_f, dev, world, rank, local_gpu, setup_s, build_s, tensor=None,
            plan_checks=(), samples=None):
    """cfg5: one full CPD-ALS iteration per step (all modes: MTTKRP, solve,
    normalisation, factor all-gather, Grams, fit)."""
    import torch
    import torch.distributed as dist

    from paper_2507_15121_b200.distributed import DistributedCpAls

    als = DistributedCpAls(plans, runner.cfg, rank=rank, world=world, device=dev)
    als.mt = runner
    for _ in range(args.warmup):
        als.run(dev_f, iterations=1)
    torch.cuda.synchronize()
    clocks = ClockSampler(local_gpu)
    clocks.start()
    time.sleep(0.3)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    e0.record()
    fits = []
    for _ in range(args.steps):
        _, _, hist = als.run(dev_f, iterations=1)
        fits.append(hist[-1])
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed = e0.elapsed_time(e1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    step_s = elapsed / args.steps
    nm = len(cfg["shape"])
    # MTTKRP kernel share (eager all-mode pass with per-kernel events)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nm)]
    runner.run(dev_f, chained=False, kernel_events=kev)
    torch.cuda.synchronize()
    kern = [a.elapsed_time(b) / 1e3 for a, b in kev]
    peak, peak_src = load_peaks()
    alg = [runner.algorithmic_bytes(i) for i in range(nm)]
    shape, R = cfg["shape"], cfg["rank"]
    comp = [runner.local_nnz(i) * (4 * nm + 4) + sum(shape[w] * R * 4 for w in range(nm) if w != plans[i].mode)
            + runner.owned_rows(i) * R * 4 for i in range(nm)]
    seq = [runner.local_nnz(i) * (4 * nm + 4) for i in range(nm)]
    roof = roofline_block(args.config, list(range(nm)), runner, dev_f, kern, alg, comp, peak, peak_src, world, seq)
    roof["mttkrp_share_of_iteration"] = sum(kern) / step_s
    parity = None
    if tensor is not None or samples is not None:
        # one more iteration with the checker hooked into every mode update:
        # sampled MTTKRP rows and the ALS update M V^-1 of those rows, in fp64
        # from the source tensor (oracle/scale.py cpd_mode_check)
        from oracle.scale import cpd_mode_check, cpd_mode_check_extracted

        checks = []
        if tensor is not None:
            src_c, src_v = tensor.device_arrays()
            als.run(dev_f, iterations=1, observe=lambda d, facs, m, new, lam: checks.append(
                cpd_mode_check(src_c, src_v, cfg["shape"], d, facs, m, new, lam,
                               rows_per_mode=args.parity_rows // 4)))
        else:  # full size on one GPU: rows extracted before the source left HBM
            by_mode = {smp["mode"]: smp for smp in samples}
            als.run(dev_f, iterations=1, observe=lambda d, facs, m, new, lam: checks.append(
                cpd_mode_check_extracted(by_mode[d], cfg["shape"], d, facs, m, new, lam)))
        worst = max(max(c["max_rel_err_mttkrp"], c["max_rel_err_update"]) for c in checks)
        parity = {"rows_checked": sum(c["rows"] for c in checks), "max_rel_err": worst, "tolerance": 1e-4,
                  "ok": worst <= 1e-4, "per_mode": checks, "plans": list(plan_checks),
                  "plans_ok": all(c["ok"] for c in plan_checks),
                  "method": "one CP-ALS iteration observed mode by mode: sampled MTTKRP rows recomputed in fp64 "
                            "from the SOURCE tensor vs the GPU's M; the ALS update of those rows (M V^-1, V = "
                            "Hadamard of fp64 Grams of the factors the GPU used, applied to the GPU's M) vs the "
                            "GPU's new*lambda (oracle/scale.py cpd_mode_check)"}
        if tensor is not None:
            tensor.drop_device()
    if rank == 0:
        line = {
            "metric": METRIC, "value": nm * cfg["nnz"] / step_s, "unit": "nnz/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["desc"], "shape": list(cfg["shape"]), "nnz": cfg["nnz"], "rank": cfg["rank"],
                       "step": "one CPD-ALS iteration (MTTKRP per mode + solve + normalise + factor all-gather + fit)",
                       "partition": f"{cfg['strategy']}, devices={world}", "accumulation": args.accumulation,
                       "layout": [p.layout for p in plans], "block_shifts": [p.block_shifts for p in plans]},
            "roofline": roof,
            "fit": fits[-1], "clocks": clk, "setup_seconds": setup_s, "plan_build_seconds": build_s,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def cpu_mode0(shape, nnz, rank, threads):
    import oracle

    idx, vals = host_sample(shape, nnz, 1)
    fac = [np.random.default_rng(0).random((s, rank)) for s in shape]
    order, counts = oracle.stable_order_c(idx, 0, shape[0])
    prefix = np.concatenate([[0], np.cumsum(counts)])
    offs = prefix[oracle.equal_index_bounds(shape[0], min(4 * threads, shape[0]))]
    sidx, svals = np.ascontiguousarray(idx[order]), np.ascontiguousarray(vals[order])
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        oracle.engine_mode(sidx, svals, 0, offs, 8192, fac, threads)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return nnz / best, best


def sample_parity(plans, init, outputs, modes, rows_per_mode=512, seed=0, nnz_budget=8_000_000, owned=None):
    """max |gpu - ref| / max(|ref|, 1) over a seeded sample of output rows
    per mode (rows added while their nonzeros fit `nnz_budget`; at least one
    row), ref recomputed in fp64 from the plan's nonzeros with the chained
    factors (cli.py:247-261 rule).  The fp64 recomputation runs on the GPU
    in torch (checker only, chunked); any execution layout works: the
    sampled rows' nonzeros are found with a row-membership mask."""
    import torch

    dev = outputs[0].device
    facs = [torch.from_numpy(f.data).to(dev) for f in init]  # fp64
    worst = 0.0
    checked = 0
    rng = np.random.default_rng(seed)
    for i, (p, d) in enumerate(zip(plans, modes)):
        col = p.coords[d]
        if owned is None:
            pool_rows = np.arange(p.shape[d])
        else:  # distributed build: only this rank's rows have their nonzeros here
            pool_rows = np.concatenate([np.arange(lo, hi) for lo, hi in owned[i]] or [np.zeros(0, np.int64)])
        cand = rng.permutation(pool_rows)[: 4 * rows_per_mode]
        member = torch.zeros(p.shape[d], dtype=torch.bool, device=dev)
        member[torch.from_numpy(np.sort(cand[:rows_per_mode]).astype(np.int64)).to(dev)] = True
        # count nonzeros of the candidate rows, drop rows beyond the budget
        hits = torch.zeros(p.shape[d], dtype=torch.int64, device=dev)
        chunk = 1 << 27
        for a in range(0, col.numel(), chunk):
            c = col[a:a + chunk].long()
            m = member[c]
            hits.index_add_(0, c[m], torch.ones(int(m.sum().item()), dtype=torch.int64, device=dev))
        rows_all = np.sort(cand[:rows_per_mode])
        if len(rows_all) == 0:
            facs = list(facs)
            facs[d] = outputs[i].double()
            continue
        h = hits[torch.from_numpy(rows_all).to(dev)].cpu().numpy()
        keep, tot = [], 0
        for r, n in zip(rows_all, h):
            if tot + n <= nnz_budget or not keep:
                keep.append(r)
                tot += n
        rows = np.array(sorted(keep), dtype=np.int64)
        member.zero_()
        member[torch.from_numpy(rows).to(dev)] = True
        expect = torch.zeros((len(rows), facs[0].shape[1]), dtype=torch.float64, device=dev)
        rows_t = torch.from_numpy(rows).to(dev)
        for a in range(0, col.numel(), chunk):
            c = col[a:a + chunk].long()
            sel = member[c].nonzero().squeeze(1)
            if sel.numel() == 0:
                continue
            for b in range(0, sel.numel(), 1 << 22):
                s_ = sel[b:b + (1 << 22)] + a
                contrib = p.vals.index_select(0, s_).double()[:, None].expand(-1, facs[0].shape[1]).clone()
                for w in range(len(facs)):
                    if w != d:
                        contrib *= facs[w].index_select(0, p.coords[w].index_select(0, s_).long())
                pos = torch.searchsorted(rows_t, p.coords[d].index_select(0, s_).long())
                expect.index_add_(0, pos, contrib)
        got = outputs[i].index_select(0, rows_t).double()
        err = float(((got - expect).abs() / expect.abs().clamp(min=1.0)).max().item()) if len(rows) else 0.0
        worst = max(worst, err)
        checked += len(rows)
        facs = list(facs)
        facs[d] = outputs[i].double()
    return {"rows_checked": checked, "max_rel_err": worst, "tolerance": 1e-4, "ok": worst <= 1e-4,
            "method": "seeded output-row sample, fp64 recomputation on the GPU (torch, checker only)"}


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--accumulation", default=None, choices=("deterministic-reduce", "atomic"),
                    help="default: the config's (atomic for uniform rows; deterministic-reduce for the Zipf configs, "
                         "whose head rows sum 10^8 nonzeros: the fp64 carry tree keeps them within 1e-4)")
    ap.add_argument("--tile", type=int, default=0, help="tile size (0 = auto)")
    ap.add_argument("--layout", default="auto", choices=("flycoo", "blocked", "panel", "cells", "auto"))
    ap.add_argument("--cell-lag", type=int, default=0, help="cells layout: lag in cells (0 = free running)")
    ap.add_argument("--cell-variant", type=int, default=1, help="cells layout: kernel variant (csrc/mttkrp_cells.cu)")
    ap.add_argument("--cell-outer-mb", type=int, default=32)
    ap.add_argument("--cell-inner-mb", type=int, default=8)
    ap.add_argument("--panel-smem-kb", type=int, default=64,
                    help="panel layout (deterministic-reduce): shared memory for the output slab")
    ap.add_argument("--l2-mb", type=int, default=192)
    ap.add_argument("--max-blocks", type=int, default=8)
    ap.add_argument("--shifts", default="", help="force block shifts per mode, e.g. '-1,19,18;19,-1,18;19,18,-1'")
    ap.add_argument("--variant", type=int, default=0, choices=(0, 1),
                    help="1: the generic scalar tile kernel (cross-check path)")
    ap.add_argument("--parity-rows", type=int, default=4096, help="sampled output rows per mode (SURVEY.md §8(c): >= 4096)")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-e2e-api", action="store_true", help="skip the drop-in API (numpy float64) e2e figure")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph per step")
    ap.add_argument("--dist-build", action="store_true", help="N>1: distributed plan build (default for cfg3-5)")
    ap.add_argument("--stream-modes", default="", help="out-of-core: stream these modes' plans from pinned host "
                                                      "memory ('all' or e.g. '0,2'; atomic accumulation)")
    ap.add_argument("--rebalance", action="store_true",
                    help="N>1: re-place shards from measured per-GPU kernel times after the warm-up")
    ap.add_argument("--rebalance-rounds", type=int, default=2, help="measure + re-place rounds for --rebalance")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="one GPU: time every rank's share of an N-GPU run alone (projected scaling line)")
    ap.add_argument("--fused-allgather", action="store_true",
                    help="N>1: panel layout whose write-back pushes rows to every rank (CUDA IPC, no collective)")
    ap.add_argument("--scheduling", default="contiguous", choices=("dynamic", "static", "contiguous", "split"),
                    help="shard placement across GPUs (contiguous: one owned row range per GPU)")
    ap.add_argument("--launch-check", action="store_true",
                    help="launch path only: join the process group, all-reduce, print the world seen (CPU ok)")
    args = ap.parse_args()
    rc = self_launch(args)
    if rc is not None:
        return rc
    if args.launch_check:
        return launch_check(args)
    if args.warmup < 3 and args.impl == "ours" and os.environ.get("BENCH_ALLOW_SHORT") != "1":
        print("note: warmup < 3 is below the timing rules; proceeding", file=sys.stderr)
    cfg = CONFIGS[args.config]
    if args.accumulation is None:
        args.accumulation = cfg.get("acc", "atomic")
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
