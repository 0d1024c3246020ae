"""Sweep the cells kernel (K1d) parameters on a bench config, one mode at a
time: the tensor is generated once on the GPU, each spec rebuilds the mode's
plan, puts it in the cells layout and times the kernel with CUDA events
(median of --reps launches).  Every result is compared with the production
tile kernel's output on the same plan (max rel diff).  One JSON line per spec.

  python tools/sweep_cells.py --config cfg2 --modes 0,1 \
      --specs '[{"lag":2},{"lag":0},{"lag":4,"flags":1}]'
"""

import argparse
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_15121_b200 as sk  # noqa: E402
from paper_2507_15121_b200 import engine  # noqa: E402


def time_exec(ex, plan, facs, out, cfg, reps):
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ex.run(plan.coords, plan.vals, plan.nnz, plan.mode, facs, out, cfg, st)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[1:]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--modes", default="0,1")
    ap.add_argument("--specs", default='[{}]')
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--baseline", action="store_true", help="also time the production auto layout")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    shape, nnz, R = cfg["shape"], cfg["nnz"], cfg["rank"]
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    tensor = sk.synth_tensor_device(shape, nnz, distribution=cfg["dist"], seed=0)
    facs = [torch.from_numpy(f.data.astype(np.float32)).to(dev) for f in sk.random_factors(shape, R, seed=0)]
    print(json.dumps({"generated_s": time.perf_counter() - t0}), flush=True)
    pcfg = sk.PartitionConfig(devices=1, strategy=cfg["strategy"])
    for d in [int(x) for x in args.modes.split(",")]:
        ref = None
        base = sk.PlatformConfig(rank=R, accumulation="atomic", layout="auto")
        p = sk.build_mode_plan(tensor, d, pcfg, keep_permutation=False)
        engine.apply_layout(p, base, R)
        ex = engine._shard_exec(p, list(range(p.shard_count)), base, R, dev)
        out = torch.zeros(shape[d], R, dtype=torch.float32, device=dev)
        ex.run(p.coords, p.vals, p.nnz, p.mode, facs, out, base, torch.cuda.current_stream().cuda_stream)
        ref = out.clone()
        ms = time_exec(ex, p, facs, out, base, args.reps)
        if args.baseline:
            print(json.dumps({"mode": d, "layout": p.layout, "kernel": sk._lib.launch_log()[-1][1], "ms": ms}),
                  flush=True)
        del p, ex, out
        gc.collect()
        torch.cuda.empty_cache()
        for spec in json.loads(args.specs):
            c = sk.PlatformConfig(rank=R, layout="cells", cell_lag=spec.get("lag", 0),
                                  cell_variant=spec.get("variant", 1), cell_outer_mb=spec.get("outer_mb", 32),
                                  cell_inner_mb=spec.get("inner_mb", 8))
            p = sk.build_mode_plan(tensor, d, pcfg, keep_permutation=False)
            prm = engine.choose_cells(p, R, c)
            if "stripe_rows" in spec:
                prm["stripe_rows"] = spec["stripe_rows"]
            tb = time.perf_counter()
            p.to_cells(range(p.shard_count), prm)
            torch.cuda.synchronize()
            tb = time.perf_counter() - tb
            ex = engine._shard_exec(p, list(range(p.shard_count)), c, R, dev)
            out = torch.full((shape[d], R), float("nan"), dtype=torch.float32, device=dev)
            ms = time_exec(ex, p, facs, out, c, args.reps)
            diff = float(((out - ref).abs() / ref.abs().clamp_min(1.0)).max())
            info = {k: v for k, v in p.cells.items() if not hasattr(v, "data_ptr") and k != "shard_ids"}
            print(json.dumps({"mode": d, "spec": spec, "ms": ms, "max_rel_diff_vs_tiles": diff,
                              "layout_s": tb, "cells": info}), flush=True)
            del p, ex, out
            gc.collect()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
