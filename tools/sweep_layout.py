#!/usr/bin/env python
"""Layout / tile / variant sweep of the tile kernel on one GPU (tuning tool).

    python tools/sweep_layout.py --config cfg2 --specs SPECFILE.json [--reps 3]

SPECFILE: list of {"mode": d, "shifts": [...], "order": [...]|null,
"tile": T, "variant": V, "acc": "atomic"}; one JSON line per spec with the
kernel time (CUDA events, mean of --reps after one warm-up launch).  The
tensor is generated once; the mode plan is rebuilt per layout.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import bench
    import paper_2507_15121_b200 as sk
    from paper_2507_15121_b200.engine import _PanelExec, _plan_arrays, _ShardExec, panel_shape

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--specs", required=True)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    specs = json.load(open(args.specs))
    dev = torch.device("cuda", 0)
    shape, nnz, R = cfg["shape"], cfg["nnz"], cfg["rank"]
    t = sk.synth_tensor_device(shape, nnz, distribution=cfg["dist"], seed=0)
    pcfg = sk.PartitionConfig(devices=1, strategy=cfg["strategy"])
    g = torch.Generator(device=dev).manual_seed(0)
    facs = [torch.rand((s, R), device=dev, generator=g) for s in shape]
    outs = {}
    fh = open(args.out, "a") if args.out else None
    cache_key = None
    plan = None
    for sp in specs:
        d = sp["mode"]
        key = (d, sp.get("layout"), sp.get("slab_shift"), tuple(sp.get("shifts") or []), tuple(sp.get("order") or []),
               json.dumps(sp.get("sweep")), sp.get("warps"))
        if key != cache_key:
            plan = None
            gc.collect()  # plans and their shards reference each other
            torch.cuda.empty_cache()
            plan = sk.build_mode_plan(t, d, pcfg, keep_permutation=False)
            t0 = time.perf_counter()
            if sp.get("layout") == "panel":
                warps = sp.get("warps") or panel_shape(len(shape), R)[0]
                plan.to_panels(sp["slab_shift"], sp["shifts"], warps, sp.get("order"),
                               sweep={int(k): v for k, v in (sp.get("sweep") or {}).items()})
            elif sp.get("shifts"):
                plan.to_blocked(sp["shifts"], sp.get("order"))
            block_s = time.perf_counter() - t0
            cache_key = key
        pl = sk.PlatformConfig(devices=1, rank=R, accumulation=sp.get("acc", "atomic"), tile_nnz=sp.get("tile", 0),
                               kernel_variant=sp.get("variant", 0), panel_lockstep=sp.get("lockstep", True))
        if plan.layout == "panel":
            ex = _PanelExec(plan, list(range(plan.shard_count)), pl, R, dev)
        else:
            ex = _ShardExec(plan, list(range(plan.shard_count)), pl, R, dev)
        coords, vals = _plan_arrays(plan, dev)
        if d not in outs:
            outs[d] = torch.empty((shape[d], R), device=dev)
        out = outs[d]
        stream = torch.cuda.current_stream(dev).cuda_stream
        times = []
        for rep in range(args.reps + 1):
            out.zero_()
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ex.run(coords, vals, plan.nnz, d, facs, out, pl, stream, events=ev)
            torch.cuda.synchronize()
            if rep:
                times.append(ev[0].elapsed_time(ev[1]))
        alg = bench.algorithmic_bytes(shape, nnz, R, d)
        ms = sum(times) / len(times)
        rec = dict(sp, ms=ms, ms_all=times, groups=(int(sum(len(x) for x in plan.groups)) if plan.groups else
                           (plan.panel["groups"] if plan.layout == "panel" else 0)),
                   tiles=ex.num_tiles, tile_nnz=ex.tile_nnz, frac_alg=alg / (ms * 1e-3) / 6457.4e9,
                   block_s=block_s, checksum=float(out.double().sum().item()))
        line = json.dumps(rec)
        print(line, flush=True)
        if fh:
            fh.write(line + "\n")
            fh.flush()
        del ex, coords, vals


if __name__ == "__main__":
    main()
