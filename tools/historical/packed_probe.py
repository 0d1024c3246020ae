"""HISTORICAL (needs the removed SKRP_FLAG_PACKED kernel; see
profiles/sweeps/r02an_packed_metadata_negative.jsonl).

A/B of the packed-metadata tile kernel (SKRP_FLAG_PACKED: one u64 per
nonzero {row | pinned-in-block | streamed} + the value = 12 B instead of
16) against the production pin-one-stream-one kernel on the same cfg2 plan,
per mode: kernel time (CUDA events, median of --reps) and max rel diff.

  python tools/packed_probe.py --modes 0,1,2
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_15121_b200 as sk  # noqa: E402
from paper_2507_15121_b200 import _lib, engine  # noqa: E402

FLAG_PACKED = 128


def pack(coords, d, js_mode, jp_mode, shift):
    n = coords[d].numel()
    out = torch.empty(n, dtype=torch.int64, device=coords[d].device)
    step = 1 << 27
    for a in range(0, n, step):
        b = min(n, a + step)
        r = coords[d][a:b].to(torch.int64) & 0xFFFFFFFF
        p = coords[jp_mode][a:b].to(torch.int64) & ((1 << shift) - 1)
        s = coords[js_mode][a:b].to(torch.int64) & 0xFFFFFFFF
        out[a:b] = (r << 39) | (p << 21) | s
    return out


def timed(ex, coords, vals, nnz, d, facs, out, cfg, reps):
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for _ in range(reps + 1):
        out.zero_()
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ex.run(coords, vals, nnz, d, facs, out, cfg, st, events=ev)
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return float(np.median(ts[1:]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--modes", default="0,1,2")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    c = bench.CONFIGS[args.config]
    shape, nnz, R = c["shape"], c["nnz"], c["rank"]
    dev = torch.device("cuda", 0)
    t = sk.synth_tensor_device(shape, nnz, distribution=c["dist"], seed=0)
    facs = [torch.from_numpy(f.data.astype(np.float32)).to(dev) for f in sk.random_factors(shape, R, seed=0)]
    pcfg = sk.PartitionConfig(devices=1, strategy=c["strategy"])
    cfg = sk.PlatformConfig(rank=R, accumulation="atomic", layout="auto")
    for d in [int(x) for x in args.modes.split(",")]:
        p = sk.build_mode_plan(t, d, pcfg, keep_permutation=False)
        engine.apply_layout(p, cfg, R)
        ex = engine._shard_exec(p, list(range(p.shard_count)), cfg, R, dev)
        coords, vals = engine._plan_arrays(p, dev)
        ins = [w for w in range(3) if w != d]
        js = 0 if ex.flags & _lib.FLAG_STREAM_INPUT0 else 1
        jsm, jpm = ins[js], ins[1 - js]
        shift = p.block_shifts[jpm]
        ok = (shape[d] < (1 << 23) and shape[jsm] < (1 << 21) and 0 <= shift <= 18
              and len(ex.segments) == 1)
        out = torch.zeros(shape[d], R, device=dev)
        ms_ref = timed(ex, coords, vals, p.nnz, d, facs, out, cfg, args.reps)
        ref = out.clone()
        rec = {"mode": d, "layout": p.layout, "block_shifts": list(p.block_shifts), "streamed_mode": jsm,
               "pinned_mode": jpm, "ms_production": ms_ref, "packable": ok}
        if ok:
            packed = pack(coords, d, jsm, jpm, shift)
            seg = ex.segments[0]
            tiles = seg["tiles"].clone()
            starts, ends = tiles[0::2], tiles[1::2]
            blk_s = (coords[jpm][starts].to(torch.int64) & 0xFFFFFFFF) >> shift
            blk_e = (coords[jpm][ends - 1].to(torch.int64) & 0xFFFFFFFF) >> shift
            rec["tiles_single_block"] = bool(torch.equal(blk_s, blk_e))
            tiles[1::2] = ends | (blk_s << 40) if shift == 18 else ends
            seg["tiles"] = tiles
            ex.flags |= FLAG_PACKED
            pc = list(coords)
            pc[d] = packed
            ms_pk = timed(ex, pc, vals, p.nnz, d, facs, out, cfg, args.reps)
            diff = float(((out - ref).abs() / ref.abs().clamp_min(1.0)).max())
            rec.update(ms_packed=ms_pk, max_rel_diff=diff, kernel=_lib.launch_log()[-1][1],
                       metadata_bytes_saved_gb=p.nnz * 4 / 1e9)
            del packed, pc
        print(json.dumps(rec), flush=True)
        del ex, p, coords, vals, out, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
