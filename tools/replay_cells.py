"""Drive tools/replay_cells.cu on a real cells layout (cfg2, one mode): the
layout's own entries replayed in three orders without the reduction, beside
the production cells kernel on the same layout.  One JSON line per run.

  python tools/replay_cells.py --config cfg2 --mode 0
"""

import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2507_15121_b200 as sk  # noqa: E402
from paper_2507_15121_b200 import engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--mode", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "bin", "libreplay_cells.so"))
    lib.replay_cells.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_float)]
    cfg = bench.CONFIGS[args.config]
    shape, nnz, R = cfg["shape"], cfg["nnz"], cfg["rank"]
    dev = torch.device("cuda", 0)
    tensor = sk.synth_tensor_device(shape, nnz, distribution=cfg["dist"], seed=0)
    facs = [torch.from_numpy(f.data.astype(np.float32)).to(dev) for f in sk.random_factors(shape, R, seed=0)]
    d = args.mode
    c = sk.PlatformConfig(rank=R, layout="cells")
    p = sk.build_mode_plan(tensor, d, sk.PartitionConfig(devices=1, strategy=cfg["strategy"]), keep_permutation=False)
    p.to_cells(range(p.shard_count), engine.choose_cells(p, R, c))
    ex = engine._shard_exec(p, list(range(p.shard_count)), c, R, dev)
    out = torch.zeros(shape[d], R, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for _ in range(args.reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ex.run(p.coords, p.vals, p.nnz, p.mode, facs, out, c, st)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"mode": d, "what": "cells kernel (production)", "ms": float(np.median(ts[1:]))}), flush=True)
    cl = p.cells
    ent, soff = cl["entries"], cl["stripe_offsets"].to(dev)
    fo, fi = facs[cl["outer_mode"]], facs[cl["inner_mode"]]
    names = {0: "GPU-wide windows", 1: "per-warp contiguous chunks", 2: "cells kernel order (stripes per warp)"}
    for nb in (4, 8):
        for order in (0, 1, 2):
            ms = ctypes.c_float()
            rc = lib.replay_cells(ent.data_ptr(), int(cl["num_entries"]), soff.data_ptr(), int(cl["stripes"]),
                                  fo.data_ptr(), fi.data_ptr(), order, nb, args.reps, ctypes.byref(ms))
            print(json.dumps({"mode": d, "what": f"replay, {names[order]}", "nb": nb, "rc": rc, "ms": ms.value}),
                  flush=True)


if __name__ == "__main__":
    main()
