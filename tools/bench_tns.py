#!/usr/bin/env python
"""GPU .tns ingestion throughput vs the host (reference-style) parser.

    python tools/bench_tns.py [--lines 20000000] [--dir /tmp]

Writes a FROSTT file of cfg2-shaped coordinates and %.17g values, parses it
with parse_tns_gpu (bytes -> device arrays) and a 1/20 slice with the host
parser (the reference's algorithm), checks they agree, prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2507_15121_b200 as sk

    ap = argparse.ArgumentParser()
    ap.add_argument("--lines", type=int, default=20_000_000)
    ap.add_argument("--dir", default="/tmp")
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    n = args.lines
    shape = (4_800_000, 1_800_000, 1_800_000)
    idx = np.stack([rng.integers(1, s + 1, n) for s in shape], 1)
    vals = rng.random(n)
    path = os.path.join(args.dir, "bench.tns")
    t0 = time.perf_counter()
    with open(path, "w") as fh:
        step = 1_000_000
        for a in range(0, n, step):
            b = min(n, a + step)
            rows = np.char.add(np.char.add(np.char.add(idx[a:b, 0].astype(str), " "),
                                           np.char.add(idx[a:b, 1].astype(str), " ")),
                               np.char.add(np.char.add(idx[a:b, 2].astype(str), " "),
                                           np.array([f"{v:.17g}" for v in vals[a:b]])))
            fh.write("\n".join(rows.tolist()) + "\n")
    write_s = time.perf_counter() - t0
    size = os.path.getsize(path)
    sk.parse_tns_gpu(path, coalesce_duplicates=True)  # warm-up (CUDA context, page cache)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tg = sk.parse_tns_gpu(path, coalesce_duplicates=True)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    # host parser on the first 1/20 of the lines
    sub = os.path.join(args.dir, "bench_sub.tns")
    with open(path, "rb") as fi, open(sub, "wb") as fo:
        for i, line in enumerate(fi):
            if i >= n // 20:
                break
            fo.write(line)
    t0 = time.perf_counter()
    th = sk.parse_tns(sub, coalesce_duplicates=True)
    host_s = time.perf_counter() - t0
    m = th.nnz
    same = (np.array_equal(tg.indices[:m], th.indices) and tg.values[:m].tobytes() == th.values.tobytes()) \
        if tg.stats.duplicates == 0 else None
    os.remove(path)
    os.remove(sub)
    print(json.dumps({"lines": n, "file_bytes": size, "gpu_parse_s": gpu_s, "gpu_gbs": size / gpu_s / 1e9,
                      "gpu_lines_per_s": n / gpu_s, "host_lines": m, "host_parse_s": host_s,
                      "host_lines_per_s": m / host_s, "speedup": (n / gpu_s) / (m / host_s),
                      "prefix_identical": same, "write_s": write_s,
                      "note": "GPU time includes reading the file (page cache), upload, parse, duplicate check and "
                              "the host copies of indices/values"}))


if __name__ == "__main__":
    main()
