"""Where the drop-in API's host time goes (cfg2): make_devices (fp64 numpy ->
HBM fp32) vs mttkrp_all_modes (compute + fp64 numpy export), and the cost
of first-touching fresh float64 output arrays.  One JSON line."""

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


def main():
    cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    c = bench.CONFIGS[cfgname]
    shape, nnz, R = c["shape"], c["nnz"], c["rank"]
    t = sk.synth_tensor_device(shape, nnz, distribution=c["dist"], seed=0)
    pcfg = sk.PartitionConfig(devices=1, strategy=c["strategy"])
    plans = [sk.build_mode_plan(t, d, pcfg, keep_permutation=False) for d in range(len(shape))]
    np_f = [f.data for f in sk.random_factors(shape, R, seed=0)]
    cfg = sk.PlatformConfig(devices=1, rank=R, layout="auto")
    sk.mttkrp_all_modes(plans, sk.make_devices(np_f, cfg), cfg)  # warm-up: layouts, staging, graphs
    res = {"config": cfgname}
    md, allm, tot = [], [], []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        devs = sk.make_devices(np_f, cfg)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        outs, _ = sk.mttkrp_all_modes(plans, devs, cfg)
        t2 = time.perf_counter()
        md.append(t1 - t0)
        allm.append(t2 - t1)
        tot.append(t2 - t0)
        del outs
    res.update(make_devices_ms=1e3 * min(md), mttkrp_all_modes_ms=1e3 * min(allm), total_ms=1e3 * min(tot))
    t0 = time.perf_counter()
    a = [np.empty((s, R)) for s in shape]
    t1 = time.perf_counter()
    for x in a:
        x.fill(0.0)
    t2 = time.perf_counter()
    res.update(np_empty_ms=1e3 * (t1 - t0), first_touch_fill_ms=1e3 * (t2 - t1),
               out_bytes=sum(x.nbytes for x in a), cores=os.cpu_count())
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
