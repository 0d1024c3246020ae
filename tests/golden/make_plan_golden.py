#!/usr/bin/env python
"""Plan-cache files written by the REFERENCE's save_plan (partition.py:270-292),
run here where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_plan_golden.py

tests/golden/plans/<name>_m<d>.plan for a few golden tensors / modes (f64 and
f32 values, both strategies) + plans/index.json (build_time of each file, so
our save_plan can be checked byte-for-byte)."""
import json
import os

import numpy as np
from shardkrp.partition import PartitionConfig, build_mode_plan, save_plan
from shardkrp.tensor import SparseTensorCOO

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    syn = np.load(os.path.join(HERE, "synth.npz"))
    out_dir = os.path.join(HERE, "plans")
    os.makedirs(out_dir, exist_ok=True)
    index = []
    for name, d, strategy, dtype in [("u3", 0, "equal-index", "float64"), ("z4", 2, "nnz-balanced", "float64"),
                                     ("u5", 4, "equal-index", "float32"), ("z3", 1, "nnz-balanced", "float32")]:
        shape = tuple(int(x) for x in syn[f"{name}_shape"])
        t = SparseTensorCOO(shape, syn[f"{name}_indices"], syn[f"{name}_values"].astype(dtype), name=name)
        p = build_mode_plan(t, d, PartitionConfig(devices=2, strategy=strategy, isp_capacity=64))
        fn = f"{name}_m{d}.plan"
        save_plan(p, os.path.join(out_dir, fn))
        index.append(dict(file=fn, tensor=name, mode=d, strategy=strategy, dtype=dtype, build_time=p.build_time,
                          devices=2, isp_capacity=64))
    with open(os.path.join(out_dir, "index.json"), "w") as fh:
        json.dump(index, fh, indent=1)
    print(len(index), "plan files")


if __name__ == "__main__":
    main()
