"""Generate the golden fixtures under tests/golden/ from the REFERENCE package.

Runs only in the build container, where the read-only reference lives at
/root/reference/pkg/src (it does not exist on the GPU box; the fixtures it
writes are committed and travel instead).  Nothing in the product imports this.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb \
        python tests/golden/make_golden.py

What is pinned:
  * spec.json         SPEC.md known-answer examples, evaluated by the reference
  * synth.npz         reference synth_tensor / random_factors outputs (small cases)
  * cfg1.json         sha256 digests of the cfg1 tensor + factors (1000^3, 1M nnz)
  * cfg1_mode0.npz    reference plan summary + dense oracle output, cfg1 mode 0
  * plans.npz         build_mode_plan: permutation, bounds, offsets, ISP bounds
  * bounds.npz        _nnz_balanced_bounds on crafted count vectors (edge cases)
  * mttkrp.npz        dense_mttkrp_oracle per mode + chained engine outputs
  * cpd.npz           cp_als fit history / lambdas (engine and oracle impls)
  * ring.json         ring_all_gather ledgers for M = 1..8
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb_cache_golden")

import shardkrp as sk  # noqa: E402  (the reference)
from shardkrp import partition as skp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# small tensors used across fixtures: (name, shape, nnz, dist, value_dist, seed)
SMALL = [
    ("u3", (50, 40, 30), 2000, "uniform", "uniform", 1),
    ("z3", (1000, 100, 100), 10000, "zipf", "uniform", 0),
    ("z4", (20, 15, 10, 8), 3000, "zipf", "normal", 3),
    ("d3", (4, 4, 4), 64, "uniform", "uniform", 2),
    ("u5", (12, 10, 8, 6, 5), 1500, "uniform", "uniform", 5),
    ("s3", (7, 300, 9), 1200, "uniform", "normal", 11),
]


def small_tensors():
    out = {}
    for name, shape, nnz, dist, vdist, seed in SMALL:
        out[name] = sk.synth_tensor(shape, nnz, distribution=dist, value_dist=vdist, seed=seed)
    return out


def gen_spec():
    res = {}
    # dense oracle, single nonzero X(0,1,2)=2 (SPEC tensor-core example)
    t = sk.SparseTensorCOO((2, 2, 3), np.array([[0, 1, 2]]), np.array([2.0]))
    a = np.array([[1.0, 2.0], [0.0, 0.0]])
    b = np.array([[0.0, 0.0], [3.0, 4.0]])
    c = np.zeros((3, 2))
    res["oracle_single_nnz_mode2"] = sk.dense_mttkrp_oracle(t, [a, b, c], 2).tolist()
    res["elementwise"] = [int(x) if i == 0 else list(map(float, x)) for i, x in enumerate(
        sk.elementwise_compute(sk.NonzeroElement((0, 1, 2), 2.0), [a, b, c], 2))]
    # 2x2x2 all-ones, R=1, d=0 through the engine
    idx = np.array([[i, j, k] for i in range(2) for j in range(2) for k in range(2)])
    t8 = sk.SparseTensorCOO((2, 2, 2), idx, np.ones(8))
    fac = [sk.FactorMatrix(w, np.ones((2, 1))) for w in range(3)]
    cfg = sk.PlatformConfig(devices=1, rank=1)
    plan = sk.build_mode_plan(t8, 0, sk.PartitionConfig())
    out, _ = sk.mttkrp_mode(plan, sk.make_devices(fac, cfg), cfg)
    res["engine_ones_2x2x2_mode0"] = out.tolist()
    res["equal_index_8_2"] = skp._equal_index_bounds(8, 2).tolist()
    res["isp_10_4"] = skp._isp_boundaries(10, 4).tolist()
    res["isp_0_4"] = skp._isp_boundaries(0, 4).tolist()
    res["khatri_rao"] = sk.khatri_rao(np.array([[1.0], [2.0]]), np.array([[3.0], [4.0]])).tolist()
    res["staging_100_3_f64"] = sk.collective.staging_nbytes(100, 3, 8)
    # zipf (1000,100,100), 10K nnz, m=4: nnz-balanced vs equal-index max shard
    z = sk.synth_tensor((1000, 100, 100), 10000, distribution="zipf", seed=0)
    maxes = {}
    for strat in ("equal-index", "nnz-balanced"):
        p = sk.build_mode_plan(z, 0, sk.PartitionConfig(devices=4, strategy=strat))
        maxes[strat] = max(s.nnz for s in p.shards)
    res["zipf_max_shard"] = maxes
    return res


def gen_synth():
    arrs = {}
    for name, t in small_tensors().items():
        arrs[f"{name}_indices"] = t.indices
        arrs[f"{name}_values"] = t.values
        arrs[f"{name}_shape"] = np.array(t.shape, dtype=np.int64)
        for r in (1, 8, 32):
            fs = sk.random_factors(t.shape, r, seed=7)
            for w, f in enumerate(fs):
                arrs[f"{name}_F{r}_{w}"] = f.data
    # float32 value opt-in
    t32 = sk.synth_tensor((30, 20, 10), 500, seed=4, value_dtype=np.float32)
    arrs["f32_indices"] = t32.indices
    arrs["f32_values"] = t32.values
    return arrs


def gen_cfg1():
    t = sk.synth_tensor((1000, 1000, 1000), 1_000_000, "uniform", value_dist="uniform", seed=0)
    fs = sk.random_factors(t.shape, 32, seed=0)
    meta = {
        "indices_sha256": sha(t.indices),
        "values_sha256": sha(t.values),
        "factor_sha256": [sha(f.data) for f in fs],
        "duplicates": int(t.stats.duplicates),
        "first_rows": t.indices[:4].tolist(),
        "first_values": t.values[:4].tolist(),
    }
    plan = sk.build_mode_plan(t, 0, sk.PartitionConfig())
    order = np.argsort(t.indices[:, 0].astype(np.int64), kind="stable")
    meta["plan_order_sha256"] = sha(order.astype(np.int64))
    meta["plan_bounds"] = [s.index_range for s in plan.shards]
    meta["plan_nnz"] = [s.nnz for s in plan.shards]
    meta["plan_isps"] = plan.isp_counts
    # oracle output (fp64, storage order) via the reference's own loop (slow, ~10 s)
    expect = sk.dense_mttkrp_oracle(t, fs, 0)
    return meta, {"mode0_oracle": expect}


PLAN_CFGS = [
    # (devices, oversub, isp_capacity, strategy)
    (1, 4, 8192, "equal-index"),
    (2, 1, 7, "equal-index"),
    (3, 2, 64, "nnz-balanced"),
    (4, 4, 100, "nnz-balanced"),
    (4, 1, 1, "equal-index"),
    (8, 4, 33, "nnz-balanced"),
    (8, 4, 33, "equal-index"),
    (2, 3, 8192, "nnz-balanced"),
]


def gen_plans():
    arrs = {}
    for name, t in small_tensors().items():
        for d in range(t.num_modes):
            for ci, (m, s, c, strat) in enumerate(PLAN_CFGS):
                cfg = sk.PartitionConfig(devices=m, oversubscription=s, isp_capacity=c, strategy=strat)
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", RuntimeWarning)
                    plan = sk.build_mode_plan(t, d, cfg)
                key = f"{name}_m{d}_c{ci}"
                arrs[key + "_ranges"] = np.array([s_.index_range for s_ in plan.shards], dtype=np.int64)
                arrs[key + "_nnz"] = np.array([s_.nnz for s_ in plan.shards], dtype=np.int64)
                arrs[key + "_isp"] = np.concatenate([s_.isp_boundaries for s_ in plan.shards])
                if ci == 0:
                    arrs[f"{name}_m{d}_sorted_indices"] = plan._indices
                    arrs[f"{name}_m{d}_sorted_values"] = plan._values
    arrs["cfgs"] = np.array([(m, s, c, 0 if st == "equal-index" else 1) for m, s, c, st in PLAN_CFGS])
    return arrs


def gen_bounds():
    rng = np.random.default_rng(123)
    arrs = {}
    cases = []
    # crafted edge cases
    cases.append((np.array([5, 0, 0, 0, 5], dtype=np.int64), 3))
    cases.append((np.array([100, 1, 1, 1, 1, 1, 1], dtype=np.int64), 4))
    cases.append((np.zeros(10, dtype=np.int64), 4))
    cases.append((np.array([1, 1, 1, 1], dtype=np.int64), 4))
    cases.append((np.array([0, 0, 7, 0, 0, 0, 3, 0], dtype=np.int64), 5))
    cases.append((np.array([3], dtype=np.int64), 1))
    cases.append((np.array([9, 9, 9, 1, 1, 1, 1, 1, 1, 1, 1, 1], dtype=np.int64), 6))
    for _ in range(150):
        n = int(rng.integers(1, 400))
        k = int(rng.integers(1, min(n, 40) + 1))
        kind = rng.integers(0, 4)
        if kind == 0:
            counts = rng.integers(0, 50, n)
        elif kind == 1:
            counts = (rng.zipf(1.3, n) - 1).clip(0, 10000)
        elif kind == 2:
            counts = np.where(rng.random(n) < 0.7, 0, rng.integers(1, 1000, n))
        else:
            counts = np.sort(rng.integers(0, 3000, n))[::-1].copy()
        cases.append((counts.astype(np.int64), k))
    for i, (counts, k) in enumerate(cases):
        arrs[f"counts_{i}"] = counts
        arrs[f"k_{i}"] = np.array(k)
        arrs[f"bounds_{i}"] = skp._nnz_balanced_bounds(counts, k)
    arrs["n_cases"] = np.array(len(cases))
    return arrs


def gen_mttkrp():
    arrs = {}
    for name, t in small_tensors().items():
        for r in (1, 8, 32):
            fs = sk.random_factors(t.shape, r, seed=7)
            for d in range(t.num_modes):
                arrs[f"{name}_R{r}_oracle_{d}"] = sk.dense_mttkrp_oracle(t, fs, d)
        # chained all-mode run through the reference engine (deterministic-reduce)
        for m in (1, 3):
            pcfg = sk.PartitionConfig(devices=m)
            cfg = sk.PlatformConfig(devices=m, rank=8)
            plans = sk.build_all_plans(t, pcfg)
            fs = sk.random_factors(t.shape, 8, seed=7)
            outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
            for d, o in enumerate(outs):
                arrs[f"{name}_chain_m{m}_{d}"] = o
    return arrs


def gen_cpd():
    arrs = {}
    t = sk.synth_tensor((30, 20, 10), 1500, seed=9)
    for impl in ("engine", "oracle"):
        model, _ = sk.cp_als(t, 4, 3, seed=1, mttkrp_impl=impl)
        arrs[f"u_{impl}_fit"] = np.array(model.fit_history)
        arrs[f"u_{impl}_lambdas"] = model.lambdas
        for w, f in enumerate(model.factors):
            arrs[f"u_{impl}_F{w}"] = f.data
    # noiseless rank-4 (SPEC acceptance #7): dense 40x30x20 kept as sparse
    rng = np.random.default_rng(5)
    a, b, c = (rng.random((n, 4)) for n in (40, 30, 20))
    dense = np.einsum("ir,jr,kr->ijk", a, b, c)
    idx = np.argwhere(np.ones_like(dense, dtype=bool))
    tr = sk.SparseTensorCOO(dense.shape, idx, dense[tuple(idx.T)])
    model, _ = sk.cp_als(tr, 4, 25, seed=0)
    arrs["r4_fit"] = np.array(model.fit_history)
    return arrs


def gen_ring():
    out = []
    rng = np.random.default_rng(2)
    for m in range(1, 9):
        rows = int(rng.integers(m, 40))
        cuts = np.sort(rng.choice(np.arange(1, rows), size=m - 1, replace=False)) if m > 1 else []
        edges = [0, *map(int, cuts), rows]
        ownership = [[(edges[j], edges[j + 1])] for j in range(m)]
        bufs = []
        for j in range(m):
            buf = np.full((rows, 2), -1.0)
            lo, hi = ownership[j][0]
            buf[lo:hi] = rng.random((hi - lo, 2))
            bufs.append(buf)
        parts = sk.FactorPartitionSet(0, ownership, bufs)
        expect = sk.gather_broadcast_oracle(parts)
        ledger = sk.TransferLedger()
        steps = sk.ring_all_gather(parts, ledger)
        out.append({
            "m": m,
            "rows": rows,
            "ownership": ownership,
            "steps": steps,
            "records": [(r.step, r.sender, r.receiver, r.byte_count, r.kind) for r in ledger.records],
            "final_equals_oracle": all(np.array_equal(b_, expect) for b_ in parts.buffers),
        })
    return out


def main():
    with open(os.path.join(HERE, "spec.json"), "w") as fh:
        json.dump(gen_spec(), fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "synth.npz"), **gen_synth())
    meta, arrs = gen_cfg1()
    with open(os.path.join(HERE, "cfg1.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "cfg1_mode0.npz"), **arrs)
    np.savez_compressed(os.path.join(HERE, "plans.npz"), **gen_plans())
    np.savez_compressed(os.path.join(HERE, "bounds.npz"), **gen_bounds())
    np.savez_compressed(os.path.join(HERE, "mttkrp.npz"), **gen_mttkrp())
    np.savez_compressed(os.path.join(HERE, "cpd.npz"), **gen_cpd())
    with open(os.path.join(HERE, "ring.json"), "w") as fh:
        json.dump(gen_ring(), fh, indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
