"""Property tests (hypothesis) of the GPU path against the CPU oracle.

Random tensors over the reference's domain -- N = 3..5 modes, ragged shapes
(size-1 modes included), 0..4000 nonzeros, uniform or Zipf draws (heavy
collisions), both partition strategies, devices/oversubscription/ISP
capacity sweeps, tile sizes from 1 -- must give:
  * the bit-exact reference plan (permutation, bounds, offsets, ISPs);
  * MTTKRP within the reference metric (<= 1e-4) for both accumulation
    disciplines and both execution layouts.
"""

import warnings

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import paper_2507_15121_b200 as sk  # noqa: E402

case = st.fixed_dictionaries({
    "shape": st.lists(st.integers(1, 60), min_size=3, max_size=5),
    "nnz": st.integers(0, 4000),
    "zipf": st.booleans(),
    "seed": st.integers(0, 10_000),
    "devices": st.integers(1, 5),
    "oversub": st.integers(1, 4),
    "cap": st.sampled_from([1, 3, 16, 100, 8192]),
    "strategy": st.sampled_from(["equal-index", "nnz-balanced"]),
    "rank": st.sampled_from([1, 3, 8, 16, 32]),
    "tile": st.sampled_from([1, 5, 32, 64, 0]),
})


def _tensor(c):
    rng = np.random.default_rng(c["seed"])
    shape = tuple(c["shape"])
    n = c["nnz"]
    if c["zipf"]:
        idx = np.stack([np.minimum(rng.zipf(1.5, n) - 1, s - 1) for s in shape], 1)
    else:
        idx = np.stack([rng.integers(0, s, n) for s in shape], 1) if n else np.zeros((0, len(shape)), np.int64)
    idx = np.unique(idx, axis=0) if n else idx  # reference tensors hold unique tuples
    rng.shuffle(idx)
    vals = rng.standard_normal(len(idx))
    return sk.SparseTensorCOO(shape, idx, vals)


@settings(max_examples=60, deadline=None, suppress_health_check=list(HealthCheck))
@given(case)
def test_plan_and_mttkrp_properties(c):
    t = _tensor(c)
    n = t.num_modes
    pcfg = sk.PartitionConfig(devices=c["devices"], oversubscription=c["oversub"], isp_capacity=c["cap"],
                              strategy=c["strategy"])
    fs = [np.random.default_rng(c["seed"] + w).random((s, c["rank"])) for w, s in enumerate(t.shape)]
    for d in range(n):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            p = sk.build_mode_plan(t, d, pcfg)
        ref = oracle.plan(t.indices, t.shape, d, c["devices"], c["oversub"], c["cap"], c["strategy"])
        assert np.array_equal(p.order(), ref["order"])
        assert np.array_equal(p.bounds, ref["bounds"])
        assert np.array_equal(p.offsets, ref["offsets"])
        assert all(np.array_equal(s_.isp_boundaries, i_) for s_, i_ in zip(p.shards, ref["isps"]))
        expect = oracle.mttkrp_seq(t.indices, t.values, fs, d)
        for acc in ("deterministic-reduce", "atomic"):
            cfg = sk.PlatformConfig(devices=c["devices"], rank=c["rank"], accumulation=acc, tile_nnz=c["tile"])
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg, update_factors=False)
            err = np.max(np.abs(out - expect) / np.maximum(np.abs(expect), 1.0)) if expect.size else 0.0
            assert err <= 1e-4, (acc, d, err)
        if c["rank"] in (8, 16, 32) and n <= 5 and t.nnz:
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                q = sk.build_mode_plan(t, d, pcfg)
            cfg = sk.PlatformConfig(devices=c["devices"], rank=c["rank"], accumulation="atomic", layout="blocked",
                                    l2_budget_mb=0, tile_nnz=c["tile"])
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                out, _ = sk.mttkrp_mode(q, sk.make_devices(fs, cfg), cfg, update_factors=False)
            err = np.max(np.abs(out - expect) / np.maximum(np.abs(expect), 1.0))
            assert err <= 1e-4, ("blocked", d, err)
            # output-stationary panel layout (small slabs, several block groups)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                q = sk.build_mode_plan(t, d, pcfg)
            cfg = sk.PlatformConfig(devices=c["devices"], rank=c["rank"], layout="panel", panel_l2_mb=0,
                                    slab_rows=64)
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                out, _ = sk.mttkrp_mode(q, sk.make_devices(fs, cfg), cfg, update_factors=False)
            err = np.max(np.abs(out - expect) / np.maximum(np.abs(expect), 1.0))
            assert err <= 1e-4, ("panel", d, err)
