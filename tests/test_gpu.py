"""GPU parity tests: the CUDA path (through the C ABI) vs the pinned oracle.

Bars:
  * partition / index work: bit-exact (permutation, sorted arrays, bounds,
    offsets, ISP boundaries);
  * MTTKRP output: max |gpu - ref| / max(|ref|, 1) <= 1e-4 per mode (fp32,
    the reference's cli.py:247-261 metric), chained replay for all-mode runs;
  * deterministic-reduce: bit-identical across device counts and runs.
"""

import hashlib
import warnings

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_15121_b200 as sk  # noqa: E402
from paper_2507_15121_b200 import _lib  # noqa: E402

TOL = 1e-4
NAMES = ["u3", "z3", "z4", "d3", "u5", "s3"]



def _plain_bits(kernel_name):
    """The PLAIN template argument of a launched mttkrp_v2_kernel<NM, LPN, U,
    MINB, PLAIN, TRED> (bit 512 = the fiber-reuse instantiation)."""
    return int(kernel_name.split("<", 1)[1].split(",")[4])

def rel_err(got, expect):
    if expect.size == 0:
        return 0.0
    return float(np.max(np.abs(got - expect) / np.maximum(np.abs(expect), 1.0)))


def tensor_from(g, name):
    s = g("synth.npz")
    return sk.SparseTensorCOO(tuple(int(x) for x in s[f"{name}_shape"]), s[f"{name}_indices"],
                              s[f"{name}_values"], name=name)


def factors_from(g, name, r, n):
    s = g("synth.npz")
    return [sk.FactorMatrix(w, s[f"{name}_F{r}_{w}"]) for w in range(n)]


def stream():
    return torch.cuda.current_stream().cuda_stream


# ------------------------------------------------------------------ primitives


@pytest.mark.parametrize("n,bits", [(1, 1), (100, 3), (4096, 8), (4097, 9), (100_003, 17),
                                    (1_000_000, 24), (300_000, 0), (65_537, 31)])
def test_stable_sort_bit_exact(n, bits):
    rng = np.random.default_rng(n + bits)
    hi = 1 << bits
    keys = rng.integers(0, hi, n, dtype=np.int64) if bits else np.zeros(n, dtype=np.int64)
    if bits > 4:  # heavy duplicates: stability matters
        keys[rng.random(n) < 0.3] = rng.integers(0, 4)
    k = torch.from_numpy(keys.astype(np.int32)).cuda()
    sk_ = torch.empty_like(k)
    perm = torch.empty_like(k)
    wsb = _lib.lib().skrp_sort_workspace_bytes(n, bits)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    _lib.call("skrp_stable_sort_by_key", k.data_ptr(), n, bits, sk_.data_ptr(), perm.data_ptr(),
              ws.data_ptr(), wsb, stream())
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(perm.cpu().numpy().astype(np.int64), order)
    assert np.array_equal(sk_.cpu().numpy().astype(np.int64), keys[order])


@pytest.mark.parametrize("n,bins", [(10, 1), (1000, 7), (500_000, 16384), (500_000, 16385),
                                    (2_000_000, 3_000_000)])
def test_histogram_and_scan(n, bins):
    rng = np.random.default_rng(bins)
    keys = (rng.zipf(1.3, n) - 1) % bins
    k = torch.from_numpy(keys.astype(np.int32)).cuda()
    counts = torch.empty(bins, dtype=torch.int64, device="cuda")
    _lib.call("skrp_histogram", k.data_ptr(), n, bins, counts.data_ptr(), stream())
    expect = np.bincount(keys, minlength=bins)
    assert np.array_equal(counts.cpu().numpy(), expect)
    pre = torch.empty(bins + 1, dtype=torch.int64, device="cuda")
    wsb = _lib.lib().skrp_scan_workspace_bytes(bins)
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    _lib.call("skrp_exclusive_scan_i64", counts.data_ptr(), bins, pre.data_ptr(), ws.data_ptr(), wsb, stream())
    assert np.array_equal(pre.cpu().numpy(), np.concatenate([[0], np.cumsum(expect)]))


# --------------------------------------------------------------------- plans


@pytest.mark.parametrize("name", NAMES)
def test_plans_bit_exact(golden, name):
    t = tensor_from(golden, name)
    plans = golden("plans.npz")
    for d in range(t.num_modes):
        for ci, (m, s, c, st) in enumerate(plans["cfgs"]):
            cfg = sk.PartitionConfig(devices=int(m), oversubscription=int(s), isp_capacity=int(c),
                                     strategy="equal-index" if st == 0 else "nnz-balanced")
            with warnings.catch_warnings():
                warnings.simplefilter("ignore", RuntimeWarning)
                p = sk.build_mode_plan(t, d, cfg)
            key = f"{name}_m{d}_c{ci}"
            assert np.array_equal(np.array([s_.index_range for s_ in p.shards]), plans[key + "_ranges"])
            assert np.array_equal(np.array([s_.nnz for s_ in p.shards]), plans[key + "_nnz"])
            assert np.array_equal(np.concatenate([s_.isp_boundaries for s_ in p.shards]), plans[key + "_isp"])
            if ci == 0:
                assert np.array_equal(p.order(), oracle.stable_order(t.indices, d))
                assert np.array_equal(p._indices, plans[f"{name}_m{d}_sorted_indices"])
                assert np.array_equal(p._values, plans[f"{name}_m{d}_sorted_values"])
                # device copy == the same permutation applied in u32 / fp32
                dev_idx = torch.stack(p.coords, 1).cpu().numpy().astype(np.uint64)
                assert np.array_equal(dev_idx, plans[f"{name}_m{d}_sorted_indices"])
                assert np.array_equal(p.vals.cpu().numpy(),
                                      plans[f"{name}_m{d}_sorted_values"].astype(np.float32))


def test_clamp_warning_matches_reference():
    t = sk.SparseTensorCOO((2, 3, 3), np.array([[0, 0, 0], [1, 2, 2]]), np.array([1.0, 2.0]))
    with pytest.warns(RuntimeWarning, match="clamping"):
        p = sk.build_mode_plan(t, 0, sk.PartitionConfig(devices=2))
    assert p.shard_count == 2


def test_cfg1_plan_digest(golden):
    meta = golden("cfg1.json")
    t = sk.synth_tensor((1000, 1000, 1000), 1_000_000, seed=0)
    assert hashlib.sha256(t.indices.tobytes()).hexdigest() == meta["indices_sha256"]
    p = sk.build_mode_plan(t, 0, sk.PartitionConfig())
    assert hashlib.sha256(p.order().tobytes()).hexdigest() == meta["plan_order_sha256"]
    assert [list(s.index_range) for s in p.shards] == meta["plan_bounds"]
    assert [s.nnz for s in p.shards] == meta["plan_nnz"]
    assert p.isp_counts == meta["plan_isps"]


# -------------------------------------------------------------------- MTTKRP


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("r", [1, 8, 32])
def test_mttkrp_matches_oracle(golden, name, r):
    t = tensor_from(golden, name)
    fs = factors_from(golden, name, r, t.num_modes)
    ref = golden("mttkrp.npz")
    for d in range(t.num_modes):
        got = sk.mttkrp(t, fs, d)
        assert got.dtype == np.float64 and got.shape == (t.shape[d], r)
        assert rel_err(got, ref[f"{name}_R{r}_oracle_{d}"]) <= TOL


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("acc", ["deterministic-reduce", "atomic"])
@pytest.mark.parametrize("tile", [1, 7, 32, 33, 1024])
def test_kernel_variants_and_tiles(golden, variant, acc, tile):
    t = tensor_from(golden, "z3")
    fs = factors_from(golden, "z3", 32, 3)
    ref = golden("mttkrp.npz")
    cfg = sk.PlatformConfig(devices=2, rank=32, accumulation=acc, tile_nnz=tile, kernel_variant=variant)
    pcfg = sk.PartitionConfig(devices=2, isp_capacity=64)
    for d in range(3):
        p = sk.build_mode_plan(t, d, pcfg)
        out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg, update_factors=False)
        assert rel_err(out, ref[f"z3_R32_oracle_{d}"]) <= TOL


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("m", [1, 3])
def test_all_modes_chained_replay(golden, name, m):
    """Chained all-mode run; mode d checked against the oracle replayed on
    the engine's own previous outputs (cli.py:247-261)."""
    t = tensor_from(golden, name)
    fs = factors_from(golden, name, 8, t.num_modes)
    cfg = sk.PlatformConfig(devices=m, rank=8)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        plans = sk.build_all_plans(t, sk.PartitionConfig(devices=m))
        outs, metrics = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
    facs = [f.data.copy() for f in fs]
    for d, out in enumerate(outs):
        expect = oracle.mttkrp_seq(t.indices, t.values, facs, d)
        assert rel_err(out, expect) <= TOL
        facs[d] = out
    # and the first mode against the reference engine's own chained output
    assert rel_err(outs[0], golden("mttkrp.npz")[f"{name}_chain_m{m}_0"]) <= TOL
    assert len(metrics.modes) == t.num_modes
    assert sum(metrics.modes[0].device_nnz) == t.nnz


def test_device_count_invariance_bit_exact(golden):
    t = tensor_from(golden, "z3")
    fs = factors_from(golden, "z3", 32, 3)
    pcfg = sk.PartitionConfig(devices=4, isp_capacity=100)
    plans = sk.build_all_plans(t, pcfg)
    results = []
    for m, sched in [(1, "dynamic"), (2, "static"), (4, "dynamic"), (4, "static"), (1, "dynamic")]:
        cfg = sk.PlatformConfig(devices=m, rank=32, scheduling=sched, tile_nnz=16)
        outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
        results.append(outs)
    for outs in results[1:]:
        for a, b in zip(results[0], outs):
            assert np.array_equal(a, b)


def test_device_count_invariance_auto_tile():
    """Default (auto) tile size: it is derived from the whole plan, so 1 and 4
    devices cut identical tiles and the deterministic carry tree is the same
    (auto_tile_nnz(10M) = 256 but auto_tile_nnz(10M / 4) = 128)."""
    from paper_2507_15121_b200.engine import auto_tile_nnz

    nnz = 10_000_000
    assert auto_tile_nnz(nnz) != auto_tile_nnz(nnz // 4)
    t = sk.synth_tensor_device((3000, 2000, 1000), nnz, seed=5)
    fs = sk.random_factors(t.shape, 32, seed=1)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=4), keep_permutation=False)
    results = []
    for m in (1, 4, 2):
        cfg = sk.PlatformConfig(devices=m, rank=32)
        outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
        results.append(outs)
    for outs in results[1:]:
        for a, b in zip(results[0], outs):
            assert np.array_equal(a, b)


def test_write_log_exclusivity(golden):
    t = tensor_from(golden, "u3")
    fs = factors_from(golden, "u3", 8, 3)
    cfg = sk.PlatformConfig(devices=4, rank=8)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=4))
    devs = sk.make_devices(fs, cfg)
    for p in plans:
        sk.mttkrp_mode(p, devs, cfg, collect_write_log=True)
        logs = [d.write_rows for d in devs]
        for i in range(4):
            for j in range(i + 1, 4):
                assert not (logs[i] & logs[j])
        assert set().union(*logs) == set(np.unique(t.indices[:, p.mode]).tolist())


def test_long_rows_many_tiles():
    """Patents-like: few output rows, each spanning many tiles and ISPs."""
    t = sk.synth_tensor((3, 300, 300), 200_000, seed=3)
    fs = sk.random_factors(t.shape, 32, seed=1)
    for acc in ("deterministic-reduce", "atomic"):
        cfg = sk.PlatformConfig(rank=32, accumulation=acc, tile_nnz=64, carry_chunk=4)
        p = sk.build_mode_plan(t, 0, sk.PartitionConfig(isp_capacity=512))
        out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg)
        expect = oracle.mttkrp_seq_c(t.indices, t.values, [f.data for f in fs], 0)
        assert rel_err(out, expect) <= TOL


def test_empty_and_single():
    t0 = sk.SparseTensorCOO((5, 4, 3), np.zeros((0, 3), dtype=np.uint64), np.zeros(0))
    fs = sk.random_factors(t0.shape, 8, seed=0)
    assert np.array_equal(sk.mttkrp(t0, fs, 1), np.zeros((4, 8)))
    t1 = sk.SparseTensorCOO((2, 2, 3), np.array([[0, 1, 2]]), np.array([2.0]))
    a = np.array([[1.0, 2.0], [0.0, 0.0]])
    b = np.array([[0.0, 0.0], [3.0, 4.0]])
    c = np.zeros((3, 2))
    got = sk.mttkrp(t1, [a, b, c], 2)
    assert got.tolist() == [[0, 0], [0, 0], [6, 16]]


def test_validation_errors_match_reference():
    t = sk.SparseTensorCOO((2, 2, 3), np.array([[0, 1, 2]]), np.array([2.0]))
    fs = sk.random_factors(t.shape, 2)
    with pytest.raises(ValueError, match="out of range"):
        sk.mttkrp(t, fs, 3)
    with pytest.raises(ValueError, match="one factor matrix per mode"):
        sk.mttkrp(t, fs[:2], 0)
    with pytest.raises(ValueError, match="ranks differ"):
        sk.mttkrp(t, [fs[0], fs[1], sk.FactorMatrix(2, np.ones((3, 3)))], 0)
    with pytest.raises(ValueError, match="rows, tensor needs"):
        sk.mttkrp(t, [fs[0], fs[1], sk.FactorMatrix(2, np.ones((4, 2)))], 0)


def test_cfg1_mode0(golden):
    t = sk.synth_tensor((1000, 1000, 1000), 1_000_000, seed=0)
    fs = sk.random_factors(t.shape, 32, seed=0)
    expect = golden("cfg1_mode0.npz")["mode0_oracle"]
    for acc in ("deterministic-reduce", "atomic"):
        cfg = sk.PlatformConfig(rank=32, accumulation=acc)
        p = sk.build_mode_plan(t, 0, sk.PartitionConfig())
        out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg)
        assert rel_err(out, expect) <= TOL


def test_host_c_abi_entry(golden):
    """skrp_mttkrp_host: dense_mttkrp_oracle's contract through one C call."""
    import ctypes

    t = tensor_from(golden, "z4")
    fs = factors_from(golden, "z4", 8, 4)
    ref = golden("mttkrp.npz")
    shape = np.array(t.shape, dtype=np.int64)
    mats = [np.ascontiguousarray(f.data) for f in fs]
    fptr = (ctypes.c_void_p * 4)(*[m.ctypes.data for m in mats])
    for d in range(4):
        out = np.empty((t.shape[d], 8))
        _lib.call("skrp_mttkrp_host", t.indices.ctypes.data, np.ascontiguousarray(t.values).ctypes.data,
                  t.nnz, 4, shape.ctypes.data, fptr, 8, d, out.ctypes.data, torch.cuda.current_device())
        assert rel_err(out, ref[f"z4_R8_oracle_{d}"]) <= TOL


# ---------------------------------------------------------------- collective


def test_ring_all_gather_device_buffers(golden):
    for case in golden("ring.json"):
        m, rows = case["m"], case["rows"]
        own = [[tuple(r) for r in o] for o in case["ownership"]]
        rng = np.random.default_rng(m)
        truth = rng.random((rows, 2)).astype(np.float32)
        bufs = []
        for j in range(m):
            b = torch.full((rows, 2), -1.0, device="cuda")
            for lo, hi in own[j]:
                b[lo:hi] = torch.from_numpy(truth[lo:hi]).cuda()
            bufs.append(b)
        parts = sk.FactorPartitionSet(0, own, bufs)
        ledger = sk.TransferLedger()
        assert sk.ring_all_gather(parts, ledger) == case["steps"]
        for b in bufs:
            assert np.array_equal(b.cpu().numpy(), truth)
        expect = [(r[0], r[1], r[2], r[3] // 2) for r in case["records"]]  # fp32 vs fp64 bytes
        assert [(r.step, r.sender, r.receiver, r.byte_count) for r in ledger.records] == expect


# --------------------------------------------------------------------- CP-ALS


def test_cp_als_rank4_recovery(golden):
    rng = np.random.default_rng(5)
    a, b, c = (rng.random((n, 4)) for n in (40, 30, 20))
    dense = np.einsum("ir,jr,kr->ijk", a, b, c)
    idx = np.argwhere(np.ones_like(dense, dtype=bool))
    t = sk.SparseTensorCOO(dense.shape, idx, dense[tuple(idx.T)])
    model, _ = sk.cp_als(t, 4, 25, seed=0)
    ref = golden("cpd.npz")["r4_fit"]
    assert model.fit_history[-1] > 0.99
    assert abs(model.fit_history[-1] - ref[-1]) < 1e-3
    assert all(b_ >= a_ - 1e-4 for a_, b_ in zip(model.fit_history, model.fit_history[1:]))


def test_cp_als_matches_reference_history(golden):
    t = sk.synth_tensor((30, 20, 10), 1500, seed=9)
    ref = golden("cpd.npz")
    for impl in ("engine", "oracle"):
        model, _ = sk.cp_als(t, 4, 3, seed=1, mttkrp_impl=impl)
        assert np.allclose(model.fit_history, ref["u_engine_fit"], rtol=0, atol=2e-4)
        assert np.allclose(model.lambdas, ref["u_engine_lambdas"], rtol=2e-3)


# ------------------------------------------------------------------ generator


def test_device_generator_laws():
    t = sk.synth_tensor_device((1000, 100, 100), 2_000_000, seed=3, unique=False)
    idx = t.indices
    assert idx.max(axis=0).tolist() == [999, 99, 99] and idx.min() == 0
    assert abs(t.values.mean() - 0.5) < 2e-3 and t.values.min() >= 0 and t.values.max() < 1
    z = sk.synth_tensor_device((1000, 100, 100), 1_000_000, distribution="zipf", seed=3, unique=False)
    cdf = sk.synth.zipf_cdf(1000, 1.2)
    head = np.mean(z.indices[:, 0] == 0)
    assert abs(head - cdf[0]) < 3e-3
    # same seed -> same tensor; other seed -> different
    t2 = sk.synth_tensor_device((1000, 100, 100), 2_000_000, seed=3, unique=False)
    assert np.array_equal(t2.indices, idx)


# ------------------------------------------------------------ runner paths


def test_runner_graph_and_host_paths(golden):
    """world == 1 runner: eager, one-graph replay and the host-buffer
    (pinned, copy-stream overlapped) path give identical chained outputs."""
    from paper_2507_15121_b200.distributed import DistributedMttkrp

    t = tensor_from(golden, "u3")
    fs = factors_from(golden, "u3", 32, 3)
    plans = sk.build_all_plans(t, sk.PartitionConfig(isp_capacity=100))
    runner = DistributedMttkrp(plans, sk.PlatformConfig(rank=32, tile_nnz=64))
    dev_f = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in fs]
    eager = [o.clone() for o in runner.run(dev_f)]
    g = runner.capture(dev_f)
    for o in runner.outputs:
        o.fill_(-7.0)
    g.replay()
    torch.cuda.synchronize()
    graphed = [o.clone() for o in runner.outputs]
    host_f = [torch.from_numpy(f.data.astype(np.float32)).pin_memory() for f in fs]
    host_o = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in eager]
    dev_f2 = [torch.zeros_like(f) for f in dev_f]
    h2d, d2h = runner.run_host(host_f, host_o, dev_f2)
    torch.cuda.synchronize()
    assert runner.needed_factors() == [1, 2]
    assert h2d == sum(host_f[w].numel() * 4 for w in (1, 2))
    assert d2h == sum(o.numel() * 4 for o in eager)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        assert torch.equal(eager[d], graphed[d])
        assert torch.equal(eager[d].cpu(), host_o[d])
        expect = oracle.mttkrp_seq(t.indices, t.values, facs, d)
        assert rel_err(eager[d].double().cpu().numpy(), expect) <= TOL
        facs[d] = eager[d].double().cpu().numpy()


# ---------------------------------------------------------- blocked layout


@pytest.mark.parametrize("name", ["u3", "z3", "z4", "u5"])
def test_blocked_layout_parity(golden, name):
    """L2-blocked execution layout (atomic, additive flushes): same outputs
    within tolerance, shard ranges unchanged, host plan views still bit-exact."""
    from paper_2507_15121_b200.engine import choose_blocking

    t = tensor_from(golden, name)
    fs = factors_from(golden, name, 32, t.num_modes)
    ref = golden("mttkrp.npz")
    plans = golden("plans.npz")
    for d in range(t.num_modes):
        p = sk.build_mode_plan(t, d, sk.PartitionConfig(devices=2))
        shards_before = [(s_.start, s_.stop, s_.index_range) for s_ in p.shards]
        shifts, _, _ = choose_blocking(p, 32, l2_bytes=1 << 10)  # tiny budget: force blocking
        shifts = shifts or [(-1 if w == d else 1) for w in range(t.num_modes)]
        p.to_blocked(shifts)
        assert p.layout == "blocked"
        assert [(s_.start, s_.stop, s_.index_range) for s_ in p.shards] == shards_before
        # every group lies inside its shard and groups tile the shard
        for s_, g in zip(p.shards, p.groups):
            if s_.nnz:
                assert g[0, 0] == s_.start and g[-1, 1] == s_.stop and np.all(g[1:, 0] == g[:-1, 1])
        assert np.array_equal(p._indices, plans[f"{name}_m{d}_sorted_indices"])
        for acc in ("atomic", "deterministic-reduce"):
            cfg = sk.PlatformConfig(devices=2, rank=32, accumulation=acc, tile_nnz=16, layout="blocked")
            out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg, update_factors=False)
            assert rel_err(out, ref[f"{name}_R32_oracle_{d}"]) <= TOL


@pytest.mark.parametrize("order_kind", ["default", "reversed"])
def test_blocked_output_blocks_parity(golden, order_kind):
    """Output-mode blocks (3-D L2 tiling: out block x input blocks) with the
    default and a reversed key order: outputs within tolerance for both
    disciplines, shard ranges and host plan views unchanged."""
    t = tensor_from(golden, "u3")
    fs = factors_from(golden, "u3", 32, t.num_modes)
    ref = golden("mttkrp.npz")
    plans = golden("plans.npz")
    for d in range(t.num_modes):
        p = sk.build_mode_plan(t, d, sk.PartitionConfig(devices=2))
        shards_before = [(s_.start, s_.stop, s_.index_range) for s_ in p.shards]
        shifts = [max(0, (s - 1).bit_length() - 2) for s in t.shape]  # ~4 blocks per mode
        order = None if order_kind == "default" else list(range(t.num_modes))[::-1]
        p.to_blocked(shifts, order)
        assert p.block_order == (order or [d] + [w for w in range(t.num_modes) if w != d])
        assert [(s_.start, s_.stop, s_.index_range) for s_ in p.shards] == shards_before
        for s_, g in zip(p.shards, p.groups):
            if s_.nnz:
                assert g[0, 0] == s_.start and g[-1, 1] == s_.stop and np.all(g[1:, 0] == g[:-1, 1])
        assert np.array_equal(p._indices, plans[f"u3_m{d}_sorted_indices"])
        for acc in ("atomic", "deterministic-reduce"):
            cfg = sk.PlatformConfig(devices=2, rank=32, accumulation=acc, tile_nnz=32, layout="blocked")
            out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg, update_factors=False)
            assert rel_err(out, ref[f"u3_R32_oracle_{d}"]) <= TOL


@pytest.mark.parametrize("name", ["u3", "z3", "z4", "u5"])
def test_panel_layout_parity(golden, name):
    """Output-stationary panel layout (slabs x block groups x warp stripes):
    every mode within tolerance of the oracle, shard ranges unchanged, host
    plan views still bit-exact, item rows tile every shard's row range."""
    from paper_2507_15121_b200.engine import panel_shape

    t = tensor_from(golden, name)
    fs = factors_from(golden, name, 32, t.num_modes)
    ref = golden("mttkrp.npz")
    plans = golden("plans.npz")
    warps, _ = panel_shape(t.num_modes, 32)
    for d in range(t.num_modes):
        p = sk.build_mode_plan(t, d, sk.PartitionConfig(devices=2))
        shards_before = [(s_.start, s_.stop, s_.index_range) for s_ in p.shards]
        shifts = [-1 if w == d else max(0, (s - 1).bit_length() - 2) for w, s in enumerate(t.shape)]
        p.to_panels(4, shifts, warps)  # 16-row slabs: many items, slabs straddle shards
        assert p.layout == "panel"
        assert [(s_.start, s_.stop, s_.index_range) for s_ in p.shards] == shards_before
        assert np.array_equal(p._indices, plans[f"{name}_m{d}_sorted_indices"])
        rows = p.panel["item_rows"]
        for j, s_ in enumerate(p.shards):
            mine = rows[p.panel["item_shard"] == j]
            lo, hi = s_.index_range
            if hi > lo:
                assert mine[0, 0] == lo and mine[-1, 1] == hi and np.all(mine[1:, 0] == mine[:-1, 1])
        offs = p.panel["item_offsets"].cpu().numpy()
        assert np.all(np.diff(offs, axis=1) >= 0)
        for acc in ("atomic", "deterministic-reduce"):
            cfg = sk.PlatformConfig(devices=2, rank=32, accumulation=acc)
            out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg, update_factors=False)
            assert rel_err(out, ref[f"{name}_R32_oracle_{d}"]) <= TOL


@pytest.mark.parametrize("rank", [8, 16, 32, 64])
def test_panel_all_modes_device_invariance(rank):
    """Panel layout through the engine (layout='panel', tiny L2 budget ->
    several block groups): chained all-mode parity for R in {8,16,32,64}, and
    bit-identical outputs for any device count / placement."""
    t = sk.synth_tensor((700, 300, 260), 300_000, seed=4)
    fs = sk.random_factors(t.shape, rank, seed=1)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=4, isp_capacity=512))
    results = []
    for m, sched in [(1, "dynamic"), (2, "static"), (4, "contiguous")]:
        cfg = sk.PlatformConfig(devices=m, rank=rank, scheduling=sched, layout="panel", panel_l2_mb=0,
                                slab_rows=64, panel_lockstep=(m != 2))
        outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
        results.append(outs)
    assert all(p.layout == "panel" and p.panel["groups"] > 1 for p in plans)
    for outs in results[1:]:
        for a, b in zip(results[0], outs):
            assert np.array_equal(a, b)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
        assert rel_err(results[0][d], expect) <= TOL
        facs[d] = results[0][d]


def test_blocked_deterministic_device_count_invariance():
    """Deterministic-reduce in the blocked layout (one launch per block group,
    read-add-write flushes, additive carry trees): bit-identical results for
    any device count / placement, like the reference's deterministic mode."""
    t = sk.synth_tensor((300, 200, 150), 400_000, seed=8)
    fs = sk.random_factors(t.shape, 32, seed=3)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=4, isp_capacity=512))
    results = []
    for m, sched in [(1, "dynamic"), (2, "static"), (4, "contiguous"), (1, "dynamic")]:
        cfg = sk.PlatformConfig(devices=m, rank=32, scheduling=sched, tile_nnz=64, layout="blocked",
                                l2_budget_mb=0)
        outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
        results.append(outs)
    assert all(p.layout == "blocked" for p in plans)
    for outs in results[1:]:
        for a, b in zip(results[0], outs):
            assert np.array_equal(a, b)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
        assert rel_err(results[0][d], expect) <= TOL
        facs[d] = results[0][d]


def test_blocked_layout_through_runner(golden):
    from paper_2507_15121_b200.distributed import DistributedMttkrp

    t = sk.synth_tensor((400, 300, 200), 300_000, seed=5)
    fs = sk.random_factors(t.shape, 32, seed=2)
    plans = sk.build_all_plans(t, sk.PartitionConfig(), keep_permutation=False)
    cfg = sk.PlatformConfig(rank=32, accumulation="atomic", layout="blocked", l2_budget_mb=0)
    runner = DistributedMttkrp(plans, cfg)
    dev_f = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in fs]
    outs = [o.double().cpu().numpy() for o in runner.run(dev_f)]
    assert all(p.layout == "blocked" for p in plans)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
        assert rel_err(outs[d], expect) <= TOL
        facs[d] = outs[d]


# ------------------------------------------------------------------- dedup


def test_dedup_mark_first_occurrence():
    rng = np.random.default_rng(3)
    n = 200_000
    idx = np.stack([rng.integers(0, s, n) for s in (20, 30, 7, 5)], 1)  # many duplicates
    cols = [torch.from_numpy(idx[:, w].astype(np.int32)).cuda() for w in range(4)]
    slots = 1 << 19
    table = torch.empty(slots, dtype=torch.int64, device="cuda")
    keep = torch.empty(n, dtype=torch.uint8, device="cuda")
    import ctypes
    cptr = (ctypes.c_void_p * 4)(*[c.data_ptr() for c in cols])
    _lib.call("skrp_dedup_mark", cptr, 4, n, table.data_ptr(), slots, keep.data_ptr(), stream())
    _, first = np.unique(idx, axis=0, return_index=True)
    expect = np.zeros(n, dtype=np.uint8)
    expect[first] = 1
    assert np.array_equal(keep.cpu().numpy(), expect)


def test_device_generator_unique_zipf():
    t = sk.synth_tensor_device((60, 50, 40), 30_000, distribution="zipf", seed=4)
    idx = t.indices
    assert len(idx) == 30_000 and len(np.unique(idx, axis=0)) == 30_000
    assert t.stats.duplicates > 0
    # deterministic in the seed
    t2 = sk.synth_tensor_device((60, 50, 40), 30_000, distribution="zipf", seed=4)
    assert np.array_equal(t2.indices, idx)


# ------------------------------------------------------- distributed CP-ALS


def test_distributed_cp_als_world1_matches_reference(golden):
    """DistributedCpAls (the cfg5 path) at world == 1 reproduces the
    reference cp_als fit history and lambdas (same init, same updates)."""
    from paper_2507_15121_b200.distributed import DistributedCpAls

    t = sk.synth_tensor((30, 20, 10), 1500, seed=9)
    ref = golden("cpd.npz")
    plans = sk.build_all_plans(t, sk.PartitionConfig())
    als = DistributedCpAls(plans, sk.PlatformConfig(rank=4))
    init = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in sk.random_factors(t.shape, 4, seed=1)]
    facs, lam, hist = als.run(init, iterations=3)
    assert np.allclose(hist, ref["u_engine_fit"], rtol=0, atol=2e-4)
    assert np.allclose(lam, ref["u_engine_lambdas"], rtol=2e-3)
    for w, f in enumerate(facs):
        assert np.allclose(f.double().cpu().numpy(), ref[f"u_engine_F{w}"], atol=2e-3)


def test_distributed_cp_als_rank4_blocked_atomic(golden):
    from paper_2507_15121_b200.distributed import DistributedCpAls

    rng = np.random.default_rng(5)
    a, b, c = (rng.random((n, 4)) for n in (40, 30, 20))
    dense = np.einsum("ir,jr,kr->ijk", a, b, c)
    idx = np.argwhere(np.ones_like(dense, dtype=bool))
    t = sk.SparseTensorCOO(dense.shape, idx, dense[tuple(idx.T)])
    plans = sk.build_all_plans(t, sk.PartitionConfig(strategy="nnz-balanced"))
    als = DistributedCpAls(plans, sk.PlatformConfig(rank=4, accumulation="atomic"))
    init = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in sk.random_factors(t.shape, 4, seed=0)]
    _, _, hist = als.run(init, iterations=25)
    assert hist[-1] > 0.99 and abs(hist[-1] - golden("cpd.npz")["r4_fit"][-1]) < 1e-3


def test_dense_cpd_kernels_vs_numpy():
    """skrp_gram / skrp_apply_rr / skrp_col_sumsq / skrp_weighted_dot / skrp_sumsq."""
    rng = np.random.default_rng(1)
    for rows, R in [(1, 8), (1000, 16), (70_001, 32), (40_000, 64), (5000, 7)]:
        y = rng.random((rows, R)).astype(np.float32)
        yt = torch.from_numpy(y).cuda()
        g = torch.empty((R, R), dtype=torch.float64, device="cuda")
        _lib.call("skrp_gram", yt.data_ptr(), rows, R, g.data_ptr(), stream())
        ref = y.astype(np.float64).T @ y.astype(np.float64)
        assert np.allclose(g.cpu().numpy(), ref, rtol=2e-5)  # fp32 partial sums over <=1024 rows, fp64 across
        w = rng.standard_normal((R, R))
        wt = torch.from_numpy(w).cuda()
        out = torch.empty_like(yt)
        _lib.call("skrp_apply_rr", yt.data_ptr(), rows, R, wt.data_ptr(), out.data_ptr(), stream())
        assert np.allclose(out.cpu().numpy(), y.astype(np.float64) @ w, rtol=1e-4, atol=1e-4)
        cs = torch.empty(R, dtype=torch.float64, device="cuda")
        _lib.call("skrp_col_sumsq", yt.data_ptr(), rows, R, cs.data_ptr(), stream())
        assert np.allclose(cs.cpu().numpy(), (y.astype(np.float64) ** 2).sum(0), rtol=1e-9)
        lam = rng.random(R)
        lt = torch.from_numpy(lam).cuda()
        o = torch.empty(1, dtype=torch.float64, device="cuda")
        _lib.call("skrp_weighted_dot", yt.data_ptr(), yt.data_ptr(), rows, R, lt.data_ptr(), o.data_ptr(), stream())
        assert np.isclose(o.item(), float((y.astype(np.float64) ** 2 @ lam).sum()), rtol=1e-9)
        _lib.call("skrp_sumsq", yt.data_ptr(), rows * R, o.data_ptr(), stream())
        assert np.isclose(o.item(), float((y.astype(np.float64) ** 2).sum()), rtol=1e-9)
        if R in (16, 32, 64):
            o2 = torch.empty_like(yt)
            sq = torch.empty(R, dtype=torch.float64, device="cuda")
            bad = torch.empty(1, dtype=torch.int32, device="cuda")
            _lib.call("skrp_apply_rr_sumsq", yt.data_ptr(), rows, R, wt.data_ptr(), o2.data_ptr(), sq.data_ptr(),
                      bad.data_ptr(), stream())
            ref2 = y.astype(np.float64) @ w
            assert np.allclose(o2.cpu().numpy(), ref2, rtol=1e-4, atol=1e-4) and int(bad.item()) == 0
            assert np.allclose(sq.cpu().numpy(), (o2.cpu().numpy().astype(np.float64) ** 2).sum(0), rtol=1e-12)
            yb = yt.clone()
            yb[rows // 2, R - 1] = float("inf")
            _lib.call("skrp_apply_rr_sumsq", yb.data_ptr(), rows, R, wt.data_ptr(), o2.data_ptr(), sq.data_ptr(),
                      bad.data_ptr(), stream())
            assert int(bad.item()) == 1
        sc = rng.random(R) + 0.5
        xs = yt.clone()
        _lib.call("skrp_scale_cols", xs.data_ptr(), rows, R, torch.from_numpy(sc).cuda().data_ptr(), stream())
        assert np.array_equal(xs.cpu().numpy(), (y.astype(np.float64) * sc).astype(np.float32))


@pytest.mark.parametrize("rows,R,offset", [(3_000_001, 64, 0), (1_234_567, 32, 0), (333_333, 16, 0),
                                           (100_003, 64, 1), (7, 64, 0), (1025 * 7, 64, 0)])
def test_gram_symmetric_kernel(rows, R, offset):
    """skrp_gram at scale (register-tiled symmetric kernel for aligned inputs,
    the 4x4-tile kernel for an unaligned base): fp64 Y^T Y within the fp32
    partial-sum tolerance, exactly symmetric."""
    rng = np.random.default_rng(rows)
    y = (rng.random((rows * R + offset)).astype(np.float32) - 0.25)
    yt = torch.from_numpy(y).cuda()
    g = torch.empty((R, R), dtype=torch.float64, device="cuda")
    _lib.call("skrp_gram", yt.data_ptr() + 4 * offset, rows, R, g.data_ptr(), stream())
    ym = y[offset:].reshape(rows, R).astype(np.float64)
    ref = ym.T @ ym
    got = g.cpu().numpy()
    if offset == 0:  # the symmetric kernel mirrors its upper triangle
        assert np.array_equal(got, got.T)
    assert np.allclose(got, ref, rtol=2e-5, atol=1e-6 * np.abs(ref).max())


def test_runner_pipelined_host_path(golden):
    from paper_2507_15121_b200.distributed import DistributedMttkrp

    t = tensor_from(golden, "z3")
    fs = factors_from(golden, "z3", 32, 3)
    plans = sk.build_all_plans(t, sk.PartitionConfig())
    runner = DistributedMttkrp(plans, sk.PlatformConfig(rank=32, accumulation="atomic", layout="blocked",
                                                        l2_budget_mb=0))
    dev_f = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in fs]
    eager = [o.clone() for o in runner.run(dev_f)]
    host_f = [torch.from_numpy(f.data.astype(np.float32)).pin_memory() for f in fs]
    host_o = [[torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in eager] for _ in range(2)]
    h2d, d2h = runner.run_host_pipelined(host_f, host_o, 5)
    torch.cuda.synchronize()
    assert h2d == sum(host_f[w].numel() * 4 for w in (1, 2)) and d2h == sum(o.numel() * 4 for o in eager)
    for b in range(2):
        for got, want in zip(host_o[b], eager):
            assert rel_err(got.double().numpy(), want.double().cpu().numpy()) <= 1e-6


# ----------------------------------------------------------- out-of-core plans


@pytest.mark.parametrize("m", [1, 2])
def test_out_of_core_streamed_modes(m):
    """Plans moved to pinned host memory are streamed
    chunk by chunk through two device buffers: chained all-mode parity with
    modes 0 and 2 out of core (many chunks, rows straddling chunks), host
    plan views unchanged, HBM freed."""
    from paper_2507_15121_b200.distributed import DistributedMttkrp

    t = sk.synth_tensor((500, 400, 300), 300_000, seed=9)
    fs = sk.random_factors(t.shape, 32, seed=4)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=m, isp_capacity=1024))
    before = [p._indices.copy() for p in plans]
    for d in (0, 2):
        plans[d].to_host()
        assert plans[d].layout == "host" and plans[d].vals.is_pinned() and not plans[d].coords[0].is_cuda
    cfg = sk.PlatformConfig(devices=m, rank=32, accumulation="atomic", stream_chunk_nnz=20_000, tile_nnz=256)
    outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
        assert rel_err(outs[d], expect) <= TOL
        facs[d] = outs[d]
        assert np.array_equal(plans[d]._indices, before[d])
    # the one-process-per-GPU runner streams the same plans
    runner = DistributedMttkrp(plans, sk.PlatformConfig(rank=32, accumulation="atomic", stream_chunk_nnz=50_000),
                               rank=0, world=1)
    dev_f = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in fs]
    got = [o.double().cpu().numpy() for o in runner.run(dev_f)]
    for d in range(3):
        assert rel_err(got[d], outs[d]) <= TOL
    # cross-mode prefetch: the runner enqueued mode 0's leading chunks for the
    # next step while mode 2 ran; a second and third step consume them
    ex0 = runner._execs[(0, 32)]
    assert ex0.pending == min(len(ex0.bufs), len(ex0.chunks)) > 0
    for _ in range(2):
        again = [o.double().cpu().numpy() for o in runner.run(dev_f)]
        for d in range(3):
            assert rel_err(again[d], outs[d]) <= TOL
    with pytest.raises(ValueError, match="atomic"):
        cfgd = sk.PlatformConfig(devices=m, rank=32, accumulation="deterministic-reduce")
        sk.mttkrp_mode(plans[0], sk.make_devices(fs, cfgd), cfgd)


# ------------------------------------------------------------- .tns on the GPU


def test_tns_gpu_golden_cases():
    """GPU .tns parser against the REFERENCE parser's outputs and exception
    messages (tests/golden/tns_cases.json): indices, values (bit-exact),
    shape, LoadStats, errors."""
    import json
    import os

    from test_host_api import _tns_check

    with open(os.path.join(os.path.dirname(__file__), "golden", "tns_cases.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            _tns_check(sk.parse_tns_gpu, c)


def test_tns_gpu_large_random_file(tmp_path):
    """A 300K-line file (comments, blank lines, CRLF, tabs, %.17g / repr
    values) parsed on the GPU == the host parser; the device arrays are kept
    and feed the plan build directly."""
    rng = np.random.default_rng(5)
    n = 300_000
    idx = np.stack([rng.integers(1, s + 1, n) for s in (5000, 3000, 2000)], 1)
    idx = np.unique(idx, axis=0)
    rng.shuffle(idx)
    vals = rng.standard_normal(len(idx)) * 10.0 ** rng.integers(-5, 5, len(idx))
    lines = ["# big", "# shape: 5000 3000 2000"]
    for k, (r, v) in enumerate(zip(idx, vals)):
        sep = "\t" if k % 7 == 0 else " "
        lines.append(sep.join(map(str, r)) + sep + (f"{v:.17g}" if k % 2 else repr(float(v))))
        if k % 1000 == 0:
            lines.append("")
    path = tmp_path / "big.tns"
    path.write_bytes(("\r\n".join(lines) + "\r\n").encode())
    t_gpu = sk.parse_tns_gpu(str(path))
    t_cpu = sk.parse_tns(str(path))
    assert t_gpu.shape == t_cpu.shape == (5000, 3000, 2000)
    assert np.array_equal(t_gpu.indices, t_cpu.indices)
    assert t_gpu.values.tobytes() == t_cpu.values.tobytes()
    assert t_gpu._dev is not None
    p = sk.build_mode_plan(t_gpu, 0, sk.PartitionConfig())
    q = sk.build_mode_plan(t_cpu, 0, sk.PartitionConfig())
    assert np.array_equal(p.order(), q.order())


def test_auto_layout_avoids_panel_on_skewed_rows():
    """deterministic-reduce + auto layout: the panel kernel sums a row in one
    warp, so a Zipf head row must route the plan to the tile layout instead;
    uniform rows take the panel."""
    from paper_2507_15121_b200.engine import _skewed_rows, apply_layout

    z = sk.synth_tensor_device((2000, 3000, 4000), 2_000_000, distribution="zipf", seed=3)
    u = sk.synth_tensor_device((200_000, 3000, 4000), 2_000_000, seed=3)
    pz = sk.build_mode_plan(z, 0, sk.PartitionConfig(strategy="nnz-balanced"))
    pu = sk.build_mode_plan(u, 0, sk.PartitionConfig())
    assert _skewed_rows(pz) and not _skewed_rows(pu)
    cfg = sk.PlatformConfig(rank=32, accumulation="deterministic-reduce", layout="auto", l2_budget_mb=0)
    apply_layout(pz, cfg, 32)
    assert pz.layout == "flycoo"  # plan order + carry tree: the fast deterministic path on skewed rows


# ------------------------------------------------------------- plan cache v1


def test_plan_cache_reference_files(golden, tmp_path):
    """GPU-direct load_plan of files written by the REFERENCE's save_plan
    (tests/golden/make_plan_golden.py): same shards, ISPs, host views
    (bit-exact, stored dtype) and device arrays as our own build; our
    save_plan reproduces the reference file byte-for-byte (from a fresh
    build and from the loaded plan); corruption / truncation / version /
    dtype errors are the reference's."""
    import json
    import os

    gdir = os.path.join(os.path.dirname(__file__), "golden", "plans")
    with open(os.path.join(gdir, "index.json")) as fh:
        index = json.load(fh)
    s = golden("synth.npz")
    for e in index:
        path = os.path.join(gdir, e["file"])
        raw = open(path, "rb").read()
        p = sk.load_plan(path)
        name = e["tensor"]
        t = sk.SparseTensorCOO(tuple(int(x) for x in s[f"{name}_shape"]), s[f"{name}_indices"],
                               s[f"{name}_values"].astype(e["dtype"]), name=name)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", RuntimeWarning)
            ref = sk.build_mode_plan(t, e["mode"], sk.PartitionConfig(devices=e["devices"], strategy=e["strategy"],
                                                                       isp_capacity=e["isp_capacity"]))
        assert [(x.index_range, x.nnz) for x in p.shards] == [(x.index_range, x.nnz) for x in ref.shards]
        assert all(np.array_equal(a.isp_boundaries, b.isp_boundaries) for a, b in zip(p.shards, ref.shards))
        assert np.array_equal(p._indices, ref._indices)
        assert p._values.dtype == np.dtype(e["dtype"]) and p._values.tobytes() == ref._values.tobytes()
        for w in range(len(t.shape)):
            assert torch.equal(p.coords[w], ref.coords[w])
        assert torch.equal(p.vals, ref.vals)
        ref.build_time = e["build_time"]
        sk.save_plan(ref, tmp_path / "a.plan")
        assert (tmp_path / "a.plan").read_bytes() == raw, e["file"]
        sk.save_plan(p, tmp_path / "b.plan")
        assert (tmp_path / "b.plan").read_bytes() == raw, e["file"]
        # loaded plans run the kernel
        fs = sk.random_factors(t.shape, 8, seed=1)
        cfg = sk.PlatformConfig(devices=2, rank=8)
        out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg, update_factors=False)
        expect = oracle.mttkrp_seq(t.indices, t.values, [f.data for f in fs], e["mode"])
        assert rel_err(out, expect) <= TOL
    # errors, in the reference's order (checksum first)
    path = os.path.join(gdir, index[0]["file"])
    raw = bytearray(open(path, "rb").read())
    bad = tmp_path / "bad.plan"
    flipped = bytearray(raw)
    flipped[len(raw) // 2] ^= 0xFF
    bad.write_bytes(bytes(flipped))
    with pytest.raises(sk.PlanIntegrityError):
        sk.load_plan(bad)
    bad.write_bytes(bytes(raw[:-100]))
    with pytest.raises(sk.PlanIntegrityError):
        sk.load_plan(bad)
    bad.write_bytes(b"not a plan at all")
    with pytest.raises(sk.PlanVersionError):
        sk.load_plan(bad)
    with pytest.raises(sk.PlanVersionError, match="expected float32"):
        sk.load_plan(path, value_dtype=np.float32)
    import struct
    import zlib

    v2 = bytearray(raw)
    v2[8:12] = struct.pack("<I", 2)
    v2[-4:] = struct.pack("<I", zlib.crc32(bytes(v2[8:-4])))
    bad.write_bytes(bytes(v2))
    with pytest.raises(sk.PlanVersionError, match="plan version 2"):
        sk.load_plan(bad)


@pytest.mark.parametrize("layout,variant", [("blocked", 0), ("panel", 0)])
def test_streamed_input_policy_parity(layout, variant):
    """Pin-one-stream-one layouts with factors > 32 MB: the streamed input is
    flagged (SKRP_FLAG_STREAM_INPUTj -> evict_first loads) in the tile and
    panel kernels; every mode matches the oracle."""
    from paper_2507_15121_b200.engine import _stream_flags, panel_shape, streamed_blocking

    shape = (2000, 300_000, 280_000)
    t = sk.synth_tensor_device(shape, 1_500_000, seed=12)
    fs = sk.random_factors(shape, 32, seed=5)
    facs = [f.data for f in fs]
    idx, vals = t.indices, t.values
    for d in range(3):
        p = sk.build_mode_plan(t, d, sk.PartitionConfig())
        sh = streamed_blocking(p, 32)
        if sh is None:  # mode 0's inputs are both > 32 MB; modes 1/2 have a small input
            sh = [-1 if w == d else (17 if w == max(w_ for w_ in range(3) if w_ != d) else -1) for w in range(3)]
        if layout == "panel":
            warps, _ = panel_shape(3, 32)
            p.to_panels(9, sh, warps)
        else:
            p.to_blocked(sh)
        flags = _stream_flags(p, 32)
        cfg = sk.PlatformConfig(rank=32, accumulation="atomic", kernel_variant=variant)
        out, _ = sk.mttkrp_mode(p, sk.make_devices(fs, cfg), cfg, update_factors=False)
        expect = oracle.mttkrp_seq_c(idx, vals, facs, d)
        assert rel_err(out, expect) <= TOL, (layout, d, flags)
        if d == 0:
            assert flags in (_lib.FLAG_STREAM_INPUT0, _lib.FLAG_STREAM_INPUT1)


def test_scaling_floor_per_rank_share():
    """SPEC acceptance 6 (scaling floor t1/t4 > 1.5), on one GPU: the kernel
    time of the whole all-mode step vs the slowest of the 4 ranks' shares of
    the same plans (each share timed alone, compute only -- what every GPU of
    a 4-GPU run executes between the all-gathers)."""
    from paper_2507_15121_b200.distributed import DistributedMttkrp

    shape = (480_000, 180_000, 180_000)
    t = sk.synth_tensor_device(shape, 40_000_000, seed=2)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=4), keep_permutation=False)
    fs = [torch.rand((s, 32), device="cuda") for s in shape]

    def kernel_seconds(runner):
        for _ in range(2):
            runner.run(fs, exchange=False)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in plans]
        runner.run(fs, kernel_events=ev, exchange=False)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in ev)

    cfg = sk.PlatformConfig(devices=4, rank=32, accumulation="atomic", scheduling="contiguous")
    t1 = kernel_seconds(DistributedMttkrp(plans, sk.PlatformConfig(devices=1, rank=32, accumulation="atomic"),
                                          rank=0, world=1))
    t4 = max(kernel_seconds(DistributedMttkrp(plans, cfg, rank=r, world=4)) for r in range(4))
    assert t1 / t4 > 1.5, (t1, t4)


# ------------------------------------------- engine API: execute_shard / measure_isolated_compute


def test_execute_shard_writes_exactly_its_rows(golden):
    """execute_shard (reference engine.py:128-212): each shard, run alone on
    its device, writes exactly its own output rows (= the oracle's rows) and
    leaves every other row untouched; a shard of another mode is refused."""
    t = tensor_from(golden, "z3")
    fs = factors_from(golden, "z3", 32, 3)
    ref = golden("mttkrp.npz")
    for acc in ("deterministic-reduce", "atomic"):
        cfg = sk.PlatformConfig(devices=2, rank=32, accumulation=acc)
        for d in range(3):
            p = sk.build_mode_plan(t, d, sk.PartitionConfig(devices=2))
            devs = sk.make_devices(fs, cfg)
            for dev in devs:
                dev.reset_for_mode(t.shape[d], 32)
            for j, shard in enumerate(p.shards):
                sk.execute_shard(shard, devs[j % 2], d, cfg)
            outs = [dev.output.double().cpu().numpy() for dev in devs]
            expect = ref[f"z3_R32_oracle_{d}"]
            owner = np.full(t.shape[d], -1)
            for j, shard in enumerate(p.shards):
                lo, hi = shard.index_range
                owner[lo:hi] = j % 2
                assert rel_err(outs[j % 2][lo:hi], expect[lo:hi]) <= TOL, (acc, d, j)
            for k in (0, 1):
                assert not outs[k][owner != k].any(), (acc, d, k)
    with pytest.raises(ValueError, match="belongs to mode"):
        sk.execute_shard(p.shards[0], devs[0], (d + 1) % 3, cfg)


def test_measure_isolated_compute_per_device_shares():
    """measure_isolated_compute (reference engine.py:403-437): one time per
    device for its static round-robin share, run alone; equal-index shares of
    a uniform tensor cost about the same, each share is cheaper than one
    device running everything, and the shares add up to at least that."""
    t = sk.synth_tensor_device((400_000, 300_000, 260_000), 8_000_000, seed=4)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=4), keep_permutation=False)
    fs = sk.random_factors(t.shape, 32, seed=1)
    for _ in range(2):  # warm-up (plan layouts, tile tables)
        four = sk.measure_isolated_compute(plans, fs, sk.PlatformConfig(devices=4, rank=32))
        one = sk.measure_isolated_compute(plans, fs, sk.PlatformConfig(devices=1, rank=32))
    assert len(four) == 4 and len(one) == 1 and all(x > 0 for x in four)
    assert max(four) / min(four) < 1.5, four
    # each quarter share runs faster than the whole, and the whole costs no
    # more than its parts (launch overheads make small shares relatively dear)
    assert max(four) < one[0] < 1.5 * sum(four), (four, one)


@pytest.mark.parametrize("acc", ["atomic", "deterministic-reduce"])
def test_fiber_layout_parity(golden, acc):
    """Fiber layout (plan.to_fibers, picked by layout='auto' where (row, c_f)
    runs are long -- the cfg3 shape): the tile kernel gathers the fiber
    input's row once per run; chained all-mode parity with the oracle, host
    plan views still the reference order, the fiber instantiation ran, and
    deterministic-reduce stays bit-identical across device counts."""
    t = sk.synth_tensor((46, 3000, 2500), 2_000_000, seed=17)
    fs = sk.random_factors(t.shape, 32, seed=8)
    ref_plans = [p._indices.copy() for p in sk.build_all_plans(t, sk.PartitionConfig(devices=2))]
    results = []
    for m in (1, 2):
        plans = sk.build_all_plans(t, sk.PartitionConfig(devices=2))
        cfg = sk.PlatformConfig(devices=m, rank=32, accumulation=acc, layout="auto", tile_nnz=1024)
        _lib.launch_log(clear=True)
        outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
        assert all(p.layout == "fibers" for p in plans), [p.layout for p in plans]
        names = [n for _, n in _lib.launch_log()]
        assert any("mttkrp_v2_kernel<" in n and _plain_bits(n) & 512 for n in names), names
        for p, before in zip(plans, ref_plans):
            assert np.array_equal(p._indices, before)
        results.append(outs)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
        assert rel_err(results[0][d], expect) <= TOL
        facs[d] = results[0][d]
    if acc == "deterministic-reduce":
        for a, b in zip(results[0], results[1]):
            assert np.array_equal(a, b)


def test_fiber_reorder_segmented_matches_whole():
    """to_fibers sorts shard run by shard run (seg_cap): the device arrays and
    the execution permutation are identical to one whole-plan sort, the
    arrays are (c_d, c_f)-sorted inside every shard and the shards keep their
    nonzeros; empty shards are fine."""
    t = sk.synth_tensor((40, 900, 700), 300_000, seed=23)
    a = sk.build_mode_plan(t, 0, sk.PartitionConfig(devices=8))  # 32 shards requested, clamped to 40 rows
    b = sk.build_mode_plan(t, 0, sk.PartitionConfig(devices=8))
    a.to_fibers(2)
    b.to_fibers(2, seg_cap=10_000)  # many runs of consecutive shards
    for x, y in zip(a.coords + [a.vals], b.coords + [b.vals]):
        assert torch.equal(x, y)
    assert torch.equal(a.exec_perm, b.exec_perm)
    rows = b.coords[0].cpu().numpy().astype(np.int64)
    fib = b.coords[2].cpu().numpy().astype(np.int64)
    key = rows * 1000 + fib
    for s_ in b.shards:
        seg = key[s_.start:s_.stop]
        assert np.all(np.diff(seg) >= 0)
        lo, hi = s_.index_range
        assert np.all((rows[s_.start:s_.stop] >= lo) & (rows[s_.start:s_.stop] < hi))
    assert np.array_equal(b._indices, sk.build_mode_plan(t, 0, sk.PartitionConfig(devices=8))._indices)


def test_fiber_layout_four_modes():
    """4-mode fiber layout (R = 64, the cfg5 shape class): every mode picks
    its smallest input as the fiber mode, the 4-mode fiber instantiation runs
    (two inputs gathered per nonzero, the fiber row once per run), chained
    all-mode parity with the oracle under both disciplines."""
    t = sk.synth_tensor((2000, 3000, 40, 30), 1_000_000, seed=29)
    fs = sk.random_factors(t.shape, 64, seed=9)
    for acc in ("atomic", "deterministic-reduce"):
        plans = sk.build_all_plans(t, sk.PartitionConfig(devices=1))
        cfg = sk.PlatformConfig(devices=1, rank=64, accumulation=acc, layout="auto")
        _lib.launch_log(clear=True)
        outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
        assert all(p.layout == "fibers" for p in plans), [p.layout for p in plans]
        names = [n for _, n in _lib.launch_log()]
        assert all("mttkrp_v2_kernel<4, 8, 2, 2, " in n and _plain_bits(n) & 512 for n in names[:4]), names
        facs = [f.data.copy() for f in fs]
        for d in range(4):
            expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
            assert rel_err(outs[d], expect) <= TOL
            facs[d] = outs[d]


@pytest.mark.gpu
@pytest.mark.parametrize("rank,tile", [(32, 33), (32, 100), (32, 1000), (64, 37), (64, 1000)])
def test_fiber_odd_tiles(rank, tile):
    """Fiber instantiations with tiles that are not a multiple of the 32-
    nonzero batch: short last batches inside fiber runs, the R = 32 two-batch
    step's end test (base + 64 <= tile end) and the metadata ring's empty
    tail groups, the R = 64 paired groups -- every mode within tolerance of
    the oracle, atomic and deterministic-reduce agreeing to tolerance."""
    nm = 3 if rank == 32 else 4
    shape = (40, 500, 60) if nm == 3 else (30, 400, 300, 20)
    t = sk.synth_tensor(shape, 400_000, seed=23)
    fs = sk.random_factors(t.shape, rank, seed=6)
    facs = [f.data.copy() for f in fs]
    outs = {}
    for acc in ("atomic", "deterministic-reduce"):
        plans = sk.build_all_plans(t, sk.PartitionConfig(devices=1))
        cfg = sk.PlatformConfig(devices=1, rank=rank, accumulation=acc, layout="fibers", tile_nnz=tile)
        _lib.launch_log(clear=True)
        outs[acc], _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
        names = [n for _, n in _lib.launch_log() if "mttkrp_v2_kernel<" in n]
        assert names and all(_plain_bits(n) & 512 for n in names), names
    f2 = [f.copy() for f in facs]
    for d in range(nm):
        expect = oracle.mttkrp_seq_c(t.indices, t.values, f2, d)
        for acc in outs:
            assert rel_err(outs[acc][d], expect) <= TOL, (acc, d)
        f2[d] = outs["atomic"][d]
