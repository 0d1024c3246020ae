"""GPU tests of the cells execution (K1d, csrc/mttkrp_cells.cu): the
GPU-synchronous 2-D blocked kernel with shared-memory output stripes.

Bars: every mode within rel 1e-4 of the oracle; host plan
views bit-exact after the in-place reorder; outputs bit-identical for any
stripe size, CTA count, lag and shard placement (each row is summed by one
warp in an order fixed by the global cell grid)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_15121_b200 as sk  # noqa: E402
from paper_2507_15121_b200 import engine  # noqa: E402

TOL = 1e-4


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


def cell_params(plan, stripe_rows, ctas, outer_rows, inner_rows, rank=32, variant=1):
    d = plan.mode
    ins = [w for w in range(3) if w != d]
    om, im = sorted(ins, key=lambda w: (plan.shape[w], w))
    shp = engine.cell_shape(rank, variant)
    if shp is None:
        variant, shp = 0, engine.cell_shape(rank, 0)
    warps, stage, _ = shp
    return {"rank": rank, "stripe_rows": stripe_rows, "ctas": ctas, "outer_mode": om, "inner_mode": im,
            "outer_shift": max(0, outer_rows.bit_length() - 1), "inner_shift": max(0, inner_rows.bit_length() - 1),
            "variant": variant, "warps": warps, "stage": stage}


def run_cells(plan, factors, rank, shard_ids=None, lag=2, out=None):
    gpu = torch.device("cuda", torch.cuda.current_device())
    cfg = sk.PlatformConfig(rank=rank, cell_lag=lag)
    ids = list(range(plan.shard_count)) if shard_ids is None else list(shard_ids)
    ex = engine._shard_exec(plan, ids, cfg, rank, gpu)
    assert isinstance(ex, engine._CellExec)
    fdev = [torch.from_numpy(np.ascontiguousarray(f, dtype=np.float32)).to(gpu) for f in factors]
    if out is None:
        out = torch.full((plan.shape[plan.mode], rank), float("nan"), dtype=torch.float32, device=gpu)
    ex.run(plan.coords, plan.vals, plan.nnz, plan.mode, fdev, out, cfg, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("name", ["u3", "z3", "d3", "s3"])
def test_cells_layout_parity_golden(golden, name):
    """Reference goldens: every mode within tolerance, host views of the plan
    still bit-exact after the in-place reorder, shard offsets unchanged."""
    t = tensor_from(golden, name)
    fs = factors_from(golden, name, 32, 3)
    ref = golden("mttkrp.npz")
    plans = golden("plans.npz")
    for d in range(3):
        p = sk.build_mode_plan(t, d, sk.PartitionConfig(devices=2))
        before = [(s_.start, s_.stop, s_.index_range) for s_ in p.shards]
        o = [w for w in range(3) if w != d]
        prm = cell_params(p, 3, 4, max(1, t.shape[o[0]] // 3), max(1, t.shape[o[1]] // 5))
        p.to_cells(range(p.shard_count), prm)
        assert p.layout == "cells" and p.cells["cells"] >= 1
        assert [(s_.start, s_.stop, s_.index_range) for s_ in p.shards] == before
        assert np.array_equal(p._indices, plans[f"{name}_m{d}_sorted_indices"])
        offs = p.cells["stripe_offsets"].cpu().numpy()
        assert offs[0] == 0 and offs[-1] == p.cells["num_entries"] >= p.nnz and np.all(np.diff(offs) >= 0)
        _layout_invariants(p)
        out = run_cells(p, [f.data for f in fs], 32)
        assert rel_err(out, ref[f"{name}_R32_oracle_{d}"]) <= TOL


def _layout_invariants(p):
    """Entries: stripes hold their own rows; cells ascend through a stripe and
    every cell's part is aligned across the slots (all slots cross a cell
    boundary in the same step); a row's nonzeros in one cell belong to one
    slot, in plan order; together the entries are exactly the nonzeros."""
    c = p.cells
    e = c["entries"][: 4 * c["num_entries"]].view(-1, 4).cpu().numpy().view(np.uint32).astype(np.int64)
    offs = c["stripe_offsets"].cpu().numpy()
    slots, rb, mask = c["slots"], c["rank"] * 4, (1 << 20) - 1
    seen = []
    for s in range(c["stripes"]):
        blk = e[offs[s]:offs[s + 1]].reshape(-1, slots, 4)
        tail = blk[:, 0, 0] == 0xFFFFFFFF
        k = int((~tail).sum())
        assert not np.any(tail[:k])  # no-cell skip entries only at the tail
        blk = blk[:k]
        cell = blk[:, :, 0] >> 20
        assert np.all(cell == cell[:, :1])  # aligned across slots
        assert np.all(np.diff(cell[:, 0]) >= 0)
        assert np.all(cell < c["cells"])
        real = (blk[:, :, 0] & mask) != mask
        for q in range(slots):
            r = blk[real[:, q], q]
            lrow = (r[:, 0] & mask) // rb
            assert np.all(lrow < c["stripe_rows"])
            seen.append(np.stack([lrow + c["row_lo"] + s * c["stripe_rows"], r[:, 1], r[:, 2]], 1))
        # one slot per (row, cell)
        rr = (blk[:, :, 0] & mask)
        for cl in np.unique(cell[:, 0]):
            sel = cell[:, 0] == cl
            for q1 in range(slots):
                a1 = set(rr[sel][real[sel][:, q1], q1].tolist())
                for q2 in range(q1 + 1, slots):
                    assert not a1 & set(rr[sel][real[sel][:, q2], q2].tolist())
    got = np.concatenate(seen) if seen else np.zeros((0, 3), np.int64)
    d, om, im = p.mode, c["outer_mode"], c["inner_mode"]
    ref = np.stack([p.coords[d].cpu().numpy(), p.coords[om].cpu().numpy(), p.coords[im].cpu().numpy()], 1)
    ref = ref.astype(np.int64) & 0xFFFFFFFF
    assert len(got) == len(ref)
    assert np.array_equal(got[np.lexsort(got.T[::-1])], ref[np.lexsort(ref.T[::-1])])


@pytest.mark.parametrize("rank", [16, 32, 64])
def test_cells_invariance_across_stripes_ctas_lag(rank):
    """The same tensor in cells layouts with different stripe sizes, CTA
    counts (rounds) and lags: bit-identical outputs, within tolerance of the
    oracle; heavy row repetition exercises the serialised duplicate steps."""
    t = sk.synth_tensor((37, 900, 700), 250_000, seed=3)  # ~6.8K nonzeros per row
    fs = sk.random_factors(t.shape, rank, seed=2)
    facs = [f.data for f in fs]
    res = {}
    for d in range(3):
        outs = []
        for sr, ctas, lag in [(1, 148, 2), (2, 3, 1), (5, 1, 3), (3, 7, 0)]:
            p = sk.build_mode_plan(t, d, sk.PartitionConfig(devices=1), keep_permutation=False)
            o = [w for w in range(3) if w != d]
            p.to_cells(range(p.shard_count),
                       cell_params(p, sr, ctas, max(1, t.shape[o[0]] // 4), max(1, t.shape[o[1]] // 7), rank))
            if sr == 2:
                _layout_invariants(p)
            outs.append(run_cells(p, facs, rank, lag=lag))
        for o_ in outs[1:]:
            assert np.array_equal(outs[0], o_)
        res[d] = outs[0]
        expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
        assert rel_err(res[d], expect) <= TOL


def test_cells_shard_subset_writes_only_its_rows():
    """A layout over shards [1, 2] of 4: those rows match the oracle, other
    rows are untouched, other shards' nonzeros keep plan order; the union of
    per-shard-set runs equals the single-set run bit for bit."""
    t = sk.synth_tensor((500, 400, 300), 300_000, seed=11)
    fs = sk.random_factors(t.shape, 32, seed=5)
    facs = [f.data for f in fs]
    expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, 0)
    full = sk.build_mode_plan(t, 0, sk.PartitionConfig(devices=4))
    full.to_cells(range(full.shard_count), cell_params(full, 2, 8, 64, 32), keep_arrays=False)
    assert full.coords is None and full.vals is None
    ref = run_cells(full, facs, 32)
    assert rel_err(ref, expect) <= TOL
    p = sk.build_mode_plan(t, 0, sk.PartitionConfig(devices=4))
    before = [c.clone() for c in p.coords]
    p.to_cells([1, 2], cell_params(p, 2, 8, 64, 32))
    got = run_cells(p, facs, 32, shard_ids=[1, 2])
    lo, hi = p.shards[1].index_range[0], p.shards[2].index_range[1]
    assert np.array_equal(got[lo:hi], ref[lo:hi])
    assert np.all(np.isnan(got[:lo])) and np.all(np.isnan(got[hi:]))
    e0, e1 = p.shards[1].start, p.shards[2].stop
    for a, b in zip(before, p.coords):
        assert torch.equal(a[:e0], b[:e0]) and torch.equal(a[e1:], b[e1:])
    with pytest.raises(ValueError):
        engine._shard_exec(p, [1], sk.PlatformConfig(rank=32), 32, torch.device("cuda", 0))


def test_cells_through_api_and_runner():
    """layout='cells' through the drop-in mttkrp_all_modes (1 device) and the
    one-process-per-GPU runner: chained all-mode parity, identical bits."""
    from paper_2507_15121_b200.distributed import DistributedMttkrp

    t = sk.synth_tensor((3000, 2000, 1000), 400_000, seed=21)
    fs = sk.random_factors(t.shape, 32, seed=4)
    cfg = sk.PlatformConfig(devices=1, rank=32, layout="cells", cell_outer_mb=1, cell_inner_mb=1)
    plans = sk.build_all_plans(t, sk.PartitionConfig(devices=1))
    outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
    assert all(p.layout == "cells" for p in plans)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
        assert rel_err(outs[d], expect) <= TOL
        facs[d] = outs[d]
    plans2 = sk.build_all_plans(t, sk.PartitionConfig(devices=1), keep_permutation=False)
    r = DistributedMttkrp(plans2, cfg, rank=0, world=1)
    dev_f = [torch.from_numpy(f.data.astype(np.float32)).cuda() for f in fs]
    got = r.run(dev_f)
    for d in range(3):
        assert np.array_equal(got[d].cpu().numpy().astype(np.float64), outs[d])


def test_cells_edge_cases():
    """One nonzero; rows beyond the last nonzero; an output mode with fewer
    rows than warps; a single cell (inputs smaller than one block)."""
    for shape, nnz in [((5, 6, 7), 1), ((3, 50, 40), 200), ((20000, 3, 3), 50)]:
        t = sk.synth_tensor(shape, nnz, seed=1)
        fs = sk.random_factors(t.shape, 32, seed=1)
        facs = [f.data for f in fs]
        for d in range(3):
            p = sk.build_mode_plan(t, d, sk.PartitionConfig(devices=1))
            cfg = sk.PlatformConfig(rank=32)
            prm = engine.choose_cells(p, 32, cfg)
            p.to_cells(range(p.shard_count), prm)
            out = run_cells(p, facs, 32)
            expect = oracle.mttkrp_seq_c(t.indices, t.values, facs, d)
            assert rel_err(out, expect) <= TOL
