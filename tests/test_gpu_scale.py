"""Parity at scale: 10^8-nonzero plans on the cfg2 and cfg4
shapes, bit-exact against the C oracle's stable counting sort + the host
bounds/ISP restatement, and sampled MTTKRP rows (chained, all modes) against
the oracle's fp64 sequential MTTKRP over the source nonzeros of those rows.
Also the full-scale property checker bench.py runs (oracle/scale.py) on the
same plans, so the bench's billion-nonzero checks are themselves pinned
against the bit-exact comparison here.
"""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2507_15121_b200 as sk  # noqa: E402
from oracle.scale import sample_parity_source, verify_plan_full  # noqa: E402

N = 100_000_000
CASES = {
    "cfg2-shape uniform": ((4_800_000, 1_800_000, 1_800_000), "uniform", "equal-index"),
    "cfg4-shape zipf": ((8_200_000, 177_000, 8_100_000), "zipf", "nnz-balanced"),
}


def _host(t):
    coords, vals = t.device_arrays()
    idx = np.empty((t.nnz, len(coords)), dtype=np.uint64)
    for w, c in enumerate(coords):
        idx[:, w] = c.cpu().numpy().view(np.uint32)
    return idx, vals.cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("case", sorted(CASES))
def test_plans_bit_exact_1e8(case):
    shape, dist, strategy = CASES[case]
    t = sk.synth_tensor_device(shape, N, distribution=dist, seed=3)
    idx, vals = _host(t)
    src_c, src_v = t.device_arrays()
    pcfg = sk.PartitionConfig(devices=2, strategy=strategy)
    k = 2 * pcfg.oversubscription
    for d in range(3):
        p = sk.build_mode_plan(t, d, pcfg, keep_permutation=True)
        order, counts = oracle.stable_order_c(idx, d, shape[d])
        assert np.array_equal(p.perm.cpu().numpy().view(np.uint32).astype(np.int64), order), (case, d, "perm")
        for w in range(3):
            got = p.coords[w].cpu().numpy().view(np.uint32)
            assert np.array_equal(got, idx[order, w].astype(np.uint32)), (case, d, w)
        assert np.array_equal(p.vals.cpu().numpy().astype(np.float64), vals[order]), (case, d, "vals")
        bounds = (oracle.equal_index_bounds(shape[d], k) if strategy == "equal-index"
                  else oracle.nnz_balanced_bounds(counts, k))
        offsets = np.concatenate([[0], np.cumsum(counts)])[bounds]
        assert np.array_equal(p.bounds, bounds) and np.array_equal(p.offsets, offsets), (case, d)
        for j, s_ in enumerate(p.shards):
            assert np.array_equal(s_.isp_boundaries,
                                  oracle.isp_boundaries(int(offsets[j + 1] - offsets[j]), pcfg.isp_capacity))
        # the bench's full-scale checker agrees on a correct plan ...
        chk = verify_plan_full(src_c, src_v, p, strategy, devices=2, isp_capacity=pcfg.isp_capacity)
        assert chk["ok"], chk
        # ... and catches a broken one: two adjacent elements of one row swapped
        # (sortedness kept, stability lost), then one element dropped
        skey = idx[order, d]
        i0 = int(np.argmax(skey[1:] == skey[:-1]))  # first pair inside one row
        saved = p.perm[i0:i0 + 2].clone()
        p.perm[i0:i0 + 2] = saved.flip(0)
        bad = verify_plan_full(src_c, src_v, p, strategy, devices=2, isp_capacity=pcfg.isp_capacity)
        assert not bad["stable"] and bad["permutation"], bad
        p.perm[i0:i0 + 2] = saved
        saved = p.perm[5].clone()
        p.perm[5] = p.perm[6]
        bad = verify_plan_full(src_c, src_v, p, strategy, devices=2, isp_capacity=pcfg.isp_capacity)
        assert not bad["permutation"], bad
        p.perm[5] = saved
        del p
        torch.cuda.empty_cache()


@pytest.mark.parametrize("case", sorted(CASES))
def test_mttkrp_sampled_rows_1e8(case):
    shape, dist, strategy = CASES[case]
    t = sk.synth_tensor_device(shape, N, distribution=dist, seed=4)
    idx, vals = _host(t)
    fs = sk.random_factors(shape, 32, seed=0)
    pcfg = sk.PartitionConfig(devices=2, strategy=strategy)
    plans = sk.build_all_plans(t, pcfg, keep_permutation=False)
    cfg = sk.PlatformConfig(devices=2, rank=32)
    outs, _ = sk.mttkrp_all_modes(plans, sk.make_devices(fs, cfg), cfg)
    # oracle: fp64 sequential MTTKRP over the source nonzeros of sampled rows
    rng = np.random.default_rng(1)
    facs = [f.data.copy() for f in fs]
    for d in range(3):
        rows = np.sort(rng.choice(shape[d], 2048, replace=False))
        if dist == "zipf":  # include the head rows (the heaviest, longest runs)
            rows = np.union1d(rows, np.arange(8))
        sel = np.isin(idx[:, d], rows.astype(np.uint64))
        expect = oracle.mttkrp_seq_c(idx[sel], vals[sel], facs, d)[rows]
        got = outs[d][rows]
        err = float(np.max(np.abs(got - expect) / np.maximum(np.abs(expect), 1.0)))
        assert err <= 1e-4, (case, d, err)
        facs[d] = outs[d]
    # the bench's source-tensor sampler agrees (same outputs, fp64 on the GPU)
    src_c, src_v = t.device_arrays()
    res = sample_parity_source(src_c, src_v, shape, [f.data for f in fs],
                               [torch.from_numpy(o).cuda() for o in outs], [0, 1, 2], rows_per_mode=512)
    assert res["ok"], res
