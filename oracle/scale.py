"""Full-scale parity checks for bench.py and the -m gpu tests -- TEST
INFRASTRUCTURE ONLY (see oracle/__init__.py: the product never imports this).

At 10^9 nonzeros the CPU oracle cannot rebuild a plan in bench time, so the
checks here use size-independent properties of the reference's
build_mode_plan (partition.py:196-257) and recompute sampled MTTKRP rows in
fp64 from the SOURCE tensor (the generator's arrays), never from the plan
arrays under test.  The elementwise work runs on the GPU in torch (checker
code, chunked); bounds, offsets and ISP boundaries are recomputed on the host
by this package's restatement (equal_index_bounds / nnz_balanced_bounds /
isp_boundaries, partition.py:127-193).

verify_plan_full(src_coords, src_vals, plan, ...) checks, for one mode plan:
  * sorted     -- the key column (c_d) is non-decreasing;
  * stable     -- inside every run of equal keys the source positions
                  (plan.perm) strictly increase (argsort(kind="stable"),
                  partition.py:219-225);
  * permutation-- plan.perm hits every source position exactly once;
  * gathered   -- every plan column and the values equal the source arrays
                  at plan.perm (bit-exact);
  * bounds     -- the shard bounds equal the host restatement on the source
                  histogram (equal-index: closed form; nnz-balanced: the C
                  routine with the reference's tie rule);
  * offsets    -- offsets == exclusive prefix of the histogram at the bounds;
  * isps       -- every shard's ISP boundaries equal isp_boundaries(nnz, P).

sample_parity_source(...) -- max |gpu - ref| / max(|ref|, 1) (cli.py:247-261)
over a seeded sample of output rows per mode, ref = fp64 MTTKRP of those rows
over the source nonzeros with the chained factors (mode d uses the GPU's own
outputs of the modes before it, as the reference's mttkrp_all_modes does).
"""

from __future__ import annotations

import numpy as np

from . import equal_index_bounds, isp_boundaries, nnz_balanced_bounds

_CHUNK = 1 << 27


def _u32(x):
    """int32 tensor holding u32 bit patterns -> int64 values."""
    return x.long() & 0xFFFFFFFF


def source_histogram(src_col, num_indices):
    import torch

    counts = torch.zeros(num_indices, dtype=torch.int64, device=src_col.device)
    for a in range(0, src_col.numel(), _CHUNK):
        counts += torch.bincount(_u32(src_col[a:a + _CHUNK]), minlength=num_indices)
    return counts


def verify_plan_full(src_coords, src_vals, plan, strategy, oversubscription=4, devices=1, isp_capacity=8192):
    import torch

    d = plan.mode
    nnz = int(src_vals.numel())
    if plan.perm is None:
        raise ValueError("verify_plan_full needs the build permutation (keep_permutation=True)")
    if plan.layout != "flycoo":
        raise ValueError("verify the plan before any execution-layout reordering")
    dev = src_vals.device
    perm, key = plan.perm, plan.coords[d]
    res = {"mode": d, "nnz": nnz, "sorted": True, "stable": True, "gathered": True}
    seen = torch.zeros(nnz, dtype=torch.bool, device=dev)
    in_range = True
    for a in range(0, nnz, _CHUNK):
        b = min(nnz, a + _CHUNK)
        e = min(nnz, b + 1)  # one element of overlap: the boundary pair
        k = _u32(key[a:e])
        p = _u32(perm[a:e])
        dk = k[1:] - k[:-1]
        dp = p[1:] - p[:-1]
        res["sorted"] &= bool((dk >= 0).all().item())
        res["stable"] &= bool(((dk > 0) | (dp > 0)).all().item())
        pc = p[: b - a]
        in_range &= bool((pc < nnz).all().item())
        pc = pc.clamp(max=nnz - 1)
        seen[pc] = True
        for w, c in enumerate(plan.coords):
            res["gathered"] &= bool((c[a:b] == src_coords[w].index_select(0, pc)).all().item())
        res["gathered"] &= bool((plan.vals[a:b].view(torch.int32)
                                 == src_vals.index_select(0, pc).view(torch.int32)).all().item())
    res["permutation"] = in_range and bool(seen.all().item())
    del seen
    n_idx = plan.shape[d]
    counts = source_histogram(src_coords[d], n_idx).cpu().numpy()
    k = min(devices * oversubscription, n_idx)
    if strategy == "equal-index":
        bounds = equal_index_bounds(n_idx, k)
    else:
        bounds = nnz_balanced_bounds(counts, k)
    prefix = np.concatenate([[0], np.cumsum(counts)])
    offsets = prefix[bounds]
    res["bounds"] = bool(np.array_equal(np.asarray(plan.bounds, dtype=np.int64), bounds))
    res["offsets"] = bool(np.array_equal(np.asarray(plan.offsets, dtype=np.int64), offsets))
    res["isps"] = all(np.array_equal(np.asarray(s_.isp_boundaries, dtype=np.int64),
                                     isp_boundaries(int(offsets[j + 1] - offsets[j]), isp_capacity))
                      for j, s_ in enumerate(plan.shards)) and len(plan.shards) == k
    res["shards"] = k
    res["ok"] = all(res[x] for x in ("sorted", "stable", "permutation", "gathered", "bounds", "offsets", "isps"))
    return res


def extract_row_samples(src_coords, src_vals, shape, modes, rows_per_mode=4096, seed=0, nnz_budget=8_000_000):
    """Phase 1 of the sampled-row parity: for every mode, a seeded sample of
    output rows (rows added while their nonzeros fit `nnz_budget`; at least
    one) and ALL their nonzeros from the SOURCE tensor, copied to host memory
    (so the source can be freed before the run -- full-size cfg3 on one GPU).
    Returns one dict per mode: rows (int64), coords (n x N int64), vals (f64)."""
    import torch

    dev = src_vals.device
    rng = np.random.default_rng(seed)
    out = []
    for d in modes:
        col = src_coords[d]
        cand = np.sort(rng.permutation(shape[d])[:rows_per_mode]).astype(np.int64)
        counts = source_histogram(col, shape[d]).index_select(0, torch.from_numpy(cand).to(dev)).cpu().numpy()
        keep, tot = [], 0
        for r, n in zip(cand, counts):
            if tot + n <= nnz_budget or not keep:
                keep.append(r)
                tot += int(n)
        rows = np.asarray(keep, dtype=np.int64)
        member = torch.zeros(shape[d], dtype=torch.bool, device=dev)
        member[torch.from_numpy(rows).to(dev)] = True
        sel_all = []
        for a in range(0, col.numel(), _CHUNK):
            sel = member[_u32(col[a:a + _CHUNK])].nonzero().squeeze(1)
            if sel.numel():
                sel_all.append(sel + a)
        sel = torch.cat(sel_all) if sel_all else torch.zeros(0, dtype=torch.int64, device=dev)
        coords = torch.stack([_u32(c.index_select(0, sel)) for c in src_coords], 1).cpu().numpy()
        vals = src_vals.index_select(0, sel).double().cpu().numpy()
        out.append({"mode": d, "rows": rows, "coords": coords, "vals": vals})
    return out


def sample_parity_extracted(samples, init_factors, outputs, tol=1e-4):
    """Phase 2: max |gpu - ref| / max(|ref|, 1) (cli.py:247-261) over the
    sampled rows, ref = fp64 MTTKRP of their source nonzeros with the chained
    factors (mode d reads the GPU's own outputs of the modes before it, as the
    reference's mttkrp_all_modes does).  fp64 arithmetic in torch on the
    outputs' GPU (checker only).  outputs: the GPU's per-mode outputs in the
    order of `samples`."""
    import torch

    dev = outputs[0].device
    facs = [torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).to(dev) for f in init_factors]
    rank = facs[0].shape[1]
    worst, checked, per_mode = 0.0, 0, []
    for i, smp in enumerate(samples):
        d = smp["mode"]
        rows_t = torch.from_numpy(smp["rows"]).to(dev)
        expect = torch.zeros((rows_t.numel(), rank), dtype=torch.float64, device=dev)
        nsel = smp["coords"].shape[0]
        for a in range(0, nsel, 1 << 22):  # bounded temporaries (a head row can hold 10^8 nonzeros)
            coords = torch.from_numpy(smp["coords"][a:a + (1 << 22)]).to(dev)
            contrib = torch.from_numpy(smp["vals"][a:a + (1 << 22)]).to(dev)[:, None].expand(-1, rank).clone()
            for w in range(coords.shape[1]):
                if w != d:
                    contrib *= facs[w].index_select(0, coords[:, w])
            expect.index_add_(0, torch.searchsorted(rows_t, coords[:, d].contiguous()), contrib)
            del coords, contrib
        got = outputs[i].index_select(0, rows_t).double()
        err = float(((got - expect).abs() / expect.abs().clamp(min=1.0)).max().item()) if rows_t.numel() else 0.0
        per_mode.append({"mode": d, "rows": int(rows_t.numel()), "nnz": int(nsel), "max_rel_err": err})
        worst = max(worst, err)
        checked += int(rows_t.numel())
        facs[d] = outputs[i].double()
    return {"rows_checked": checked, "max_rel_err": worst, "tolerance": tol, "ok": worst <= tol,
            "per_mode": per_mode,
            "method": "seeded output-row sample; fp64 recomputation from the SOURCE tensor's nonzeros of those "
                      "rows (generator arrays, not the plan), chained factors; torch on the GPU as checker "
                      "(oracle/scale.py)"}


def sample_parity_source(src_coords, src_vals, shape, init_factors, outputs, modes, rows_per_mode=4096, seed=0,
                         nnz_budget=8_000_000, tol=1e-4):
    """Both phases at once (source still on the device)."""
    samples = extract_row_samples(src_coords, src_vals, shape, modes, rows_per_mode, seed, nnz_budget)
    return sample_parity_extracted(samples, init_factors, outputs, tol)


def cpd_mode_check(src_coords, src_vals, shape, d, facs, m, new, lambdas, rows_per_mode=1024, seed=0,
                   nnz_budget=8_000_000):
    """One CP-ALS mode update (cpd.py:39-67 / 108-167) checked on sampled rows:
    facs = the factors the GPU used for mode d (torch, I_w x R), m = its MTTKRP
    output, new = its normalised updated factor, lambdas = its column norms.
    Expected, in fp64 from the SOURCE tensor: M[rows] (MTTKRP), and
    M[rows] @ V^-1 with V = Hadamard of the other modes' Grams (computed here
    in fp64 from facs) applied to the GPU's own M rows -- compared with
    new[rows] * lambdas (the GPU's update before normalisation), the error
    scaled by sum_k |M_k| |W_kj| (the bound of a dot product in finite
    precision: the update is checked to working accuracy).  Returns
    {max_rel_err_mttkrp, max_rel_err_update, ...}; the update error against a
    fully fp64 chain and cond(V) are reported alongside."""
    import torch

    dev = m.device
    R = m.shape[1]
    rng = np.random.default_rng(seed + 7919 * d)
    col = src_coords[d]
    cand = np.sort(rng.permutation(shape[d])[:rows_per_mode]).astype(np.int64)
    counts = source_histogram(col, shape[d]).index_select(0, torch.from_numpy(cand).to(dev)).cpu().numpy()
    keep, tot = [], 0
    for r, n in zip(cand, counts):
        if n > 0 and (tot + n <= nnz_budget or not keep):
            keep.append(r)
            tot += int(n)
    rows_t = torch.from_numpy(np.asarray(keep, dtype=np.int64)).to(dev)
    member = torch.zeros(shape[d], dtype=torch.bool, device=dev)
    member[rows_t] = True
    f64 = [f.double() for f in facs]
    expect = torch.zeros((rows_t.numel(), R), dtype=torch.float64, device=dev)
    for a in range(0, col.numel(), _CHUNK):
        sel = member[_u32(col[a:a + _CHUNK])].nonzero().squeeze(1)
        if sel.numel() == 0:
            continue
        s_ = sel + a
        contrib = src_vals.index_select(0, s_).double()[:, None].expand(-1, R).clone()
        for w in range(len(shape)):
            if w != d:
                contrib *= f64[w].index_select(0, _u32(src_coords[w].index_select(0, s_)))
        expect.index_add_(0, torch.searchsorted(rows_t, _u32(col.index_select(0, s_))), contrib)
    return _cpd_update_check(rows_t, expect, tot, shape, d, f64, m, new, lambdas)


def _cpd_update_check(rows_t, expect, tot, shape, d, f64, m, new, lambdas):
    """The MTTKRP and ALS-update comparisons of cpd_mode_check for the sampled
    rows `rows_t` with their fp64 MTTKRP `expect` (f64: the factors the GPU
    used, in fp64)."""
    import torch

    dev = m.device
    R = m.shape[1]
    got_m = m.index_select(0, rows_t).double()
    err_m = float(((got_m - expect).abs() / expect.abs().clamp(min=1.0)).max().item())
    v = torch.ones((R, R), dtype=torch.float64, device=dev)
    for w in range(len(shape)):
        if w != d:
            v *= f64[w].T @ f64[w]
    lam = torch.from_numpy(np.asarray(lambdas, dtype=np.float64)).to(dev)
    got_u = new.index_select(0, rows_t).double() * lam[None, :]
    # the update step itself: fp64 M_gpu V^-1 from the GPU's own M.  V^-1 has
    # large entries of both signs when V is ill-conditioned, so the result is
    # a cancelling sum; its error is measured against the scale fp arithmetic
    # guarantees, sum_k |M_k| |W_kj| (|fl(sum a_k b_k) - sum a_k b_k| <=
    # gamma_n sum |a_k||b_k|), i.e. the update must be exact to working accuracy
    w = torch.linalg.inv(v)
    upd = got_m @ w
    scale = got_m.abs() @ w.abs()
    err_u = float(((got_u - upd).abs() / scale.clamp(min=1e-300)).max().item())
    # end to end (info): fp64 M V^-1 from the source -- M's fp32 rounding
    # (err_m) amplified by cond(V), a property of fp32 arithmetic, not gated
    upd64 = torch.linalg.solve(v, expect.T).T
    err_e2e = float(((got_u - upd64).abs() / upd64.abs().clamp(min=1.0)).max().item())
    return {"mode": d, "rows": int(rows_t.numel()), "nnz": tot, "max_rel_err_mttkrp": err_m,
            "max_rel_err_update": err_u, "max_rel_err_update_vs_fp64_source": err_e2e,
            "cond_V": float(torch.linalg.cond(v).item())}


def cpd_mode_check_extracted(sample, shape, d, facs, m, new, lambdas):
    """cpd_mode_check from rows extracted before the source left HBM
    (extract_row_samples: full-size cfg5 on one GPU): the sampled rows'
    MTTKRP in fp64 from their SOURCE nonzeros with the factors the GPU used,
    then the same MTTKRP and update comparisons."""
    import torch

    dev = m.device
    R = m.shape[1]
    f64 = [f.double() for f in facs]
    rows_t = torch.from_numpy(sample["rows"]).to(dev)
    expect = torch.zeros((rows_t.numel(), R), dtype=torch.float64, device=dev)
    nsel = sample["coords"].shape[0]
    for a in range(0, nsel, 1 << 22):
        coords = torch.from_numpy(sample["coords"][a:a + (1 << 22)]).to(dev)
        contrib = torch.from_numpy(sample["vals"][a:a + (1 << 22)]).to(dev)[:, None].expand(-1, R).clone()
        for w in range(coords.shape[1]):
            if w != d:
                contrib *= f64[w].index_select(0, coords[:, w])
        expect.index_add_(0, torch.searchsorted(rows_t, coords[:, d].contiguous()), contrib)
        del coords, contrib
    return _cpd_update_check(rows_t, expect, int(nsel), shape, d, f64, m, new, lambdas)
