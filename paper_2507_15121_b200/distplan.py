"""Distributed mode-plan build: one process per GPU (SURVEY.md §8(e) "Plan build").

Each rank starts from a CONTIGUOUS chunk of the global nonzero order
(``synth.synth_tensor_chunk`` or any caller-provided split) and ends with
the exact slice of the reference plan (partition.py:196-257) that it owns:

  1. histogram of c_d over the local chunk (skrp_histogram), all-reduced ->
     global counts; exclusive scan -> prefix;
  2. shard bounds from the global counts (equal-index formula or the
     bit-exact nnz-balanced search) -- identical on every rank;
  3. shard -> rank placement with engine.assign_shards on the GLOBAL shard
     sizes (the same call DistributedMttkrp makes, so both agree);
  4. route: dest = owner(shard(c_d)) (skrp_route_by_bounds), stable
     partition of the chunk by dest (radix sort on the dest key), counts
     exchanged, one all-to-all per array (coordinates, values);
  5. the received elements arrive grouped by source rank, i.e. in GLOBAL
     order (chunks are contiguous and the partition was stable), so a local
     stable sort by c_d reproduces ``argsort(kind="stable")`` restricted to
     the owned shards bit-for-bit.

No rank ever holds the whole tensor, so totals beyond 2^32 nonzeros and
beyond one GPU's HBM (cfg3/cfg4) build in parallel.  The returned plan keeps
every shard's global index range and global size; non-owned shards are empty
locally.
"""

from __future__ import annotations

import time
import warnings

import numpy as np

from . import _lib
from .engine import assign_shards
from .partition import ModePartitionPlan, PartitionConfig, _key_bits


def _dist():
    import torch.distributed as dist

    return dist


def _backend_is_nccl(group):
    dist = _dist()
    return dist.get_backend(group) == "nccl"


def _all_reduce_(t, group):
    dist = _dist()
    if _backend_is_nccl(group):
        dist.all_reduce(t, group=group)
        return t
    c = t.cpu()
    dist.all_reduce(c, group=group)
    t.copy_(c)
    return t


def _all_to_all(send, send_counts, recv_counts, group):
    """all_to_all_single over variable splits (device tensors)."""
    import torch

    dist = _dist()
    out = torch.empty(int(sum(recv_counts)), dtype=send.dtype, device=send.device)
    if _backend_is_nccl(group):
        dist.all_to_all_single(out, send, [int(x) for x in recv_counts], [int(x) for x in send_counts], group=group)
        return out
    # gloo: point-to-point over CPU staging (used by the single-GPU smoke of this path)
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    s_off = np.concatenate([[0], np.cumsum(send_counts)])
    r_off = np.concatenate([[0], np.cumsum(recv_counts)])
    send_c = send.cpu()
    recv_c = torch.empty(int(sum(recv_counts)), dtype=send.dtype)
    ops = []
    for r in range(world):
        if r == me:
            recv_c[r_off[r]:r_off[r + 1]] = send_c[s_off[r]:s_off[r + 1]]
            continue
        if send_counts[r]:
            ops.append(dist.isend(send_c[s_off[r]:s_off[r + 1]].contiguous(), r, group=group))
        if recv_counts[r]:
            buf = torch.empty(int(recv_counts[r]), dtype=send.dtype)
            ops.append((r, buf, dist.irecv(buf, r, group=group)))
    for op in ops:
        if isinstance(op, tuple):
            r, buf, w = op
            w.wait()
            recv_c[r_off[r]:r_off[r + 1]] = buf
        else:
            op.wait()
    out.copy_(recv_c)
    return out


def _stable_sort(keys, bits, stream):
    import torch

    n = keys.numel()
    sk = torch.empty_like(keys)
    perm = torch.empty_like(keys)
    ws_bytes = _lib.lib().skrp_sort_workspace_bytes(n, bits)
    ws = torch.empty(max(int(ws_bytes), 16), dtype=torch.uint8, device=keys.device)
    _lib.call("skrp_stable_sort_by_key", keys.data_ptr(), n, bits, sk.data_ptr(), perm.data_ptr(), ws.data_ptr(),
              ws_bytes, stream)
    return sk, perm


def _gather(src, perm, stream):
    import torch

    out = torch.empty_like(src)
    _lib.call("skrp_gather_u32", src.data_ptr(), perm.data_ptr(), perm.numel(), out.data_ptr(), stream)
    return out


def _histogram(keys, bins, stream):
    import torch

    counts = torch.empty(bins, dtype=torch.int64, device=keys.device)
    _lib.call("skrp_histogram", keys.data_ptr(), keys.numel(), bins, counts.data_ptr(), stream)
    return counts


def _prefix(counts, stream):
    import torch

    n = counts.numel()
    pre = torch.empty(n + 1, dtype=torch.int64, device=counts.device)
    wsb = _lib.lib().skrp_scan_workspace_bytes(n)
    ws = torch.empty(max(int(wsb), 16), dtype=torch.uint8, device=counts.device)
    _lib.call("skrp_exclusive_scan_i64", counts.data_ptr(), n, pre.data_ptr(), ws.data_ptr(), wsb, stream)
    return pre


def build_mode_plan_distributed(chunk, mode: int, cfg: PartitionConfig, scheduling: str = "dynamic",
                                group=None) -> ModePartitionPlan:
    """This rank's slice of the mode-`mode` plan from its chunk (see module doc).

    ``scheduling="split"`` (element-split placement):
    rank r receives the global sorted positions [r*nnz/m, (r+1)*nnz/m), so a
    heavy row is cut across ranks exactly like engine.assign_elements cuts a
    replicated plan -- no rank needs the whole plan."""
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    if not 0 <= mode < chunk.num_modes:
        raise ValueError(f"mode {mode} out of range")
    t0 = time.perf_counter()
    shape = chunk.shape
    num_indices = shape[mode]
    k = cfg.devices * cfg.oversubscription
    if k > num_indices:
        warnings.warn(f"mode {mode}: requested {k} shards exceeds {num_indices} indices; clamping",
                      RuntimeWarning, stacklevel=2)
        k = num_indices
    coords, vals = chunk.device_arrays()
    dev = vals.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    n_local = vals.numel()

    # 1-2: global histogram -> bounds, global shard sizes
    counts = _all_reduce_(_histogram(coords[mode], num_indices, stream), group)
    prefix = _prefix(counts, stream)
    bounds = np.empty(k + 1, dtype=np.int64)
    if cfg.strategy == "equal-index":
        _lib.call("skrp_equal_index_bounds", num_indices, k, _lib.ptr(bounds))
    else:
        c_host = np.ascontiguousarray(counts.cpu().numpy())
        _lib.call("skrp_nnz_balanced_bounds", _lib.ptr(c_host), num_indices, k, _lib.ptr(bounds))
    bounds_d = torch.from_numpy(bounds).to(dev)
    global_offsets = prefix[bounds_d].cpu().numpy()
    global_sizes = np.diff(global_offsets)

    if scheduling == "split":
        return _build_split(chunk, mode, cfg, group, coords, vals, counts, prefix, bounds, bounds_d, global_offsets,
                            global_sizes, t0, stream)

    # 3: placement on global sizes (the runner recomputes the same)
    class _Shape:  # minimal plan view for assign_shards
        shard_count = k
        shards = [type("S", (), {"nnz": int(x)})() for x in global_sizes]

    assignment = assign_shards(_Shape, world, scheduling, weights=global_sizes)
    owner = np.empty(k, dtype=np.int32)
    for r, ids in enumerate(assignment):
        owner[ids] = r
    owner_d = torch.from_numpy(owner).to(dev)

    # 4: route, stable partition by destination, exchange
    dest = torch.empty(n_local, dtype=torch.int32, device=dev)
    _lib.call("skrp_route_by_bounds", coords[mode].data_ptr(), n_local, bounds_d.data_ptr(), k,
              owner_d.data_ptr(), dest.data_ptr(), stream)
    send_counts = _histogram(dest, world, stream)
    _, perm = _stable_sort(dest, max(1, _key_bits(world)), stream)
    del dest
    recv_counts = send_counts.clone()
    if _backend_is_nccl(group):
        dist.all_to_all_single(recv_counts, send_counts, group=group)
    else:
        gathered = [torch.empty(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, send_counts.cpu(), group=group)
        me = dist.get_rank(group)
        rc = torch.stack([g[me] for g in gathered])
        recv_counts = rc.to(dev)
    sc = send_counts.cpu().numpy()
    rcn = recv_counts.cpu().numpy()
    recv = []
    for arr in list(coords) + [vals]:
        moved = _gather(arr, perm, stream)
        recv.append(_all_to_all(moved, sc, rcn, group))
        del moved
    del perm
    r_coords, r_vals = recv[:-1], recv[-1]

    # 5: local stable sort by c_d (arrivals are in global order)
    n_mine = r_vals.numel()
    bits = _key_bits(num_indices)
    key_sorted, order = _stable_sort(r_coords[mode], bits, stream)
    sorted_coords = [key_sorted if w == mode else _gather(r_coords[w], order, stream) for w in range(len(shape))]
    svals = _gather(r_vals, order, stream)
    del r_coords, r_vals, order
    local_counts = _histogram(sorted_coords[mode], num_indices, stream)
    local_offsets = _prefix(local_counts, stream)[bounds_d].cpu().numpy()
    torch.cuda.current_stream(dev).synchronize()
    plan = ModePartitionPlan(mode, shape, cfg.strategy, cfg.isp_capacity, chunk.name, sorted_coords, svals, None,
                             bounds, local_offsets, build_time=time.perf_counter() - t0)
    plan.global_shard_nnz = global_sizes
    plan.global_offsets = global_offsets
    plan.shard_owner = owner
    plan.local_nnz = n_mine
    return plan


def _build_split(chunk, mode, cfg, group, coords, vals, counts, prefix, bounds, bounds_d, global_offsets,
                 global_sizes, t0, stream):
    """Split routing: an element of row c with within-row global rank j sits at
    global sorted position prefix[c] + j; it goes to the rank whose element
    range holds that position.  Rows inside one range route by their start
    (skrp_route_by_bounds on the row cuts); only the <= m-1 rows cut by a
    range edge need j: this rank's rank among the row's elements in its chunk
    plus the row's counts on lower ranks (an all-gather of m-1 integers)."""
    import torch

    dist = _dist()
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = vals.device
    shape = chunk.shape
    num_indices = shape[mode]
    n = int(prefix[-1].item())
    cuts = np.array([r * n // world for r in range(world + 1)], dtype=np.int64)
    pre_h = prefix.cpu().numpy()
    # row at global position p: last c with prefix[c] <= p
    def row_at(p):
        return int(np.searchsorted(pre_h, p, side="right") - 1)

    inner = [c for c in cuts[1:-1] if 0 < c < n]
    rcut = [0] + [row_at(c) if 0 < c < n else num_indices for c in cuts[1:-1]] + [num_indices]
    boundary = sorted({row_at(c) for c in inner if row_at(c - 1) == row_at(c)})
    # route whole rows by the row cuts (rows [rcut[r], rcut[r+1]) -> r; a cut
    # row routes to the higher rank here and is fixed up below)
    n_local = vals.numel()
    keys = coords[mode]
    rb = torch.from_numpy(np.asarray(rcut, dtype=np.int64)).to(dev)
    ident = torch.arange(world, dtype=torch.int32, device=dev)
    dest = torch.empty(n_local, dtype=torch.int32, device=dev)
    _lib.call("skrp_route_by_bounds", keys.data_ptr(), n_local, rb.data_ptr(), world, ident.data_ptr(),
              dest.data_ptr(), stream)
    if boundary:
        mine = torch.stack([(keys == b).sum() for b in boundary]).to(torch.int64)
        allc = [torch.empty_like(mine.cpu()) for _ in range(world)]
        dist.all_gather(allc, mine.cpu(), group=group)
        lower = torch.stack(allc[:me]).sum(0) if me else torch.zeros_like(mine.cpu())
        cuts_d = torch.from_numpy(cuts).to(dev)
        for bi, b in enumerate(boundary):
            m = keys == b
            idx = torch.nonzero(m).squeeze(1)
            if idx.numel() == 0:
                continue
            pos = int(pre_h[b]) + int(lower[bi]) + torch.arange(idx.numel(), device=dev, dtype=torch.int64)
            dest[idx] = (torch.searchsorted(cuts_d, pos, right=True) - 1).to(torch.int32)
    send_counts = _histogram(dest, world, stream)
    _, perm = _stable_sort(dest, max(1, _key_bits(world)), stream)
    del dest
    if _backend_is_nccl(group):
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=group)
    else:
        gathered = [torch.empty(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, send_counts.cpu(), group=group)
        recv_counts = torch.stack([g[me] for g in gathered]).to(dev)
    sc = send_counts.cpu().numpy()
    rcn = recv_counts.cpu().numpy()
    recv = []
    for arr in list(coords) + [vals]:
        moved = _gather(arr, perm, stream)
        recv.append(_all_to_all(moved, sc, rcn, group))
        del moved
    del perm
    r_coords, r_vals = recv[:-1], recv[-1]
    bits = _key_bits(num_indices)
    key_sorted, order = _stable_sort(r_coords[mode], bits, stream)
    sorted_coords = [key_sorted if w == mode else _gather(r_coords[w], order, stream) for w in range(len(shape))]
    svals = _gather(r_vals, order, stream)
    del r_coords, r_vals, order
    local_counts = _histogram(sorted_coords[mode], num_indices, stream)
    local_offsets = _prefix(local_counts, stream)[bounds_d].cpu().numpy()
    torch.cuda.current_stream(dev).synchronize()
    plan = ModePartitionPlan(mode, shape, cfg.strategy, cfg.isp_capacity, chunk.name, sorted_coords, svals, None,
                             bounds, local_offsets, build_time=time.perf_counter() - t0)
    plan.global_shard_nnz = global_sizes
    plan.global_offsets = global_offsets
    plan.local_nnz = int(svals.numel())
    # the element-split placement of the GLOBAL plan (engine.assign_elements)
    plan.split_info = {"ranges": [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)],
                       "boundary": boundary, "rcut": rcut}
    assert plan.local_nnz == int(cuts[me + 1] - cuts[me]), "split routing lost elements"
    return plan
