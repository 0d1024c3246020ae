"""Synthetic tensors: the reference's generator law, on the host and on the GPU.

``synth_tensor`` reproduces ``shardkrp.synth.synth_tensor`` (synth.py:25-93)
array-for-array: same numpy Generator call sequence (per-mode uniform
``integers`` or Zipf inverse-CDF ``searchsorted`` draws, batch sizing, first-
occurrence dedup rounds, values drawn after coordinates).  Dedup uses a packed
1-D key when the shape's capacity fits in int64 -- the same first-occurrence
set as the reference's row-wise ``np.unique(axis=0)``, ~20x faster.  Pinned
by tests/test_host_api.py against tests/golden/ (cfg1 digests included).

``synth_tensor_device`` is the billion-scale generator:
the same laws drawn with a counter-based Philox stream inside a CUDA kernel,
written straight into the device mirror (int32 coordinates per mode + fp32
values).  It cannot reproduce numpy's stream; it reproduces the law, and the
bench's parity checks run on the arrays it produced.
"""

from __future__ import annotations

import numpy as np

from .tensor import DEFAULT_VALUE_DTYPE, LoadStats, SparseTensorCOO

_MAX_ROUNDS = 200


def zipf_cdf(size: int, exponent: float) -> np.ndarray:
    """Normalised cumulative i^-s over i = 1..size (synth.py:17-22)."""
    w = np.arange(1, size + 1, dtype=np.float64) ** (-exponent)
    return np.cumsum(w) / w.sum()


def _first_occurrence(pool: np.ndarray, shape) -> np.ndarray:
    cap = 1
    for s in shape:
        cap *= int(s)
    if cap < 2 ** 62:
        key = np.zeros(len(pool), dtype=np.int64)
        for w, s in enumerate(shape):
            key = key * int(s) + pool[:, w]
        _, first = np.unique(key, return_index=True)
    else:
        _, first = np.unique(pool, axis=0, return_index=True)
    return first


def synth_tensor(shape, nnz, distribution="uniform", zipf_exponent=1.2, value_dist="uniform",
                 seed=0, value_dtype=DEFAULT_VALUE_DTYPE, name=""):
    """Tensor with `nnz` unique coordinates, deterministic in `seed`."""
    shape = tuple(int(s) for s in shape)
    nnz = int(nnz)
    if nnz < 0:
        raise ValueError("nnz must be >= 0")
    capacity = 1
    for s in shape:
        capacity *= s
    if nnz > capacity:
        raise ValueError(f"nnz={nnz} infeasible for shape {shape} (capacity {capacity})")
    if distribution not in ("uniform", "zipf"):
        raise ValueError(f"unknown distribution {distribution!r}")
    if value_dist not in ("uniform", "normal"):
        raise ValueError(f"unknown value_dist {value_dist!r}")

    gen = np.random.default_rng(seed)
    cdfs = [zipf_cdf(s, zipf_exponent) for s in shape] if distribution == "zipf" else None

    def draw(count):
        cols = []
        for w, s in enumerate(shape):
            if cdfs is None:
                cols.append(gen.integers(0, s, count, dtype=np.int64))
            else:
                cols.append(np.searchsorted(cdfs[w], gen.random(count)).astype(np.int64))
        return np.stack(cols, axis=1)

    kept = np.empty((0, len(shape)), dtype=np.int64)
    dups = 0
    rounds = 0
    while len(kept) < nnz:
        if rounds >= _MAX_ROUNDS - 1:  # the reference's for/else gives up at its 200th draw
            raise ValueError(
                f"could not collect {nnz} unique coordinates in {_MAX_ROUNDS} rounds; "
                "distribution too concentrated for requested nnz")
        rounds += 1
        short = nnz - len(kept)
        pool = np.concatenate([kept, draw(max(short + short // 4 + 16, 64))], axis=0)
        first = _first_occurrence(pool, shape)
        dups += len(pool) - len(first)
        kept = pool[np.sort(first)]
    coords = kept[:nnz]
    if value_dist == "uniform":
        vals = gen.random(nnz).astype(value_dtype)
    else:
        vals = gen.standard_normal(nnz).astype(value_dtype)
    t = SparseTensorCOO(shape, coords, vals, name=name or f"synth-{distribution}-{seed}")
    t.stats = LoadStats(nnz=nnz, zero_values=int(np.count_nonzero(vals == 0)), duplicates=dups)
    return t


def synth_tensor_device(shape, nnz, distribution="uniform", zipf_exponent=1.2,
                        value_dist="uniform", seed=0, name="", device=None, unique=True):
    """Billion-scale generator on the GPU (Philox, the reference's laws).

    Coordinates of draw g are a pure function of (seed, mode, g).  With
    ``unique`` (default, like the reference) duplicate tuples are removed
    keeping first occurrences and the pool is topped up with further draws
    until `nnz` unique tuples exist -- the reference's rounds (synth.py:68-84:
    batch = short + short//4 + 16, first occurrences kept, <= 200 rounds) run
    on the GPU with a hash-table first-occurrence filter (skrp_dedup_mark).
    Values are drawn after the coordinates, one per kept nonzero.
    """
    import torch

    from . import _lib

    shape = tuple(int(s) for s in shape)
    nnz = int(nnz)
    if distribution not in ("uniform", "zipf"):
        raise ValueError(f"unknown distribution {distribution!r}")
    if value_dist not in ("uniform", "normal"):
        raise ValueError(f"unknown value_dist {value_dist!r}")
    capacity = 1
    for s_ in shape:
        capacity *= s_
    if nnz > capacity:
        raise ValueError(f"nnz={nnz} infeasible for shape {shape} (capacity {capacity})")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    stream = torch.cuda.current_stream(dev).cuda_stream
    cdfs = ([torch.from_numpy(zipf_cdf(s_, zipf_exponent)).to(dev) for s_ in shape]
            if distribution == "zipf" else None)

    def draw(count, offset):
        cols = [torch.empty(count, dtype=torch.int32, device=dev) for _ in shape]
        for w, s_ in enumerate(shape):
            if cdfs is None:
                _lib.call("skrp_synth_uniform_coords", _lib.ptr(cols[w]), count, s_, seed, w, offset, stream)
            else:
                _lib.call("skrp_synth_zipf_coords", _lib.ptr(cols[w]), count, _lib.ptr(cdfs[w]), s_, seed, w,
                          offset, stream)
        return cols

    dups = 0
    if not unique:
        coords = draw(nnz, 0)
    else:
        coords = [torch.empty(0, dtype=torch.int32, device=dev) for _ in shape]
        drawn = 0
        rounds = 0
        while coords[0].numel() < nnz:
            if rounds >= _MAX_ROUNDS - 1:
                raise ValueError(
                    f"could not collect {nnz} unique coordinates in {_MAX_ROUNDS} rounds; "
                    "distribution too concentrated for requested nnz")
            rounds += 1
            short = nnz - coords[0].numel()
            count = max(short + short // 4 + 16, 64)
            batch = draw(count, drawn)
            drawn += count
            if coords[0].numel() == 0:  # first round: no copy of the batch
                pool = batch
            else:
                pool = [torch.cat([c, b]) for c, b in zip(coords, batch)]
            del batch
            n = pool[0].numel()
            # open-addressing table at load factor <= 1/2, or <= 2/3 past 2^31
            # entries (10^9-scale pools: the table is the largest buffer)
            slots = 1
            while slots < (2 * n if n < (1 << 31) else (3 * n) // 2):
                slots *= 2
            table = torch.empty(slots, dtype=torch.int64, device=dev)
            keep = torch.empty(n, dtype=torch.uint8, device=dev)
            cptr = (_lib.vp * len(pool))(*[c.data_ptr() for c in pool])
            _lib.call("skrp_dedup_mark", cptr, len(pool), n, table.data_ptr(), slots, keep.data_ptr(), stream)
            del table
            mask = keep.bool()
            kept = int(mask.sum().item())
            dups += n - kept
            coords = [c[mask] for c in pool]  # stable compaction: first occurrences, draw order
            del pool, mask, keep
        coords = [c[:nnz].contiguous() for c in coords]
    vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("skrp_synth_values", _lib.ptr(vals), nnz, 1 if value_dist == "normal" else 0, seed, 0, stream)
    return SparseTensorCOO.from_device(shape, coords, vals,
                                       name=name or f"synth-{distribution}-{seed}-device",
                                       stats=LoadStats(nnz=nnz, duplicates=dups))


def _draw_coords(shape, count, offset, cdfs, seed, dev, stream):
    """Coordinates of global draws [offset, offset + count) (Philox, K7)."""
    import torch

    from . import _lib

    cols = [torch.empty(count, dtype=torch.int32, device=dev) for _ in shape]
    for w, s_ in enumerate(shape):
        if cdfs is None:
            _lib.call("skrp_synth_uniform_coords", _lib.ptr(cols[w]), count, s_, seed, w, offset, stream)
        else:
            _lib.call("skrp_synth_zipf_coords", _lib.ptr(cols[w]), count, _lib.ptr(cdfs[w]), s_, seed, w, offset,
                      stream)
    return cols


def _tuple_owner(cols, world):
    """Owner rank of each coordinate tuple (a hash of the whole tuple), so all
    copies of a tuple meet on one rank."""
    import torch

    h = torch.zeros(cols[0].numel(), dtype=torch.int64, device=cols[0].device)
    for w, c in enumerate(cols):
        h = (h ^ (c.long() + 0x9E3779B9 + (w << 20))) * 0x100000001B3
        h = h ^ (h >> 29)
    return torch.remainder(h, world).to(torch.int32)


def synth_tensor_chunk(shape, nnz, rank, world, distribution="uniform", zipf_exponent=1.2,
                       value_dist="uniform", seed=0, device=None, unique=True, group=None):
    """Rank `rank`'s contiguous chunk [nnz*rank//world, nnz*(rank+1)//world) of
    the global nonzero order, for the distributed plan build (distplan.py).

    ``unique=False``: the raw draw stream (counter-based, identical to the
    single-GPU draws of those positions; no collective).

    ``unique=True`` (default, the reference law, synth.py:68-84): the tensor is
    the first `nnz` DISTINCT tuples of the global draw stream -- exactly what
    ``synth_tensor_device(unique=True)`` returns on one GPU -- built without any
    rank holding the tensor.  Rounds follow the reference's schedule (batch =
    short + short//4 + 16 draws, split across ranks in rank order).  Every draw
    is hash-routed to the rank owning its tuple (all-to-all); the owner keeps
    the tuples of earlier rounds, so a first-occurrence pass over [its kept
    tuples | arrivals in global draw order] (skrp_dedup_mark) decides which
    draws survive; the verdicts travel back.  After the last round every
    survivor's global position (prefix over (round, rank)) routes it to the
    rank whose chunk holds that position, and values are drawn per position
    (values after coordinates, like the reference)."""
    import torch

    from . import _lib

    shape = tuple(int(s) for s in shape)
    nnz = int(nnz)
    lo = nnz * rank // world
    hi = nnz * (rank + 1) // world
    n = hi - lo
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    stream = torch.cuda.current_stream(dev).cuda_stream
    cdfs = ([torch.from_numpy(zipf_cdf(s_, zipf_exponent)).to(dev) for s_ in shape]
            if distribution == "zipf" else None)
    dups = 0
    if not unique or world == 1:
        if unique:  # one rank: the single-GPU generator is the global one
            t = synth_tensor_device(shape, nnz, distribution, zipf_exponent, value_dist, seed, device=dev)
            coords, _ = t.device_arrays(dev)
            dups = t.stats.duplicates
        else:
            coords = _draw_coords(shape, n, lo, cdfs, seed, dev, stream)
    else:
        coords, dups = _unique_chunk(shape, nnz, rank, world, cdfs, seed, dev, stream, group)
    vals = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.call("skrp_synth_values", _lib.ptr(vals), n, 1 if value_dist == "normal" else 0, seed, lo, stream)
    t = SparseTensorCOO.from_device(shape, coords, vals, name=f"synth-{distribution}-{seed}-chunk{rank}of{world}",
                                    stats=LoadStats(nnz=n, duplicates=dups))
    t.global_offset = lo
    t.global_nnz = nnz
    return t


def _unique_chunk(shape, nnz, rank, world, cdfs, seed, dev, stream, group):
    import torch

    from . import _lib
    from .distplan import _all_reduce_, _all_to_all, _dist, _stable_sort

    dist = _dist()
    capacity = 1
    for s_ in shape:
        capacity *= s_
    if nnz > capacity:
        raise ValueError(f"nnz={nnz} infeasible for shape {shape} (capacity {capacity})")
    nm = len(shape)
    owned = [torch.empty(0, dtype=torch.int32, device=dev) for _ in shape]  # tuples I own, kept so far
    kept_parts = []   # per round: this rank's surviving draws (coords), in draw order
    round_counts = []  # per round: survivors on every rank (world,)
    total, drawn, rounds, dups = 0, 0, 0, 0

    def exchange(x, send_counts, recv_counts):
        return _all_to_all(x, send_counts, recv_counts, group)

    while total < nnz:
        if rounds >= _MAX_ROUNDS - 1:
            raise ValueError(
                f"could not collect {nnz} unique coordinates in {_MAX_ROUNDS} rounds; "
                "distribution too concentrated for requested nnz")
        rounds += 1
        short = nnz - total
        count = max(short + short // 4 + 16, 64)
        a, b = drawn + count * rank // world, drawn + count * (rank + 1) // world
        drawn += count
        mine = _draw_coords(shape, b - a, a, cdfs, seed, dev, stream)
        # route every draw to its tuple's owner, stably (draw order kept per dest)
        dest = _tuple_owner(mine, world)
        _, perm = _stable_sort(dest, max(1, (world - 1).bit_length()), stream)
        send_counts = torch.bincount(dest.long(), minlength=world).cpu().numpy().astype(np.int64)
        allc = [None] * world
        dist.all_gather_object(allc, send_counts.tolist(), group=group)
        recv_counts = np.asarray([allc[r][rank] for r in range(world)], dtype=np.int64)
        perm_l = perm.long()
        arrivals = [exchange(c.index_select(0, perm_l), send_counts, recv_counts) for c in mine]
        # arrivals are grouped by source rank = global draw order (rank slices are
        # consecutive draw ranges): first occurrences over [owned | arrivals]
        pool = [torch.cat([o, x]) for o, x in zip(owned, arrivals)]
        npool = pool[0].numel()
        slots = 1
        while slots < 2 * max(npool, 1):
            slots *= 2
        table = torch.empty(slots, dtype=torch.int64, device=dev)
        keep = torch.empty(npool, dtype=torch.uint8, device=dev)
        cptr = (_lib.vp * nm)(*[c.data_ptr() for c in pool])
        _lib.call("skrp_dedup_mark", cptr, nm, npool, table.data_ptr(), slots, keep.data_ptr(), stream)
        del table
        k_new = keep[owned[0].numel():]
        owned = [torch.cat([o, x[k_new.bool()]]) for o, x in zip(owned, arrivals)]
        del pool, arrivals
        # verdicts back to the drawing ranks, then back into draw order
        back = exchange(k_new, recv_counts, send_counts)
        verdict = torch.empty_like(back)
        verdict[perm_l] = back
        sel = verdict.bool()
        kept_parts.append([c[sel] for c in mine])
        cnt = torch.zeros(world, dtype=torch.int64, device=dev)
        cnt[rank] = int(sel.sum().item())
        _all_reduce_(cnt, group)
        cnt = cnt.cpu().numpy()
        dups += int(b - a - cnt[rank])
        round_counts.append(cnt)
        total += int(cnt.sum())
        del mine, dest, perm, perm_l, back, verdict, sel
    # global position of every survivor: rounds in order, ranks in order inside a round
    base = 0
    pos_parts, coord_parts = [], []
    for cnt, part in zip(round_counts, kept_parts):
        start = base + int(cnt[:rank].sum())
        m = part[0].numel()
        pos_parts.append(torch.arange(start, start + m, dtype=torch.int64, device=dev))
        coord_parts.append(part)
        base += int(cnt.sum())
    pos = torch.cat(pos_parts)
    cols = [torch.cat([p_[w] for p_ in coord_parts]) for w in range(nm)]
    keep = pos < nnz
    pos = pos[keep]
    cols = [c[keep] for c in cols]
    bounds = torch.tensor([nnz * r // world for r in range(world + 1)], dtype=torch.int64, device=dev)
    dest = (torch.searchsorted(bounds, pos, right=True) - 1).to(torch.int32)
    _, perm = _stable_sort(dest, max(1, (world - 1).bit_length()), stream)
    perm_l = perm.long()
    send_counts = torch.bincount(dest.long(), minlength=world).cpu().numpy().astype(np.int64)
    allc = [None] * world
    dist.all_gather_object(allc, send_counts.tolist(), group=group)
    recv_counts = np.asarray([allc[r][rank] for r in range(world)], dtype=np.int64)
    rpos = _all_to_all(pos.index_select(0, perm_l), send_counts, recv_counts, group)
    lo = nnz * rank // world
    n = nnz * (rank + 1) // world - lo
    if rpos.numel() != n:
        raise RuntimeError(f"unique chunk routing: rank {rank} received {rpos.numel()} of {n} positions")
    slot = rpos - lo
    out = []
    for c in cols:
        x = _all_to_all(c.index_select(0, perm_l), send_counts, recv_counts, group)
        y = torch.empty(n, dtype=torch.int32, device=dev)
        y[slot] = x
        out.append(y)
    return out, dups
