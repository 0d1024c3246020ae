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
            pool = [torch.cat([c, b]) for c, b in zip(coords, batch)]
            del batch
            n = pool[0].numel()
            slots = 1
            while slots < 2 * n:
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


def synth_tensor_chunk(shape, nnz, rank, world, distribution="uniform", zipf_exponent=1.2,
                       value_dist="uniform", seed=0, device=None):
    """Rank `rank`'s contiguous chunk [nnz*rank//world, nnz*(rank+1)//world) of
    the global draw stream (counter-based: identical to the single-GPU draws
    of those elements), for the distributed plan build (distplan.py).  No
    de-duplication across the chunk boundary is possible here; see DESIGN.md."""
    import torch

    from . import _lib

    shape = tuple(int(s) for s in shape)
    lo = nnz * rank // world
    hi = nnz * (rank + 1) // world
    n = hi - lo
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    stream = torch.cuda.current_stream(dev).cuda_stream
    coords = [torch.empty(n, dtype=torch.int32, device=dev) for _ in shape]
    for w, s_ in enumerate(shape):
        if distribution == "uniform":
            _lib.call("skrp_synth_uniform_coords", _lib.ptr(coords[w]), n, s_, seed, w, lo, stream)
        else:
            cdf = torch.from_numpy(zipf_cdf(s_, zipf_exponent)).to(dev)
            _lib.call("skrp_synth_zipf_coords", _lib.ptr(coords[w]), n, _lib.ptr(cdf), s_, seed, w, lo, stream)
    vals = torch.empty(n, dtype=torch.float32, device=dev)
    _lib.call("skrp_synth_values", _lib.ptr(vals), n, 1 if value_dist == "normal" else 0, seed, lo, stream)
    t = SparseTensorCOO.from_device(shape, coords, vals, name=f"synth-{distribution}-{seed}-chunk{rank}of{world}",
                                    stats=LoadStats(nnz=n))
    t.global_offset = lo
    t.global_nnz = nnz
    return t
