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
                        value_dist="uniform", seed=0, name="", device=None):
    """Billion-scale generator on the GPU (Philox, same laws); see module doc.

    Coordinates are drawn independently per nonzero; duplicates are NOT
    removed here (expected count for uniform draws is nnz^2 / (2 * prod(shape)),
    0.09 for the Amazon-shaped config).  Returns a device-resident tensor.
    """
    import torch

    from . import _lib

    shape = tuple(int(s) for s in shape)
    if distribution not in ("uniform", "zipf"):
        raise ValueError(f"unknown distribution {distribution!r}")
    if value_dist not in ("uniform", "normal"):
        raise ValueError(f"unknown value_dist {value_dist!r}")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    coords = [torch.empty(nnz, dtype=torch.int32, device=dev) for _ in shape]
    vals = torch.empty(nnz, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    for w, s in enumerate(shape):
        if distribution == "uniform":
            _lib.call("skrp_synth_uniform_coords", _lib.ptr(coords[w]), nnz, s, seed, w, stream)
        else:
            cdf = torch.from_numpy(zipf_cdf(s, zipf_exponent)).to(dev)
            _lib.call("skrp_synth_zipf_coords", _lib.ptr(coords[w]), nnz, _lib.ptr(cdf), s, seed, w,
                      stream)
    _lib.call("skrp_synth_values", _lib.ptr(vals), nnz, 1 if value_dist == "normal" else 0, seed,
              stream)
    return SparseTensorCOO.from_device(shape, coords, vals,
                                       name=name or f"synth-{distribution}-{seed}-device",
                                       stats=LoadStats(nnz=nnz))
