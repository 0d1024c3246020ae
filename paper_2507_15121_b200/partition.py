"""Per-mode shard/ISP plans built on the GPU (drop-in for shardkrp.partition).

Same types, fields and semantics as the reference (partition.py:44-262):
``PartitionConfig``, ``TensorShard``, ``ModePartitionPlan``,
``build_mode_plan``, ``build_all_plans`` -- including the shard-count clamp
with its RuntimeWarning (partition.py:209-217), ``index_range`` bounds from
the equal-index or nnz-balanced strategy, element offsets
(``searchsorted(sorted_col, bounds, 'left')`` == ``prefix[bounds]``), and ISP
boundaries ``[0, c, 2c, ..., count]`` (partition.py:127-131).

What moved to the GPU (libshardkrp_cuda.so, csrc/partition.cu):
  * the stable sort by c_d -- LSD radix on (c_d, position), 8-bit digits;
    the permutation equals numpy's ``argsort(kind="stable")`` bit-for-bit;
  * the permuted copy -- SoA u32 coordinates + fp32 values, resident in HBM
    (the layout the MTTKRP kernel streams);
  * ``bincount`` + prefix -- histogram and exclusive scan kernels.
The nnz-balanced cut search runs on the host inside the same library (it is
O(k log I log nnz) on the prefix array).

Host-visible ``_indices`` (nnz, N) uint64 / ``_values`` are materialised
lazily on first access (bit-exact: the source tensor's arrays permuted by the
GPU order), so billion-scale plans never round-trip through host memory.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .tensor import INDEX_DTYPE, SparseTensorCOO

PLAN_MAGIC = b"SKRPPLN\x00"
CELL_TAIL_STAGES = 8  # skip entries after the last stripe (csrc/mttkrp_cells.cu CELL_TAIL_STAGES)
PLAN_VERSION = 1
STRATEGIES = ("equal-index", "nnz-balanced")


class PlanError(Exception):
    """Base class for plan cache problems (partition.py:32-41)."""


class PlanVersionError(PlanError):
    pass


class PlanIntegrityError(PlanError):
    pass


@dataclass(frozen=True)
class PartitionConfig:
    devices: int = 1
    workers_per_device: int = 1
    oversubscription: int = 4
    isp_capacity: int = 8192
    strategy: str = "equal-index"

    def __post_init__(self):
        for name in ("devices", "workers_per_device", "oversubscription", "isp_capacity"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be a positive integer")
        if self.strategy not in STRATEGIES:
            raise ValueError(f"strategy must be one of {STRATEGIES}, got {self.strategy!r}")


def isp_boundaries(count: int, capacity: int) -> np.ndarray:
    """[0, c, 2c, ..., count]; [0] for an empty shard (partition.py:127-131)."""
    if count == 0:
        return np.zeros(1, dtype=np.int64)
    return np.append(np.arange(0, count, capacity, dtype=np.int64), np.int64(count))


class TensorShard:
    """Contiguous run of plan elements owning one output-index range."""

    def __init__(self, plan, mode, shard_id, index_range, start, stop, isp_bounds):
        self._plan = plan
        self.mode = mode
        self.shard_id = shard_id
        self.index_range = index_range
        self.start = start  # element offset of the shard inside the plan
        self.stop = stop
        self.isp_boundaries = isp_bounds

    @property
    def nnz(self) -> int:
        return self.stop - self.start

    @property
    def isp_count(self) -> int:
        return max(len(self.isp_boundaries) - 1, 0)

    def isp_slices(self):
        b = self.isp_boundaries
        for q in range(self.isp_count):
            yield int(b[q]), int(b[q + 1])

    @property
    def indices(self) -> np.ndarray:
        return self._plan._indices[self.start:self.stop]

    @property
    def values(self) -> np.ndarray:
        return self._plan._values[self.start:self.stop]

    @property
    def byte_size(self) -> int:
        return self.nnz * (len(self._plan.shape) * 8 + np.dtype(self._plan.value_dtype).itemsize)

    def __repr__(self):
        return (f"TensorShard(mode={self.mode}, shard_id={self.shard_id}, "
                f"index_range={self.index_range}, nnz={self.nnz}, isps={self.isp_count})")


class ModePartitionPlan:
    """Reordered, sharded copy of a tensor for one output mode.

    Device side (HBM): ``coords[w]`` int32 (== u32) sorted by c_mode,
    ``vals`` fp32, ``perm`` the stable order (int32), ``offsets`` (k+1).
    """

    def __init__(self, mode, shape, strategy, isp_capacity, name, coords, vals, perm, bounds,
                 offsets, source=None, build_time=0.0):
        self.mode = mode
        self.shape = tuple(shape)
        self.strategy = strategy
        self.isp_capacity = isp_capacity
        self.name = name
        self.build_time = build_time
        self.coords = coords
        self.vals = vals
        self.perm = perm
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.offsets = np.asarray(offsets, dtype=np.int64)
        self._source = source
        self._host_idx = None
        self._host_vals = None
        self._exec_cache = {}
        # execution layout of the device arrays: "flycoo" (plan order) or
        # "blocked" (see to_blocked); groups: per shard, [start, stop) ranges
        self.layout = "flycoo"
        self.block_shifts = None
        self.block_order = None
        self.groups = None
        self.panel = None
        self.cells = None
        self.shards = [
            TensorShard(self, mode, j, (int(self.bounds[j]), int(self.bounds[j + 1])),
                        int(self.offsets[j]), int(self.offsets[j + 1]),
                        isp_boundaries(int(self.offsets[j + 1] - self.offsets[j]), isp_capacity))
            for j in range(len(self.bounds) - 1)
        ]

    @property
    def shard_count(self) -> int:
        return len(self.shards)

    @property
    def nnz(self) -> int:
        return int(self.offsets[-1] - self.offsets[0]) if len(self.offsets) else 0

    @property
    def isp_counts(self) -> list:
        return [s.isp_count for s in self.shards]

    @property
    def total_isps(self) -> int:
        return sum(self.isp_counts)

    @property
    def value_dtype(self):
        if getattr(self, "_file_src", None) is not None:
            return self._file_src["dtype"]
        if self._source is not None and self._source._values is not None and self.perm is not None:
            return self._source._values.dtype
        # built without its permutation: host views come from the fp32 device
        # copy, so that is the value type a host view or a saved file carries
        return np.dtype(np.float32)

    @property
    def byte_size(self) -> int:
        return self.nnz * (len(self.shape) * 8 + np.dtype(self.value_dtype).itemsize)

    @property
    def device_bytes(self) -> int:
        return self.nnz * 4 * (len(self.shape) + 1)

    # -------------------------------------------------------- host views
    def order(self) -> np.ndarray:
        """The stable permutation (== argsort(c_mode, kind="stable"))."""
        if self.perm is None:
            raise ValueError("plan was built with keep_permutation=False")
        return self.perm.cpu().numpy().astype(np.int64)

    def _file_view(self, what):
        """Host views of a plan loaded from a cache file: memory-mapped from
        the file itself (exact stored values, no HBM round trip)."""
        f = self._file_src
        if what == "idx":
            return np.memmap(f["path"], dtype=INDEX_DTYPE, mode="r", offset=f["idx_off"],
                             shape=(f["nnz"], f["nmodes"]))
        return np.memmap(f["path"], dtype=f["dtype"], mode="r", offset=f["val_off"], shape=(f["nnz"],))

    @property
    def _indices(self) -> np.ndarray:
        if self._host_idx is None and getattr(self, "_file_src", None) is not None and self.layout == "flycoo":
            self._host_idx = np.asarray(self._file_view("idx"))
        if self._host_idx is None:
            src = self._source
            if src is not None and src._indices is not None and self.perm is not None:
                self._host_idx = src._indices[self.order()]
            else:
                import torch
                if self.coords is None:
                    raise ValueError("cells plan: host views need the source tensor and the permutation")
                arr = torch.stack(self.coords, 1).cpu().numpy().astype(INDEX_DTYPE)
                self._host_idx = self._to_plan_order(arr)
            self._host_idx.setflags(write=False)
        return self._host_idx

    @property
    def _values(self) -> np.ndarray:
        if self._host_vals is None and getattr(self, "_file_src", None) is not None and self.layout == "flycoo":
            self._host_vals = np.asarray(self._file_view("val"))
        if self._host_vals is None:
            src = self._source
            if src is not None and src._values is not None and self.perm is not None:
                self._host_vals = src._values[self.order()]
            else:
                if self.vals is None:
                    raise ValueError("cells plan: host views need the source tensor and the permutation")
                self._host_vals = self._to_plan_order(self.vals.cpu().numpy())
            self._host_vals.setflags(write=False)
        return self._host_vals

    def _to_plan_order(self, arr):
        if self.layout in ("flycoo", "host", "cells"):  # cells: the plan-order arrays are untouched
            return arr
        if getattr(self, "exec_perm", None) is None:
            if self.layout == "cells":
                raise ValueError("cells plan: host views need the source tensor and the permutation")
            raise ValueError("blocked plan built without its permutation: host views unavailable")
        out = np.empty_like(arr)
        out[self.exec_perm.cpu().numpy().astype(np.int64)] = arr
        return out

    def to_blocked(self, shifts, order=None):
        """Reorder the device arrays IN PLACE into the L2-blocked execution
        layout: inside every shard, nonzeros are grouped by the blocks
        (c_w >> shifts[w]) of the blocked modes and stay sorted by c_d inside
        each group (stable sort by [shard | blocks]).  ``shifts[mode] >= 0``
        also cuts the OUTPUT rows into blocks, so a run of groups shares one
        L2-resident output block.  ``order`` = blocked modes by key
        significance (default: the output mode first, then the input modes
        ascending): the work queue runs groups in that order, so the last
        mode's block changes fastest.  Shard offsets are unchanged; the
        host-visible plan (``_indices``, ``_values``, ISPs) keeps the
        reference order (it is derived from the source tensor + order)."""
        import torch

        if self.layout != "flycoo":
            raise ValueError("plan is already in a blocked layout")
        n = len(self.shape)
        shifts = [int(x) for x in shifts]
        if len(shifts) != n:
            raise ValueError("need one shift per mode")
        if all(x < 0 for x in shifts):
            return self
        if order is None:
            order = ([self.mode] if shifts[self.mode] >= 0 else []) + [w for w in range(n) if w != self.mode]
        order = [int(w) for w in order if shifts[int(w)] >= 0]
        if sorted(order) != [w for w in range(n) if shifts[w] >= 0]:
            raise ValueError("order must list every blocked mode once")
        widths = [0] * n
        for w in range(n):
            if shifts[w] >= 0:
                widths[w] = max(1, _key_bits(-(-self.shape[w] // (1 << shifts[w]))))
        k = self.shard_count
        shard_bits = max(1, _key_bits(k))
        total_bits = shard_bits + sum(widths)
        if total_bits > 32:
            raise ValueError(f"blocked key needs {total_bits} > 32 bits")
        sorted_keys = self._reorder_by_key([(self.coords[w], shifts[w], widths[w]) for w in order], shard_bits)
        dev = self.vals.device
        stream = torch.cuda.current_stream(dev).cuda_stream
        # group sizes: histogram of the sorted keys (bins = 2^total_bits)
        counts = torch.empty(1 << total_bits, dtype=torch.int64, device=dev)
        _lib.call("skrp_histogram", sorted_keys.data_ptr(), self.nnz, 1 << total_bits, counts.data_ptr(), stream)
        del sorted_keys
        c = counts.cpu().numpy()
        per_shard = 1 << (total_bits - shard_bits)
        self.groups = []
        for j in range(k):
            cnt = c[j * per_shard:(j + 1) * per_shard]
            ends = self.offsets[j] + np.cumsum(cnt)
            begins = ends - cnt
            keep = cnt > 0
            gkey = np.arange(per_shard, dtype=np.int64)[keep]  # block-tuple id of each group
            self.groups.append(np.stack([begins[keep], ends[keep], gkey], axis=1).astype(np.int64))
        self.layout = "blocked"
        self.block_shifts = shifts
        self.block_order = order
        self._exec_cache.clear()
        torch.cuda.current_stream(dev).synchronize()
        return self

    def _reorder_by_key(self, parts, shard_bits, need_keys=True, seg_cap=1 << 29):
        """Stable-sort the device arrays IN PLACE by [shard | parts...] (parts:
        (coordinate array, shift, width) in key order); returns the sorted keys.
        Keeps ``exec_perm`` (device position -> plan position) when the plan
        keeps its permutation (host views).  ``need_keys=False``: the keys
        never reorder across shards, so runs of consecutive shards of at most
        ``seg_cap`` nonzeros (or one larger shard) are sorted one at a time --
        temporaries scale with the run, not the plan (full-size cfg3 sorts
        beside its source tensor) -- and nothing is returned."""
        import torch

        nnz = self.nnz
        dev = self.vals.device
        stream = torch.cuda.current_stream(dev).cuda_stream
        total_bits = shard_bits + sum(p[2] for p in parts)
        if need_keys or nnz <= seg_cap:
            segs = [(0, self.shard_count)]
        else:
            segs, j0 = [], 0
            while j0 < self.shard_count:
                j1 = j0 + 1
                while j1 < self.shard_count and self.offsets[j1 + 1] - self.offsets[j0] <= seg_cap:
                    j1 += 1
                segs.append((j0, j1))
                j0 = j1
        keep_perm = self.perm is not None
        full_perm = torch.empty(nnz, dtype=torch.int32, device=dev) if keep_perm and len(segs) > 1 else None
        sorted_keys = None
        for j0, j1 in segs:
            e0, e1 = int(self.offsets[j0]), int(self.offsets[j1])
            n = e1 - e0
            if n == 0:
                continue
            starts = torch.from_numpy(np.ascontiguousarray(self.offsets[j0:j1 + 1] - e0)).to(dev)
            keys = torch.empty(n, dtype=torch.int32, device=dev)
            cptr = (_lib.vp * len(parts))(*[p[0][e0:].data_ptr() for p in parts])
            sh = np.ascontiguousarray([p[1] for p in parts], dtype=np.int32)
            wd = np.ascontiguousarray([p[2] for p in parts], dtype=np.int32)
            _lib.call("skrp_block_keys", cptr, len(parts), sh.ctypes.data, wd.ctypes.data, starts.data_ptr(),
                      j1 - j0, shard_bits, n, keys.data_ptr(), stream)
            sk = torch.empty_like(keys)
            perm = torch.empty_like(keys)
            ws_bytes = _lib.lib().skrp_sort_workspace_bytes(n, total_bits)
            ws = torch.empty(max(int(ws_bytes), 16), dtype=torch.uint8, device=dev)
            _lib.call("skrp_stable_sort_by_key", keys.data_ptr(), n, total_bits, sk.data_ptr(), perm.data_ptr(),
                      ws.data_ptr(), ws_bytes, stream)
            del ws, keys
            if not need_keys:
                del sk
                sk = None
            for w in range(len(self.shape)):
                out = torch.empty(n, dtype=self.coords[w].dtype, device=dev)
                _lib.call("skrp_gather_u32", self.coords[w][e0:].data_ptr(), perm.data_ptr(), n, out.data_ptr(),
                          stream)
                if n == nnz:
                    self.coords[w] = out
                else:
                    self.coords[w][e0:e1].copy_(out)
                del out
            out = torch.empty(n, dtype=self.vals.dtype, device=dev)
            _lib.call("skrp_gather_u32", self.vals[e0:].data_ptr(), perm.data_ptr(), n, out.data_ptr(), stream)
            if n == nnz:
                self.vals = out
            else:
                self.vals[e0:e1].copy_(out)
            del out
            if full_perm is not None:
                full_perm[e0:e1] = perm + e0
            elif keep_perm:
                full_perm = perm  # one segment covering the plan
            sorted_keys = sk
        # device position i holds plan-order element exec_perm[i] (kept only when
        # the plan keeps its permutation, i.e. host views are wanted)
        self.exec_perm = full_perm if keep_perm else None
        return sorted_keys

    def to_fibers(self, fiber_mode, seg_cap=1 << 29):
        """Reorder the device arrays IN PLACE into the FIBER execution layout:
        inside every shard the nonzeros are sorted by (c_d, c_f) (stable), so
        each run of one row is cut into FIBERS of one c_f -- the tile kernel
        gathers F_f's row once per fiber instead of once per nonzero (CSF-style
        reuse; cfg3: ~325 nonzeros per fiber in every mode).  Rows stay
        contiguous inside shards and tiles; shard offsets and host views
        (through the permutation) are unchanged.  Sorted shard run by shard
        run: the temporaries scale with a run, not the plan."""
        import torch

        if self.layout != "flycoo":
            raise ValueError("plan is already in a reordered layout")
        n, d, f = len(self.shape), self.mode, int(fiber_mode)
        if not (0 <= f < n) or f == d:
            raise ValueError("fiber_mode must be an input mode")
        shard_bits = max(1, _key_bits(self.shard_count))
        rb, fb = max(1, _key_bits(self.shape[d])), max(1, _key_bits(self.shape[f]))
        if shard_bits + rb + fb > 32:
            raise ValueError(f"fiber key needs {shard_bits + rb + fb} > 32 bits")
        self._reorder_by_key([(self.coords[d], 0, rb), (self.coords[f], 0, fb)], shard_bits, need_keys=False,
                             seg_cap=seg_cap)
        self.layout = "fibers"
        self.fiber_mode = f
        self.groups = None
        self.block_shifts = None
        self._exec_cache.clear()
        torch.cuda.current_stream(self.vals.device).synchronize()
        return self

    def to_panels(self, slab_shift, shifts, warps, order=None, sweep=None):
        """Reorder the device arrays IN PLACE into the PANEL execution layout
        of the output-stationary kernel (csrc/mttkrp_panel.cuh): key =
        [shard | slab (c_d >> slab_shift) | input blocks (c_w >> shifts[w], in
        ``order``) | warp stripe ((c_d >> stripe_shift) mod warps)].  Rows stay
        sorted inside every (slab, group, stripe) range.  Builds the item
        table: one ITEM per (shard, slab) intersection with its row range and
        groups*warps+1 element offsets (``self.panel``).  Shard offsets and
        the host-visible plan are unchanged, as in to_blocked."""
        import torch

        if self.layout != "flycoo":
            raise ValueError("plan is already in a reordered layout")
        n, d = len(self.shape), self.mode
        shifts = [int(x) for x in shifts]
        if len(shifts) != n or shifts[d] >= 0:
            raise ValueError("need one shift per mode (-1 = unblocked), none for the output mode")
        if warps < 1 or warps & (warps - 1) or (1 << slab_shift) < warps:
            raise ValueError("warps must be a power of two <= slab rows")
        if order is None:
            order = [w for w in range(n) if w != d]
        order = [int(w) for w in order if w != d and shifts[int(w)] >= 0]
        stripe_bits = _key_bits(warps)
        stripe_shift = slab_shift - stripe_bits
        slab_w = max(1, _key_bits(-(-self.shape[d] // (1 << slab_shift))))
        in_w = [max(1, _key_bits(-(-self.shape[w] // (1 << shifts[w])))) for w in order]
        parts = ([(self.coords[d], slab_shift, slab_w)] + [(self.coords[w], shifts[w], b) for w, b in zip(order, in_w)]
                 + ([(self.coords[d], stripe_shift, stripe_bits)] if stripe_bits else []))
        # sweep = {mode: shift}: sub-blocks sorted INSIDE every (group, stripe)
        # range, so all CTAs walk that input in ascending order together
        sweep = dict(sweep or {})
        sweep_w = [max(1, _key_bits(-(-self.shape[w] // (1 << sft)))) for w, sft in sweep.items()]
        parts += [(self.coords[w], sft, b) for (w, sft), b in zip(sweep.items(), sweep_w)]
        sweep_bits = sum(sweep_w)
        k = self.shard_count
        shard_bits = max(1, _key_bits(k))
        group_bits = sum(in_w)
        total_bits = shard_bits + slab_w + group_bits + stripe_bits + sweep_bits
        if total_bits > 31:
            raise ValueError(f"panel key needs {total_bits} > 31 bits (use larger slabs or blocks)")
        dev = self.vals.device
        sorted_keys = self._reorder_by_key(parts, shard_bits)
        # items: (shard, slab) intersections, in row order
        rows, bases = [], []
        for j, sh in enumerate(self.shards):
            lo, hi = sh.index_range
            if hi <= lo:
                continue
            for s_ in range(lo >> slab_shift, ((hi - 1) >> slab_shift) + 1):
                rows.append((max(lo, s_ << slab_shift), min(hi, (s_ + 1) << slab_shift)))
                bases.append(((j << slab_w) | s_) << (group_bits + stripe_bits + sweep_bits))
        groups = 1 << group_bits
        per = groups * warps
        base = torch.tensor(bases, dtype=torch.int64, device=dev)
        q = (base[:, None] + (torch.arange(per + 1, dtype=torch.int64, device=dev)[None, :] << sweep_bits))
        q[:, per] = base + (1 << (group_bits + stripe_bits + sweep_bits))  # end = the next slab's first key
        offs = torch.searchsorted(sorted_keys, q.to(torch.int32).reshape(-1)).reshape(len(bases), per + 1)
        del sorted_keys
        self.panel = {
            "slab_shift": slab_shift, "warps": warps, "groups": groups, "order": order,
            "item_rows": np.asarray(rows, dtype=np.int64).reshape(-1, 2),
            "item_shard": np.asarray([b >> (group_bits + stripe_bits + sweep_bits + slab_w) for b in bases],
                                     dtype=np.int64),
            "item_offsets": offs.to(torch.int64).contiguous(),
        }
        self.groups = None
        self.layout = "panel"
        self.block_shifts = shifts
        self.block_order = order
        self._exec_cache.clear()
        torch.cuda.current_stream(dev).synchronize()
        return self

    def to_cells(self, shard_ids, params, keep_arrays=True):
        """Build the CELLS execution layout of the GPU-synchronous 2-D blocked
        kernel (csrc/mttkrp_cells.cu) for the shards `shard_ids` (consecutive:
        one output row range and one element range).

        A stable GPU sort by [stripe | cell] (stripe = the rows one warp owns;
        cell = the snake-ordered (outer block, inner block) pair) makes every
        (stripe, cell) SEGMENT contiguous with rows ascending; every run of
        one row inside a segment goes whole to the least-loaded slot of the
        warp (skrp_cell_assign), and the nonzeros are written as 16-byte
        entries {cell | panel row offset, outer index, inner index, value},
        each segment's slots interleaved and padded to equal length with skip
        entries of that cell, so all slots of a warp cross every cell boundary
        in the same step.  ``params``: dict with rank, stripe_rows, ctas,
        outer_mode, inner_mode, outer_shift, inner_shift, variant, warps, stage
        (engine.choose_cells).
        ``keep_arrays=False`` frees the plan-order device arrays (the entries
        replace them; host views then need the source tensor + permutation)."""
        import torch

        if self.layout != "flycoo":
            raise ValueError("plan is already in a reordered layout")
        if len(self.shape) != 3:
            raise ValueError("the cells layout covers 3-mode tensors")
        ids = sorted(int(j) for j in shard_ids)
        if not ids or ids != list(range(ids[0], ids[-1] + 1)):
            raise ValueError("the cells layout needs a run of consecutive shards")
        d = self.mode
        lo, hi = int(self.bounds[ids[0]]), int(self.bounds[ids[-1] + 1])
        e0, e1 = int(self.offsets[ids[0]]), int(self.offsets[ids[-1] + 1])
        n = e1 - e0
        p = dict(params)
        rank = int(p["rank"])
        if rank not in (16, 32, 64):
            raise ValueError("the cells layout needs R in {16, 32, 64}")
        slots = 128 // rank
        sr, om, im = int(p["stripe_rows"]), int(p["outer_mode"]), int(p["inner_mode"])
        so, si = int(p["outer_shift"]), int(p["inner_shift"])
        nout = -(-self.shape[om] // (1 << so))
        nin = -(-self.shape[im] // (1 << si))
        cells = nout * nin
        rows = hi - lo
        stripes = -(-rows // sr) if rows > 0 else 0
        nseg = stripes * cells
        stripe_bits = _key_bits(max(stripes, 1))
        cell_bits = _key_bits(cells)
        if cells > 1024 or stripe_bits + cell_bits > 31 or sr * rank * 4 >= (1 << 20):
            raise ValueError(f"cells layout key too wide ({stripes} stripes, {cells} cells)")
        dev = self.vals.device
        stream = torch.cuda.current_stream(dev).cuda_stream
        rowc, co, ci = self.coords[d], self.coords[om], self.coords[im]
        seg_len = torch.zeros(max(nseg, 1), dtype=torch.int32, device=dev)
        sk = perm = slot_t = None
        if n > 0:
            keys = torch.empty(n, dtype=torch.int32, device=dev)
            _lib.call("skrp_cell_keys", rowc[e0:].data_ptr(), co[e0:].data_ptr(), ci[e0:].data_ptr(), n, lo, sr, so,
                      si, nin, cell_bits, keys.data_ptr(), stream)
            sk = torch.empty_like(keys)
            perm = torch.empty_like(keys)
            bits = stripe_bits + cell_bits
            ws_bytes = _lib.lib().skrp_sort_workspace_bytes(n, bits)
            ws = torch.empty(max(int(ws_bytes), 16), dtype=torch.uint8, device=dev)
            _lib.call("skrp_stable_sort_by_key", keys.data_ptr(), n, bits, sk.data_ptr(), perm.data_ptr(),
                      ws.data_ptr(), ws_bytes, stream)
            del ws
            rows_sorted = keys  # reuse
            _lib.call("skrp_gather_u32", rowc[e0:].data_ptr(), perm.data_ptr(), n, rows_sorted.data_ptr(), stream)
            g = torch.arange(nseg + 1, dtype=torch.int64, device=dev)
            q = ((g // cells) << cell_bits) + g % cells
            q[-1] = (1 << 31) - 1
            seg_off = torch.searchsorted(sk, q.to(torch.int32)).to(torch.int64)
            seg_off[-1] = n
            del g, q
            slot_t = torch.empty(n, dtype=torch.int32, device=dev)
            _lib.call("skrp_cell_assign", seg_off.data_ptr(), nseg, rows_sorted.data_ptr(), slots, slot_t.data_ptr(),
                      seg_len.data_ptr(), stream)
            del rows_sorted, keys, seg_off
        # segment g of stripe s: [seg_base[g], + slots*seg_len[g]); every stripe
        # rounded up to whole pipeline stages (params["stage"] steps); skip
        # entries at the end of the array (the kernel reads ahead)
        seg_n = seg_len[:nseg].to(torch.int64).reshape(stripes, cells) * slots
        tot = seg_n.sum(dim=1)
        unit = int(p["stage"]) * slots
        tot = (tot + unit - 1) // unit * unit
        base = torch.zeros(stripes + 1, dtype=torch.int64, device=dev)
        if stripes:
            base[1:] = torch.cumsum(tot, 0)
        seg_base = (base[:-1, None] + torch.cumsum(seg_n, 1) - seg_n).reshape(-1).contiguous()
        num = int(base[-1].item())
        total = num + CELL_TAIL_STAGES * unit
        entries = torch.empty(total * 4, dtype=torch.int32, device=dev)
        _lib.call("skrp_cell_entries", _lib.ptr(sk), _lib.ptr(perm), _lib.ptr(slot_t), n, cell_bits, cells,
                  seg_base.data_ptr(), seg_len.data_ptr(), nseg, slots, rowc[e0:].data_ptr(), co[e0:].data_ptr(),
                  ci[e0:].data_ptr(), self.vals[e0:].data_ptr(), lo, sr, rank * 4, entries.data_ptr(), total, stream)
        del sk, perm, slot_t, seg_base, seg_len, seg_n
        torch.cuda.current_stream(dev).synchronize()
        p.update({"rank": rank, "row_lo": lo, "rows": rows, "stripes": stripes, "stripe_rows": sr,
                  "slots": slots, "inner_blocks": nin, "outer_blocks": nout, "cells": cells,
                  "shard_ids": tuple(ids), "stripe_offsets": base, "entries": entries, "num_entries": num,
                  "elements": (e0, e1), "pad_entries": num - n})
        self.cells = p
        self.groups = None
        self.layout = "cells"
        self.block_shifts = None
        self.exec_perm = None  # host views come from the source tensor + permutation
        if not keep_arrays:
            self.coords = None
            self.vals = None
        self._exec_cache.clear()
        return self

    def to_host(self, pinned=True):
        """Out-of-core execution (the B200 form of the
        reference's per-mode staging, engine.py:103-105): move the sorted
        arrays to PINNED host memory and free their HBM; the stream executor
        (engine._StreamExec) copies them back chunk by chunk, overlapped with
        the kernel, every time the mode runs.  Plan order only.
        ``pinned=False`` parks the arrays in pageable memory of their exact
        size (a build parking finished plans; see to_device) -- in any
        execution layout except cells, which to_device restores."""
        import torch

        if pinned and self.layout != "flycoo":
            raise ValueError("out-of-core execution streams the plan (FLYCOO) order")
        if self.layout in ("host", "cells"):
            raise ValueError(f"cannot park a plan in the {self.layout!r} layout")
        self._parked_layout = self.layout if not pinned else "flycoo"

        def pin(t):
            if not pinned:
                return t.cpu()
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
            h.copy_(t)
            return h

        self.coords = [pin(c) for c in self.coords]
        self.vals = pin(self.vals)
        if self.perm is not None:
            self.perm = self.perm.cpu()
        if getattr(self, "exec_perm", None) is not None:
            self.exec_perm = self.exec_perm.cpu()
        self.layout = "host"
        self._exec_cache.clear()
        return self

    def to_device(self, device=None):
        """Inverse of to_host: the pinned arrays back into HBM (plan order).
        Lets a build park finished plans on the host while the next mode's
        sort needs the HBM (full-size cfg3 on one GPU, bench.py)."""
        import torch

        if self.layout != "host":
            raise ValueError("plan is not host-resident")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.coords = [c.to(dev, non_blocking=True) for c in self.coords]
        self.vals = self.vals.to(dev, non_blocking=True)
        if self.perm is not None:
            self.perm = self.perm.to(dev)
        if getattr(self, "exec_perm", None) is not None and not self.exec_perm.is_cuda:
            self.exec_perm = self.exec_perm.to(dev)
        torch.cuda.current_stream(dev).synchronize()
        self.layout = getattr(self, "_parked_layout", "flycoo")
        self._exec_cache.clear()
        return self

    def release_device(self):
        self.coords = self.vals = self.perm = None
        self.cells = None
        self._exec_cache.clear()

    def __repr__(self):
        return (f"ModePartitionPlan(mode={self.mode}, shape={self.shape}, shards={self.shard_count}, "
                f"nnz={self.nnz}, strategy={self.strategy!r})")


def _key_bits(n: int) -> int:
    bits = 0
    while (1 << bits) < n:
        bits += 1
    return bits


def _shard_bounds(counts_host_fn, num_indices, k, strategy):
    bounds = np.empty(k + 1, dtype=np.int64)
    if strategy == "equal-index":
        _lib.call("skrp_equal_index_bounds", num_indices, k, _lib.ptr(bounds))
    else:
        counts = np.ascontiguousarray(counts_host_fn(), dtype=np.int64)
        _lib.call("skrp_nnz_balanced_bounds", _lib.ptr(counts), num_indices, k, _lib.ptr(bounds))
    return bounds


def build_mode_plan(tensor: SparseTensorCOO, mode: int, cfg: PartitionConfig, *,
                    keep_permutation: bool = True) -> ModePartitionPlan:
    """GPU build of the mode-`mode` plan (partition.py:196-257 semantics)."""
    import torch

    if not 0 <= mode < tensor.num_modes:
        raise ValueError(f"mode {mode} out of range")
    t0 = time.perf_counter()
    num_indices = tensor.shape[mode]
    k = cfg.devices * cfg.oversubscription
    if k > num_indices:
        warnings.warn(f"mode {mode}: requested {k} shards exceeds {num_indices} indices; clamping",
                      RuntimeWarning, stacklevel=2)
        k = num_indices
    coords, vals = tensor.device_arrays()
    nnz = tensor.nnz
    if nnz >= 2 ** 32:
        raise ValueError("per-GPU plan build needs nnz < 2^32 (shard the tensor across GPUs)")
    dev = vals.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    bits = _key_bits(num_indices)

    sorted_coords = [None] * tensor.num_modes
    key_sorted = torch.empty(nnz, dtype=torch.int32, device=dev)
    perm = torch.empty(nnz, dtype=torch.int32, device=dev)
    ws_bytes = _lib.lib().skrp_sort_workspace_bytes(nnz, bits)
    ws = torch.empty(max(int(ws_bytes), 16), dtype=torch.uint8, device=dev)
    _lib.call("skrp_stable_sort_by_key", _lib.ptr(coords[mode]), nnz, bits, _lib.ptr(key_sorted),
              _lib.ptr(perm), _lib.ptr(ws), ws_bytes, stream)
    del ws
    sorted_coords[mode] = key_sorted
    for w in range(tensor.num_modes):
        if w != mode:
            out = torch.empty(nnz, dtype=torch.int32, device=dev)
            _lib.call("skrp_gather_u32", _lib.ptr(coords[w]), _lib.ptr(perm), nnz, _lib.ptr(out), stream)
            sorted_coords[w] = out
    svals = torch.empty(nnz, dtype=torch.float32, device=dev)
    _lib.call("skrp_gather_u32", _lib.ptr(vals), _lib.ptr(perm), nnz, _lib.ptr(svals), stream)

    # bincount + exclusive prefix on the GPU; offsets = prefix[bounds]
    counts = torch.empty(num_indices, dtype=torch.int64, device=dev)
    _lib.call("skrp_histogram", _lib.ptr(coords[mode]), nnz, num_indices, _lib.ptr(counts), stream)
    prefix = torch.empty(num_indices + 1, dtype=torch.int64, device=dev)
    sws_bytes = _lib.lib().skrp_scan_workspace_bytes(num_indices)
    sws = torch.empty(max(int(sws_bytes), 16), dtype=torch.uint8, device=dev)
    _lib.call("skrp_exclusive_scan_i64", _lib.ptr(counts), num_indices, _lib.ptr(prefix), _lib.ptr(sws),
              sws_bytes, stream)
    bounds = _shard_bounds(lambda: counts.cpu().numpy(), num_indices, k, cfg.strategy)
    offsets = prefix[torch.from_numpy(bounds).to(dev)].cpu().numpy()
    torch.cuda.current_stream(dev).synchronize()
    plan = ModePartitionPlan(
        mode, tensor.shape, cfg.strategy, cfg.isp_capacity, tensor.name, sorted_coords, svals,
        perm if keep_permutation else None, bounds, offsets, source=tensor,
        build_time=time.perf_counter() - t0)
    return plan


def build_all_plans(tensor: SparseTensorCOO, cfg: PartitionConfig, *,
                    keep_permutation: bool = True) -> list:
    """One independent plan per mode (partition.py:260-262)."""
    return [build_mode_plan(tensor, d, cfg, keep_permutation=keep_permutation)
            for d in range(tensor.num_modes)]


# ------------------------------------------------------------- work tables


def tile_table(plan: ModePartitionPlan, shard_ids, tile_nnz: int, group_key=None, clip=None):
    """[start, end) element ranges of the TILES of the given shards, in order.

    A tile is a slice of one ISP of at most ``tile_nnz`` elements; tiles
    never straddle an ISP (hence never a shard).  Also returns, per shard,
    its number of tiles (for the carry-tree chunk tables).  ``clip`` =
    (e0, e1) keeps only the parts of tiles inside that element range (the
    element-split placement, engine.assign_elements).
    """
    cap = plan.isp_capacity
    step = max(1, min(tile_nnz, cap))
    starts, stops, per_shard = [], [], []
    blocked = getattr(plan, "layout", "flycoo") == "blocked"
    for j in shard_ids:
        sh = plan.shards[j]
        n = sh.nnz
        if n == 0:
            per_shard.append(0)
            continue
        if blocked:
            # blocked layout: tiles slice the shard's block groups instead
            g = plan.groups[j]
            if group_key is not None:
                g = g[g[:, 2] == group_key]
                if len(g) == 0:
                    per_shard.append(0)
                    continue
            isp0 = g[:, 0] - sh.start
            isp1 = g[:, 1] - sh.start
        else:
            isp0 = np.arange(0, n, cap, dtype=np.int64)
            isp1 = np.minimum(isp0 + cap, n)
        pieces = (isp1 - isp0 + step - 1) // step
        total = int(pieces.sum())
        first = np.repeat(np.cumsum(pieces) - pieces, pieces)
        s = np.repeat(isp0, pieces) + (np.arange(total, dtype=np.int64) - first) * step
        e = np.minimum(s + step, np.repeat(isp1, pieces))
        s, e = s + sh.start, e + sh.start
        if clip is not None:
            s, e = np.maximum(s, clip[0]), np.minimum(e, clip[1])
            keep = e > s
            s, e = s[keep], e[keep]
            total = int(keep.sum())
        starts.append(s)
        stops.append(e)
        per_shard.append(total)
    if starts:
        s = np.concatenate(starts)
        e = np.concatenate(stops)
    else:
        s = e = np.zeros(0, dtype=np.int64)
    if blocked and len(s):
        # work-queue order: block tuple major, shard minor -- every shard's
        # group of the same factor blocks runs back to back, so a block pair
        # is loaded into L2 once per device instead of once per shard
        gkeys = []
        for j in shard_ids:
            sh = plan.shards[j]
            if sh.nnz == 0:
                continue
            g = plan.groups[j]
            if group_key is not None:
                g = g[g[:, 2] == group_key]
            glen = ((g[:, 1] - g[:, 0]) + step - 1) // step
            gkeys.append(np.repeat(g[:, 2], glen))
        gk = np.concatenate(gkeys)
        order = np.argsort(gk, kind="stable")
        s, e = s[order], e[order]
    tiles = np.empty(2 * len(s), dtype=np.int64)
    tiles[0::2] = s
    tiles[1::2] = e
    return tiles, np.asarray(per_shard, dtype=np.int64)


def carry_levels(tiles_per_shard: np.ndarray, chunk: int = 256):
    """Chunk tables of the fixed carry-reduction tree.

    Level 1 has 2 entries per tile; a shard's entries are cut into chunks of
    <= ``chunk`` entries (never crossing shards).  A shard whose entries fit
    one chunk is FINAL at that level (its rows are complete); otherwise each
    chunk emits a head and a tail partial to the next level.  The tree is a
    function of the shard's tile count only, so results do not depend on
    which device ran the shard.
    Returns a list of (chunks (2*n int64), final_flags (n uint8)).
    """
    levels = []
    counts = 2 * np.asarray(tiles_per_shard, dtype=np.int64)
    base = np.concatenate([[0], np.cumsum(counts)[:-1]]) if len(counts) else counts
    while True:
        live = counts > 0
        if not live.any():
            break
        nch = np.where(live, (counts + chunk - 1) // chunk, 0)
        total = int(nch.sum())
        first = np.repeat(np.cumsum(nch) - nch, nch)
        local = np.arange(total, dtype=np.int64) - first
        c0 = np.repeat(base, nch) + local * chunk
        c1 = np.minimum(c0 + chunk, np.repeat(base + counts, nch))
        final = np.repeat(nch <= 1, nch).astype(np.uint8)
        table = np.empty(2 * total, dtype=np.int64)
        table[0::2] = c0
        table[1::2] = c1
        levels.append((table, final))
        chunk_first = np.cumsum(nch) - nch  # global chunk index of each shard's first chunk
        counts = np.where(nch > 1, 2 * nch, 0)
        base = 2 * chunk_first
    return levels


# ------------------------------------------------------------- plan cache
# Format v1 of partition.py:265-379 (reference), byte-compatible: magic,
# version, value tag, strategy tag, mode, shape, nnz, capacity, build time,
# shard table, u64 indices, values, CRC32.

_VALUE_TAG = {np.dtype(np.float64): 8, np.dtype(np.float32): 4}
_TAG_VALUE = {v: k for k, v in _VALUE_TAG.items()}


_CRC_SUB = 1 << 12        # CRC sub-chunk (bytes) computed per GPU thread
_IO_RECORDS = 1 << 22     # index records / values per streamed chunk


def _header(plan) -> bytes:
    import struct

    body = bytearray()
    body += struct.pack("<I", PLAN_VERSION)
    body += struct.pack("<B", _VALUE_TAG[np.dtype(plan.value_dtype)])
    body += struct.pack("<B", STRATEGIES.index(plan.strategy))
    body += struct.pack("<I", plan.mode)
    body += struct.pack("<I", len(plan.shape))
    body += struct.pack(f"<{len(plan.shape)}Q", *plan.shape)
    body += struct.pack("<QQd", plan.nnz, plan.isp_capacity, plan.build_time)
    body += struct.pack("<I", plan.shard_count)
    name = plan.name.encode("utf-8")
    body += struct.pack("<I", len(name)) + name
    for sh in plan.shards:
        body += struct.pack("<QQQ", sh.index_range[0], sh.index_range[1], sh.nnz)
    return bytes(body)


def _crc_device(buf, n, crc, stream):
    """zlib.crc32 continued over the first n bytes of device buffer `buf`:
    per-thread raw CRCs of 4-KB sub-chunks on the GPU, folded on the host."""
    import ctypes

    import torch

    if n == 0:
        return crc
    cnt = -(-n // _CRC_SUB)
    raws = torch.empty(cnt, dtype=torch.int32, device=buf.device)
    _lib.call("skrp_crc32_chunks", buf.data_ptr(), n, _CRC_SUB, raws.data_ptr(), stream)
    h = raws.cpu().numpy()
    out = ctypes.c_uint32()
    _lib.call("skrp_crc32_fold_host", h.ctypes.data, cnt, _CRC_SUB, n, crc & 0xFFFFFFFF, ctypes.byref(out))
    return out.value


def save_plan(plan: ModePartitionPlan, path):
    """Write the reference's v1 plan file (partition.py:270-292), byte-for-byte
    the same layout.  GPU-direct: the u64 AoS index section is packed from the
    device coordinates and checksummed on the GPU, then streamed to disk;
    values come from their exact source (host f64 or the device f32 copy)."""
    import struct
    import zlib

    import torch

    if plan.layout != "flycoo" or plan.coords is None:
        return _save_plan_host(plan, path)
    dev = plan.vals.device
    stream = torch.cuda.current_stream(dev).cuda_stream
    nm, nnz = len(plan.shape), plan.nnz
    head = _header(plan)
    crc = zlib.crc32(head)
    dtype = np.dtype(plan.value_dtype)
    with open(path, "wb") as fh:
        fh.write(PLAN_MAGIC)
        fh.write(head)
        aos = torch.empty(min(nnz, _IO_RECORDS) * nm, dtype=torch.int64, device=dev)
        host = torch.empty(aos.numel(), dtype=torch.int64, pin_memory=True)
        for r0 in range(0, nnz, _IO_RECORDS):
            k = min(_IO_RECORDS, nnz - r0)
            cptr = (_lib.vp * nm)(*[c.data_ptr() + 4 * r0 for c in plan.coords])
            _lib.call("skrp_plan_pack_indices", cptr, k, nm, aos.data_ptr(), stream)
            crc = _crc_device(aos, k * nm * 8, crc, stream)
            host[:k * nm].copy_(aos[:k * nm])
            fh.write(host[:k * nm].numpy().tobytes())
        if dtype == np.float32 and getattr(plan, "_file_src", None) is None and (
                plan._source is None or plan._source._values is None):
            for r0 in range(0, nnz, _IO_RECORDS):
                k = min(_IO_RECORDS, nnz - r0)
                chunk = plan.vals[r0:r0 + k]
                crc = _crc_device(chunk, k * 4, crc, stream)
                fh.write(chunk.cpu().numpy().tobytes())
        else:  # exact stored dtype from the host source (f64 values never round-trip through fp32)
            vals = np.ascontiguousarray(plan._values, dtype=dtype)
            for r0 in range(0, nnz, _IO_RECORDS):
                b = vals[r0:r0 + _IO_RECORDS].tobytes()
                crc = zlib.crc32(b, crc)
                fh.write(b)
        fh.write(struct.pack("<I", crc & 0xFFFFFFFF))


def _save_plan_host(plan, path):
    import struct
    import zlib

    body = bytearray(_header(plan))
    body += np.ascontiguousarray(plan._indices, dtype=INDEX_DTYPE).tobytes()
    body += np.ascontiguousarray(plan._values, dtype=plan.value_dtype).tobytes()
    with open(path, "wb") as fh:
        fh.write(PLAN_MAGIC)
        fh.write(body)
        fh.write(struct.pack("<I", zlib.crc32(bytes(body))))


def _file_crc_host(path, size):
    import zlib

    crc = 0
    with open(path, "rb") as fh:
        fh.seek(len(PLAN_MAGIC))
        left = size - len(PLAN_MAGIC) - 4
        while left > 0:
            b = fh.read(min(left, 1 << 26))
            if not b:
                break
            crc = zlib.crc32(b, crc)
            left -= len(b)
    return crc & 0xFFFFFFFF


def load_plan(path, value_dtype=None, *, device=None) -> ModePartitionPlan:
    """Read a v1 plan file (partition.py:295-379: checksum, then version and
    value-type checks, same exceptions) straight into HBM.  GPU-direct: the
    index and value sections stream through a pinned buffer into device
    staging buffers where the GPU checksums them (4-KB sub-chunk CRCs folded
    on the host) and splits the u64 AoS records into per-mode u32 arrays;
    host views (_indices / _values) are memory-mapped from the file."""
    import os
    import struct

    import torch

    size = os.path.getsize(path)
    with open(path, "rb") as fh:
        head = fh.read(min(size, 1 << 22))
    if size < len(PLAN_MAGIC) + 4 or head[:len(PLAN_MAGIC)] != PLAN_MAGIC:
        raise PlanVersionError(f"{path}: not a plan cache file")
    with open(path, "rb") as fh:
        fh.seek(size - 4)
        (crc_stored,) = struct.unpack("<I", fh.read(4))
    body = head[len(PLAN_MAGIC):]
    pos = 0

    def take(fmt):
        nonlocal pos
        out = struct.unpack_from(fmt, body, pos)
        pos += struct.calcsize(fmt)
        return out

    def integrity_then(exc):
        # the reference checks the CRC before anything else
        if _file_crc_host(path, size) != crc_stored:
            raise PlanIntegrityError(f"{path}: checksum mismatch (truncated or corrupted)")
        raise exc

    try:
        (version,) = take("<I")
        (vtag,) = take("<B")
        (stag,) = take("<B")
        (mode,) = take("<I")
        (nmodes,) = take("<I")
        shape = take(f"<{nmodes}Q")
        nnz, capacity, build_time = take("<QQd")
        (shards,) = take("<I")
        (nlen,) = take("<I")
        name = body[pos:pos + nlen].decode("utf-8")
        pos += nlen
        table = np.array([take("<QQQ") for _ in range(shards)], dtype=np.int64).reshape(-1, 3)
    except (struct.error, UnicodeDecodeError, ValueError, MemoryError):
        integrity_then(PlanIntegrityError(f"{path}: checksum mismatch (truncated or corrupted)"))
    if version != PLAN_VERSION:
        integrity_then(PlanVersionError(f"{path}: plan version {version}, expected {PLAN_VERSION}"))
    if vtag not in _TAG_VALUE:
        integrity_then(PlanVersionError(f"{path}: unknown value-type tag {vtag}"))
    dtype = _TAG_VALUE[vtag]
    if value_dtype is not None and np.dtype(value_dtype) != dtype:
        integrity_then(PlanVersionError(f"{path}: plan stores {dtype} values, expected {np.dtype(value_dtype)}"))
    hdr_len = pos
    idx_off = len(PLAN_MAGIC) + hdr_len
    val_off = idx_off + nnz * nmodes * 8
    if val_off + nnz * dtype.itemsize + 4 != size or any(x >= 2 ** 32 for x in shape):
        integrity_then(PlanIntegrityError(f"{path}: checksum mismatch (truncated or corrupted)"))

    gpu = device or torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(gpu).cuda_stream
    import zlib

    crc = zlib.crc32(body[:hdr_len])
    coords = [torch.empty(nnz, dtype=torch.int32, device=gpu) for _ in range(nmodes)]
    dvals = torch.empty(nnz, dtype=torch.float32, device=gpu)
    rec = nmodes * 8
    k_max = max(1, min(nnz, _IO_RECORDS))
    pinned = torch.empty(k_max * max(rec, 8), dtype=torch.uint8, pin_memory=True)
    stage = torch.empty(k_max * max(rec, 8), dtype=torch.uint8, device=gpu)
    bad = torch.zeros(1, dtype=torch.int64, device=gpu)
    with open(path, "rb") as fh:
        fh.seek(idx_off)
        for r0 in range(0, nnz, _IO_RECORDS):
            k = min(_IO_RECORDS, nnz - r0)
            n = fh.readinto(pinned[:k * rec].numpy())
            stage[:n].copy_(pinned[:n], non_blocking=True)
            crc = _crc_device(stage, k * rec, crc, stream)
            cptr = (_lib.vp * nmodes)(*[c.data_ptr() + 4 * r0 for c in coords])
            _lib.call("skrp_plan_unpack_indices", stage.data_ptr(), k, nmodes, cptr, bad.data_ptr(), stream)
        for r0 in range(0, nnz, _IO_RECORDS):
            k = min(_IO_RECORDS, nnz - r0)
            n = fh.readinto(pinned[:k * dtype.itemsize].numpy())
            stage[:n].copy_(pinned[:n], non_blocking=True)
            crc = _crc_device(stage, k * dtype.itemsize, crc, stream)
            if dtype == np.float64:
                _lib.call("skrp_f64_to_f32", stage.data_ptr(), k, dvals.data_ptr() + 4 * r0, stream)
            else:
                dvals[r0:r0 + k].copy_(stage[:k * 4].view(torch.float32))
    if (crc & 0xFFFFFFFF) != crc_stored:
        raise PlanIntegrityError(f"{path}: checksum mismatch (truncated or corrupted)")
    if int(bad.item()):
        raise ValueError(f"{path}: indices >= 2^32 cannot live on the device")
    bounds = np.concatenate([table[:, 0], table[-1:, 1]]) if shards else np.zeros(1, dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(table[:, 2])]).astype(np.int64)
    plan = ModePartitionPlan(int(mode), tuple(int(x) for x in shape), STRATEGIES[stag], int(capacity), name,
                             coords, dvals, None, bounds, offsets, build_time=float(build_time))
    plan._file_src = {"path": os.fspath(path), "idx_off": idx_off, "val_off": val_off, "nnz": int(nnz),
                      "nmodes": int(nmodes), "dtype": dtype}
    return plan
