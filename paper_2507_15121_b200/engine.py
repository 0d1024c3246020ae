"""Multi-device MTTKRP execution on B200 (drop-in for shardkrp.engine).

Same public surface and semantics as the reference engine (engine.py:45-437):
``PlatformConfig``, ``DeviceState``, ``make_devices``, ``execute_shard``,
``mttkrp_mode``, ``mttkrp_all_modes``, ``measure_isolated_compute``,
``elementwise_compute`` -- plus ``mttkrp(tensor, factors, mode)``, the
per-mode call with ``dense_mttkrp_oracle``'s contract (reference.py:32-68).

What a "device" is: a logical owner of shards with its own factor replicas
and output buffer on a physical GPU (device_id mod #GPUs).  Compute is the
tile kernel (csrc/mttkrp.cu) over the device's shards: a device-side work
queue of ISP tiles claimed with atomics (the reference's worker pool,
engine.py:162-209), per-row register accumulation, and the deterministic-
reduce or atomic discipline for rows shared by two tiles.  Shards are placed
on devices by the host balancer ``assign_shards``: static round-robin
(engine.py:291-293) or "dynamic" -- a deterministic replay of the
reference's claim-next-shard queue (engine.py:267-277) with nnz as the cost,
i.e. greedy list scheduling in shard order.  After compute, owned rows are
all-gathered (collective.ring_all_gather in one process; NCCL broadcast of
owned row ranges across processes, see distributed.py) and, when chained,
become the mode's factor on every device (engine.py:350-352).

Data stays on the GPU between modes; results come back to the host (float64,
like the reference) only when asked (``as_numpy=True``, the default).
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .collective import FactorPartitionSet, TransferLedger, ring_all_gather
from .metrics import ModeMetrics, RunMetrics
from .partition import ModePartitionPlan, PartitionConfig, TensorShard, build_mode_plan, carry_levels, tile_table
from .tensor import FactorMatrix, NonzeroElement

ACCUMULATION_MODES = ("deterministic-reduce", "atomic")
# "contiguous" (B200 addition): each device gets one run of consecutive shards
# cut at the cumulative-nnz targets, so its output rows form ONE range and the
# inter-mode all-gather is one broadcast per device
# "split" (B200 addition): equal-NONZERO element ranges per
# device; the <= devices-1 rows cut by a range boundary (heavy rows included)
# are summed across devices -- perfect balance under any skew, at the price
# of a tiny cross-device reduction (one-process-per-GPU runner only)
SCHEDULING_MODES = ("dynamic", "static", "contiguous", "split")


@dataclass(frozen=True)
class PlatformConfig:
    devices: int = 1
    workers_per_device: int = 1
    column_width: int = 32
    rank: int = 32
    accumulation: str = "deterministic-reduce"
    scheduling: str = "dynamic"
    # B200 knobs (defaults keep the reference's fields and meaning intact)
    tile_nnz: int = 0           # nonzeros per work-queue tile (a slice of one ISP); 0 = auto
    kernel_variant: int = 0     # 0 = production kernel, 1 = generic scalar tile kernel (cross-check path)
    carry_chunk: int = 256      # carry-tree fan-in
    layout: str = "flycoo"      # "flycoo" (plan order), "blocked" (L2-blocked), "auto" (cost model)
    l2_budget_mb: int = 192     # L2 bytes the blocked layout plans on (B200-calibrated)
    max_blocks: int = 8         # blocks per input mode the layout search may use (B200-tuned)
    panel_l2_mb: int = -1       # panel layout: >= 0 cuts input modes to this L2 budget; -1 = blocked cost model
    slab_rows: int = 0          # panel layout: output rows per slab (0 = auto, see panel_smem_kb)
    panel_smem_kb: int = 64     # panel layout: shared memory for the output panel (auto slab size)
    panel_lockstep: bool = True  # panel layout: items in grid-synchronised rounds (uniform item sizes)
    stream_chunk_nnz: int = 1 << 27  # out-of-core plans: nonzeros per streamed chunk (2 device buffers)
    fused_allgather: bool = False  # N>1, panel layout: push finished rows into peers' outputs (CUDA IPC)
    fibers: bool = True         # auto layout: the fiber layout where (row, c_f) runs are long (3 modes, R = 32)
    cell_outer_mb: int = 32     # cells layout: outer input block (MB of factor rows)
    cell_inner_mb: int = 8      # cells layout: inner input block
    cell_lag: int = 0           # cells layout: cells a warp may run ahead of the slowest CTA (0 = free running:
                                #   measured 2-5 % faster on cfg2 -- every warp crosses the cells at the same rate)
    cell_variant: int = 1       # cells layout: kernel variant (warps per CTA, pipeline depth; see csrc/mttkrp_cells.cu)
    cell_keep_arrays: bool = True  # cells layout: keep the plan-order device arrays beside the entries

    def __post_init__(self):
        if self.devices < 1 or self.workers_per_device < 1:
            raise ValueError("devices and workers_per_device must be >= 1")
        if self.column_width < 1 or self.rank < 1:
            raise ValueError("column_width and rank must be >= 1")
        if self.accumulation not in ACCUMULATION_MODES:
            raise ValueError(f"accumulation must be one of {ACCUMULATION_MODES}")
        if self.scheduling not in SCHEDULING_MODES:
            raise ValueError(f"scheduling must be one of {SCHEDULING_MODES}")
        if self.kernel_variant not in (0, 1):
            raise ValueError("kernel_variant must be 0 (production) or 1 (generic scalar)")
        if self.tile_nnz < 0 or self.carry_chunk < 2:
            raise ValueError("tile_nnz must be >= 0 (0 = auto) and carry_chunk >= 2")
        if self.layout not in ("flycoo", "blocked", "panel", "cells", "fibers", "auto"):
            raise ValueError("layout must be 'flycoo', 'blocked', 'panel', 'cells', 'fibers' or 'auto'")
        if self.cell_outer_mb < 1 or self.cell_inner_mb < 1:
            raise ValueError("cell_outer_mb and cell_inner_mb must be >= 1")



def _torch():
    import torch

    return torch


class DeviceState:
    """One logical device: factor replicas + output buffer on a GPU."""

    def __init__(self, device_id, factors, output=None, cuda_device=None):
        torch = _torch()
        self.device_id = device_id
        self.cuda_device = cuda_device if cuda_device is not None else (
            factors[0].device if factors else torch.device("cuda", 0))
        self.factors = list(factors)
        self.output = output
        self.compute_seconds = 0.0
        self.staging_seconds = 0.0
        self.shards_processed = 0
        self.nnz_processed = 0
        self.owned_ranges = []
        self.write_rows = None

    def reset_for_mode(self, rows, rank, dtype=None, collect_write_log=False):
        torch = _torch()
        self.output = torch.zeros((rows, rank), dtype=dtype or torch.float32, device=self.cuda_device)
        self.owned_ranges = []
        self.write_rows = set() if collect_write_log else None

    def __repr__(self):
        return f"DeviceState(device_id={self.device_id}, gpu={self.cuda_device})"


def _as_device_factor(f, dev):
    torch = _torch()
    if isinstance(f, FactorMatrix):
        f = f.data
    if isinstance(f, torch.Tensor):
        return f.to(dev, dtype=torch.float32).contiguous()
    from .hostio import upload_f64

    return upload_f64(f, dev)


def make_devices(factors, cfg: PlatformConfig) -> list:
    """One DeviceState per device, each with its own fp32 factor replicas
    (engine.py:83-88); device j lives on GPU j mod torch.cuda.device_count().
    Host factors cross PCIe once per physical GPU (pinned staging, converted
    on the GPU, hostio.upload_f64); further replicas on that GPU are device
    copies."""
    torch = _torch()
    ngpu = torch.cuda.device_count()
    if ngpu == 0:
        raise RuntimeError("make_devices: no CUDA device visible (the B200 engine has no CPU path)")
    devs, first = [], {}
    for j in range(cfg.devices):
        gpu = torch.device("cuda", j % ngpu)
        if gpu.index in first:
            facs = [f.clone() for f in first[gpu.index]]
        else:
            facs = [_as_device_factor(f, gpu) for f in factors]
            first[gpu.index] = facs
        devs.append(DeviceState(j, facs, cuda_device=gpu))
    return devs


def elementwise_compute(x: NonzeroElement, factors, mode: int):
    """Single-element update (engine.py:91-100): (row, length-R contribution)."""
    mats = [f.data if isinstance(f, FactorMatrix) else np.asarray(f) for f in factors]
    contrib = x.value * np.ones(mats[0].shape[1])
    for w, m in enumerate(mats):
        if w != mode:
            contrib = contrib * m[x.indices[w]]
    return x.indices[mode], contrib


# ----------------------------------------------------------------- balancer


def assign_elements(plan: ModePartitionPlan, m: int, cuts=None):
    """Element-split placement: device r processes plan elements
    [cuts[r], cuts[r+1]) (plan order; default r*n//m, equal nonzeros).
    Returns (ranges, shard ids per device, boundary rows cut by a range edge,
    row cuts R_0..R_m)."""
    torch = _torch()
    n = plan.nnz
    cuts = [r * n // m for r in range(m + 1)] if cuts is None else [int(c) for c in cuts]
    rowc = plan.coords[plan.mode]
    probe = sorted({c for c in cuts if 0 < c < n} | {c - 1 for c in cuts if 0 < c < n})
    val = {}
    if probe:
        got = rowc[torch.tensor(probe, device=rowc.device, dtype=torch.int64)].cpu().tolist()
        val = dict(zip(probe, got))
    rows = plan.shape[plan.mode]
    rcut = [0] + [val[c] if 0 < c < n else rows for c in cuts[1:-1]] + [rows]
    boundary = sorted({val[c] for c in cuts[1:-1] if 0 < c < n and val[c - 1] == val[c]})
    ranges = [(cuts[r], cuts[r + 1]) for r in range(m)]
    ids = []
    for e0, e1 in ranges:
        ids.append([s.shard_id for s in plan.shards if s.nnz and s.start < e1 and s.stop > e0])
    return ranges, ids, boundary, rcut


def assign_shards(plan: ModePartitionPlan, m: int, scheduling: str, weights=None) -> list:
    """Shard ids per device.

    static     -- round-robin j::m (engine.py:291-293);
    contiguous -- one run of consecutive shards per device, cut at the
                  cumulative-cost targets (one owned row range per device);
    dynamic -- the reference's shared claim queue replayed deterministically:
               shards in order, each to the device that frees up first under
               cost = nnz (or ``weights``); ties to the lowest device id.
    """
    k = plan.shard_count
    if scheduling == "static":
        return [list(range(j, k, m)) for j in range(m)]
    cost = np.array([s.nnz for s in plan.shards] if weights is None else weights, dtype=np.float64)
    if scheduling == "contiguous":
        # cut the shard sequence at the prefix closest to j*total/m (every
        # device gets at least one shard while shards remain)
        pre = np.concatenate([[0.0], np.cumsum(cost)])
        total = pre[-1]
        cuts = [0]
        for j in range(1, m):
            lo = cuts[-1] + (1 if cuts[-1] < k - (m - j) else 0)
            hi = max(lo, k - (m - j))
            window = pre[lo:hi + 1]
            cuts.append(lo + int(np.argmin(np.abs(window - j * total / m))) if len(window) else lo)
        cuts.append(k)
        return [list(range(cuts[j], cuts[j + 1])) for j in range(m)]
    load = np.zeros(m)
    out = [[] for _ in range(m)]
    for j in range(k):
        dev = int(np.argmin(load))
        out[dev].append(j)
        load[dev] += cost[j]
    return out


# --------------------------------------------------------- resident tables


# ------------------------------------------------------ L2-blocked layouts

_V2_RANKS = (8, 16, 32, 64, 128)


def blocking_cost(plan, rank, shifts, shard_ids=None, l2_bytes=96 << 20):
    """Modelled HBM bytes of one mode in the layout given by `shifts`
    (shifts[w] >= 0: input mode w cut into blocks of 2^shifts[w] rows).

    stream: nnz*(4N+4).  gathers: if the input blocks of a group fit the L2
    budget, each group loads them once; otherwise random rows miss with
    probability 1 - L2/working-set.  output: each group re-reads and rewrites
    (red) the rows it touches: min(shard rows, group nnz) rows."""
    n = len(plan.shape)
    d = plan.mode
    ids = range(plan.shard_count) if shard_ids is None else shard_ids
    nnz = sum(plan.shards[j].nnz for j in ids)
    row_b = rank * 4
    ws = 0.0
    groups = 1
    for w in range(n):
        if w == d:
            continue
        if shifts[w] >= 0:
            rows = min(plan.shape[w], 1 << shifts[w])
            groups *= -(-plan.shape[w] // rows)
        else:
            rows = plan.shape[w]
        ws += rows * row_b
    gathers = 0.0
    out = 0.0
    for j in ids:
        sh = plan.shards[j]
        if sh.nnz == 0:
            continue
        rows = sh.index_range[1] - sh.index_range[0]
        out += groups * min(rows, sh.nnz / groups) * row_b * (2 if groups > 1 else 1)
        if ws <= l2_bytes:
            gathers += groups * ws
        else:
            gathers += sh.nnz * (n - 1) * row_b * (1.0 - l2_bytes / ws)
    return nnz * (4 * n + 4) + gathers + out


def choose_blocking(plan, rank, shard_ids=None, l2_bytes=96 << 20, max_blocks=64, force=False):
    """Block counts (powers of two, up to max_blocks per input mode) that
    minimise blocking_cost.  Returns (shifts for plan.to_blocked or None,
    modelled bytes, modelled bytes of the unblocked plan order).
    force: never return the unblocked layout."""
    import itertools

    n = len(plan.shape)
    d = plan.mode
    ins = [w for w in range(n) if w != d]
    none = [-1] * n
    base = blocking_cost(plan, rank, none, shard_ids, l2_bytes)
    best, best_sh = (float("inf"), None) if force else (base, None)
    opts = [1 << i for i in range(1, max_blocks.bit_length()) if (1 << i) <= max_blocks]
    for combo in itertools.product([1] + opts, repeat=len(ins)):
        if all(b == 1 for b in combo):
            continue
        sh = list(none)
        for w, b in zip(ins, combo):
            if b > 1 and plan.shape[w] > 1:
                rows = -(-plan.shape[w] // b)
                sh[w] = max(0, (rows - 1).bit_length())
        if all(x < 0 for x in sh):
            continue
        c = blocking_cost(plan, rank, sh, shard_ids, l2_bytes)
        if c < best * 0.999:
            best, best_sh = c, sh
    if best_sh is None:
        return None, base, base
    return best_sh, best, base


def _skewed_rows(plan, shard_ids=None, warps=16) -> bool:
    """True when one output row holds more than a quarter of a warp's fair
    share of the nonzeros (#SM x 16 warps): the panel kernel sums a row in one
    warp, so a Zipf head row would serialise it (cfg4s: 3.2 s per mode); the
    tile kernel splits such rows across tiles (carries / atomics)."""
    torch = _torch()
    ids = range(plan.shard_count) if shard_ids is None else shard_ids
    nnz = sum(plan.shards[j].nnz for j in ids)
    if nnz == 0:
        return False
    rows = plan.coords[plan.mode]
    dev = rows.device
    counts = torch.empty(plan.shape[plan.mode], dtype=torch.int64, device=dev)
    _lib.call("skrp_histogram", rows.data_ptr(), rows.numel(), counts.numel(), counts.data_ptr(),
              torch.cuda.current_stream(dev).cuda_stream)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    return int(counts.max().item()) * 4 * sms * warps > nnz


def streamed_blocking(plan, rank, block_mb=32, stream_mb=256):
    """'Pin one, stream one' block shapes (measured best on cfg2 for every
    mode, profiles/sweeps/r01d_sweep_o.jsonl: 48.3/49.0/49.1 ms vs 52.5/51.7/
    51.5 for the cost model's two-block shapes): the smallest input factor
    larger than one block but at most `stream_mb` streams through L2
    unblocked, every other large input is cut into `block_mb` blocks that stay
    L2-resident while a group runs; few groups keep the output re-sweeps and
    the runs short-run free.  None when no input qualifies."""
    n, d = len(plan.shape), plan.mode
    row_b = rank * 4
    big = [w for w in range(n) if w != d and plan.shape[w] * row_b > (block_mb << 20)]
    if not big:
        return None
    cand = [w for w in big if plan.shape[w] * row_b <= (stream_mb << 20)]
    if not cand:
        return None
    stream = min(cand, key=lambda w: plan.shape[w])
    shifts = [-1] * n
    rows = max(1, (block_mb << 20) // row_b)
    for w in big:
        if w != stream:
            shifts[w] = max(0, rows.bit_length() - 1)
    return shifts if any(x >= 0 for x in shifts) else None


def apply_layout(plan, cfg: PlatformConfig, rank: int, shard_ids=None):
    """Put `plan` in the execution layout `cfg.layout` asks for (once)."""
    if cfg.layout == "flycoo" or plan.layout != "flycoo" or cfg.scheduling == "split":
        return plan
    if cfg.layout == "cells":
        prm = choose_cells(plan, rank, cfg, shard_ids)
        if prm is None:
            raise ValueError("cells layout needs a 3-mode tensor, R in {16,32,64} and consecutive shards")
        plan.to_cells(_cell_shards(plan, shard_ids), prm, keep_arrays=cfg.cell_keep_arrays)
        return plan
    if cfg.layout == "panel":
        prm = choose_panels(plan, rank, cfg, shard_ids)
        if prm is None:
            raise ValueError("panel layout needs R in {8,16,32,64} and 3..5 modes")
        plan.to_panels(*prm)
        return plan
    if cfg.layout == "fibers" or (cfg.layout == "auto" and cfg.fibers and cfg.scheduling != "split"):
        f = choose_fibers(plan, rank)
        if f is not None:
            plan.to_fibers(f)
            return plan
        if cfg.layout == "fibers":
            raise ValueError("fiber layout needs a 3-mode tensor, R = 32 and long (row, c_f) runs")
    if rank not in _V2_RANKS or len(plan.shape) > 5:
        if cfg.layout == "blocked":
            raise ValueError("blocked layout needs R in {8,16,32,64,128} and N <= 5")
        return plan
    skewed = _skewed_rows(plan, shard_ids)
    if cfg.layout == "auto" and cfg.accumulation == "deterministic-reduce" and skewed:
        # skewed rows under deterministic-reduce: plan order + carry tree runs at
        # the atomic speed (cfg4s 28.4 vs 29.2 ms/step, cfg5s 56.6 vs 56.7),
        # the blocked carry path pays per-group launches (123 / 191 ms)
        return plan
    if cfg.layout == "auto" and not skewed and len(plan.shape) == 3:
        sh = streamed_blocking(plan, rank)
        if sh is not None:
            if cfg.accumulation == "deterministic-reduce" and panel_shape(len(plan.shape), rank) is not None:
                prm = choose_panels(plan, rank, cfg, shard_ids)
                plan.to_panels(prm[0], sh, prm[2])
            else:
                plan.to_blocked(sh)
            return plan
    shifts, cost, base = choose_blocking(plan, rank, shard_ids, cfg.l2_budget_mb << 20,
                                         max_blocks=cfg.max_blocks, force=cfg.layout == "blocked")
    if shifts is not None and (cfg.layout == "blocked" or cost < 0.8 * base):
        if (cfg.layout == "auto" and cfg.accumulation == "deterministic-reduce"
                and panel_shape(len(plan.shape), rank) is not None):
            # deterministic-reduce: the output-stationary panel kernel sums every
            # row in a fixed order with no carry pass, per-group launches or
            # output zeroing -- bit-identical across device counts, 5 % behind
            # the atomic blocked tiles on cfg2 (157.7 vs 149.6 ms/step) where
            # the blocked deterministic path needs 175 ms
            plan.to_panels(*choose_panels(plan, rank, cfg, shard_ids))
        else:
            plan.to_blocked(shifts)
    return plan


def plan_global_nnz(plan) -> int:
    """Nonzeros of the WHOLE mode plan (all shards, all ranks): the auto tile
    size must not depend on the placement, or tile cuts -- and with them the
    deterministic-reduce carry tree -- would change with the device count."""
    g = getattr(plan, "global_shard_nnz", None)
    if g is not None:
        return int(np.sum(g))
    return int(sum(s_.nnz for s_ in plan.shards))


def auto_tile_nnz(nnz: int, gpu=None) -> int:
    """Tile size giving every resident warp (~#SM x 24) at least ~8 tiles,
    clamped to [128, 4096] (a power of two): big tiles amortise the claim and
    the carries on billion-nonzero modes, small ones keep small modes busy."""
    torch = _torch()
    sms = 148
    try:
        sms = torch.cuda.get_device_properties(gpu or 0).multi_processor_count
    except Exception:
        pass
    want = max(1, nnz // (sms * 24 * 8))
    tile = 128
    while tile * 2 <= want and tile < 4096:
        tile *= 2
    return tile


class _ShardExec:
    """Device-resident tile tables + carry-tree buffers for a set of shards.

    One SEGMENT = one kernel launch (+ its carry tree).  Plan order and the
    atomic blocked layout need one segment; the deterministic blocked layout
    runs one segment per block group (rows are exclusive inside a segment,
    flushes read-add-write in segment order -> bit-reproducible)."""

    def __init__(self, plan, shard_ids, cfg: PlatformConfig, rank, gpu, clip=None):
        torch = _torch()
        self.gpu = gpu
        self.rank = rank
        self.det = cfg.accumulation == "deterministic-reduce"
        self.blocked = plan.layout == "blocked"
        if clip is not None and self.blocked:
            raise ValueError("element-split placement needs the plan-order (flycoo) layout")
        self.flags = (_lib.FLAG_ADDITIVE if self.blocked else 0) | _stream_flags(plan, rank) | _fiber_flags(plan, rank)
        self.nnz = (int(clip[1] - clip[0]) if clip is not None
                    else int(sum(plan.shards[j].nnz for j in shard_ids)))
        self.tile_nnz = cfg.tile_nnz or auto_tile_nnz(plan_global_nnz(plan), gpu)
        if self.blocked and self.det:
            keys = sorted({int(k) for j in shard_ids if plan.shards[j].nnz for k in plan.groups[j][:, 2]})
        else:
            keys = [None]
        self.segments = []
        for key in keys:
            tiles, per_shard = tile_table(plan, shard_ids, self.tile_nnz, group_key=key, clip=clip)
            if len(tiles) == 0:
                continue
            seg = {"n": len(tiles) // 2, "tiles": torch.from_numpy(tiles).to(gpu), "levels": [], "key": key}
            if self.det:
                for table, final in carry_levels(per_shard, cfg.carry_chunk):
                    nch = len(final)
                    lvl = {"n": nch, "chunks": torch.from_numpy(table).to(gpu),
                           "final": torch.from_numpy(final).to(gpu), "rows_out": None, "vals_out": None}
                    if not final.all():
                        lvl["rows_out"] = torch.empty(2 * nch, dtype=torch.int32, device=gpu)
                        lvl["vals_out"] = torch.empty(2 * nch * rank, dtype=torch.float64, device=gpu)
                    seg["levels"].append(lvl)
            self.segments.append(seg)
        self.passes = 1
        self.num_tiles = sum(sg["n"] for sg in self.segments)
        self.counter = torch.zeros(1, dtype=torch.int64, device=gpu)
        mx = max((sg["n"] for sg in self.segments), default=0)
        if self.det and mx:
            self.carry_rows = torch.empty(2 * mx, dtype=torch.int32, device=gpu)
            self.carry_vals = torch.empty(2 * mx * rank, dtype=torch.float32, device=gpu)
        else:
            self.carry_rows = self.carry_vals = None

    @property
    def levels(self):  # carry-tree launches of the first segment (reporting)
        return self.segments[0]["levels"] if self.segments else []

    @property
    def launches(self) -> int:
        return sum(1 + len(sg["levels"]) for sg in self.segments)

    def run(self, coords, vals, nnz_total, mode, factors, out, cfg: PlatformConfig, stream, events=None):
        """Launch the tile kernel(s) (+ carry trees).  `events` (start, end) CUDA
        events, if given, bracket all launches of this mode on `stream`."""
        if self.num_tiles == 0:
            return
        a = _lib.MttkrpArgs()
        a.nmodes = len(coords)
        a.mode = mode
        a.rank = self.rank
        a.accumulation = _lib.ACC_DETERMINISTIC if self.det else _lib.ACC_ATOMIC
        a.nnz = nnz_total
        for w, c in enumerate(coords):
            a.coords[w] = c.data_ptr()
            a.factors[w] = None if w == mode else factors[w].data_ptr()
        a.values = vals.data_ptr()
        a.out = out.data_ptr()
        a.carry_rows = self.carry_rows.data_ptr() if self.det else None
        a.carry_vals = self.carry_vals.data_ptr() if self.det else None
        a.work_counter = self.counter.data_ptr()
        a.persistent_ctas = 0
        a.variant = cfg.kernel_variant
        a.flags = self.flags

        if events is not None:
            events[0].record()  # current stream == `stream` (callers launch on it)
        for seg in self.segments:
            a.tiles = seg["tiles"].data_ptr()
            a.num_tiles = seg["n"]
            _lib.check(_lib.lib().skrp_mttkrp_tiles(ctypes.byref(a), stream), "skrp_mttkrp_tiles")
            if not self.det:
                continue
            rows_in, vals_in, in_f64 = self.carry_rows, self.carry_vals, 0
            for lvl in seg["levels"]:
                _lib.call("skrp_carry_fixup", rows_in.data_ptr(), vals_in.data_ptr(), in_f64,
                          lvl["chunks"].data_ptr(), lvl["final"].data_ptr(), lvl["n"], self.rank,
                          out.data_ptr(), _lib.ptr(lvl["rows_out"]), _lib.ptr(lvl["vals_out"]),
                          1 if self.blocked else 0, stream)
                if lvl["rows_out"] is None:
                    break
                rows_in, vals_in, in_f64 = lvl["rows_out"], lvl["vals_out"], 1
        if events is not None:
            events[1].record()


def _fiber_flags(plan, rank) -> int:
    """SKRP_FLAG_FIBER_INPUTj for a plan in the fiber layout (tile kernel,
    R = 32, 3 modes): j = position of the fiber mode among the inputs."""
    if plan.layout != "fibers" or (len(plan.shape), rank) not in _FIBER_SHAPES:
        return 0
    ins = [w for w in range(len(plan.shape)) if w != plan.mode]
    return (_lib.FLAG_FIBER_INPUT0, _lib.FLAG_FIBER_INPUT1, _lib.FLAG_FIBER_INPUT2)[ins.index(plan.fiber_mode)]


# (modes, rank) with a fiber-reuse kernel instantiation (csrc/mttkrp.cu choose)
_FIBER_SHAPES = ((3, 32), (4, 64))


def choose_fibers(plan, rank, min_fiber=8.0):
    """Fiber mode for the fiber layout, or None: the input mode with the
    fewest rows (the longest (row, c_f) runs), if the expected fiber length
    -- nnz / sum_rows I_f (1 - exp(-n_row / I_f)), the uniform-draw number
    of distinct (row, c_f) pairs -- is at least `min_fiber` (cfg3: ~325 in
    every mode; cfg5 full: ~20 in modes 2 and 3; cfg2, cfg4: ~1)."""
    torch = _torch()
    n, d = len(plan.shape), plan.mode
    if (n, rank) not in _FIBER_SHAPES or plan.nnz == 0:
        return None
    f = min((w for w in range(n) if w != d), key=lambda w: (plan.shape[w], w))
    rows = plan.coords[d]
    counts = torch.empty(plan.shape[d], dtype=torch.int64, device=rows.device)
    _lib.call("skrp_histogram", rows.data_ptr(), rows.numel(), counts.numel(), counts.data_ptr(),
              torch.cuda.current_stream(rows.device).cuda_stream)
    i_f = float(plan.shape[f])
    pairs = float((i_f * (1.0 - torch.exp(-counts.double() / i_f))).sum().item())
    return f if pairs > 0 and plan.nnz / pairs >= min_fiber else None


def _stream_flags(plan, rank) -> int:
    """SKRP_FLAG_STREAM_INPUTj for a pin-one-stream-one layout (one large input
    left unblocked next to a blocked one): that input's rows are loaded
    L2::evict_first so they do not push the pinned blocks out (cfg2: 48.1 ->
    46.2, 49.5 -> 47.3, 49.2 -> 46.8 ms per mode; profiles/sweeps/r01d_sweep_p.jsonl)."""
    sh = getattr(plan, "block_shifts", None)
    if sh is None or plan.layout not in ("blocked", "panel") or len(plan.shape) != 3 or rank != 32:
        return 0
    ins = [w for w in range(3) if w != plan.mode]
    if not any(sh[w] >= 0 for w in ins):
        return 0
    flags = 0
    for j, w in enumerate(ins):
        if sh[w] < 0 and plan.shape[w] * rank * 4 > (32 << 20):
            flags |= 2 << j
    return flags if flags in (_lib.FLAG_STREAM_INPUT0, _lib.FLAG_STREAM_INPUT1) else 0


class _StreamExec:
    """Out-of-core executor: the plan lives in pinned
    host memory (plan.to_host()); each run copies it to two device buffers
    chunk by chunk on a copy stream while the tile kernel processes the
    previous chunk (double buffering, events both ways).  A chunk is a
    contiguous element range of whole tiles; rows may straddle chunks, so
    every flush adds (atomic discipline).  HBM holds only 2 chunks + the
    factors + the output, whatever the tensor size; the rate is bound by the
    host->device link (PCIe), not HBM."""

    writes_all_rows = False

    def __init__(self, plan, shard_ids, cfg: PlatformConfig, rank, gpu):
        torch = _torch()
        if cfg.accumulation != "atomic":
            raise ValueError("out-of-core (streamed) plans run under accumulation='atomic' (rows straddle chunks)")
        self.gpu = gpu
        self.rank = rank
        self.det = False
        self.passes = 1
        self.levels = []
        self.nnz = int(sum(plan.shards[j].nnz for j in shard_ids))
        self.tile_nnz = cfg.tile_nnz or auto_tile_nnz(plan_global_nnz(plan), gpu)
        tiles, _ = tile_table(plan, shard_ids, self.tile_nnz)
        s_, e_ = tiles[0::2], tiles[1::2]
        cap = max(int(cfg.stream_chunk_nnz), self.tile_nnz)
        self.chunks = []  # (elem start, elem end, device tile table (chunk-local))
        i, n = 0, len(s_)
        while i < n:
            j = i + 1
            while j < n and s_[j] == e_[j - 1] and e_[j] - s_[i] <= cap:
                j += 1
            c0, c1 = int(s_[i]), int(e_[j - 1])
            t = np.empty(2 * (j - i), dtype=np.int64)
            t[0::2] = s_[i:j] - c0
            t[1::2] = e_[i:j] - c0
            self.chunks.append((c0, c1, torch.from_numpy(t).to(gpu)))
            i = j
        self.num_tiles = n
        self.h2d_bytes = sum(c1 - c0 for c0, c1, _ in self.chunks) * 4 * (len(plan.shape) + 1)
        big = max((c1 - c0 for c0, c1, _ in self.chunks), default=0)
        nmodes = len(plan.shape)
        self.bufs = [([torch.empty(big, dtype=torch.int32, device=gpu) for _ in range(nmodes)],
                      torch.empty(big, dtype=torch.float32, device=gpu)) for _ in range(2 if len(self.chunks) > 1 else 1)]
        self.copy_stream = torch.cuda.Stream(gpu)
        self.ready = [torch.cuda.Event() for _ in self.bufs]
        self.free = [torch.cuda.Event() for _ in self.bufs]
        self.pending = 0  # leading chunks of the next run already enqueued (prefetch)
        self.counter = torch.zeros(1, dtype=torch.int64, device=gpu)

    @property
    def launches(self) -> int:
        return len(self.chunks)

    def _copy_chunk(self, i, coords, vals):
        """Enqueue chunk i's host->device copy on the copy stream (into buffer
        i % nb, once the kernel that last read that buffer is done)."""
        torch = _torch()
        c0, c1, _ = self.chunks[i]
        b = i % len(self.bufs)
        bc, bv = self.bufs[b]
        n = c1 - c0
        self.copy_stream.wait_event(self.free[b])  # no-op before the buffer's first use
        with torch.cuda.stream(self.copy_stream):
            for w in range(len(coords)):
                bc[w][:n].copy_(coords[w][c0:c1], non_blocking=True)
            bv[:n].copy_(vals[c0:c1], non_blocking=True)
            self.ready[b].record(self.copy_stream)

    def prefetch(self, coords, vals):
        """Start the next run's leading chunk copies now (the runner calls it
        right after the previous mode's kernel is enqueued), so this mode's
        partition streaming overlaps that mode's tail and its factor
        all-gather instead of starting after them (north_star (4))."""
        k = min(len(self.bufs), len(self.chunks))
        for i in range(self.pending, k):
            self._copy_chunk(i, coords, vals)
        self.pending = max(self.pending, k)

    def run(self, coords, vals, nnz_total, mode, factors, out, cfg: PlatformConfig, stream, events=None):
        torch = _torch()
        if not self.chunks:
            return
        cur = torch.cuda.current_stream(self.gpu)
        a = _lib.MttkrpArgs()
        a.nmodes = len(coords)
        a.mode = mode
        a.rank = self.rank
        a.accumulation = _lib.ACC_ATOMIC
        for w in range(len(coords)):
            a.factors[w] = None if w == mode else factors[w].data_ptr()
        a.out = out.data_ptr()
        a.work_counter = self.counter.data_ptr()
        a.variant = cfg.kernel_variant
        a.flags = _lib.FLAG_ADDITIVE
        if events is not None:
            events[0].record()
        nb = len(self.bufs)
        for i, (c0, c1, tiles) in enumerate(self.chunks):
            b = i % nb
            bc, bv = self.bufs[b]
            if i >= self.pending:  # not prefetched: copy now (double-buffered)
                self._copy_chunk(i, coords, vals)
            cur.wait_event(self.ready[b])
            for w in range(len(coords)):
                a.coords[w] = bc[w].data_ptr()
            a.values = bv.data_ptr()
            a.nnz = c1 - c0
            a.tiles = tiles.data_ptr()
            a.num_tiles = tiles.numel() // 2
            _lib.check(_lib.lib().skrp_mttkrp_tiles(ctypes.byref(a), cur.cuda_stream), "skrp_mttkrp_tiles")
            self.free[b].record(cur)
        self.pending = 0
        if events is not None:
            events[1].record()


class _PanelExec:
    """Item tables of the output-stationary panel kernel (plan.to_panels) for
    a set of shards: the items of those shards, in row order.  One launch per
    mode (per column pass); every owned row is written once, so the output
    needs no zeroing; the result does not depend on the placement."""

    writes_all_rows = True

    def __init__(self, plan, shard_ids, cfg: PlatformConfig, rank, gpu):
        torch = _torch()
        pn = plan.panel
        self.gpu = gpu
        self.rank = rank
        self.det = cfg.accumulation == "deterministic-reduce"
        self.passes = 1
        mine = np.isin(pn["item_shard"], np.asarray(list(shard_ids), dtype=np.int64))
        idx = np.nonzero(mine)[0]
        self.num_items = int(len(idx))
        self.num_tiles = self.num_items  # "work units" for the runner's accounting
        self.tile_nnz = 0
        self.levels = []
        self.nnz = int(sum(plan.shards[j].nnz for j in shard_ids))
        self.item_rows = torch.from_numpy(np.ascontiguousarray(pn["item_rows"][idx])).to(gpu)
        ti = torch.from_numpy(idx).to(pn["item_offsets"].device)
        self.item_offsets = pn["item_offsets"].index_select(0, ti).to(gpu).contiguous()
        self.groups = pn["groups"]
        self.warps = pn["warps"]
        self.slab_rows = 1 << pn["slab_shift"]
        self.stream_flags = _stream_flags(plan, rank)
        self.counter = torch.zeros(1, dtype=torch.int64, device=gpu)
        # grid-synchronised rounds only pay when items are about equal
        # (uniform tensors); skewed items are claimed dynamically
        sizes = (self.item_offsets[:, -1] - self.item_offsets[:, 0]).double() if self.num_items else None
        self.lockstep = bool(cfg.panel_lockstep and self.num_items
                             and float(sizes.max()) <= 1.5 * float(sizes.mean()) + 1.0)

    @property
    def launches(self) -> int:
        return 1 if self.num_items else 0

    def run(self, coords, vals, nnz_total, mode, factors, out, cfg: PlatformConfig, stream, events=None,
            peers=None):
        """``peers`` = (device uint64 table of peer output pointers, count):
        the fused all-gather (every finished row is also stored there)."""
        if self.num_items == 0:
            return
        a = _lib.MttkrpArgs()
        a.nmodes = len(coords)
        a.mode = mode
        a.rank = self.rank
        a.accumulation = _lib.ACC_DETERMINISTIC if self.det else _lib.ACC_ATOMIC
        a.nnz = nnz_total
        for w, c in enumerate(coords):
            a.coords[w] = c.data_ptr()
            a.factors[w] = None if w == mode else factors[w].data_ptr()
        a.values = vals.data_ptr()
        a.out = out.data_ptr()
        a.work_counter = self.counter.data_ptr()
        a.variant = cfg.kernel_variant
        a.flags = self.stream_flags
        pa = _lib.PanelArgs()
        pa.item_rows = self.item_rows.data_ptr()
        pa.item_offsets = self.item_offsets.data_ptr()
        pa.num_items = self.num_items
        pa.groups = self.groups
        pa.slab_rows = self.slab_rows
        pa.warps = self.warps
        pa.flags = _lib.PANEL_LOCKSTEP if self.lockstep else 0
        if peers is not None and peers[1]:
            pa.peer_out = peers[0].data_ptr()
            pa.num_peers = peers[1]
        if events is not None:
            events[0].record()
        _lib.check(_lib.lib().skrp_mttkrp_panels(ctypes.byref(a), ctypes.byref(pa), stream), "skrp_mttkrp_panels")
        if events is not None:
            events[1].record()


def panel_shape(nmodes: int, rank: int):
    """(warps per CTA, largest slab rows) of the panel kernel, or None."""
    w = ctypes.c_int32()
    m = ctypes.c_int32()
    rc = _lib.lib().skrp_panel_shape(nmodes, rank, ctypes.byref(w), ctypes.byref(m))
    if rc != _lib.SKRP_OK:
        return None
    return int(w.value), int(m.value)


def choose_panels(plan, rank, cfg: PlatformConfig, shard_ids=None):
    """Panel layout parameters (slab_shift, input shifts, warps) or None.

    Input blocks: the blocked layout's cost model (choose_blocking with
    cfg.l2_budget_mb / max_blocks -- the same blocks, measured equally fast on
    cfg2) unless cfg.panel_l2_mb >= 0, which cuts every input mode whose factor
    exceeds its share of that budget (tuning / tests).  Slab: the largest power
    of two whose panel fits cfg.panel_smem_kb of shared memory (the rest of the
    SM's L1 holds the gathers in flight), capped by the kernel and the mode."""
    n, d = len(plan.shape), plan.mode
    shp = panel_shape(n, rank)
    if shp is None:
        return None
    warps, max_slab = shp
    if cfg.slab_rows:
        slab = cfg.slab_rows
    else:
        slab = warps
        while slab * 2 * rank * 4 <= cfg.panel_smem_kb * 1024 and slab * 2 <= max_slab:
            slab *= 2
    slab = min(slab, max(warps, 1 << max(0, (plan.shape[d] - 1).bit_length())))
    ins = [w for w in range(n) if w != d]
    row_b = rank * 4
    shifts = [-1] * n
    if cfg.panel_l2_mb < 0:
        sh, _, _ = choose_blocking(plan, rank, shard_ids, cfg.l2_budget_mb << 20, max_blocks=cfg.max_blocks, force=True)
        if sh is not None:
            shifts = list(sh)
    else:
        share = (cfg.panel_l2_mb << 20) / max(1, len(ins))
        for w in ins:
            if plan.shape[w] * row_b > share:
                rows = max(1, int(share // row_b))
                shift = max(0, rows.bit_length() - 1)
                while -(-plan.shape[w] // (1 << shift)) > 64:  # bounds the item table
                    shift += 1
                shifts[w] = shift
    # key budget of to_panels: shard | slab | groups | stripe <= 30 bits, and
    # at most 2^12 group slots per item (bounds the item table): coarsen the
    # input mode with the most blocks until both hold
    slab_shift = slab.bit_length() - 1

    def width(w):
        return max(1, (-(-plan.shape[w] // (1 << shifts[w])) - 1).bit_length()) if shifts[w] >= 0 else 0

    fixed = (max(1, (plan.shard_count - 1).bit_length()) + max(1, (-(-plan.shape[d] // slab) - 1).bit_length())
             + (warps.bit_length() - 1))
    while True:
        gb = sum(width(w) for w in ins)
        if (fixed + gb <= 30 and gb <= 12) or gb == 0:
            break
        w = max(ins, key=width)
        shifts[w] = shifts[w] + 1
        if (1 << shifts[w]) >= plan.shape[w]:
            shifts[w] = -1
    return (slab_shift, shifts, warps)


def cell_shape(rank: int, variant: int = 1):
    """(warps per CTA, steps per pipeline stage, largest stripe rows) of a
    cells kernel variant, or None."""
    w = ctypes.c_int32()
    b = ctypes.c_int32()
    m = ctypes.c_int32()
    rc = _lib.lib().skrp_cell_shape(rank, variant, ctypes.byref(w), ctypes.byref(b), ctypes.byref(m))
    if rc != _lib.SKRP_OK:
        return None
    return int(w.value), int(b.value), int(m.value)


def _cell_shards(plan, shard_ids):
    return list(range(plan.shard_count)) if shard_ids is None else sorted(int(j) for j in shard_ids)


def choose_cells(plan, rank, cfg: PlatformConfig, shard_ids=None, sms=None):
    """Parameters of the cells layout (plan.to_cells) or None.

    Outer input = the smaller factor (per round the GPU reads it once and the
    inner factor once per outer block: rounds x (|outer| + outer_blocks x
    |inner|)), cut into cfg.cell_outer_mb blocks; inner input in
    cfg.cell_inner_mb blocks (coarsened until <= 1024 cells).  Stripes: the
    fewest ROUNDS of #SM x 16 stripes whose panels fit shared memory, rows
    spread evenly over them."""
    torch = _torch()
    n, d = len(plan.shape), plan.mode
    if n != 3:
        return None
    variant = cfg.cell_variant
    shp = cell_shape(rank, variant)
    if shp is None and variant != 0:
        variant, shp = 0, cell_shape(rank, 0)  # the tuned variants are built for R = 32
    if shp is None:
        return None
    warps, stage, max_sr = shp
    ids = _cell_shards(plan, shard_ids)
    if not ids or ids != list(range(ids[0], ids[-1] + 1)):
        return None
    if sms is None:
        sms = torch.cuda.get_device_properties(plan.vals.device).multi_processor_count
    lo, hi = int(plan.bounds[ids[0]]), int(plan.bounds[ids[-1] + 1])
    rows = max(1, hi - lo)
    per_round = sms * warps * max_sr
    rounds = -(-rows // per_round)
    sr = -(-rows // (rounds * sms * warps))
    ins = [w for w in range(n) if w != d]
    om, im = sorted(ins, key=lambda w: (plan.shape[w], w))
    row_b = rank * 4

    def shift_for(mb, extent):
        rws = max(1, (mb << 20) // row_b)
        sh = max(0, rws.bit_length() - 1)
        return min(sh, max(0, (extent - 1).bit_length()))

    so = shift_for(cfg.cell_outer_mb, plan.shape[om])
    si = shift_for(cfg.cell_inner_mb, plan.shape[im])
    nout = -(-plan.shape[om] // (1 << so))
    while nout * -(-plan.shape[im] // (1 << si)) > 1024:
        si += 1
    return {"rank": rank, "stripe_rows": sr, "ctas": sms, "outer_mode": om, "inner_mode": im, "outer_shift": so,
            "inner_shift": si, "variant": variant, "warps": warps, "stage": stage}


class _CellExec:
    """The cells kernel over the shards the layout was built for: one launch
    per mode; every owned row is written once (no output zeroing); the result
    does not depend on the placement."""

    writes_all_rows = True

    def __init__(self, plan, shard_ids, cfg: PlatformConfig, rank, gpu):
        torch = _torch()
        c = plan.cells
        if tuple(_cell_shards(plan, shard_ids)) != c["shard_ids"]:
            raise ValueError("the cells layout was built for another shard set")
        self.gpu = gpu
        self.rank = rank
        self.c = c
        self.passes = 1
        self.levels = []
        self.tile_nnz = 0
        self.nnz = int(sum(plan.shards[j].nnz for j in shard_ids))
        if c["rank"] != rank:
            raise ValueError(f"the cells layout was built for R={c['rank']}, not R={rank}")
        self.num_tiles = int(c["stripes"]) if self.nnz else 0
        self.offsets = c["stripe_offsets"].to(gpu)
        self.entries = c["entries"].to(gpu)
        panels = -(-c["stripes"] // c["warps"])
        rounds = -(-panels // c["ctas"]) if panels else 0
        self.done = torch.zeros(max(1, rounds * c["cells"]), dtype=torch.int32, device=gpu)
        self.lag = cfg.cell_lag

    @property
    def launches(self) -> int:
        return 1 if self.num_tiles else 0

    def run(self, coords, vals, nnz_total, mode, factors, out, cfg: PlatformConfig, stream, events=None):
        if self.num_tiles == 0:
            return
        c = self.c
        a = _lib.MttkrpArgs()
        a.nmodes = len(factors)
        a.mode = mode
        a.rank = self.rank
        a.accumulation = _lib.ACC_DETERMINISTIC
        a.nnz = nnz_total
        for w in range(len(factors)):
            a.factors[w] = None if w == mode else factors[w].data_ptr()
        a.values = None
        a.out = out.data_ptr()
        ca = _lib.CellArgs()
        ca.row_lo = c["row_lo"]
        ca.rows = c["rows"]
        ca.out_row_base = 0
        ca.stripe_offsets = self.offsets.data_ptr()
        ca.stripes = c["stripes"]
        ca.stripe_rows = c["stripe_rows"]
        ca.ctas = c["ctas"]
        ca.outer_mode = c["outer_mode"]
        ca.inner_mode = c["inner_mode"]
        ca.outer_shift = c["outer_shift"]
        ca.inner_shift = c["inner_shift"]
        ca.inner_blocks = c["inner_blocks"]
        ca.cells = c["cells"]
        ca.lag = self.lag
        ca.variant = c["variant"]
        ca.done = self.done.data_ptr()
        ca.entries = self.entries.data_ptr()
        if events is not None:
            events[0].record()
        _lib.check(_lib.lib().skrp_mttkrp_cells(ctypes.byref(a), ctypes.byref(ca), stream), "skrp_mttkrp_cells")
        if events is not None:
            events[1].record()


def _plan_arrays(plan: ModePartitionPlan, gpu):
    """The plan's sorted arrays on `gpu` (copied once and cached if the plan
    was built on another GPU); host-resident (out-of-core) plans are returned
    as they are -- their executor streams them."""
    if plan.layout == "cells" and plan.vals is None:
        return None, None  # the cells executor reads the layout's entries
    if plan.vals is None:
        raise ValueError("plan has no device arrays (released)")
    if plan.layout == "host":
        return plan.coords, plan.vals
    if plan.vals.device == gpu:
        return plan.coords, plan.vals
    key = ("arrays", str(gpu))
    if key not in plan._exec_cache:
        plan._exec_cache[key] = ([c.to(gpu) for c in plan.coords], plan.vals.to(gpu))
    return plan._exec_cache[key]


def _shard_exec(plan, shard_ids, cfg, rank, gpu, clip=None):
    key = ("exec", tuple(shard_ids), cfg.tile_nnz, cfg.carry_chunk, cfg.accumulation, rank, str(gpu), plan.layout,
           cfg.cell_lag,
           clip)
    ex = plan._exec_cache.get(key)
    if ex is None:
        if plan.layout == "panel":
            if clip is not None:
                raise ValueError("element-split placement needs the plan-order (flycoo) layout")
            ex = _PanelExec(plan, shard_ids, cfg, rank, gpu)
        elif plan.layout == "cells":
            if clip is not None:
                raise ValueError("element-split placement needs the plan-order (flycoo) layout")
            ex = _CellExec(plan, shard_ids, cfg, rank, gpu)
        elif plan.layout == "host":
            if clip is not None:
                raise ValueError("element-split placement is not streamed")
            ex = _StreamExec(plan, shard_ids, cfg, rank, gpu)
        else:
            ex = _ShardExec(plan, shard_ids, cfg, rank, gpu, clip)
        plan._exec_cache[key] = ex
    return ex


def _normalize_ranges(ranges):
    merged = []
    for lo, hi in sorted(ranges):
        if merged and merged[-1][1] == lo:
            merged[-1] = (merged[-1][0], hi)
        else:
            merged.append((lo, hi))
    return merged


def _write_rows(plan, shard_ids, gpu):
    torch = _torch()
    coords, _ = _plan_arrays(plan, gpu)
    rows = set()
    for j in shard_ids:
        sh = plan.shards[j]
        if sh.nnz:
            rows.update(torch.unique_consecutive(coords[plan.mode][sh.start:sh.stop]).cpu().tolist())
    return rows


def _check_factors(plan, factors):
    for w, size in enumerate(plan.shape):
        if factors[w].shape[0] != size:
            raise ValueError(f"factor for mode {w} has {factors[w].shape[0]} rows, plan needs {size}")


def execute_shard(shard: TensorShard, device: DeviceState, mode: int, cfg: PlatformConfig, *,
                  stream=None, collect_write_log: bool = False, **_ignored):
    """Run every ISP of one shard on one device (engine.py:128-212).

    The shard's rows are exclusively owned, so its tiles write them directly
    into ``device.output`` (which must be zero on those rows)."""
    if shard.mode != mode:
        raise ValueError(f"shard belongs to mode {shard.mode}, not {mode}")
    if device.output is None or device.output.shape[1] != device.factors[0].shape[1]:
        raise ValueError("device output accumulator not initialized for this mode")
    if shard.nnz == 0:
        return
    torch = _torch()
    plan = shard._plan
    gpu = device.cuda_device
    coords, vals = _plan_arrays(plan, gpu)
    ex = _shard_exec(plan, [shard.shard_id], cfg, device.output.shape[1], gpu)
    s = stream or torch.cuda.current_stream(gpu)
    with torch.cuda.device(gpu):
        ex.run(coords, vals, plan.nnz, mode, device.factors, device.output, cfg, s.cuda_stream)
    if collect_write_log and device.write_rows is not None:
        device.write_rows.update(_write_rows(plan, [shard.shard_id], gpu))


def mttkrp_mode(plan: ModePartitionPlan, devices: list, cfg: PlatformConfig,
                ledger: TransferLedger | None = None, *, update_factors: bool = True,
                collect_write_log: bool = False, as_numpy: bool = True, assignment=None):
    """One output mode end to end: compute, barrier, all-gather, barrier.

    Returns (gathered output, ModeMetrics) -- float64 numpy like the
    reference (engine.py:366), or the fp32 device tensor with as_numpy=False.
    """
    torch = _torch()
    m = len(devices)
    if m != cfg.devices:
        raise ValueError(f"{m} device states but config says {cfg.devices}")
    mode = plan.mode
    rows = plan.shape[mode]
    rank = devices[0].factors[0].shape[1]
    _check_factors(plan, devices[0].factors)
    if m > plan.shard_count:
        warnings.warn(f"mode {mode}: {m} devices but only {plan.shard_count} shards; surplus devices idle",
                      RuntimeWarning, stacklevel=2)
    t_mode = time.perf_counter()
    ledger = ledger if ledger is not None else TransferLedger()
    if cfg.scheduling == "split":
        raise ValueError("scheduling='split' needs the one-process-per-GPU runner (distributed.DistributedMttkrp)")
    if assignment is None:
        assignment = assign_shards(plan, m, cfg.scheduling)
    apply_layout(plan, cfg, rank)

    torch.cuda.nvtx.range_push(f"skrp mttkrp_mode {mode}")
    events = []
    for dev in devices:
        dev.reset_for_mode(rows, rank, collect_write_log=collect_write_log)
        dev.compute_seconds = dev.staging_seconds = 0.0
        dev.shards_processed = dev.nnz_processed = 0
    for dev, shard_ids in zip(devices, assignment):
        gpu = dev.cuda_device
        stream = torch.cuda.current_stream(gpu)
        coords, vals = _plan_arrays(plan, gpu)
        ex = _shard_exec(plan, shard_ids, cfg, rank, gpu)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(gpu):
            e0.record(stream)
            ex.run(coords, vals, plan.nnz, mode, dev.factors, dev.output, cfg, stream.cuda_stream)
            e1.record(stream)
        events.append((e0, e1))
        dev.owned_ranges = [plan.shards[j].index_range for j in shard_ids]
        dev.shards_processed = len(shard_ids)
        dev.nnz_processed = ex.nnz
        if collect_write_log:
            dev.write_rows = _write_rows(plan, shard_ids, gpu)
    for (e0, e1), dev in zip(events, devices):
        e1.synchronize()
        dev.compute_seconds = e0.elapsed_time(e1) / 1e3  # barrier 1: all shards drained

    ownership = [_normalize_ranges(dev.owned_ranges) for dev in devices]
    parts = FactorPartitionSet(mode, ownership, [dev.output for dev in devices])
    gather_before = ledger.total_bytes("allgather")
    t0 = time.perf_counter()
    ring_all_gather(parts, ledger)
    for dev in devices:
        torch.cuda.current_stream(dev.cuda_device).synchronize()  # barrier 2
    allgather_seconds = time.perf_counter() - t0
    if update_factors:
        for dev in devices:
            dev.factors[mode] = dev.output
    metrics = ModeMetrics(
        mode=mode,
        device_compute_seconds=[dev.compute_seconds for dev in devices],
        device_nnz=[dev.nnz_processed for dev in devices],
        device_shards=[dev.shards_processed for dev in devices],
        staging_bytes=0,  # plans are resident in HBM: nothing is staged per mode
        staging_seconds=0.0,
        allgather_bytes=ledger.total_bytes("allgather") - gather_before,
        allgather_seconds=allgather_seconds,
        barrier_count=2,
        wall_seconds=time.perf_counter() - t_mode,
        algorithmic_bytes=plan.nnz * (4 * len(plan.shape) + 4) + plan.nnz * (len(plan.shape) - 1) * rank * 4
        + rows * rank * 4,
    )
    torch.cuda.nvtx.range_pop()
    out = devices[0].output
    if as_numpy:
        from .hostio import ExportQueue

        q = ExportQueue(out.device)
        q.push(out)
        return q.results()[0], metrics
    return out, metrics


def mttkrp_all_modes(plans: list, devices: list, cfg: PlatformConfig, ledger: TransferLedger | None = None,
                     *, collect_write_log: bool = False, as_numpy: bool = True):
    """All modes in ascending order, chained: each mode's gathered output
    replaces that mode's factor on every device (engine.py:369-400)."""
    plans = sorted(plans, key=lambda p: p.mode)
    metrics = RunMetrics(devices=cfg.devices)
    metrics.preprocessing_seconds = [p.build_time for p in plans]
    outputs = []
    t0 = time.perf_counter()
    export = None
    if as_numpy and devices:
        # each mode's float64 copy leaves on a side stream while the next
        # modes compute (hostio.ExportQueue), not after the last one
        from .hostio import ExportQueue

        export = ExportQueue(devices[0].cuda_device)
    for plan in plans:
        out, mm = mttkrp_mode(plan, devices, cfg, ledger, update_factors=True,
                              collect_write_log=collect_write_log, as_numpy=False)
        if export is not None:
            export.push(out)
        outputs.append(out)
        metrics.modes.append(mm)
    if export is not None:
        outputs = export.results()
    metrics.wall_seconds = time.perf_counter() - t0
    return outputs, metrics


def measure_isolated_compute(plans: list, factors, cfg: PlatformConfig) -> list:
    """Per-device compute seconds with each device's static round-robin
    share run alone on the GPU (engine.py:403-437), timed with CUDA events."""
    torch = _torch()
    totals = [0.0] * cfg.devices
    gpu = torch.device("cuda", torch.cuda.current_device())
    for plan in sorted(plans, key=lambda p: p.mode):
        rows = plan.shape[plan.mode]
        facs = [_as_device_factor(f, gpu) for f in factors]
        rank = facs[0].shape[1]
        coords, vals = _plan_arrays(plan, gpu)
        for j in range(cfg.devices):
            ids = list(range(j, plan.shard_count, cfg.devices))
            out = torch.zeros((rows, rank), dtype=torch.float32, device=gpu)
            ex = _shard_exec(plan, ids, cfg, rank, gpu)
            s = torch.cuda.current_stream(gpu)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ex.run(coords, vals, plan.nnz, plan.mode, facs, out, cfg, s.cuda_stream)
            e1.record(s)
            e1.synchronize()
            totals[j] += e0.elapsed_time(e1) / 1e3
    return totals


def _factor_arrays(factors):
    return [f.data if isinstance(f, FactorMatrix) else f for f in factors]


def mttkrp(tensor, factors, mode: int, *, platform: PlatformConfig | None = None,
           partition: PartitionConfig | None = None, as_numpy: bool = True):
    """Per-mode MTTKRP with dense_mttkrp_oracle's contract (reference.py:32-68):
    same validation and messages; float64 (I_mode, R) result computed on the
    GPU in fp32."""
    if not 0 <= mode < tensor.num_modes:
        raise ValueError(f"mode {mode} out of range for {tensor.num_modes}-mode tensor")
    mats = _factor_arrays(factors)
    if len(mats) != tensor.num_modes:
        raise ValueError("need one factor matrix per mode")
    ranks = {int(m.shape[1]) for m in mats}
    if len(ranks) != 1:
        raise ValueError(f"factor ranks differ: {sorted(ranks)}")
    for w, mtx in enumerate(mats):
        if mtx.shape[0] != tensor.shape[w]:
            raise ValueError(f"factor for mode {w} has {mtx.shape[0]} rows, tensor needs {tensor.shape[w]}")
    rank = ranks.pop()
    cfg = platform or PlatformConfig(rank=rank)
    pcfg = partition or PartitionConfig(devices=cfg.devices)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", RuntimeWarning)
        plan = build_mode_plan(tensor, mode, pcfg, keep_permutation=False)
        out, _ = mttkrp_mode(plan, make_devices(mats, cfg), cfg, update_factors=False, as_numpy=as_numpy)
    return out
