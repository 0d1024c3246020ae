"""One process per GPU: the all-mode MTTKRP across ranks (Alg. 1 of the paper).

Each rank owns the shards ``assign_shards(plan, world, scheduling)[rank]``
of every mode plan (output-row ranges are disjoint by construction, so no
cross-GPU reduction exists -- partition.py:1-9).  Per mode:

  1. zero the rank's owned output rows;
  2. tile kernel over the rank's shards (device work queue, csrc/mttkrp.cu)
     and, for deterministic-reduce, the carry tree;
  3. exchange: every owner broadcasts its owned row ranges in place
     (collective.allgather_owned_rows: NCCL over NVLink/NVSwitch, gloo on CPU);
  4. chained: the gathered output is the mode's factor for later modes
     (engine.py:350-352).

``world == 1`` needs no torch.distributed at all; the same object is the
single-GPU runner used by bench.py.  The compute callable is injectable only
so tests/test_distributed.py can drive the host logic under gloo on CPU;
the default is the CUDA kernel and there is no other product path.
"""

from __future__ import annotations

import numpy as np

from .collective import TransferLedger, allgather_owned_rows
from .engine import (PlatformConfig, _normalize_ranges, _plan_arrays, _shard_exec, apply_layout, assign_elements,
                     assign_shards)


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


class DistributedMttkrp:
    def __init__(self, plans, cfg: PlatformConfig, rank: int | None = None, world: int | None = None,
                 group=None, device=None, compute=None):
        import torch

        d = _dist()
        self.rank = rank if rank is not None else (d.get_rank(group) if d else 0)
        self.world = world if world is not None else (d.get_world_size(group) if d else 1)
        self.group = group
        self.cfg = cfg
        self.plans = sorted(plans, key=lambda p: p.mode)
        self.shape = self.plans[0].shape
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self.compute = compute
        self.assignment = []
        self.ownership = []
        self.mine = []
        for p in self.plans:
            # plans built by distplan carry GLOBAL shard sizes (local ones are
            # zero for shards other ranks own): place on those, like the build did
            a = assign_shards(p, self.world, cfg.scheduling, weights=getattr(p, "global_shard_nnz", None))
            self.assignment.append(a)
            self.ownership.append([_normalize_ranges([p.shards[j].index_range for j in a[r]])
                                   for r in range(self.world)])
            self.mine.append(a[self.rank])
        self.erange = [None] * len(self.plans)   # element range (split placement)
        self.boundary = [[] for _ in self.plans]  # rows summed across ranks (split)
        self.touch = [None] * len(self.plans)    # rows this rank writes (split)
        self._cuts = [None] * len(self.plans)
        if cfg.scheduling == "split":
            for d in range(len(self.plans)):
                self._set_split(d)
        self._execs = {}
        self.outputs = None

    def _set_split(self, d, cuts=None):
        """Element-split placement of mode d (cut positions in plan order;
        default equal nonzeros): element range, shards, boundary rows summed
        across ranks, owned row ranges, rows this rank writes."""
        p = self.plans[d]
        info = getattr(p, "split_info", None)
        if info is not None:  # split-routed distributed plan: local = my element range
            bnd, rcut = info["boundary"], info["rcut"]
            self.erange[d] = (0, p.nnz)
            self.mine[d] = [s_.shard_id for s_ in p.shards if s_.nnz]
        else:
            ranges, ids, bnd, rcut = assign_elements(p, self.world, cuts=cuts)
            self._cuts[d] = [r[0] for r in ranges] + [ranges[-1][1]]
            self.erange[d] = ranges[self.rank]
            self.mine[d] = ids[self.rank]
        self.boundary[d] = bnd
        bset = set(bnd)
        own = []
        for r in range(self.world):
            lo, hi = rcut[r], rcut[r + 1]
            rr, cur = [], lo
            for b in bnd:  # boundary rows are all-reduced, not broadcast
                if lo <= b < hi:
                    if b > cur:
                        rr.append((cur, b))
                    cur = b + 1
            if hi > cur:
                rr.append((cur, hi))
            own.append(rr)
        self.ownership[d] = own
        lo, hi = rcut[self.rank], rcut[self.rank + 1]
        if hi in bset:
            hi += 1
        self.touch[d] = (lo, min(hi, p.shape[p.mode]))

    # ----------------------------------------------------------- rebalancing
    def measure_mode_seconds(self, factors, chained=True):
        """This rank's kernel seconds per mode (one eager all-mode pass with
        CUDA events on the launching stream)."""
        import torch

        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in self.plans]
        self.run(factors, chained=chained, kernel_events=ev)
        torch.cuda.synchronize(self.device)
        return [a.elapsed_time(b) / 1e3 for a, b in ev]

    def rebalance(self, factors=None, rank_seconds=None):
        """Host-side rebalancing across the GPUs from MEASURED per-GPU times
        (SURVEY.md §8(e)): each rank's per-nonzero cost in mode d is its
        measured kernel time over its nonzeros; a shard is then weighted by
        nnz x the cost of the GPU that ran it, and the placement (contiguous
        cut or the dynamic claim replay) is recomputed on those weights -- a
        GPU that ran slow (heavier rows, worse locality, a slower device)
        sheds work.  ``rank_seconds[r][d]`` may be given (tests); otherwise
        every rank measures one pass and the times are all-gathered.  Only
        replicated plans move (the data of distributed plans stays put);
        returns the modes whose placement changed."""
        if rank_seconds is None:
            mine = self.measure_mode_seconds(factors)
            if self.world > 1:
                allt = [None] * self.world
                _dist().all_gather_object(allt, mine, group=self.group)
            else:
                allt = [mine]
            rank_seconds = allt
        changed = []
        for d, p in enumerate(self.plans):
            if self.cfg.scheduling == "split" and self._cuts[d] is not None:
                # cost-weighted element cuts: per-element cost is piecewise
                # constant (each rank's measured time / its elements); cut the
                # cumulative cost into equal parts
                cuts = self._cuts[d]
                t = np.array([rank_seconds[r][d] for r in range(self.world)], dtype=np.float64)
                n_r = np.diff(np.asarray(cuts, dtype=np.float64))
                if not np.all(t > 0):
                    continue
                cum = np.concatenate([[0.0], np.cumsum(t)])
                new = [0]
                for j in range(1, self.world):
                    target = j * cum[-1] / self.world
                    r = int(np.searchsorted(cum, target, side="right") - 1)
                    r = min(max(r, 0), self.world - 1)
                    pos = cuts[r] + (target - cum[r]) / t[r] * n_r[r] if t[r] > 0 else cuts[r]
                    new.append(int(min(max(round(pos), new[-1]), p.nnz)))
                new.append(p.nnz)
                if new != list(cuts):
                    self._set_split(d, new)
                    for key in [k for k in self._execs if k[0] == d]:
                        del self._execs[key]
                    changed.append(d)
                continue
            if self.cfg.scheduling not in ("contiguous", "dynamic") or getattr(p, "global_shard_nnz", None) is not None:
                continue
            owner = np.empty(p.shard_count, dtype=np.int64)
            for r, ids in enumerate(self.assignment[d]):
                owner[ids] = r
            nnz_r = np.array([sum(p.shards[j].nnz for j in ids) for ids in self.assignment[d]], dtype=np.float64)
            rate = np.array([rank_seconds[r][d] for r in range(self.world)], dtype=np.float64) / np.maximum(nnz_r, 1)
            if not np.all(rate > 0):
                continue
            w = np.array([s_.nnz for s_ in p.shards], dtype=np.float64) * rate[owner]
            new = assign_shards(p, self.world, self.cfg.scheduling, weights=w)
            if [list(x) for x in new] != [list(x) for x in self.assignment[d]]:
                self.assignment[d] = new
                self.ownership[d] = [_normalize_ranges([p.shards[j].index_range for j in new[r]])
                                     for r in range(self.world)]
                self.mine[d] = new[self.rank]
                for key in [k for k in self._execs if k[0] == d]:
                    del self._execs[key]
                changed.append(d)
        if changed and self.outputs is not None and self.compute is None:
            for d in changed:
                self._exec(d, self._rank_r)
        return changed

    # ------------------------------------------------------------ accounting
    def local_nnz(self, d) -> int:
        if self.erange[d] is not None:
            return int(self.erange[d][1] - self.erange[d][0])
        p = self.plans[d]
        return int(sum(p.shards[j].nnz for j in self.mine[d]))

    def owned_rows(self, d) -> int:
        return int(sum(hi - lo for lo, hi in self.ownership[d][self.rank]))

    def algorithmic_bytes(self, d) -> int:
        """Alg. 2 traffic of this rank's mode-d kernel:
        nnz*(4N+4) streamed + nnz*(N-1)*R*4 gathered + owned rows written."""
        n = len(self.shape)
        r = self._rank_r
        nnz = self.local_nnz(d)
        return nnz * (4 * n + 4) + nnz * (n - 1) * r * 4 + self.owned_rows(d) * r * 4

    # ---------------------------------------------------------------- running
    def _exec(self, d, rank_r):
        key = (d, rank_r)
        if key not in self._execs:
            self._execs[key] = _shard_exec(self.plans[d], self.mine[d], self.cfg, rank_r, self.device,
                                           clip=self.erange[d])
        return self._execs[key]

    def launches_per_mode(self, d) -> int:
        ex = self._execs.get((d, self._rank_r))
        if ex is None or ex.num_tiles == 0:
            return 0
        return ex.launches

    def prepare(self, rank_r, dtype=None):
        import torch

        self._rank_r = rank_r
        self.outputs = [torch.empty((p.shape[p.mode], rank_r), dtype=dtype or torch.float32, device=self.device)
                        for p in self.plans]
        self._close_peers()
        self._peers = [None] * len(self.plans)
        if self.compute is None:
            for d in range(len(self.plans)):
                apply_layout(self.plans[d], self.cfg, rank_r, self.mine[d])
                self._exec(d, rank_r)
            if self.cfg.fused_allgather and self.world > 1:
                self._open_peers()

    # ------------------------------------------------- fused all-gather (IPC)
    def _open_peers(self):
        """Map every other rank's output buffers (CUDA IPC) for the modes that
        run the panel kernel: its write-back then stores each finished row to
        all ranks (NVLink P2P), and the all-gather collective disappears."""
        import ctypes

        import torch

        from . import _lib

        d_ = _dist()
        self._ipc_bases = []
        for d, out in enumerate(self.outputs):
            if self.plans[d].layout not in ("panel", "slots"):
                continue
            h = (ctypes.c_uint8 * 64)()
            off = ctypes.c_int64()
            _lib.call("skrp_ipc_get_handle", out.data_ptr(), h, ctypes.byref(off))
            allh = [None] * self.world
            d_.all_gather_object(allh, (bytes(h), int(off.value)), group=self.group)
            ptrs = []
            for r, (hb, o) in enumerate(allh):
                if r == self.rank:
                    continue
                ptr, base = ctypes.c_void_p(), ctypes.c_void_p()
                buf = (ctypes.c_uint8 * 64).from_buffer_copy(hb)
                _lib.call("skrp_ipc_open_handle", buf, o, ctypes.byref(ptr), ctypes.byref(base))
                ptrs.append(ptr.value)
                self._ipc_bases.append(base.value)
            table = torch.tensor(np.asarray(ptrs, dtype=np.uint64).view(np.int64), device=self.device)
            self._peers[d] = (table, len(ptrs))

    def _close_peers(self):
        from . import _lib

        for b in getattr(self, "_ipc_bases", []):
            _lib.call("skrp_ipc_close_handle", b)
        self._ipc_bases = []

    def _peer_sync(self):
        """All ranks' pushes of this mode are complete before anyone goes on
        (stream-ordered under NCCL; host barrier under gloo).  The panel
        kernel ends every item's write-back with __threadfence_system(), so
        its NVLink stores are visible before its completion -- which the
        1-element all-reduce (queued behind the kernel on every rank) orders
        ahead of the next mode's kernel on every rank."""
        import torch

        d_ = _dist()
        if d_.get_backend(self.group) == "nccl":
            t = torch.zeros(1, device=self.device)
            d_.all_reduce(t, group=self.group)
        else:
            torch.cuda.synchronize(self.device)
            d_.barrier(group=self.group)

    def run(self, factors, chained=True, kernel_events=None, ledger: TransferLedger | None = None,
            after_mode=None, outputs=None, exchange=True):
        """All modes; `factors` are this rank's full fp32 factor replicas.
        Returns the list of gathered outputs (device tensors, reused).
        ``after_mode(i, out)`` is called once mode i's output is gathered
        (stream-ordered), e.g. to start its device-to-host copy.
        ``exchange=False`` skips the all-gather (one rank's compute alone:
        bench.py --emulate-world runs every rank's share on one GPU)."""
        import torch
        from torch.cuda import nvtx

        rank_r = factors[0].shape[1]
        if self.outputs is None or self._rank_r != rank_r or self.outputs[0].dtype != factors[0].dtype:
            self.prepare(rank_r, factors[0].dtype)
        self._exchange = exchange
        facs = list(factors)
        for d, plan in enumerate(self.plans):
            nvtx.range_push(f"skrp mode {plan.mode} mttkrp")
            out = self.mode_output(d, facs, None if kernel_events is None else kernel_events[d],
                                   out=None if outputs is None else outputs[d])
            nvtx.range_pop()
            self._prefetch_next(d + 1 if d + 1 < len(self.plans) else 0)
            if self.world > 1 and exchange:
                nvtx.range_push(f"skrp mode {plan.mode} all-gather")
                if outputs is None and self._fused(d):
                    self._peer_sync()  # rows were pushed by every rank's kernel
                else:
                    allgather_owned_rows(out, self.ownership[d], self.group, ledger, step=d)
                nvtx.range_pop()
            if after_mode is not None:
                after_mode(d, out)
            if chained:
                facs[plan.mode] = out
        return self.outputs

    def _prefetch_next(self, d):
        """Out-of-core plans: enqueue mode d's leading chunk copies now, so its
        partition streaming overlaps the all-gather of the mode just launched
        (north_star (4)); resident plans have nothing to stream."""
        if self.compute is not None or getattr(self, "_rank_r", None) is None:
            return
        ex = self._execs.get((d, self._rank_r))
        if ex is not None and hasattr(ex, "prefetch"):
            coords, vals = _plan_arrays(self.plans[d], self.device)
            ex.prefetch(coords, vals)

    def _fused(self, d) -> bool:
        peers = getattr(self, "_peers", None)
        return bool(peers) and peers[d] is not None

    def mode_output(self, d, factors, events=None, out=None):
        """Mode d's MTTKRP on this rank's shards into self.outputs[d] (or
        `out`): owned rows valid, nothing exchanged yet."""
        import torch

        rank_r = factors[0].shape[1]
        if self.outputs is None or self._rank_r != rank_r or self.outputs[0].dtype != factors[0].dtype:
            self.prepare(rank_r, factors[0].dtype)
        plan = self.plans[d]
        out = self.outputs[d] if out is None else out
        writes_all = self.compute is None and getattr(self._exec(d, rank_r), "writes_all_rows", False)
        if self.touch[d] is not None:
            lo, hi = self.touch[d]
            out[lo:hi].zero_()
        if not writes_all:  # the panel kernel writes every owned row itself
            for lo, hi in self.ownership[d][self.rank]:
                out[lo:hi].zero_()
        if self.compute is not None:
            self.compute(plan, self.mine[d], factors, out)
        else:
            coords, vals = _plan_arrays(plan, self.device)
            stream = torch.cuda.current_stream(self.device)
            ex = self._exec(d, rank_r)
            if out is self.outputs[d] and self._fused(d):
                ex.run(coords, vals, plan.nnz, plan.mode, factors, out, self.cfg, stream.cuda_stream, events=events,
                       peers=self._peers[d])
            else:
                ex.run(coords, vals, plan.nnz, plan.mode, factors, out, self.cfg, stream.cuda_stream, events=events)
        if self.boundary[d] and getattr(self, "_exchange", True):
            self._reduce_boundary(d, out)
        return out

    def _reduce_boundary(self, d, out):
        """Split placement: rows cut by a range edge hold per-rank partial sums;
        sum them across ranks (all ranks end with the full rows)."""
        import torch

        rows = torch.tensor(self.boundary[d], dtype=torch.int64, device=out.device)
        lo, hi = self.touch[d]
        mine = ((rows >= lo) & (rows < hi)).to(out.dtype).unsqueeze(1)
        part = out.index_select(0, rows) * mine
        if self.world > 1:
            import torch.distributed as dist

            if dist.get_backend(self.group) == "nccl" or part.device.type == "cpu":
                dist.all_reduce(part, group=self.group)
            else:
                c = part.cpu()
                dist.all_reduce(c, group=self.group)
                part.copy_(c)
        out.index_copy_(0, rows, part)

    def needed_factors(self, chained=True):
        """Modes whose INPUT factor is actually read: with chaining, factor w
        is replaced by mode w's output before any later mode reads it, so
        only factors read by an earlier mode (or never recomputed) count."""
        order = [p.mode for p in self.plans]
        need = set()
        for i, d in enumerate(order):
            for w in range(len(self.shape)):
                if w == d:
                    continue
                if chained and w in order[:i]:
                    continue
                need.add(w)
        return sorted(need)

    def capture(self, factors, chained=True):
        """CUDA-graph the whole all-mode step (single process only): every
        memset, tile kernel and carry-tree launch of all modes replays as one
        graph launch.  Returns the torch.cuda.CUDAGraph."""
        import torch

        if self.world > 1:
            raise ValueError("graph capture is for world == 1 (NCCL groups are launched eagerly)")
        self.run(factors, chained=chained)  # allocate + warm the tables outside capture
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.run(factors, chained=chained)
        return g

    def run_host_pipelined(self, host_factors, host_outputs, steps, chained=True):
        """`steps` end-to-end steps with HOST buffers, double-buffered: step
        k+1's factor upload (copy stream) and step k's result download (second
        copy stream) run while step k / k+1 compute, like a loader feeding a
        pipeline.  Every step still moves its inputs H2D and its outputs D2H
        inside the caller's timed region; only the overlap changes.
        host_outputs: two sets of pinned (rows x R) tensors (alternating).
        Returns (h2d bytes per step, d2h bytes per step)."""
        import torch

        dev = self.device
        comp = torch.cuda.current_stream(dev)
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        need = self.needed_factors(chained)
        rank_r = host_factors[0].shape[1]
        if self.outputs is None or self._rank_r != rank_r:
            self.prepare(rank_r)
        if not hasattr(self, "_pipe"):
            fac_sets = [[torch.empty(h.shape, dtype=h.dtype, device=dev) for h in host_factors] for _ in range(2)]
            out_sets = [self.outputs, [torch.empty_like(o) for o in self.outputs]]
            self._pipe = (fac_sets, out_sets)
        fac_sets, out_sets = self._pipe
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_comp = [torch.cuda.Event(), torch.cuda.Event()]
        ev_out = [torch.cuda.Event(), torch.cuda.Event()]
        h2d = sum(host_factors[w].numel() * host_factors[w].element_size() for w in need)
        # the gathered result is replicated on every rank: each rank reads back
        # the rows it owns (the whole matrix at world == 1)
        spans = [[(lo, hi) for lo, hi in self.ownership[d][self.rank] if hi > lo] + [(b, b + 1) for b in
                 (self.boundary[d] if self.rank == 0 else [])] for d in range(len(self.plans))]
        row_b = [o.shape[1] * o.element_size() for o in self.outputs]
        d2h = sum(sum(hi - lo for lo, hi in spans[d]) * row_b[d] for d in range(len(self.plans)))

        def upload(b):
            with torch.cuda.stream(s_in):
                for w in need:
                    fac_sets[b][w].copy_(host_factors[w], non_blocking=True)
                ev_in[b].record(s_in)

        s_in.wait_stream(comp)
        upload(0)
        for k in range(steps):
            b = k % 2
            comp.wait_event(ev_in[b])
            if k >= 2:
                comp.wait_event(ev_out[b])  # step k-2's download of this output set is done

            def download(d, o, b=b):
                # mode d's rows leave as soon as they are final, so only the
                # last mode's download is left to drain after the step
                s_out.wait_stream(comp)
                with torch.cuda.stream(s_out):
                    for lo, hi in spans[d]:
                        host_outputs[b][d][lo:hi].copy_(o[lo:hi], non_blocking=True)

            self.run(fac_sets[b], chained=chained, outputs=out_sets[b], after_mode=download)
            ev_comp[b].record(comp)
            ev_out[b].record(s_out)
            if k + 1 < steps:
                nb = 1 - b
                if k >= 1:
                    s_in.wait_event(ev_comp[nb])  # step k-1 finished reading that factor set
                upload(nb)
        comp.wait_stream(s_out)
        comp.wait_stream(s_in)
        return h2d, d2h

    def run_host(self, host_factors, host_outputs, dev_factors, chained=True, copy_streams=None):
        """End-to-end step with HOST buffers (pinned): upload the factors the
        chain actually reads, run all modes, download every gathered output.
        Downloads of mode i overlap the compute of mode i+1 on a copy stream.
        Returns bytes moved (h2d, d2h)."""
        import torch

        comp = torch.cuda.current_stream(self.device)
        s_in, s_out = copy_streams or (torch.cuda.Stream(self.device), torch.cuda.Stream(self.device))
        h2d = d2h = 0
        s_in.wait_stream(comp)
        with torch.cuda.stream(s_in):
            for w in self.needed_factors(chained):
                dev_factors[w].copy_(host_factors[w], non_blocking=True)
                h2d += host_factors[w].numel() * host_factors[w].element_size()
        comp.wait_stream(s_in)
        moved = []

        def download(i, out):
            s_out.wait_stream(comp)
            with torch.cuda.stream(s_out):
                host_outputs[i].copy_(out, non_blocking=True)
            moved.append(out.numel() * out.element_size())

        self.run(dev_factors, chained=chained, after_mode=download)
        comp.wait_stream(s_out)
        d2h = sum(moved)
        return h2d, d2h


class DistributedCpAls:
    """CP-ALS with one process per GPU (cpd.py:108-167 semantics; cfg5).

    Per mode d, on every rank: MTTKRP of its own shards (owned output rows
    only), V = Hadamard of the other modes' Grams (R x R, identical on all
    ranks), W = V^-1 with the reference's jitter/pinv fallback (host, fp64),
    new rows = M[owned] @ W (GPU), column norms = sqrt(all-reduce of per-rank
    column sums of squares) -> lambdas, owned rows normalised, then the
    FACTOR ALL-GATHER of the owned rows (every rank holds the full updated
    factor) and Gram_d = all-reduce of the per-rank partial Grams.  The fit
    sums <X, Xhat> and ||X||^2 over each rank's share of the nonzeros (the
    mode-0 plan's owned shards partition them) and all-reduces the pair.
    """

    def __init__(self, plans, cfg: PlatformConfig, rank=None, world=None, group=None, device=None):
        self.mt = DistributedMttkrp(plans, cfg, rank=rank, world=world, group=group, device=device)
        self.group = group

    def _allreduce(self, t):
        if self.mt.world > 1:
            import torch.distributed as dist

            dist.all_reduce(t, group=self.group)
        return t

    def _owned(self, d, count_once=False):
        """Rows this rank updates.  Under split placement the boundary rows
        (full after the cross-rank sum) are updated redundantly by every rank
        and, for partial sums (count_once), counted by rank 0 only."""
        own = list(self.mt.ownership[d][self.mt.rank])
        if self.mt.boundary[d] and (not count_once or self.mt.rank == 0):
            own += [(b, b + 1) for b in self.mt.boundary[d]]
        return own

    def _partial_gram(self, y, d):
        import torch

        from . import _lib

        R = y.shape[1]
        g = torch.zeros((R, R), dtype=torch.float64, device=y.device)
        tmp = torch.empty((R, R), dtype=torch.float64, device=y.device)
        stream = torch.cuda.current_stream(y.device).cuda_stream
        for lo, hi in self._owned(d, count_once=True):
            if hi > lo:
                _lib.call("skrp_gram", y[lo:hi].data_ptr(), hi - lo, R, tmp.data_ptr(), stream)
                g += tmp
        return self._allreduce(g).cpu().numpy()

    def _col_sumsq(self, x, d):
        import torch

        from . import _lib

        R = x.shape[1]
        acc = torch.zeros(R, dtype=torch.float64, device=x.device)
        tmp = torch.empty(R, dtype=torch.float64, device=x.device)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        for lo, hi in self._owned(d, count_once=True):
            if hi > lo:
                _lib.call("skrp_col_sumsq", x[lo:hi].data_ptr(), hi - lo, R, tmp.data_ptr(), stream)
                acc += tmp
        return self._allreduce(acc).cpu().numpy()

    def _x_sq(self):
        """||X||^2 over this rank's nonzeros (mode-0 plan's owned shards), summed."""
        import torch

        from . import _lib

        if getattr(self, "_xsq", None) is None:
            plan = self.mt.plans[0]
            _, vals = _plan_arrays(plan, self.mt.device)
            total = torch.zeros(1, dtype=torch.float64, device=self.mt.device)
            out = torch.empty(1, dtype=torch.float64, device=self.mt.device)
            stream = torch.cuda.current_stream(self.mt.device).cuda_stream
            if self.mt.erange[0] is not None:
                spans = [self.mt.erange[0]]
            else:
                spans = [(plan.shards[j].start, plan.shards[j].stop) for j in self.mt.mine[0]]
            for a, b in spans:
                if b > a:
                    _lib.call("skrp_sumsq", vals.data_ptr() + 4 * a, b - a, out.data_ptr(), stream)
                    total += out
            self._xsq = float(self._allreduce(total).item())
        return self._xsq

    def _inner_fused(self, d, new, m, lambdas):
        """<X, Xhat> = sum_r lambda_r sum_i F_d[i, r] M_d[i, r] over owned rows of
        the LAST mode d (M_d computed with the already-updated other factors):
        the fit without a second pass over the nonzeros."""
        import torch

        from . import _lib

        R = new.shape[1]
        lam = torch.from_numpy(np.ascontiguousarray(lambdas, dtype=np.float64)).to(new.device)
        total = torch.zeros(1, dtype=torch.float64, device=new.device)
        out = torch.empty(1, dtype=torch.float64, device=new.device)
        stream = torch.cuda.current_stream(new.device).cuda_stream
        for lo, hi in self._owned(d, count_once=True):
            if hi > lo:
                _lib.call("skrp_weighted_dot", new[lo:hi].data_ptr(), m[lo:hi].data_ptr(), hi - lo, R,
                          lam.data_ptr(), out.data_ptr(), stream)
                total += out
        return float(self._allreduce(total).item())

    def run(self, factors, iterations=1, fit_tol=None, timings=None, observe=None):
        """ALS sweeps from the given full fp32 factor replicas (device).
        Returns (factors, lambdas, fit_history).  ``observe(d, factors, m,
        new, lambdas)``, if given, sees every mode update (the factors the
        mode read, its MTTKRP output, the normalised new factor) before the
        all-gather -- the parity checker's hook."""
        import torch

        from . import _lib
        from .cpd import _fit_value, _hadamard, _solve_matrix, mm_fp32

        facs = [f.clone() for f in factors]
        nm = len(facs)
        R = facs[0].shape[1]
        grams = [self._partial_gram(f, w) for w, f in enumerate(facs)]
        lambdas = np.ones(R)
        history = []
        stream = torch.cuda.current_stream(self.mt.device).cuda_stream
        for _ in range(iterations):
            for d in range(nm):
                m = self.mt.mode_output(d, facs)
                v = _hadamard([grams[w] for w in range(nm) if w != d], R)
                owned = [r for r in self._owned(d) if r[1] > r[0]]
                # the same decision on every rank (collective sequences must
                # match): no split boundary rows, whose partial sums count once
                fused = (R in (16, 32, 64) and m.is_contiguous() and m.data_ptr() % 16 == 0 and np.isfinite(v).all()
                         and not self.mt.boundary[d])
                new = torch.empty_like(m)
                if fused:
                    # owned rows times the R x R inverse fused with the new
                    # columns' sums of squares and the non-finite probe of M
                    # (skrp_apply_rr_sumsq: one pass instead of GEMM + 2 norms)
                    w64 = torch.from_numpy(np.ascontiguousarray(_solve_matrix(v))).to(m.device)
                    acc = torch.zeros(R + 1, dtype=torch.float64, device=m.device)
                    sq = torch.empty(R, dtype=torch.float64, device=m.device)
                    bad = torch.empty(1, dtype=torch.int32, device=m.device)
                    for lo, hi in owned:
                        _lib.call("skrp_apply_rr_sumsq", m[lo:hi].data_ptr(), hi - lo, R, w64.data_ptr(),
                                  new[lo:hi].data_ptr(), sq.data_ptr(), bad.data_ptr(), stream)
                        acc[:R] += sq
                        acc[R] += bad[0].double()
                    acc = self._allreduce(acc).cpu().numpy()
                    if acc[R] > 0:
                        raise FloatingPointError("non-finite MTTKRP output")
                    lambdas = np.sqrt(acc[:R])
                else:
                    if not np.isfinite(self._col_sumsq(m, d)).all():
                        raise FloatingPointError("non-finite MTTKRP output")
                    if not np.isfinite(v).all():
                        raise FloatingPointError("non-finite Gram product")
                    # owned rows times the R x R inverse: a plain GEMM -> cuBLAS
                    # (fp32, no TF32)
                    w_t = torch.from_numpy(np.ascontiguousarray(_solve_matrix(v))).to(m.device, dtype=torch.float32)
                    for lo, hi in owned:
                        mm_fp32(m[lo:hi], w_t, out=new[lo:hi])
                    lambdas = np.sqrt(self._col_sumsq(new, d))
                if not np.isfinite(lambdas).all():
                    raise FloatingPointError("non-finite entries in updated factor matrix")
                scale = torch.from_numpy(1.0 / np.where(lambdas > 0, lambdas, 1.0)).to(m.device)
                for lo, hi in self._owned(d):
                    if hi > lo:
                        _lib.call("skrp_scale_cols", new[lo:hi].data_ptr(), hi - lo, R, scale.data_ptr(), stream)
                if d == nm - 1:
                    inner = self._inner_fused(d, new, m, lambdas)
                if observe is not None:
                    observe(d, facs, m, new, lambdas)
                if self.mt.world > 1:
                    allgather_owned_rows(new, self.mt.ownership[d], self.group)
                facs[d] = new
                grams[d] = self._partial_gram(new, d)
            history.append(_fit_value(self._x_sq(), inner, grams, lambdas))
            if fit_tol is not None and len(history) > 1 and history[-1] - history[-2] < fit_tol:
                break
        return facs, lambdas, history


def ownership_table(plan, world: int, scheduling: str = "dynamic"):
    """Per-rank owned [lo, hi) row ranges of a plan (host-only helper)."""
    a = assign_shards(plan, world, scheduling)
    return [_normalize_ranges([plan.shards[j].index_range for j in a[r]]) for r in range(world)]


def rows_cover(ownership, rows: int) -> bool:
    cover = np.zeros(rows, dtype=np.int64)
    for ranges in ownership:
        for lo, hi in ranges:
            cover[lo:hi] += 1
    return bool(np.all(cover == 1))
