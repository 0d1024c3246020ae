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
from .engine import PlatformConfig, _normalize_ranges, _plan_arrays, _shard_exec, apply_layout, assign_shards


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
            a = assign_shards(p, self.world, cfg.scheduling)
            self.assignment.append(a)
            self.ownership.append([_normalize_ranges([p.shards[j].index_range for j in a[r]])
                                   for r in range(self.world)])
            self.mine.append(a[self.rank])
        self._execs = {}
        self.outputs = None

    # ------------------------------------------------------------ accounting
    def local_nnz(self, d) -> int:
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
            self._execs[key] = _shard_exec(self.plans[d], self.mine[d], self.cfg, rank_r, self.device)
        return self._execs[key]

    def launches_per_mode(self, d) -> int:
        ex = self._execs.get((d, self._rank_r))
        if ex is None or ex.num_tiles == 0:
            return 0
        return 1 + (len(ex.levels) if ex.det else 0)

    def prepare(self, rank_r, dtype=None):
        import torch

        self._rank_r = rank_r
        self.outputs = [torch.empty((p.shape[p.mode], rank_r), dtype=dtype or torch.float32, device=self.device)
                        for p in self.plans]
        if self.compute is None:
            for d in range(len(self.plans)):
                apply_layout(self.plans[d], self.cfg, rank_r, self.mine[d])
                self._exec(d, rank_r)

    def run(self, factors, chained=True, kernel_events=None, ledger: TransferLedger | None = None,
            after_mode=None):
        """All modes; `factors` are this rank's full fp32 factor replicas.
        Returns the list of gathered outputs (device tensors, reused).
        ``after_mode(i, out)`` is called once mode i's output is gathered
        (stream-ordered), e.g. to start its device-to-host copy."""
        import torch

        rank_r = factors[0].shape[1]
        if self.outputs is None or self._rank_r != rank_r or self.outputs[0].dtype != factors[0].dtype:
            self.prepare(rank_r, factors[0].dtype)
        facs = list(factors)
        stream = torch.cuda.current_stream(self.device) if self.device.type == "cuda" else None
        for d, plan in enumerate(self.plans):
            out = self.outputs[d]
            for lo, hi in self.ownership[d][self.rank]:
                out[lo:hi].zero_()
            if self.compute is not None:
                self.compute(plan, self.mine[d], facs, out)
            else:
                coords, vals = _plan_arrays(plan, self.device)
                ev = kernel_events[d] if kernel_events is not None else None
                self._exec(d, rank_r).run(coords, vals, plan.nnz, plan.mode, facs, out, self.cfg,
                                          stream.cuda_stream, events=ev)
            if self.world > 1:
                allgather_owned_rows(out, self.ownership[d], self.group, ledger, step=d)
            if after_mode is not None:
                after_mode(d, out)
            if chained:
                facs[plan.mode] = out
        return self.outputs

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
