"""N>1 host logic under torch.distributed (gloo, world_size 2, CPU).

The multi-GPU path (distributed.DistributedMttkrp) is one process per GPU:
shard placement per rank, zeroing of owned rows, per-rank compute, in-place
broadcast of owned row ranges, chained factor replacement.  Here the same
object runs on CPU tensors under gloo with the per-shard compute supplied by
the CPU oracle (injected; the product default is the CUDA kernel), and the
gathered chained outputs must equal the single-process oracle chain exactly.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2507_15121_b200.collective import TransferLedger, allgather_owned_rows
from paper_2507_15121_b200.distributed import DistributedMttkrp, ownership_table, rows_cover
from paper_2507_15121_b200.engine import PlatformConfig
from paper_2507_15121_b200.partition import ModePartitionPlan


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cpu_plans(idx, vals, shape, devices, cap, strategy):
    plans = []
    for d in range(len(shape)):
        p = oracle.plan(idx, shape, d, devices, 4, cap, strategy)
        sidx = idx[p["order"]]
        coords = [torch.from_numpy(sidx[:, w].astype(np.int32)) for w in range(len(shape))]
        plan = ModePartitionPlan(d, shape, strategy, cap, "cpu", coords, torch.from_numpy(vals[p["order"]]),
                                 None, p["bounds"], p["offsets"])
        plan._host_idx = sidx
        plan._host_vals = vals[p["order"]]
        plans.append(plan)
    return plans


def _oracle_compute(cap):
    def compute(plan, shard_ids, facs, out):
        mats = [f.numpy() for f in facs]
        for j in shard_ids:
            sh = plan.shards[j]
            if sh.nnz == 0:
                continue
            part = oracle.engine_mode(plan._host_idx[sh.start:sh.stop], plan._host_vals[sh.start:sh.stop],
                                      plan.mode, np.array([0, sh.nnz]), cap, mats, 1)
            lo, hi = sh.index_range
            out[lo:hi] += torch.from_numpy(part[lo:hi])
    return compute


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = np.load(os.path.join(os.path.dirname(__file__), "golden", "synth.npz"))
        for name, strategy, sched in [("z3", "nnz-balanced", "dynamic"), ("u5", "equal-index", "static"),
                                      ("u3", "equal-index", "contiguous")]:
            idx, vals = s[f"{name}_indices"], s[f"{name}_values"]
            shape = tuple(int(x) for x in s[f"{name}_shape"])
            facs0 = [s[f"{name}_F8_{w}"] for w in range(len(shape))]
            cap = 37
            plans = _cpu_plans(idx, vals, shape, world, cap, strategy)
            cfg = PlatformConfig(devices=world, rank=8, scheduling=sched)
            runner = DistributedMttkrp(plans, cfg, device=torch.device("cpu"), compute=_oracle_compute(cap))
            for d, p in enumerate(plans):
                assert rows_cover(runner.ownership[d], p.shape[d])
                assert runner.ownership[d] == ownership_table(p, world, sched)
            outs = runner.run([torch.from_numpy(f.copy()) for f in facs0])
            expect = oracle.all_modes_chained(idx, vals, shape, facs0, devices=world, isp_capacity=cap,
                                              strategy=strategy)
            for o, e in zip(outs, expect):
                assert np.array_equal(o.numpy(), e), name
            if sched in ("dynamic", "contiguous"):
                # rebalancing from measured per-GPU times: rank 0 "ran" 3x slower,
                # so it sheds nonzeros; the outputs stay exact
                before = [sum(plans[d].shards[j].nnz for j in runner.assignment[d][0]) for d in range(len(plans))]
                secs = [[3.0 * max(b, 1) for b in before],
                        [float(max(sum(plans[d].shards[j].nnz for j in runner.assignment[d][1]), 1))
                         for d in range(len(plans))]]
                changed = runner.rebalance(rank_seconds=secs)
                after = [sum(plans[d].shards[j].nnz for j in runner.assignment[d][0]) for d in range(len(plans))]
                assert changed and all(a_ <= b_ for a_, b_ in zip(after, before)) and sum(after) < sum(before)
                for d, p in enumerate(plans):
                    assert rows_cover(runner.ownership[d], p.shape[d])
                outs = runner.run([torch.from_numpy(f.copy()) for f in facs0])
                for o, e in zip(outs, expect):
                    assert np.array_equal(o.numpy(), e), (name, "rebalanced")
        # ragged all-gather with a ledger: every rank ends with every row
        rows = 23
        own = [[(0, 5), (9, 14)], [(5, 9), (14, 23)]]
        buf = torch.full((rows, 3), -1.0, dtype=torch.float64)
        truth = torch.arange(rows * 3, dtype=torch.float64).reshape(rows, 3)
        for lo, hi in own[rank]:
            buf[lo:hi] = truth[lo:hi]
        ledger = TransferLedger()
        allgather_owned_rows(buf, own, ledger=ledger)
        assert torch.equal(buf, truth)
        sent = sum(hi - lo for lo, hi in own[rank]) * 3 * 8
        assert ledger.total_bytes("allgather") == sent
        q.put((rank, "ok"))
    except Exception as exc:  # pragma: no cover - reported to the parent
        q.put((rank, repr(exc)))
    finally:
        dist.destroy_process_group()


def test_two_rank_chained_all_modes_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: "ok", 1: "ok"}, results


def test_bench_self_launches_world_of_gpus():
    """`python bench.py --gpus 2` without torchrun's environment re-launches
    itself as 2 ranks (torch.distributed.run) and the group really has 2
    members (gloo here; NCCL on the GPU box)."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["BENCH_DIST_BACKEND"] = "gloo"
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["world_size"] == 2 and line["backend"] == "gloo"
    assert line["self_launched"] is True


def test_bench_refuses_world_mismatch():
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)
