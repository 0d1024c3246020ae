"""N > 1 ranks over NCCL, one GPU per rank (skipped with fewer than 2 GPUs).

The same checks as tests/test_gpu_dist.py (which shares one GPU between two
gloo ranks), but with the production transport: NCCL broadcasts of owned
row ranges, the NCCL all-to-all of the distributed plan build, the fused
peer push over NVLink (CUDA IPC between two real GPUs) with its NCCL
completion barrier -- and bench.py's own self-launch of `--gpus 2`.
Reference semantics: engine.py:225-366 (devices, barrier, all-gather) and
collective.py:94-124 (ring all-gather == every rank ends with every row).
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 CUDA devices (one per NCCL rank)", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        import oracle
        import paper_2507_15121_b200 as sk
        from paper_2507_15121_b200.distplan import build_mode_plan_distributed
        from paper_2507_15121_b200.distributed import DistributedMttkrp

        assert dist.get_backend() == "nccl" and dist.get_world_size() == world
        shape, nnz = (3000, 2000, 1000), 2_000_000
        full = sk.synth_tensor_device(shape, nnz, seed=3, device=dev)
        fc, fv = full.device_arrays()
        lo, hi = nnz * rank // world, nnz * (rank + 1) // world
        chunk = sk.SparseTensorCOO.from_device(shape, [c[lo:hi].contiguous() for c in fc], fv[lo:hi].contiguous())
        pcfg = sk.PartitionConfig(devices=world)
        fs = sk.random_factors(shape, 32, seed=1)
        dev_f = [torch.from_numpy(f.data.astype(np.float32)).to(dev) for f in fs]
        host_idx, host_val = full.indices, full.values
        outs_by = {}
        for name, cfg in [("det", sk.PlatformConfig(devices=world, rank=32)),
                          ("atomic-contig", sk.PlatformConfig(devices=world, rank=32, accumulation="atomic",
                                                              scheduling="contiguous", layout="auto")),
                          ("fused", sk.PlatformConfig(devices=world, rank=32, layout="panel", fused_allgather=True,
                                                      scheduling="contiguous"))]:
            plans = [build_mode_plan_distributed(chunk, d, pcfg) for d in range(3)]
            runner = DistributedMttkrp(plans, cfg, device=dev)
            outs = [o.double().cpu().numpy() for o in runner.run(dev_f)]
            if name == "fused":
                assert all(runner._fused(d) for d in range(3))
            facs = [f.data.copy() for f in fs]
            for d in range(3):
                expect = oracle.mttkrp_seq_c(host_idx, host_val, facs, d)
                err = np.max(np.abs(outs[d] - expect) / np.maximum(np.abs(expect), 1.0))
                assert err <= 1e-4, (name, d, err)
                facs[d] = outs[d]
            outs_by[name] = outs
            runner._close_peers()
        # deterministic-reduce: bit-identical to the single-GPU run of the same plans
        single = DistributedMttkrp(sk.build_all_plans(full, pcfg), sk.PlatformConfig(devices=1, rank=32),
                                   rank=0, world=1, device=dev)
        one = [o.double().cpu().numpy() for o in single.run(dev_f)]
        assert all(np.array_equal(a, b) for a, b in zip(one, outs_by["det"]))
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()[-3000:]))
    finally:
        dist.destroy_process_group()


def test_two_nccl_ranks_build_run_and_fused_push():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_bench_gpus2_self_launch_over_nccl():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["BENCH_DIST_BACKEND"] = "nccl"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "cfg1",
                        "--steps", "3", "--warmup", "3", "--no-cpu"], capture_output=True, text=True, env=env,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["config"]["dist_backend"] == "nccl"
    assert line["parity"]["ok"]
    assert "nRanks 2" in r.stderr or "nranks 2" in r.stderr.lower()
