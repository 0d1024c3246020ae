"""Host <-> HBM transfers for the drop-in (numpy, float64) API.

The reference API takes and returns float64 numpy factor matrices
(engine.py:83-88 make_devices, engine.py:366 / 400 mttkrp_mode /
mttkrp_all_modes).  The device path computes in fp32, so every call converts.
Doing that conversion on the host (numpy astype, one thread) or copying
through pageable memory costs more than the MTTKRP itself at cfg2 sizes
(~1.2 GB of fp64 per 4.8 M x 32 factor), so the transfers here are:

* upload: fp64 rows are narrowed to fp32 by the host threads straight into a
  ring of pinned staging chunks (round to nearest even, as the GPU's
  conversion), and each chunk crosses PCIe as fp32 -- half the bytes --
  while the host fills the next one;
* download: the fp32 result crosses PCIe as fp32 chunk by chunk on a side
  stream into pinned staging, and the host threads widen landed chunks into
  the fresh float64 array (exact) while the next chunks are in flight --
  started right after the mode's kernel, so it overlaps the next mode's
  compute (ExportQueue).  Host memory traffic per element: 12 B instead of
  16, PCIe 4 B instead of 8 (profiles/r02/r02aj_e2e_api_breakdown.json: the
  drop-in call is host-memory bound).

Staging buffers are cached per device and reused across calls (no pinned
allocation on the hot path).
"""

from __future__ import annotations

import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import _lib

_CHUNK_BYTES = 64 << 20   # per staging chunk
_NBUF = 3                 # staging ring depth
_POOL = None         # memcpy workers
_EXPORTS = None      # one export thread (exports share the staging ring anyway)
_STAGING = {}
_LOCK = threading.Lock()


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=max(2, min(16, os.cpu_count() or 2)))
    return _POOL


def _exports():
    global _EXPORTS
    if _EXPORTS is None:
        _EXPORTS = ThreadPoolExecutor(max_workers=1)
    return _EXPORTS


def _copyto(dst: np.ndarray, src: np.ndarray):
    # fp64 -> fp32 narrowing: out-of-range values become +-inf silently, as
    # the device conversion does (the caller's finiteness checks decide)
    with np.errstate(over="ignore", invalid="ignore"):
        np.copyto(dst, src, casting="unsafe")


def _par_copy(dst: np.ndarray, src: np.ndarray):
    """dst[...] = src (with a dtype cast) for two flat same-length arrays,
    split across threads (numpy releases the GIL on large copies)."""
    n = dst.shape[0]
    parts = max(1, min(_pool()._max_workers, n // (1 << 20)))
    if parts == 1:
        _copyto(dst, src)
        return
    cuts = [n * i // parts for i in range(parts + 1)]
    futs = [_pool().submit(_copyto, dst[cuts[i]:cuts[i + 1]], src[cuts[i]:cuts[i + 1]]) for i in range(parts)]
    for f in futs:
        f.result()


class _Staging:
    """Ring of pinned host chunks + device fp64 chunks + events for one GPU."""

    def __init__(self, dev):
        import torch

        self.dev = dev
        n = _CHUNK_BYTES // 8
        self.host = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(_NBUF)]
        self.hnp = [h.numpy() for h in self.host]
        # fp32 views of the same pinned chunks (n elements use half a chunk)
        self.host32 = [h.view(torch.float32) for h in self.host]
        self.hnp32 = [h.numpy() for h in self.host32]
        self.ev = [torch.cuda.Event() for _ in range(_NBUF)]
        self.stream = torch.cuda.Stream(dev)
        self.n = n
        self.lock = threading.Lock()


def staging(dev) -> _Staging:
    key = str(dev)
    with _LOCK:
        st = _STAGING.get(key)
        if st is None:
            st = _Staging(dev)
            _STAGING[key] = st
    return st


def upload_f64(arr, dev):
    """float64 numpy (rows x R) -> new fp32 device tensor (contiguous)."""
    import torch

    a = np.ascontiguousarray(arr, dtype=np.float64)
    out = torch.empty(a.shape, dtype=torch.float32, device=dev)
    flat = a.reshape(-1)
    total = flat.shape[0]
    if total == 0:
        return out
    st = staging(dev)
    cur = torch.cuda.current_stream(dev)
    with st.lock:
        st.stream.wait_stream(cur)
        k = 0
        for a0 in range(0, total, st.n):
            b = k % _NBUF
            n = min(st.n, total - a0)
            st.ev[b].synchronize()  # the chunk's previous H2D is done
            _par_copy(st.hnp32[b][:n], flat[a0:a0 + n])  # fp64 -> fp32, round to nearest even
            with torch.cuda.stream(st.stream):
                out.view(-1)[a0:a0 + n].copy_(st.host32[b][:n], non_blocking=True)
                st.ev[b].record(st.stream)
            k += 1
        cur.wait_stream(st.stream)
    return out


class ExportQueue:
    """Device fp32 matrices -> fresh float64 numpy arrays, overlapped with
    later GPU work: ``push(t)`` enqueues the conversion + D2H on the staging
    stream right away (after the work already on the current stream) and a
    host thread copies the landed chunks out; ``results()`` waits and returns
    the arrays in push order."""

    def __init__(self, dev):
        self.dev = dev
        self.jobs = []

    def push(self, t):
        import torch

        st = staging(self.dev)
        src = t.detach()
        if src.dtype != torch.float32 or not src.is_contiguous():
            src = src.float().contiguous()
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.dev))
        out = np.empty(tuple(src.shape), dtype=np.float64)
        job = _exports().submit(self._export, st, src, ready, out)
        self.jobs.append((job, out))

    @staticmethod
    def _export(st, src, ready, out):
        import torch

        flat_out = out.reshape(-1)
        total = flat_out.shape[0]
        if total == 0:
            return
        flat = src.view(-1)
        with st.lock, torch.cuda.device(st.dev):
            st.stream.wait_event(ready)
            pend = []
            k = 0
            for a0 in range(0, total, st.n):
                b = k % _NBUF
                n = min(st.n, total - a0)
                if len(pend) == _NBUF:  # ring full: drain the oldest chunk
                    pb, pa, pn = pend.pop(0)
                    st.ev[pb].synchronize()
                    _par_copy(flat_out[pa:pa + pn], st.hnp32[pb][:pn])  # fp32 -> fp64, exact
                with torch.cuda.stream(st.stream):
                    st.host32[b][:n].copy_(flat[a0:a0 + n], non_blocking=True)
                    st.ev[b].record(st.stream)
                pend.append((b, a0, n))
                k += 1
            for pb, pa, pn in pend:
                st.ev[pb].synchronize()
                _par_copy(flat_out[pa:pa + pn], st.hnp32[pb][:pn])

    def results(self):
        outs = []
        for job, out in self.jobs:
            job.result()
            outs.append(out)
        self.jobs = []
        return outs
