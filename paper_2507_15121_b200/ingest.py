"""GPU .tns ingestion.

``parse_tns_gpu`` has the contract of the reference's ``parse_tns``
(tensor.py:173-247; host restatement in tensor.py here): same arrays, shape,
LoadStats and the same exceptions/messages, but the bytes are split into
lines, classified and converted on the GPU (csrc/tns.cu).  Tokens outside the
kernel's fast grammar (underscores, hex, over-long significands whose rounding
the kernel cannot decide, anything invalid) come back FLAGGED and only those
tokens are converted here with Python's int()/float() -- which is also what
produces the reference's error messages.  Duplicate coalescing (rare; the
reference sums them in first-occurrence order with np.add.at) runs on the
host.  The returned tensor keeps its device arrays (int32 coordinates, fp32
values), so plan building needs no second upload.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .tensor import DEFAULT_VALUE_DTYPE, LoadStats, SparseTensorCOO, TnsFormatError

_CHUNK = 1 << 16


def _read_bytes(source):
    if isinstance(source, (str, os.PathLike)):
        return np.fromfile(source, dtype=np.uint8), str(source)
    if isinstance(source, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytes(source), dtype=np.uint8), ""
    data = source.read()
    if isinstance(data, str):
        data = data.encode()
    return np.frombuffer(data, dtype=np.uint8), ""


def _line_text(host, starts, n_nl, i):
    lo = int(starts[i])
    hi = int(starts[i + 1]) - 1 if i < n_nl else len(host)
    return bytes(host[lo:hi]).decode(errors="replace")


def parse_tns_gpu(source, coalesce_duplicates: bool = False, shape=None, value_dtype=DEFAULT_VALUE_DTYPE,
                  name: str = "", device=None) -> SparseTensorCOO:
    """FROSTT text -> tensor on the GPU; see the module docstring."""
    import torch

    host, src_name = _read_bytes(source)
    name = name or src_name
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev).cuda_stream
    n = int(host.size)
    if n == 0:
        raise TnsFormatError("no data lines")
    if not host.flags.writeable:
        host = host.copy()
    text = torch.from_numpy(np.ascontiguousarray(host)).to(dev)
    nch = -(-n // _CHUNK)
    counts = torch.empty(nch, dtype=torch.int64, device=dev)
    _lib.call("skrp_tns_count_lines", text.data_ptr(), n, _CHUNK, counts.data_ptr(), stream)
    offs = torch.empty(nch + 1, dtype=torch.int64, device=dev)
    wsb = _lib.lib().skrp_scan_workspace_bytes(nch)
    ws = torch.empty(max(int(wsb), 16), dtype=torch.uint8, device=dev)
    _lib.call("skrp_exclusive_scan_i64", counts.data_ptr(), nch, offs.data_ptr(), ws.data_ptr(), wsb, stream)
    n_nl = int(offs[-1].item())
    starts = torch.zeros(n_nl + 1, dtype=torch.int64, device=dev)
    _lib.call("skrp_tns_line_starts", text.data_ptr(), n, _CHUNK, offs.data_ptr(), starts.data_ptr(), stream)
    nlines = n_nl + (1 if host[-1] != ord("\n") else 0)
    kind = torch.empty(nlines, dtype=torch.int8, device=dev)
    ntok = torch.empty(nlines, dtype=torch.int32, device=dev)
    _lib.call("skrp_tns_classify", text.data_ptr(), n, starts.data_ptr(), n_nl, nlines, kind.data_ptr(),
              ntok.data_ptr(), stream)
    starts_h = starts.cpu().numpy()

    # the reference walks lines in order and raises at the first bad one:
    # a malformed '# shape:' comment, the first data line's column count, or
    # the first data line whose column count differs
    data_lines = torch.nonzero(kind == 2).squeeze(1)
    first_data = int(data_lines[0].item()) if data_lines.numel() else nlines
    ncols = int(ntok[first_data].item()) if data_lines.numel() else None
    first_bad = nlines
    if ncols is not None:
        if ncols < 4:
            first_bad = first_data
        else:
            bad = torch.nonzero((kind == 2) & (ntok != ncols)).squeeze(1)
            if bad.numel():
                first_bad = int(bad[0].item())
    header = None
    for i in torch.nonzero(kind == 1).squeeze(1).cpu().numpy():
        if i > first_bad:
            break
        body = _line_text(host, starts_h, n_nl, int(i)).strip()[1:].strip()
        if body.lower().startswith("shape:"):
            header = tuple(int(t) for t in body[len("shape:"):].split())
    if first_bad < nlines:
        if first_bad == first_data:
            raise TnsFormatError(f"line {first_bad + 1}: expected at least 3 index columns and a value, "
                                 f"got {ncols} columns")
        got = int(ntok[first_bad].item())
        raise TnsFormatError(f"line {first_bad + 1}: inconsistent column count ({got} vs {ncols})")
    if ncols is None:
        raise TnsFormatError("no data lines")

    nm = ncols - 1
    idx_all = torch.empty((nlines, nm), dtype=torch.int64, device=dev)
    vals_all = torch.empty(nlines, dtype=torch.float64, device=dev)
    flags_all = torch.zeros(nlines, dtype=torch.int32, device=dev)
    _lib.call("skrp_tns_parse", text.data_ptr(), n, starts.data_ptr(), n_nl, nlines, kind.data_ptr(), nm,
              idx_all.data_ptr(), vals_all.data_ptr(), flags_all.data_ptr(), stream)
    idx = idx_all.index_select(0, data_lines)
    vals = vals_all.index_select(0, data_lines)
    flags = flags_all.index_select(0, data_lines)
    del idx_all, vals_all, flags_all
    flagged = torch.nonzero(flags != 0).squeeze(1).cpu().numpy()
    if len(flagged):
        fl = flags.index_select(0, torch.from_numpy(flagged).to(dev)).cpu().numpy().astype(np.uint32)
        lines = data_lines.index_select(0, torch.from_numpy(flagged).to(dev)).cpu().numpy()
        toks = [_line_text(host, starts_h, n_nl, int(li)).split() for li in lines]
        # indices first, then values -- the reference's conversion order
        fixed_i = {}
        try:
            for r, f, tk in zip(flagged, fl, toks):
                for w in range(nm):
                    if f & (1 << w):
                        v = int(tk[w])
                        np.array([v], dtype=np.int64)  # OverflowError like the reference's np.array
                        fixed_i[(int(r), w)] = v
            fixed_v = {}
            for r, f, tk in zip(flagged, fl, toks):
                if f & (1 << 31):
                    fixed_v[int(r)] = float(tk[nm])
        except ValueError as exc:
            raise TnsFormatError(f"non-numeric token: {exc}") from None
        if fixed_i:
            rr = torch.tensor([k[0] for k in fixed_i], dtype=torch.int64, device=dev)
            ww = torch.tensor([k[1] for k in fixed_i], dtype=torch.int64, device=dev)
            idx[rr, ww] = torch.tensor(list(fixed_i.values()), dtype=torch.int64, device=dev)
        if fixed_v:
            rr = torch.tensor(list(fixed_v), dtype=torch.int64, device=dev)
            vals[rr] = torch.tensor(list(fixed_v.values()), dtype=torch.float64, device=dev)
    nonpos = torch.nonzero((idx <= 0).any(dim=1)).squeeze(1)
    if nonpos.numel():
        raise TnsFormatError(f"data line {int(nonpos[0].item()) + 1}: index must be >= 1 (1-based format)")
    idx -= 1
    vt = torch.float64 if np.dtype(value_dtype) == np.float64 else torch.float32
    vals = vals.to(vt)
    stats = LoadStats(nnz=int(vals.numel()), zero_values=int((vals == 0).sum().item()))
    ndup = int(idx.shape[0] - torch.unique(idx, dim=0).shape[0])
    idx_h = idx.cpu().numpy()
    vals_h = vals.cpu().numpy()
    if ndup:
        if not coalesce_duplicates:
            raise TnsFormatError(f"{ndup} duplicate coordinate tuple(s); pass coalesce_duplicates=True to sum them")
        uniq, first, inv = np.unique(idx_h, axis=0, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")
        rank_of = np.empty(len(uniq), dtype=np.int64)
        rank_of[order] = np.arange(len(uniq))
        summed = np.zeros(len(uniq), dtype=vals_h.dtype)
        np.add.at(summed, rank_of[inv.reshape(-1)], vals_h)
        idx_h, vals_h = uniq[order], summed
        stats.coalesced = True
    stats.duplicates = ndup
    stats.nnz = len(vals_h)
    if shape is None:
        shape = header if header is not None else tuple(int(m) + 1 for m in idx_h.max(axis=0))
    t = SparseTensorCOO(shape, idx_h, vals_h, name=name)
    t.stats = stats
    if not ndup and all(s < 2 ** 31 for s in t.shape):
        # keep the parsed arrays resident: plan building reads them directly
        t._dev = ([idx[:, w].to(torch.int32).contiguous() for w in range(nm)], vals.to(torch.float32))
    return t
