"""CP-ALS on the B200 engine (drop-in for shardkrp.cpd).

Same API and update rule as the reference (cpd.py:22-167): per mode, the
engine MTTKRP (not chained), V = Hadamard product of the other modes' Grams,
the normal-equations solve with the 1e-12*tr(V)/R jitter then pinv fallback,
column normalisation into lambdas (zero norms left unscaled), and the fit
1 - ||X - Xhat|| / ||X|| through the sparse identity.

Placement: every I x R quantity stays on the GPU (MTTKRP output, Grams'
inputs, the solved factor, normalisation, the <X, Xhat> pass over the
nonzeros); only R x R matrices and R-vectors cross to the host, where the
R x R solve runs in float64 exactly as the reference does it.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import PlatformConfig, make_devices, mttkrp, mttkrp_mode
from .metrics import RunMetrics
from .partition import PartitionConfig, build_all_plans
from .tensor import FactorMatrix, SparseTensorCOO, random_factors


@dataclass
class CpModel:
    factors: list
    lambdas: np.ndarray
    fit_history: list = field(default_factory=list)

    @property
    def rank(self) -> int:
        return len(self.lambdas)


def _is_torch(x) -> bool:
    return hasattr(x, "data_ptr") and hasattr(x, "device")


def gram(factor) -> np.ndarray:
    """Y^T Y (cpd.py:33-36).  Device tensors are reduced on the GPU in fp64."""
    if _is_torch(factor):
        return _gram_device(factor)
    y = factor.data if isinstance(factor, FactorMatrix) else np.asarray(factor)
    return y.T @ y


def _gram_device(y) -> np.ndarray:
    import torch

    rows, rank = y.shape
    g = torch.empty((rank, rank), dtype=torch.float64, device=y.device)
    _lib.call("skrp_gram", y.data_ptr(), rows, rank, g.data_ptr(), torch.cuda.current_stream(y.device).cuda_stream)
    return g.cpu().numpy()


def _solve_matrix(v: np.ndarray) -> np.ndarray:
    """W with M @ W == solve(V, M^T)^T, with the reference's fallbacks."""
    rank = v.shape[0]
    eye = np.eye(rank)
    try:
        return np.linalg.solve(v, eye).T
    except np.linalg.LinAlgError:
        jitter = 1e-12 * np.trace(v) / rank
        try:
            return np.linalg.solve(v + jitter * eye, eye).T
        except np.linalg.LinAlgError:
            return np.linalg.pinv(v)


def _hadamard(grams, rank):
    v = np.ones((rank, rank))
    for g in grams:
        v = v * g
    return v


def als_update(mttkrp_out, grams):
    """Solve the mode's least-squares problem and normalise (cpd.py:39-67).

    Host arrays follow the reference exactly; a device tensor stays on the
    GPU (M @ W on the GPU with W from the host R x R solve)."""
    if _is_torch(mttkrp_out):
        return _als_update_device(mttkrp_out, grams)
    if not np.isfinite(mttkrp_out).all():
        raise FloatingPointError("non-finite MTTKRP output")
    rank = mttkrp_out.shape[1]
    v = _hadamard(grams, rank)
    if not np.isfinite(v).all():
        raise FloatingPointError("non-finite Gram product")
    solved = mttkrp_out @ _solve_matrix(v)
    lambdas = np.linalg.norm(solved, axis=0)
    safe = np.where(lambdas > 0, lambdas, 1.0)
    return solved / safe, lambdas


def mm_fp32(a, b, out=None):
    """Plain fp32 GEMM through cuBLAS with TF32 forced off (a global TF32
    switch would break the reference's 1e-4 tolerance)."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return torch.mm(a, b, out=out)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def _col_sumsq(x) -> np.ndarray:
    import torch

    rows, rank = x.shape
    out = torch.empty(rank, dtype=torch.float64, device=x.device)
    _lib.call("skrp_col_sumsq", x.data_ptr(), rows, rank, out.data_ptr(), torch.cuda.current_stream(x.device).cuda_stream)
    return out.cpu().numpy()


def _als_update_device(m, grams):
    import torch

    rows, rank = m.shape
    stream = torch.cuda.current_stream(m.device).cuda_stream
    v = _hadamard(grams, rank)
    fused = rank in (16, 32, 64) and m.is_contiguous() and m.data_ptr() % 16 == 0
    if not fused or not np.isfinite(v).all():
        # reference order (cpd.py): the MTTKRP output is checked before V
        if not np.isfinite(_col_sumsq(m)).all():
            raise FloatingPointError("non-finite MTTKRP output")
        if not np.isfinite(v).all():
            raise FloatingPointError("non-finite Gram product")
    if fused:
        # M @ W, the new columns' sums of squares and the non-finite probe of M
        # in one pass (skrp_apply_rr_sumsq)
        w64 = torch.from_numpy(np.ascontiguousarray(_solve_matrix(v))).to(m.device)
        solved = torch.empty_like(m)
        sq = torch.empty(rank, dtype=torch.float64, device=m.device)
        bad = torch.empty(1, dtype=torch.int32, device=m.device)
        _lib.call("skrp_apply_rr_sumsq", m.data_ptr(), rows, rank, w64.data_ptr(), solved.data_ptr(),
                  sq.data_ptr(), bad.data_ptr(), stream)
        if int(bad.item()):
            raise FloatingPointError("non-finite MTTKRP output")
        lambdas = np.sqrt(sq.cpu().numpy())
    else:
        w = torch.from_numpy(np.ascontiguousarray(_solve_matrix(v))).to(m.device, dtype=torch.float32)
        solved = mm_fp32(m, w)  # plain GEMM (rows x R) @ (R x R): cuBLAS fp32
        lambdas = np.sqrt(_col_sumsq(solved))
    if not np.isfinite(lambdas).all():
        raise FloatingPointError("non-finite entries in updated factor matrix")
    scale = torch.from_numpy(1.0 / np.where(lambdas > 0, lambdas, 1.0)).to(m.device)
    _lib.call("skrp_scale_cols", solved.data_ptr(), rows, rank, scale.data_ptr(), stream)
    return solved, lambdas


def _device_inner(tensor: SparseTensorCOO, dev_factors, lambdas):
    """(<X, Xhat>, ||X||^2) with Xhat = sum_r lambda_r prod_w F_w[:, r]."""
    import torch

    coords, vals = tensor.device_arrays(dev_factors[0].device)
    rank = dev_factors[0].shape[1]
    out = torch.empty(2, dtype=torch.float64, device=vals.device)
    lam = torch.from_numpy(np.ascontiguousarray(lambdas, dtype=np.float64)).to(vals.device)
    cptr = (_lib.vp * len(coords))(*[c.data_ptr() for c in coords])
    fptr = (_lib.vp * len(dev_factors))(*[f.data_ptr() for f in dev_factors])
    _lib.call("skrp_model_inner", cptr, vals.data_ptr(), tensor.nnz, len(coords), fptr, lam.data_ptr(), rank,
              out.data_ptr(), torch.cuda.current_stream(vals.device).cuda_stream)
    inner, sq = out.cpu().numpy()
    return float(inner), float(sq)


def _fused_inner(new, m_out, lambdas) -> float:
    """<X, Xhat> = sum_r lambda_r sum_i F_last[i, r] M_last[i, r]: the last
    mode's MTTKRP output already holds sum over its nonzeros of
    v * prod_{w < last} F_w, so the fit needs no pass over the nonzeros."""
    import torch

    rows, rank = new.shape
    lam = torch.from_numpy(np.ascontiguousarray(lambdas, dtype=np.float64)).to(new.device)
    out = torch.empty(1, dtype=torch.float64, device=new.device)
    _lib.call("skrp_weighted_dot", new.data_ptr(), m_out.data_ptr(), rows, rank, lam.data_ptr(), out.data_ptr(),
              torch.cuda.current_stream(new.device).cuda_stream)
    return float(out.item())


def _device_sumsq(tensor) -> float:
    import torch

    _, vals = tensor.device_arrays()
    out = torch.empty(1, dtype=torch.float64, device=vals.device)
    _lib.call("skrp_sumsq", vals.data_ptr(), tensor.nnz, out.data_ptr(),
              torch.cuda.current_stream(vals.device).cuda_stream)
    return float(out.item())


def _fit_value(x_sq, inner, grams, lambdas):
    if x_sq == 0.0:
        raise ValueError("tensor has zero Frobenius norm; fit undefined")
    g = _hadamard(grams, len(lambdas))
    model_sq = float(lambdas @ g @ lambdas)
    resid = max(x_sq - 2.0 * inner + model_sq, 0.0)
    return 1.0 - np.sqrt(resid) / np.sqrt(x_sq)


def _x_sq(tensor, device_sq):
    if tensor._values is not None:
        v = tensor._values.astype(np.float64)
        return float(np.dot(v, v))
    return device_sq


def fit(tensor: SparseTensorCOO, model: CpModel) -> float:
    """1 - relative reconstruction error (cpd.py:84-105), <X, Xhat> on the GPU."""
    import torch

    gpu = torch.device("cuda", torch.cuda.current_device())
    facs = [torch.from_numpy(np.ascontiguousarray(f.data)).to(gpu, dtype=torch.float32) for f in model.factors]
    inner, sq = _device_inner(tensor, facs, model.lambdas)
    return _fit_value(_x_sq(tensor, sq), inner, [gram(f) for f in model.factors], np.asarray(model.lambdas))


def cp_als(tensor: SparseTensorCOO, rank: int, iterations: int, platform: PlatformConfig | None = None,
           seed: int = 0, partition: PartitionConfig | None = None, mttkrp_impl: str = "engine",
           fit_tol: float | None = None):
    """Alternating least squares CP decomposition (cpd.py:108-167).

    mttkrp_impl: "engine" -- the sharded multi-device engine; "oracle" --
    the single-call per-mode ``mttkrp`` (one device, its own plan), kept as
    the reference's cross-check switch (both run on the GPU).
    """
    import torch

    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    if mttkrp_impl not in ("engine", "oracle"):
        raise ValueError("mttkrp_impl must be 'engine' or 'oracle'")
    platform = platform or PlatformConfig(rank=rank)
    partition = partition or PartitionConfig(devices=platform.devices,
                                             workers_per_device=platform.workers_per_device)
    init = random_factors(tensor.shape, rank, seed)
    metrics = RunMetrics(devices=platform.devices)
    devices = make_devices(init, platform)
    plans = []
    if mttkrp_impl == "engine":
        plans = build_all_plans(tensor, partition, keep_permutation=False)
        metrics.preprocessing_seconds = [p.build_time for p in plans]
    cur = list(devices[0].factors)  # fp32 device factors (replicated on devices)
    grams = [_gram_device(f) for f in cur]
    lambdas = np.ones(rank)
    history = []
    x_sq = None
    for _ in range(iterations):
        for d in range(tensor.num_modes):
            if mttkrp_impl == "engine":
                m_out, mm = mttkrp_mode(plans[d], devices, platform, update_factors=False, as_numpy=False)
                metrics.modes.append(mm)
            else:
                m_out = mttkrp(tensor, cur, d, as_numpy=False)
            new, lambdas = _als_update_device(m_out, [grams[w] for w in range(tensor.num_modes) if w != d])
            if d == tensor.num_modes - 1:
                inner = _fused_inner(new, m_out, lambdas)
            cur[d] = new
            grams[d] = _gram_device(new)
            for dev in devices:
                dev.factors[d] = new if new.device == dev.cuda_device else new.to(dev.cuda_device)
        if x_sq is None:
            x_sq = _x_sq(tensor, None) if tensor._values is not None else _device_sumsq(tensor)
        history.append(_fit_value(x_sq, inner, grams, lambdas))
        if fit_tol is not None and len(history) > 1 and history[-1] - history[-2] < fit_tol:
            break
    factors = [FactorMatrix(w, f.double().cpu().numpy()) for w, f in enumerate(cur)]
    return CpModel(factors, lambdas, fit_history=history), metrics
