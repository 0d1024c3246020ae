"""ctypes binding of libshardkrp_cuda.so (include/shardkrp_cuda.h).

The product path has exactly one compute backend: this library.  There is no
CPU fallback -- if the .so is missing or a call fails, an exception is raised
(status codes map to the reference's exception types: SKRP_ERR_INVALID ->
ValueError, SKRP_ERR_NONFINITE -> FloatingPointError, SKRP_ERR_NOMEM ->
MemoryError, SKRP_ERR_CUDA -> RuntimeError).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libshardkrp_cuda.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "shardkrp_cuda.h")

SKRP_OK, SKRP_ERR_INVALID, SKRP_ERR_CUDA, SKRP_ERR_NOMEM, SKRP_ERR_NONFINITE = 0, 1, 2, 3, 4
SKRP_MAX_MODES = 8
ACC_DETERMINISTIC, ACC_ATOMIC = 0, 1
FLAG_ADDITIVE = 1
FLAG_STREAM_INPUT0 = 2
FLAG_STREAM_INPUT1 = 4
FLAG_FIBER_INPUT0 = 16
FLAG_FIBER_INPUT1 = 32
FLAG_FIBER_INPUT2 = 64
PANEL_LOCKSTEP = 1

vp = ctypes.c_void_p
i64 = ctypes.c_int64
i32 = ctypes.c_int32
u64 = ctypes.c_uint64
sz = ctypes.c_size_t


ABI_VERSION = 12  # bumped whenever a struct or signature in include/shardkrp_cuda.h changes


class MttkrpArgs(ctypes.Structure):
    _fields_ = [
        ("nmodes", i32),
        ("mode", i32),
        ("rank", i32),
        ("accumulation", i32),
        ("nnz", i64),
        ("coords", vp * SKRP_MAX_MODES),
        ("values", vp),
        ("factors", vp * SKRP_MAX_MODES),
        ("out", vp),
        ("tiles", vp),
        ("num_tiles", i64),
        ("carry_rows", vp),
        ("carry_vals", vp),
        ("work_counter", vp),
        ("persistent_ctas", i32),
        ("variant", i32),
        ("flags", i32),
        ("factor_ld", i32),
        ("out_ld", i32),
        ("reserved2", i32 * 2),
    ]


class PanelArgs(ctypes.Structure):
    _fields_ = [
        ("item_rows", vp),
        ("item_offsets", vp),
        ("num_items", i64),
        ("groups", i32),
        ("slab_rows", i32),
        ("warps", i32),
        ("flags", i32),
        ("peer_out", vp),
        ("num_peers", i32),
        ("reserved", i32),
    ]


class CellArgs(ctypes.Structure):
    _fields_ = [
        ("row_lo", i64),
        ("rows", i64),
        ("out_row_base", i64),
        ("stripe_offsets", vp),
        ("stripes", i64),
        ("stripe_rows", i32),
        ("ctas", i32),
        ("outer_mode", i32),
        ("inner_mode", i32),
        ("outer_shift", i32),
        ("inner_shift", i32),
        ("inner_blocks", i32),
        ("cells", i32),
        ("lag", i32),
        ("variant", i32),
        ("done", vp),
        ("entries", vp),
    ]


# name -> (restype, argtypes)
SIGNATURES = {
    "skrp_last_error": (i32, [ctypes.c_char_p, sz]),
    "skrp_abi_version": (i32, []),
    "skrp_launch_log": (i32, [i64, ctypes.c_char_p, sz, ctypes.POINTER(i64)]),
    "skrp_crc32_chunks": (i32, [vp, i64, i64, vp, vp]),
    "skrp_crc32_fold_host": (i32, [vp, i64, i64, i64, ctypes.c_uint32, vp]),
    "skrp_crc32_raw_host": (i32, [vp, i64, vp]),
    "skrp_plan_unpack_indices": (i32, [vp, i64, i32, vp, vp, vp]),
    "skrp_plan_pack_indices": (i32, [vp, i64, i32, vp, vp]),
    "skrp_f64_to_f32": (i32, [vp, i64, vp, vp]),
    "skrp_ipc_get_handle": (i32, [vp, vp, vp]),
    "skrp_ipc_open_handle": (i32, [vp, i64, vp, vp]),
    "skrp_ipc_close_handle": (i32, [vp]),
    "skrp_tns_count_lines": (i32, [vp, i64, i64, vp, vp]),
    "skrp_tns_line_starts": (i32, [vp, i64, i64, vp, vp, vp]),
    "skrp_tns_classify": (i32, [vp, i64, vp, i64, i64, vp, vp, vp]),
    "skrp_tns_parse": (i32, [vp, i64, vp, i64, i64, vp, i32, vp, vp, vp, vp]),
    "skrp_tns_parse_token_host": (i32, [ctypes.c_char_p, i64, i32, vp, vp]),
    "skrp_mttkrp_panels": (i32, [vp, vp, vp]),
    "skrp_panel_shape": (i32, [i32, i32, vp, vp]),
    "skrp_mttkrp_cells": (i32, [vp, vp, vp]),
    "skrp_cell_shape": (i32, [i32, i32, vp, vp, vp]),
    "skrp_cell_keys": (i32, [vp, vp, vp, i64, i64, i32, i32, i32, i32, i32, vp, vp]),
    "skrp_cell_assign": (i32, [vp, i64, vp, i32, vp, vp, vp]),
    "skrp_cell_entries": (i32, [vp, vp, vp, i64, i32, i32, vp, vp, i64, i32, vp, vp, vp, vp, i64, i32, i32, vp, i64,
                                vp]),
    "skrp_device_sm_count": (i32, [ctypes.POINTER(i32)]),
    "skrp_histogram": (i32, [vp, i64, i64, vp, vp]),
    "skrp_scan_workspace_bytes": (sz, [i64]),
    "skrp_exclusive_scan_i64": (i32, [vp, i64, vp, vp, sz, vp]),
    "skrp_equal_index_bounds": (i32, [i64, i64, vp]),
    "skrp_nnz_balanced_bounds": (i32, [vp, i64, i64, vp]),
    "skrp_sort_workspace_bytes": (sz, [i64, ctypes.c_int]),
    "skrp_stable_sort_by_key": (i32, [vp, i64, ctypes.c_int, vp, vp, vp, sz, vp]),
    "skrp_gather_u32": (i32, [vp, vp, i64, vp, vp]),
    "skrp_block_keys": (i32, [vp, i32, vp, vp, vp, i64, i32, i64, vp, vp]),
    "skrp_mttkrp_tiles": (i32, [ctypes.POINTER(MttkrpArgs), vp]),
    "skrp_carry_fixup": (i32, [vp, vp, i32, vp, vp, i64, i32, vp, vp, vp, i32, vp]),
    "skrp_mttkrp_host": (i32, [vp, vp, i64, i32, vp, vp, i32, i32, vp, i32]),
    "skrp_synth_uniform_coords": (i32, [vp, i64, i64, u64, i32, i64, vp]),
    "skrp_synth_zipf_coords": (i32, [vp, i64, vp, i64, u64, i32, i64, vp]),
    "skrp_synth_values": (i32, [vp, i64, i32, u64, i64, vp]),
    "skrp_route_by_bounds": (i32, [vp, i64, vp, i64, vp, vp, vp]),
    "skrp_dedup_mark": (i32, [vp, i32, i64, vp, i64, vp, vp]),
    "skrp_gram": (i32, [vp, i64, i32, vp, vp]),
    "skrp_apply_rr": (i32, [vp, i64, i32, vp, vp, vp]),
    "skrp_apply_rr_sumsq": (i32, [vp, i64, i32, vp, vp, vp, vp, vp]),
    "skrp_col_sumsq": (i32, [vp, i64, i32, vp, vp]),
    "skrp_scale_cols": (i32, [vp, i64, i32, vp, vp]),
    "skrp_model_inner": (i32, [vp, vp, i64, i32, vp, vp, i32, vp, vp]),
    "skrp_weighted_dot": (i32, [vp, vp, i64, i32, vp, vp, vp]),
    "skrp_sumsq": (i32, [vp, i64, vp, vp]),
}

_LIB = None


def launch_log(clear=False):
    """(mode, demangled kernel name) of the MTTKRP kernels launched so far, in
    launch order; clear=True empties the log and returns []."""
    h = lib()
    cnt = i64()
    if clear:
        h.skrp_launch_log(-1, None, 0, ctypes.byref(cnt))
        return []
    buf = ctypes.create_string_buffer(1024)
    h.skrp_launch_log(1 << 62, buf, 1024, ctypes.byref(cnt))  # out of range: reports the count only
    out = []
    for k in range(cnt.value):
        check(h.skrp_launch_log(k, buf, 1024, None), "skrp_launch_log")
        m, name = buf.value.decode().split("\t", 1)
        out.append((int(m), name))
    return out


def build(force: bool = False):
    """Compile the library in-tree for sm_100a (make; nvcc cross-compiles)."""
    args = ["make", "-s", "-C", _HERE, "-j8"]
    if force:
        subprocess.run(["make", "-s", "-C", _HERE, "clean"], check=True)
    subprocess.run(args, check=True)


def lib():
    """Load the library (fail loudly if absent -- no fallback path exists)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                "(or __graft_entry__.build()); the shardkrp B200 path has no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        if handle.skrp_abi_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {handle.skrp_abi_version()}, this package needs {ABI_VERSION}: "
                              f"rebuild it with `make -C {_HERE}`")
        _LIB = handle
    return _LIB


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    lib().skrp_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def check(rc: int, name: str):
    if rc == SKRP_OK:
        return
    msg = f"{name}: {last_error()}"
    if rc == SKRP_ERR_INVALID:
        raise ValueError(msg)
    if rc == SKRP_ERR_NONFINITE:
        raise FloatingPointError(msg)
    if rc == SKRP_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    rc = getattr(lib(), name)(*args)
    check(rc, name)
    return rc


def ptr(t) -> int:
    """Raw device (or host) address of a torch tensor / numpy array."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_handle(stream=None) -> int:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream
