"""ctypes binding of ``include/ragsched_b200.h`` (``libragsched_b200.so``).

The library is the only compute path of this package: if it is missing or
the device is not an sm_100 part, every entry point raises — there is no CPU
fallback.  Struct layouts below mirror the header (static size asserts in
``tests/test_abi.py``).
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# RAGSCHED_B200_LIB selects a tuning variant built by build.build(defines=..., out=...)
LIB_PATH = os.environ.get("RAGSCHED_B200_LIB") or os.path.join(HERE, "libragsched_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "ragsched_b200.h")

RS_OK, RS_ERR_INVALID_ARG, RS_ERR_CUDA, RS_ERR_UNSUPPORTED, RS_ERR_OOM, RS_ERR_OVERFLOW = range(6)
RS_MAP_RERANK, RS_STUFF, RS_MAP_REDUCE = 1, 2, 4
RS_SELECT_BEST_FIT, RS_SELECT_FALLBACK, RS_SELECT_MUST_QUEUE, RS_SELECT_OVERFLOW = range(4)
RS_F32, RS_BF16 = 0, 1
RS_ALGO_AUTO, RS_ALGO_SIMT, RS_ALGO_TCGEN05, RS_ALGO_TCGEN05_1SM = 0, 1, 2, 3
WINDOW_CAPACITY = 10

# numpy mirrors of the C structs (packed exactly like the C layout)
PROFILE_DTYPE = np.dtype([("complexity_high", "u1"), ("needs_joint_reasoning", "u1"),
                          ("pieces_required", "<u2"), ("summary_lo", "<u2"), ("summary_hi", "<u2"),
                          ("confidence", "<f8")])
SPACE_DTYPE = np.dtype([("methods", "<u2"), ("num_chunks_lo", "<u2"), ("num_chunks_hi", "<u2"),
                        ("interlen_lo", "<u2"), ("interlen_hi", "<u2"), ("gate_fallback", "<u2"),
                        ("reserved", "<u4")])
CONFIG_DTYPE = np.dtype([("kv_bytes", "<i8"), ("method", "u1"), ("status", "u1"),
                         ("num_chunks", "<u2"), ("interlen", "<u2"), ("reserved", "<u2")])
WINDOW_DTYPE = np.dtype([("spaces", SPACE_DTYPE, (WINDOW_CAPACITY,)), ("len", "<i4"),
                         ("reserved", "<i4", (3,))])
CALL_DTYPE = np.dtype([("kv_bytes", "<i8"), ("prompt_tokens", "<i4"), ("max_output_tokens", "<i4"),
                       ("index", "<u2"), ("kind", "u1"), ("reserved0", "u1"), ("reserved1", "<u4")])
CALL_KINDS = ("single", "mapper", "reducer", "rerank")  # rs_call.kind -> CallKind value (memory.py:29-33)
RS_PLAN_OK, RS_PLAN_NONE, RS_PLAN_INVALID_CHUNKS, RS_PLAN_CONTEXT_OVERFLOW, RS_PLAN_BAD_INTERLEN = range(5)
assert CALL_DTYPE.itemsize == 24
CANDIDATE_DTYPE = np.dtype([("kv_bytes", "<i8"), ("delay", "<f8"), ("method", "u1"), ("reserved0", "u1"),
                            ("num_chunks", "<u2"), ("interlen", "<u2"), ("reserved1", "<u2")])
assert CANDIDATE_DTYPE.itemsize == 24
ADMIT_INFO_DTYPE = np.dtype([("admitted_bytes", "<i8"), ("admitted_calls", "<i4"), ("fixed_path", "<i4")])
ADMIT_RESULT_DTYPE = np.dtype([("admitted", "<i8"), ("used_bytes", "<i8"), ("stop", "<i4"), ("reserved", "<i4")])
(RS_ADMIT_DRAINED, RS_ADMIT_BLOCKED, RS_ADMIT_NO_PROFILE, RS_ADMIT_IMPOSSIBLE, RS_ADMIT_FIXED_SPACE,
 RS_ADMIT_INVALID_CHUNKS, RS_ADMIT_CONTEXT_OVERFLOW, RS_ADMIT_BAD_INTERLEN, RS_ADMIT_OVERFLOW) = range(9)
assert ADMIT_INFO_DTYPE.itemsize == 16 and ADMIT_RESULT_DTYPE.itemsize == 24
assert PROFILE_DTYPE.itemsize == 16 and SPACE_DTYPE.itemsize == 16
assert CONFIG_DTYPE.itemsize == 16 and WINDOW_DTYPE.itemsize == 176


class SpaceC(ctypes.Structure):
    _fields_ = [("methods", ctypes.c_uint16), ("num_chunks_lo", ctypes.c_uint16),
                ("num_chunks_hi", ctypes.c_uint16), ("interlen_lo", ctypes.c_uint16),
                ("interlen_hi", ctypes.c_uint16), ("gate_fallback", ctypes.c_uint16),
                ("reserved", ctypes.c_uint32)]


class SelectParamsC(ctypes.Structure):
    _fields_ = [("per_token_bytes", ctypes.c_int64), ("chunk_size", ctypes.c_int32),
                ("out_budget", ctypes.c_int32), ("template_tokens", ctypes.c_int32),
                ("max_chunks", ctypes.c_int32), ("chunk_step", ctypes.c_int32),
                ("interlen_step", ctypes.c_int32), ("allow_fallback", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class CostModelC(ctypes.Structure):
    _fields_ = [("prefill_secs_per_token", ctypes.c_double),
                ("decode_secs_per_token_base", ctypes.c_double),
                ("batch_slowdown_per_seq", ctypes.c_double)]


class GateParamsC(ctypes.Structure):
    _fields_ = [("threshold", ctypes.c_double), ("default_space", SpaceC),
                ("max_chunks", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class AdmitParamsC(ctypes.Structure):
    _fields_ = [("capacity_bytes", ctypes.c_int64), ("used_bytes", ctypes.c_int64),
                ("max_context_tokens", ctypes.c_int64)]


assert ctypes.sizeof(SelectParamsC) == 40 and ctypes.sizeof(GateParamsC) == 32

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32

PEER_MAX = 64
PEER_HANDLE_BYTES = 64


class PeerExchangeC(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("k", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("slice_cap", ctypes.c_int64), ("region", _P * PEER_MAX)]


_PX = ctypes.POINTER(PeerExchangeC)

# exported symbol -> (restype, argtypes)
SIGNATURES = {
    "rs_abi_version": (ctypes.c_int, []),
    "rs_last_error": (ctypes.c_char_p, []),
    "rs_device_supported": (ctypes.c_int, [ctypes.c_int]),
    "rs_prune_gate_workspace_size": (ctypes.c_size_t, [_I64]),
    "rs_prune_gate": (ctypes.c_int, [_P, _I64, ctypes.POINTER(GateParamsC), _P, _P, _P, ctypes.c_size_t, _P]),
    "rs_select": (ctypes.c_int, [_P, _P, _P, _P, _I64, ctypes.POINTER(SelectParamsC),
                                 ctypes.POINTER(CostModelC), _P, _P, _P, _P]),
    "rs_call_latency": (ctypes.c_int, [_P, _P, _P, _I64, ctypes.POINTER(CostModelC), _P, _P]),
    "rs_plan_bytes": (ctypes.c_int, [_P, _P, _P, _P, _I64, ctypes.POINTER(SelectParamsC), _P, _P]),
    "rs_index_create": (ctypes.c_int, [_I32, _I32, _I64, _I32, ctypes.POINTER(_P)]),
    "rs_index_destroy": (ctypes.c_int, [_P]),
    "rs_index_add": (ctypes.c_int, [_P, _P, _I64, _P]),
    "rs_index_reset": (ctypes.c_int, [_P]),
    "rs_index_ntotal": (ctypes.c_int, [_P, ctypes.POINTER(_I64)]),
    "rs_index_data": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(_P)]),
    "rs_index_set_algo": (ctypes.c_int, [_P, _I32]),
    "rs_index_set_walk_bias": (ctypes.c_int, [_P, _I32]),
    "rs_index_set_segment_rows": (ctypes.c_int, [_P, _I32]),
    "rs_index_set_burst_merge": (ctypes.c_int, [_P, _I32]),
    "rs_index_set_probe": (ctypes.c_int, [_P, _I32]),
    "rs_index_last_probe_rows": (ctypes.c_int, [_P, _P]),
    "rs_index_burst_merge_active": (ctypes.c_int, [_P, _P]),
    "rs_index_reserve": (ctypes.c_int, [_P, _I64, _I32]),
    "rs_index_search": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _P, _P, _P, _P]),
    "rs_index_search_keys": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _P, _P]),
    "rs_index_last_plan": (ctypes.c_int, [_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                          ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "rs_merge_topk": (ctypes.c_int, [_P, _I64, _I32, _I32, _I64, _I32, _P, _P, _P, _P]),
    "rs_row_norms": (ctypes.c_int, [_P, _I64, _I32, _I32, _P, _P]),
    "rs_plan_calls_workspace_size": (ctypes.c_size_t, [_I64]),
    "rs_plan_calls": (ctypes.c_int, [_P, _P, _I64, ctypes.POINTER(SelectParamsC), _I64, _P, _P, _P, _P, _P,
                                     ctypes.c_size_t, _P]),
    "rs_candidate_costs_workspace_size": (ctypes.c_size_t, [_I64]),
    "rs_candidate_costs": (ctypes.c_int, [_P, _P, _P, _I64, ctypes.POINTER(SelectParamsC), ctypes.POINTER(CostModelC),
                                          _P, _P, _P, ctypes.c_size_t, _P]),
    "rs_parse_profiles": (ctypes.c_int, [ctypes.c_char_p, _P, _I64, _P, _P, _P, _P, _P, _I32]),
    "rs_field_confidences": (ctypes.c_int, [ctypes.c_char_p, _P, _I64, _P, ctypes.c_char_p, _P, _P, _P, _P, _I32]),
    "rs_admit_fifo": (ctypes.c_int, [_P, _P, _P, _P, _I64, ctypes.POINTER(SelectParamsC),
                                     ctypes.POINTER(AdmitParamsC), _P, _P, _P, _P]),
    "rs_peer_region_bytes": (ctypes.c_int, [_I32, _I64, _I32, ctypes.POINTER(ctypes.c_uint64)]),
    "rs_peer_alloc": (ctypes.c_int, [ctypes.c_uint64, _I32, ctypes.POINTER(_P), _P]),
    "rs_peer_open": (ctypes.c_int, [_P, _I32, ctypes.POINTER(_P)]),
    "rs_peer_close": (ctypes.c_int, [_P]),
    "rs_peer_free": (ctypes.c_int, [_P]),
    "rs_peer_scatter_keys": (ctypes.c_int, [_PX, _P, _I64, ctypes.c_uint32, _P]),
    "rs_peer_merge_topk": (ctypes.c_int, [_PX, _I64, ctypes.c_uint32, _I32, _P, _P, _P, _I32, _P]),
    "rs_peer_error": (ctypes.c_int, [_PX, _I32, ctypes.POINTER(_I32)]),
    "rs_index_search_scatter": (ctypes.c_int, [_P, _P, _I64, _I32, _I64, _PX, ctypes.c_uint32, _P]),
    "rs_launch_count": (ctypes.c_uint64, []),
    "rs_index_enable_timing": (ctypes.c_int, [_P, _I32]),
    "rs_index_kernel_times": (ctypes.c_int, [_P, _P, _I32, ctypes.POINTER(_I32)]),
}


def launch_count() -> int:
    """Kernels launched by libragsched_b200 in this process."""
    return int(load().rs_launch_count())


class RagschedError(RuntimeError):
    """A CUDA / library failure reported through the C ABI."""


class LibraryUnavailable(ImportError):
    """libragsched_b200.so is missing or cannot run here (no CPU fallback)."""


_lib = None
_lock = threading.Lock()


def header_symbols() -> list[str]:
    """Function names declared in include/ragsched_b200.h."""
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(rs_\w+)\s*\(", text, re.M)))


def load(path: str = LIB_PATH):
    """Load the shared library (does not touch the GPU)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise LibraryUnavailable(
                    f"{path} not built — run `python -m paper_2412_10543_b200.build`; "
                    "this package has no CPU fallback")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


_checked_devices: set[int] = set()


def lib_for_device(device_index: int):
    """The library, after verifying the CUDA device is a supported B200."""
    lib = load()
    if device_index not in _checked_devices:
        if not lib.rs_device_supported(int(device_index)):
            raise LibraryUnavailable(
                f"CUDA device {device_index} is not an sm_100 (B200) part; "
                "libragsched_b200 is compiled for sm_100a only and has no fallback")
        _checked_devices.add(device_index)
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == RS_OK:
        return
    msg = load().rs_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == RS_ERR_INVALID_ARG:
        raise ValueError(text)
    if rc == RS_ERR_OVERFLOW:
        raise OverflowError(text)
    if rc == RS_ERR_OOM:
        raise MemoryError(text)
    raise RagschedError(f"[rc={rc}] {text}")


def ptr(t) -> int:
    """Raw device pointer of a torch tensor (or 0 for None)."""
    return 0 if t is None else int(t.data_ptr())


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
