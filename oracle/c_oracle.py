"""ctypes wrapper of the C restatement (oracle/csrc/oracle_select.c) — TEST
INFRASTRUCTURE / CPU BASELINE ONLY."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle_select.so")
_lib = None


class _Params(ctypes.Structure):
    _fields_ = [("per_token_bytes", ctypes.c_int64), ("chunk_size", ctypes.c_int32),
                ("out_budget", ctypes.c_int32), ("template_tokens", ctypes.c_int32),
                ("max_chunks", ctypes.c_int32), ("chunk_step", ctypes.c_int32),
                ("interlen_step", ctypes.c_int32)]


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, "csrc", f) for f in ("oracle_select.c", "synth.c")]
    outs = [_SO, os.path.join(_HERE, "_build", "libsynth.so")]
    if force or any(not os.path.exists(o) for o in outs) or \
            max(os.path.getmtime(s) for s in srcs) > min(os.path.getmtime(o) for o in outs):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _SO


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        _lib = ctypes.CDLL(_SO)
        _lib.oracle_select_batch.restype = ctypes.c_int
        _lib.oracle_gate_batch.restype = ctypes.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def select_batch(spaces, joint, qlen, free_bytes, params, allow_fallback=True, nthreads=0):
    """spaces int32 [n,5]; joint uint8 [n]; qlen int32 [n]; free int64 [n].
    Returns (cfg int32 [n,3], bytes int64 [n], status uint8 [n])."""
    spaces = np.ascontiguousarray(spaces, dtype=np.int32)
    joint = np.ascontiguousarray(joint, dtype=np.uint8)
    qlen = np.ascontiguousarray(qlen, dtype=np.int32)
    free_bytes = np.ascontiguousarray(free_bytes, dtype=np.int64)
    n = spaces.shape[0]
    cfg = np.zeros((n, 3), dtype=np.int32)
    b = np.zeros(n, dtype=np.int64)
    st = np.zeros(n, dtype=np.uint8)
    p = _Params(params.per_token_bytes, params.chunk_size, params.out_budget,
                params.template_tokens, params.max_chunks, params.chunk_step, params.interlen_step)
    rc = lib().oracle_select_batch(ctypes.c_int64(n), _p(spaces), _p(joint), _p(qlen), _p(free_bytes),
                                   ctypes.byref(p), ctypes.c_int(int(allow_fallback)), _p(cfg), _p(b),
                                   _p(st), ctypes.c_int(nthreads))
    if rc:
        raise MemoryError("oracle_select_batch failed")
    return cfg, b, st


def gate_batch(profiles, conf, threshold=0.90, default_space=(2, 1, 5, 0, 0), max_chunks=35,
               window=()):
    """profiles int32 [n,5] (cx, joint, pieces, s_lo, s_hi); conf float64 [n].
    Returns (spaces int32 [n,5], used_fallback uint8 [n], window list)."""
    profiles = np.ascontiguousarray(profiles, dtype=np.int32)
    conf = np.ascontiguousarray(conf, dtype=np.float64)
    n = profiles.shape[0]
    win = np.zeros((10, 5), dtype=np.int32)
    wl = ctypes.c_int32(len(window))
    if len(window):
        win[:len(window)] = np.asarray(window, dtype=np.int32)
    ds = np.ascontiguousarray(default_space, dtype=np.int32)
    out = np.zeros((n, 5), dtype=np.int32)
    fb = np.zeros(n, dtype=np.uint8)
    lib().oracle_gate_batch(ctypes.c_int64(n), _p(profiles), _p(conf), ctypes.c_double(threshold),
                            _p(ds), ctypes.c_int(max_chunks), _p(win), ctypes.byref(wl), _p(out), _p(fb))
    return out, fb, [tuple(int(x) for x in r) for r in win[:wl.value]]
