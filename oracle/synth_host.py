"""ctypes wrapper of oracle/csrc/synth.c: the host copy of tools/synth.py's
"iso" corpus generator — TEST INFRASTRUCTURE / CPU ARMS ONLY (the CPU
baseline and ``bench.py --impl reference`` build the same corpus the GPU arm
searches, bit for bit)."""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import c_oracle

_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libsynth.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            c_oracle.build(force=True)
        _lib = ctypes.CDLL(_SO)
        _lib.synth_rows.restype = ctypes.c_int
        _lib.synth_rows.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_uint32, ctypes.c_int,
                                    ctypes.c_void_p, ctypes.c_int]
    return _lib


def corpus_rows(r0: int, r1: int, d: int, seed: int, bf16: bool, out: np.ndarray | None = None,
                nthreads: int | None = None) -> np.ndarray:
    """Rows [r0, r1) as float32 [r1 - r0, d] (bf16-rounded values when ``bf16``)."""
    if out is None:
        out = np.empty((r1 - r0, d), dtype=np.float32)
    assert out.dtype == np.float32 and out.flags.c_contiguous and out.shape == (r1 - r0, d)
    rc = lib().synth_rows(r0, r1 - r0, d, seed & 0xFFFFFFFF, int(bf16), out.ctypes.data,
                          int(nthreads or os.cpu_count()))
    if rc:
        raise ValueError("synth_rows: bad arguments")
    return out
