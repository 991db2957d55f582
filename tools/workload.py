"""Loader of the committed config-path workloads (``tests/golden/workload_<cfg>.npz``,
made by RUNNING THE REFERENCE in ``tests/golden/make_workload.py``):
per-query profile fields, query lengths, free KV bytes, and the reference's
own gate / select decisions on them (``exp_*``)."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def load(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, f"workload_{name}.npz"))
    w = {k: z[k] for k in z.files}
    for k in ("chunk_size", "out_budget"):
        w[k] = int(w[k])
    return w


def profiles_int5(w: dict) -> np.ndarray:
    """int32 [n, 5]: complexity_high, joint, pieces, summary lo, summary hi."""
    return np.stack([w["cx"], w["joint"], w["pieces"], w["s_lo"], w["s_hi"]], 1).astype(np.int32)


def full_space(w: dict) -> bool:
    return bool(int(w["fixed_space"][0]))
