"""The AS-SHIPPED reference config path over a batch — TEST INFRASTRUCTURE /
CPU ARMS ONLY.

Drives the reference package ``ragsched`` itself (no restatement): for each
query in order, ``gate_profile`` (profiler.py:467-486, one shared
``RecentSpaceWindow``), then the decision order of
``Scheduler._try_admit_new`` (scheduler.py:340-378): ``best_fit_select``
(scheduler.py:127-156) -> ``fallback_config`` (scheduler.py:159-191) ->
MustQueue.  Used by

* ``tests/golden/make_workload.py`` (dev container, ``/root/reference``) to
  make the committed workload fixtures and their expected decisions;
* ``bench.py --impl reference`` and bench's CPU baseline (GPU box: the
  reference installed into ``baseline/_ref`` by ``tools/install_reference.sh``),
  single-threaded as shipped and under ``multiprocessing.Pool``.
"""

from __future__ import annotations

import importlib
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")
REF_SRC = "/root/reference/pkg/src"
BIT = {"map_rerank": 1, "stuff": 2, "map_reduce": 4}


def import_ragsched(prefer: str | None = None):
    """The reference package: ``baseline/_ref`` (the pip --target install that
    travels to the GPU box), else ``/root/reference/pkg/src`` (dev container).
    Raises ImportError when neither exists."""
    for path in ([prefer] if prefer else []) + [REF_INSTALL, REF_SRC]:
        if path and os.path.isdir(os.path.join(path, "ragsched")):
            if path not in sys.path:
                sys.path.insert(0, path)
            mod = importlib.import_module("ragsched")
            if os.path.dirname(os.path.dirname(os.path.abspath(mod.__file__))) != os.path.abspath(path):
                raise ImportError(f"ragsched already imported from {mod.__file__}, wanted {path}")
            for sub in ("config", "mapping", "memory", "profiler", "scheduler", "sim", "types", "workload",
                        "metrics"):
                importlib.import_module("ragsched." + sub)
            return mod
    raise ImportError(f"reference package not found (looked in {REF_INSTALL} and {REF_SRC}); "
                      "run tools/install_reference.sh")


def source_of(rs) -> str:
    return os.path.dirname(os.path.abspath(rs.__file__))


def enc_space(rs, s) -> tuple:
    m = 0
    for x in s.synthesis_methods:
        m |= BIT[x.value]
    il = s.intermediate_length_range
    return (m, s.num_chunks_range.low, s.num_chunks_range.high, il.low if il else 0, il.high if il else 0)


def dec_space(rs, t):
    T, M = rs.types, rs.mapping
    m, lo, hi, a, b = (int(x) for x in t)
    inv = {v: k for k, v in BIT.items()}
    methods = frozenset(T.SynthesisMethod(inv[bit]) for bit in (1, 2, 4) if m & bit)
    return M.PrunedConfigSpace(methods, T.IntRange(lo, hi), T.IntRange(a, b) if m & 4 else None)


class Batch:
    """Reference objects for one workload fixture (``tests/golden/workload_*.npz``)."""

    def __init__(self, rs, w: dict):
        T, M = rs.types, rs.mapping
        self.rs = rs
        n = len(w["qlen"])
        self.n = n
        self.profiles = [M.QueryProfile(complexity_high=bool(w["cx"][i]), needs_joint_reasoning=bool(w["joint"][i]),
                                        pieces_required=int(w["pieces"][i]),
                                        summary_len_range=T.IntRange(int(w["s_lo"][i]), int(w["s_hi"][i])),
                                        confidence=float(w["conf"][i])) for i in range(n)]
        self.queries = [T.QueryRecord(id=f"q{i}", text="t", query_token_len=int(w["qlen"][i])) for i in range(n)]
        self.free = [int(x) for x in w["free"]]
        self.model = rs.config.DEFAULT_MODEL
        self.meta = T.DatasetMeta(description="bench workload", chunk_size=int(w["chunk_size"]))
        self.out_budget = int(w["out_budget"])
        self.fixed_space = dec_space(rs, w["fixed_space"]) if "fixed_space" in w and int(w["fixed_space"][0]) \
            else None
        self.spaces = None

    def gate(self):
        """gate_profile over the batch in order with a fresh window.
        Returns (spaces int32 [n,5], used_fallback uint8 [n])."""
        P = self.rs.profiler
        if self.fixed_space is not None:
            self.spaces = [self.fixed_space] * self.n
            enc = np.tile(np.array(enc_space(self.rs, self.fixed_space), dtype=np.int32), (self.n, 1))
            return enc, np.zeros(self.n, dtype=np.uint8)
        window = P.RecentSpaceWindow()
        spaces, fb = [], np.zeros(self.n, dtype=np.uint8)
        for i, prof in enumerate(self.profiles):
            out = P.ProfilerOutput(profile=prof, raw_text="", per_field_confidence={})
            dec = P.gate_profile(out, window)
            spaces.append(dec.space)
            fb[i] = dec.used_fallback
        self.spaces = spaces
        return np.array([enc_space(self.rs, s) for s in spaces], dtype=np.int32), fb

    def select_range(self, lo: int, hi: int) -> np.ndarray:
        """best_fit_select -> fallback_config -> MustQueue for queries [lo, hi).
        Returns int64 [hi - lo, 5]: method bit, num_chunks, interlen (0 = None),
        status (0 best fit, 1 fallback, 2 must queue), plan bytes."""
        rs = self.rs
        S, Mem = rs.scheduler, rs.memory
        per_tok = Mem.bytes_per_kv_token(self.model)
        out = np.zeros((hi - lo, 5), dtype=np.int64)
        kw = dict(model=self.model, meta=self.meta, out_budget=self.out_budget)
        for i in range(lo, hi):
            q = self.queries[i]
            cfg = S.best_fit_select(self.spaces[i], q, self.free[i], **kw)
            status = 0
            if cfg is None:
                cfg = S.fallback_config(self.profiles[i], q, self.free[i], **kw)
                status = 1 if cfg is not None else 2
            if cfg is not None:
                b = Mem.plan_bytes(q.query_token_len, cfg, self.meta.chunk_size, per_tok, self.out_budget)
                out[i - lo] = (BIT[cfg.synthesis_method.value], cfg.num_chunks, cfg.intermediate_length or 0,
                               status, b)
            else:
                out[i - lo, 3] = status
        return out


_POOL_BATCH: Batch | None = None


def _pool_select(args):
    lo, hi = args
    return _POOL_BATCH.select_range(lo, hi)


class PoolSelect:
    """``multiprocessing.Pool(cores)`` over query chunks.
    The workers fork with the batch already built; ``gate`` must have run
    in the parent first (the spaces are inherited)."""

    def __init__(self, batch: Batch, cores: int):
        global _POOL_BATCH
        _POOL_BATCH = batch
        self.cores = cores
        self.n = batch.n
        self.pool = mp.get_context("fork").Pool(cores)

    def run(self, lo: int = 0, hi: int | None = None) -> np.ndarray:
        hi = self.n if hi is None else hi
        step = max(1, -(-(hi - lo) // (4 * self.cores)))
        parts = self.pool.map(_pool_select, [(a, min(hi, a + step)) for a in range(lo, hi, step)])
        return np.concatenate(parts) if parts else np.zeros((0, 5), dtype=np.int64)

    def close(self):
        self.pool.terminate()
        self.pool.join()
