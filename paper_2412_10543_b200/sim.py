"""Prefill/decode delay model (reference ``sim.py:42-92``) on the GPU."""

from __future__ import annotations

from . import batch as _b
from . import scalar as _scalar
from .batch import CostModel  # sim.py:42-57

__all__ = ["CostModel", "call_latency"]


_COST_C: dict = {}  # (prefill, decode base, slowdown) -> rs_cost_model struct (a sim passes one CostModel)


def call_latency(call, concurrent_seqs: int, cost: CostModel) -> float:
    """sim.py:84-92 — bit-exact IEEE double via ``rs_call_latency`` (scalar
    fast path, scalar.py)."""
    key = (cost.prefill_secs_per_token, cost.decode_secs_per_token_base, cost.batch_slowdown_per_seq)
    c = _COST_C.get(key)
    if c is None:
        c = _b.cost_c(_b.CostModel(*key))
        if len(_COST_C) < 64:
            _COST_C[key] = c
    return _scalar.call_latency_one(int(call.prompt_tokens), int(call.max_output_tokens), int(concurrent_seqs), c)
