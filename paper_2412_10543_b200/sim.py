"""Prefill/decode delay model (reference ``sim.py:42-92``) on the GPU."""

from __future__ import annotations

import torch

from . import batch as _b
from .batch import CostModel  # sim.py:42-57

__all__ = ["CostModel", "call_latency"]


def call_latency(call, concurrent_seqs: int, cost: CostModel) -> float:
    """sim.py:84-92 — bit-exact IEEE double via ``rs_call_latency``."""
    dev = _b.default_device()
    t = lambda v: torch.tensor([int(v)], dtype=torch.int64, device=dev)  # noqa: E731
    out = _b.call_latency_batch(t(call.prompt_tokens), t(call.max_output_tokens), t(concurrent_seqs),
                                _b.CostModel(cost.prefill_secs_per_token, cost.decode_secs_per_token_base,
                                             cost.batch_slowdown_per_seq))
    return float(out.item())
