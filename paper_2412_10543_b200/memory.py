"""KV-cache memory model (reference ``memory.py``).

``plan_bytes`` — the per-candidate cost the selection maximises — is
evaluated by the ``rs_plan_bytes`` kernel (the same int64 device routine the
select kernel inlines).  ``bytes_per_kv_token`` and ``buffered_bytes`` are the
host-side scalars that parameterise the kernels.
"""

from __future__ import annotations

import torch

from . import batch as _b
from .types import DEFAULT_TEMPLATE_TOKENS, SynthesisMethod, method_bit

BUFFER_NUMERATOR = 102   # memory.py:25
BUFFER_DENOMINATOR = 100  # memory.py:26

bytes_per_kv_token = _b.bytes_per_kv_token  # memory.py:70-73


def buffered_bytes(tokens: int, per_token_bytes: int) -> int:
    """memory.py:76-78 — integer ceil of the 2% buffer."""
    return (BUFFER_NUMERATOR * tokens * per_token_bytes + BUFFER_DENOMINATOR - 1) // BUFFER_DENOMINATOR


def plan_bytes(query_token_len: int, cfg, chunk_size: int, per_token_bytes: int, out_budget: int,
               template_tokens: int = DEFAULT_TEMPLATE_TOKENS) -> int:
    """memory.py:164-195, computed on the GPU (``rs_plan_bytes``)."""
    m = method_bit(cfg.synthesis_method)
    il = cfg.intermediate_length
    if m == method_bit(SynthesisMethod.MAP_REDUCE) and (il is None or il <= 0):
        raise ValueError("map_reduce config requires a positive intermediate_length")
    dev = _b.default_device()
    params = _b.SelectParams(int(per_token_bytes), int(chunk_size), int(out_budget), int(template_tokens))
    t = lambda v, dt: torch.tensor([v], dtype=dt, device=dev)  # noqa: E731
    out = _b.plan_bytes_batch(t(m, torch.uint8), t(int(cfg.num_chunks), torch.int32), t(int(il or 0), torch.int32),
                              t(int(query_token_len), torch.int32), params)
    return int(out.item())
