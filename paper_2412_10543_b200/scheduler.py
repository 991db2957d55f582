"""Best-fit + fallback selection (reference ``scheduler.py:127-191``), on the
GPU.  Scalar drop-ins with the reference signatures; the batched fast path is
:func:`paper_2412_10543_b200.batch.select`.
"""

from __future__ import annotations

import numpy as np
import torch

from . import batch as _b
from ._lib import SPACE_DTYPE
from .mapping import EnumGranularity
from .types import DEFAULT_MAX_CHUNKS, DEFAULT_TEMPLATE_TOKENS, RagConfig, SynthesisMethod


class SchedulingImpossible(RuntimeError):
    """scheduler.py:41."""


def _run_select(space_rec, profile, q, free_bytes, params, config_cls, method_enum):
    dev = _b.default_device()
    spaces = _b.to_device(space_rec, dev)
    prof = _b.to_device(_b.pack_profiles([profile]), dev) if profile is not None else None
    qlen = torch.tensor([int(q.query_token_len)], dtype=torch.int32, device=dev)
    free = torch.tensor([int(free_bytes)], dtype=torch.int64, device=dev)
    out, _ = _b.select(spaces, prof, qlen, free, params)
    return _b.unpack_config(_b.from_device(out, _b.CONFIG_DTYPE)[0], config_cls=config_cls, method_enum=method_enum)


def best_fit_select(space, q, free_bytes: int, *, model, meta, out_budget: int,
                    template_tokens: int = DEFAULT_TEMPLATE_TOKENS, granularity=EnumGranularity(),
                    config_cls=RagConfig, method_enum=SynthesisMethod):
    """scheduler.py:127-156 — the candidate with the largest whole-plan bytes
    that fits ``free_bytes`` (byte ties -> latest grid position); None if none
    fits."""
    params = _b.SelectParams.from_model(model, meta, out_budget, template_tokens, DEFAULT_MAX_CHUNKS, granularity,
                                        allow_fallback=False)
    return _run_select(_b.pack_spaces([space]), None, q, free_bytes, params, config_cls, method_enum)


def fallback_config(profile, q, free_bytes: int, *, model, meta, out_budget: int,
                    template_tokens: int = DEFAULT_TEMPLATE_TOKENS, max_chunks: int = DEFAULT_MAX_CHUNKS,
                    config_cls=RagConfig, method_enum=SynthesisMethod):
    """scheduler.py:159-191 — rerank with as many chunks as fit (non-joint) or
    the largest fitting stuff (joint); never map_reduce; None = MustQueue."""
    params = _b.SelectParams.from_model(model, meta, out_budget, template_tokens, max_chunks, None,
                                        allow_fallback=True)
    empty = np.zeros(1, dtype=SPACE_DTYPE)  # no candidates: the kernel goes straight to the fallback
    return _run_select(empty, profile, q, free_bytes, params, config_cls, method_enum)
