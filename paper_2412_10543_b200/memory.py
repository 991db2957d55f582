"""KV-cache memory model (reference ``memory.py``).

``plan_bytes`` — the per-candidate cost the selection maximises — is
evaluated by the ``rs_plan_bytes`` kernel (the same int64 device routine the
select kernel inlines).  ``bytes_per_kv_token`` and ``buffered_bytes`` are the
host-side scalars that parameterise the kernels.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _lib
from . import batch as _b
from . import scalar as _scalar
from .types import DEFAULT_MAX_CHUNKS, ContextOverflow, InvalidChunkCount
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
    params = _b.SelectParams(int(per_token_bytes), int(chunk_size), int(out_budget), int(template_tokens))
    return _scalar.plan_bytes_one(m, int(cfg.num_chunks), int(il or 0), int(query_token_len), _b.params_c(params))


# -- per-call expansion (memory.py:29-67, :89-150) -----------------------------


class CallKind(str, Enum):
    """memory.py:29-33."""

    SINGLE = "single"
    MAPPER = "mapper"
    REDUCER = "reducer"
    RERANK = "rerank"


class AdmissionMode(str, Enum):
    """memory.py:36-40."""

    WHOLE = "whole"
    PER_CALL = "per_call"


@dataclass(frozen=True)
class LlmCall:
    """memory.py:43-56."""

    kind: CallKind
    prompt_tokens: int
    max_output_tokens: int
    kv_bytes: int
    index: int = 0
    depends_on: frozenset = field(default_factory=frozenset)


@dataclass(frozen=True)
class CallPlan:
    """memory.py:59-67."""

    calls: tuple
    total_bytes: int

    def independent_calls(self) -> list[int]:
        return [i for i, c in enumerate(self.calls) if not c.depends_on]


def memory_requirement(plan, admission=AdmissionMode.WHOLE) -> int:
    """memory.py:153-161."""
    if getattr(admission, "value", admission) == AdmissionMode.WHOLE.value:
        return plan.total_bytes
    return max(c.kv_bytes for c in plan.calls)


PLAN_ERRORS = {
    _lib.RS_PLAN_INVALID_CHUNKS: (InvalidChunkCount, "num_chunks {n} outside [1, {mc}]"),
    _lib.RS_PLAN_CONTEXT_OVERFLOW: (ContextOverflow, "a call of {cfg} exceeds the context window of {ctx} tokens"),
    _lib.RS_PLAN_BAD_INTERLEN: (ValueError, "map_reduce config requires a positive intermediate_length"),
}


def plans_from_device(offsets, calls, totals, status, *, call_cls=LlmCall, plan_cls=CallPlan,
                      kind_enum=CallKind) -> list:
    """Host objects of an ``rs_plan_calls`` result (device tensors): one
    CallPlan per query, or the RS_PLAN_* status (int) where the reference raises."""
    rec = _b.from_device(calls, _lib.CALL_DTYPE) if calls.numel() else np.zeros(0, _lib.CALL_DTYPE)
    return plans_from_host(offsets.cpu().numpy(), rec, totals.cpu().numpy(), status.cpu().numpy(),
                           call_cls=call_cls, plan_cls=plan_cls, kind_enum=kind_enum)


def plans_from_host(off, rec, tot, st, *, call_cls=LlmCall, plan_cls=CallPlan, kind_enum=CallKind) -> list:
    """``plans_from_device`` over host arrays (offsets [n+1], rs_call records,
    totals [n], status [n])."""
    kinds = [kind_enum(v) for v in _lib.CALL_KINDS]
    out = []
    for i in range(len(st)):
        if st[i] != _lib.RS_PLAN_OK:
            out.append(int(st[i]))
            continue
        cs = []
        mappers = frozenset()
        for r in rec[int(off[i]):int(off[i + 1])]:
            kind = kinds[int(r["kind"])]
            if kind.value == "reducer":
                deps = mappers
            else:
                deps = frozenset()
            if kind.value == "mapper":
                mappers = mappers | {int(r["index"])}
            cs.append(call_cls(kind, int(r["prompt_tokens"]), int(r["max_output_tokens"]), int(r["kv_bytes"]),
                               index=int(r["index"]), depends_on=deps))
        out.append(plan_cls(calls=tuple(cs), total_bytes=int(tot[i])))
    return out


def context_overflow_message(qlen: int, cfg, chunk_size: int, template_tokens: int, out_budget: int,
                             max_context_tokens: int) -> str:
    """The message of the reference's first failing ``_check_context``
    (memory.py:81-86, :117-145) for this config."""
    C, T, O, ctx = chunk_size, template_tokens, out_budget, max_context_tokens
    n, m = cfg.num_chunks, cfg.synthesis_method.value
    if m == "stuff":
        checks = [("stuff call", qlen + n * C + T, O)]
    elif m == "map_rerank":
        checks = [("rerank call", qlen + C + T, O)]
    else:
        il = cfg.intermediate_length
        checks = [("mapper call", qlen + C + T, il), ("reducer call", qlen + n * il + T, O)]
    for label, prompt, out in checks:
        if prompt + out > ctx:
            return f"{label} needs {prompt + out} tokens, context window is {ctx}"
    return "context window exceeded"


def raise_plan_error(code: int, cfg, *, max_chunks: int, max_context_tokens: int, qlen: int = 0,
                     chunk_size: int = 0, template_tokens: int = DEFAULT_TEMPLATE_TOKENS, out_budget: int = 0):
    """Raise the reference's exception (and message) for an RS_PLAN_* status."""
    if code == _lib.RS_PLAN_CONTEXT_OVERFLOW:
        raise ContextOverflow(context_overflow_message(qlen, cfg, chunk_size, template_tokens, out_budget,
                                                       max_context_tokens))
    exc, fmt = PLAN_ERRORS[code]
    desc = cfg.describe() if hasattr(cfg, "describe") else str(cfg)
    raise exc(fmt.format(n=getattr(cfg, "num_chunks", "?"), mc=max_chunks, cfg=desc, ctx=max_context_tokens))


def plan_calls(q, cfg, meta, model, out_budget: int, *, template_tokens: int = DEFAULT_TEMPLATE_TOKENS,
               max_chunks: int = DEFAULT_MAX_CHUNKS, call_cls=LlmCall, plan_cls=CallPlan, kind_enum=CallKind):
    """memory.py:89-150 on the GPU (``rs_plan_calls``): the config's LLM calls
    with their KV bytes.  Raises InvalidChunkCount / ContextOverflow /
    ValueError exactly where the reference does."""
    # the reference's check order (memory.py:108-111): chunk count, then out_budget
    if not 1 <= int(cfg.num_chunks) <= max_chunks:
        raise InvalidChunkCount(f"num_chunks {cfg.num_chunks} outside [1, {max_chunks}]")
    if out_budget <= 0:
        raise ValueError("out_budget must be positive")
    dev = _b.default_device()
    rec = np.zeros(1, dtype=_lib.CONFIG_DTYPE)
    rec["method"] = method_bit(cfg.synthesis_method)
    rec["num_chunks"] = min(max(int(cfg.num_chunks), 0), 0xFFFF)
    il = cfg.intermediate_length
    rec["interlen"] = 0 if il is None or il <= 0 else min(int(il), 0xFFFF)
    params = _b.SelectParams(_b.bytes_per_kv_token(model), int(meta.chunk_size), int(out_budget),
                             int(template_tokens), int(max_chunks))
    qlen = torch.tensor([int(q.query_token_len)], dtype=torch.int32, device=dev)
    res = _b.plan_calls(_b.to_device(rec, dev), qlen, params, int(model.max_context_tokens))
    plan = plans_from_device(*res, call_cls=call_cls, plan_cls=plan_cls, kind_enum=kind_enum)[0]
    if isinstance(plan, int):
        raise_plan_error(plan, cfg, max_chunks=max_chunks, max_context_tokens=model.max_context_tokens,
                         qlen=int(q.query_token_len), chunk_size=int(meta.chunk_size),
                         template_tokens=int(template_tokens), out_budget=int(out_budget))
    return plan
