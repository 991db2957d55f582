"""Batched SoA entry points of the config path (the fast path).

Inputs and outputs are device tensors holding the C structs of
``include/ragsched_b200.h`` as raw bytes (``uint8 [n, 16]``); the helpers here
pack / unpack them from the reference-style objects.  Every compute step is a
kernel of ``libragsched_b200.so``:

* :func:`prune_gate`  — ``gate_profile`` over a batch in order
  (profiler.py:467-486) → ``rs_prune_gate``
* :func:`select`      — ``best_fit_select`` → ``fallback_config`` per query
  (scheduler.py:127-191, :335-378) + optional delay → ``rs_select``
"""

from __future__ import annotations

import ctypes
import functools
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import CONFIG_DTYPE, PROFILE_DTYPE, SPACE_DTYPE, WINDOW_DTYPE
from .types import (
    BIT_METHOD,
    DEFAULT_MAX_CHUNKS,
    DEFAULT_TEMPLATE_TOKENS,
    IntRange,
    RagConfig,
    SynthesisMethod,
    method_bit,
)

GATE_THRESHOLD = 0.90  # profiler.py:30


def bytes_per_kv_token(model) -> int:
    """memory.py:70-73 (host scalar: a parameter of the select kernel)."""
    return int(2 * model.num_layers * model.num_kv_heads * model.head_dim * model.bytes_per_element)


@dataclass(frozen=True)
class SelectParams:
    """Host mirror of ``rs_select_params`` (the scalars of best_fit_select /
    fallback_config, scheduler.py:127-191)."""

    per_token_bytes: int
    chunk_size: int
    out_budget: int
    template_tokens: int = DEFAULT_TEMPLATE_TOKENS
    max_chunks: int = DEFAULT_MAX_CHUNKS
    chunk_step: int = 1
    interlen_step: int = 10
    allow_fallback: bool = True

    @classmethod
    def from_model(cls, model, meta, out_budget, template_tokens=DEFAULT_TEMPLATE_TOKENS,
                   max_chunks=DEFAULT_MAX_CHUNKS, granularity=None, allow_fallback=True):
        cs = granularity.chunk_step if granularity is not None else 1
        ist = granularity.interlen_step if granularity is not None else 10
        return cls(bytes_per_kv_token(model), int(meta.chunk_size), int(out_budget), int(template_tokens),
                   int(max_chunks), int(cs), int(ist), bool(allow_fallback))

    def c(self) -> _lib.SelectParamsC:
        return _lib.SelectParamsC(self.per_token_bytes, self.chunk_size, self.out_budget, self.template_tokens,
                                  self.max_chunks, self.chunk_step, self.interlen_step,
                                  int(self.allow_fallback), 0)


@dataclass(frozen=True)
class CostModel:
    """sim.py:42-57 (the latency terms; the profiler latency is not a kernel input)."""

    prefill_secs_per_token: float = 1.0e-4
    decode_secs_per_token_base: float = 4.0e-3
    batch_slowdown_per_seq: float = 0.01
    profiler_latency_secs: float = 0.015

    def c(self) -> _lib.CostModelC:
        return _lib.CostModelC(self.prefill_secs_per_token, self.decode_secs_per_token_base,
                               self.batch_slowdown_per_seq)


# -- packing -------------------------------------------------------------------

def pack_profiles(profiles) -> np.ndarray:
    """QueryProfile-like objects -> structured array of rs_profile."""
    a = np.zeros(len(profiles), dtype=PROFILE_DTYPE)
    for i, p in enumerate(profiles):
        a[i] = profile_tuple(p)
    return a


def profile_tuple(p) -> tuple:
    """QueryProfile-like -> one rs_profile record as a tuple."""
    return (bool(p.complexity_high), bool(p.needs_joint_reasoning), int(p.pieces_required),
            int(p.summary_len_range.low), int(p.summary_len_range.high), float(p.confidence))


@functools.lru_cache(maxsize=256)
def params_c(params: SelectParams) -> _lib.SelectParamsC:
    """The (cached) C struct of a SelectParams (scalar calls reuse it)."""
    return params.c()


@functools.lru_cache(maxsize=64)
def cost_c(cost: CostModel) -> _lib.CostModelC:
    return cost.c()


def profiles_from_arrays(complexity_high, joint, pieces, summary_lo, summary_hi, confidence) -> np.ndarray:
    n = len(confidence)
    a = np.zeros(n, dtype=PROFILE_DTYPE)
    a["complexity_high"] = np.asarray(complexity_high, dtype=np.uint8)
    a["needs_joint_reasoning"] = np.asarray(joint, dtype=np.uint8)
    a["pieces_required"] = np.asarray(pieces, dtype=np.uint16)
    a["summary_lo"] = np.asarray(summary_lo, dtype=np.uint16)
    a["summary_hi"] = np.asarray(summary_hi, dtype=np.uint16)
    a["confidence"] = np.asarray(confidence, dtype=np.float64)
    return a


def _u16(v, what):
    v = int(v)
    if not 0 <= v <= 0xFFFF:
        raise ValueError(f"{what} {v} outside the supported range [0, 65535]")
    return v


def space_record(space) -> tuple:
    """PrunedConfigSpace-like -> (methods, n_lo, n_hi, il_lo, il_hi)."""
    m = 0
    for x in space.synthesis_methods:
        m |= method_bit(x)
    il = space.intermediate_length_range
    if m & 4 and il is not None and il.low <= 0:
        raise ValueError("map_reduce config requires a positive intermediate_length")
    return (m, _u16(space.num_chunks_range.low, "num_chunks"), _u16(space.num_chunks_range.high, "num_chunks"),
            _u16(il.low, "intermediate_length") if (m & 4 and il is not None) else 0,
            _u16(il.high, "intermediate_length") if (m & 4 and il is not None) else 0)


def pack_spaces(spaces) -> np.ndarray:
    a = np.zeros(len(spaces), dtype=SPACE_DTYPE)
    for i, s in enumerate(spaces):
        m, lo, hi, a0, b0 = space_record(s)
        a[i]["methods"], a[i]["num_chunks_lo"], a[i]["num_chunks_hi"] = m, lo, hi
        a[i]["interlen_lo"], a[i]["interlen_hi"] = a0, b0
    return a


def spaces_from_arrays(methods, n_lo, n_hi, il_lo, il_hi) -> np.ndarray:
    a = np.zeros(len(methods), dtype=SPACE_DTYPE)
    for f, v in (("methods", methods), ("num_chunks_lo", n_lo), ("num_chunks_hi", n_hi),
                 ("interlen_lo", il_lo), ("interlen_hi", il_hi)):
        a[f] = np.asarray(v, dtype=np.uint16)
    return a


def unpack_space(rec, *, space_cls=None, method_enum=SynthesisMethod, range_cls=IntRange):
    from .mapping import PrunedConfigSpace

    space_cls = space_cls or PrunedConfigSpace
    m = int(rec["methods"])
    methods = frozenset(method_enum(BIT_METHOD[b].value) for b in (1, 2, 4) if m & b)
    il = range_cls(int(rec["interlen_lo"]), int(rec["interlen_hi"])) if m & 4 else None
    return space_cls(methods, range_cls(int(rec["num_chunks_lo"]), int(rec["num_chunks_hi"])), il)


def unpack_config(rec, *, config_cls=RagConfig, method_enum=SynthesisMethod):
    """rs_config record -> RagConfig (None for MustQueue)."""
    st = int(rec["status"])
    if st == _lib.RS_SELECT_OVERFLOW:
        raise OverflowError("KV byte arithmetic exceeds int64 for this query")
    if st == _lib.RS_SELECT_MUST_QUEUE:
        return None
    m = BIT_METHOD[int(rec["method"])]
    me = method_enum(m.value)
    il = int(rec["interlen"]) if m is SynthesisMethod.MAP_REDUCE else None
    return config_cls(me, int(rec["num_chunks"]), il)


RS_PARSE_OK, RS_PARSE_UNPARSEABLE = 0, 1
RS_CLAMPED_PIECES, RS_CLAMPED_SUMMARY = 1, 2


def parse_profiles(texts, confidences=None, *, nthreads: int = 0):
    """parse_profile_text (profiler.py:203-254) for a batch of estimator
    answers, on the host (``rs_parse_profiles``, multi-threaded native code).
    Returns (rs_profile structured array, clamped bits u8 [n], status u8 [n],
    field line numbers int32 [n, 4])."""
    n = len(texts)
    enc = [t.encode("utf-8", "surrogatepass") for t in texts]
    offsets = np.zeros(n + 1, dtype=np.int64)
    if n:
        offsets[1:] = np.cumsum([len(b) for b in enc])
    buf = b"".join(enc) + b"\0"
    conf = np.ones(n, dtype=np.float64) if confidences is None else np.asarray(confidences, dtype=np.float64)
    out = np.zeros(n, dtype=PROFILE_DTYPE)
    clamped = np.zeros(n, dtype=np.uint8)
    status = np.zeros(n, dtype=np.uint8)
    lines = np.zeros((n, 4), dtype=np.int32)
    lib = _lib.load()
    _lib.check(lib.rs_parse_profiles(buf, offsets.ctypes.data, n, conf.ctypes.data, out.ctypes.data,
                                     clamped.ctypes.data, lines.ctypes.data, status.ctypes.data, int(nthreads)),
               "rs_parse_profiles")
    return out, clamped, status, lines


def field_confidences(texts, token_lists, *, nthreads: int = 0) -> np.ndarray:
    """_per_field_confidences (profiler.py:427-464) for a batch of estimator
    answers and their token streams (each a list of ``{"token", "logprob"}``
    dicts, or None), on the host (``rs_field_confidences``, multi-threaded
    native code).  Returns float64 [n, 4] in PROFILE_FIELDS order."""
    n = len(texts)
    if len(token_lists) != n:
        raise ValueError("texts and token_lists differ in length")
    enc = [t.encode("utf-8", "surrogatepass") for t in texts]
    offsets = np.zeros(n + 1, dtype=np.int64)
    if n:
        offsets[1:] = np.cumsum([len(b) for b in enc])
    tok_offsets = np.zeros(n + 1, dtype=np.int64)
    tok_enc, lps, has = [], [], []
    for i, toks in enumerate(token_lists):
        for tok in toks or ():
            text = tok.get("token", "")
            if not isinstance(text, str):
                raise TypeError(f"object of type {type(text).__name__!r} has no len()")  # len(text), :454
            lp = tok.get("logprob")
            tok_enc.append(text.encode("utf-8", "surrogatepass"))
            lps.append(0.0 if lp is None else float(lp))
            has.append(lp is not None)
        tok_offsets[i + 1] = len(tok_enc)
    tt_off = np.zeros(len(tok_enc) + 1, dtype=np.int64)
    if tok_enc:
        tt_off[1:] = np.cumsum([len(b) for b in tok_enc])
    lp_arr = np.asarray(lps, dtype=np.float64)
    has_arr = np.asarray(has, dtype=np.uint8)
    out = np.empty((n, 4), dtype=np.float64)
    lib = _lib.load()
    _lib.check(lib.rs_field_confidences(b"".join(enc) + b"\0", offsets.ctypes.data, n, tok_offsets.ctypes.data,
                                        b"".join(tok_enc) + b"\0", tt_off.ctypes.data, lp_arr.ctypes.data,
                                        has_arr.ctypes.data, out.ctypes.data, int(nthreads)),
               "rs_field_confidences")
    return out


def clamped_names(bits) -> frozenset:
    bits = int(bits)
    return frozenset(n for b, n in ((RS_CLAMPED_PIECES, "pieces"), (RS_CLAMPED_SUMMARY, "summary_range"))
                     if bits & b)


def unpack_profile(rec, *, profile_cls=None, range_cls=IntRange):
    """rs_profile record -> QueryProfile (this package's or the reference's)."""
    from .mapping import QueryProfile

    cls = profile_cls or QueryProfile
    return cls(complexity_high=bool(rec["complexity_high"]), needs_joint_reasoning=bool(rec["needs_joint_reasoning"]),
               pieces_required=int(rec["pieces_required"]),
               summary_len_range=range_cls(int(rec["summary_lo"]), int(rec["summary_hi"])),
               confidence=float(rec["confidence"]))


def to_device(arr: np.ndarray, device) -> torch.Tensor:
    """Structured numpy array -> device uint8 tensor [n, itemsize]."""
    raw = np.ascontiguousarray(arr).view(np.uint8).reshape(len(arr), arr.dtype.itemsize)
    return torch.from_numpy(raw).to(device, non_blocking=False)


def from_device(t: torch.Tensor, dtype: np.dtype) -> np.ndarray:
    return t.detach().to("cpu").contiguous().numpy().reshape(-1).view(dtype)


def _dev_index(t: torch.Tensor) -> int:
    if t.device.type != "cuda":
        raise ValueError(f"expected a CUDA tensor, got {t.device}")
    return t.device.index if t.device.index is not None else torch.cuda.current_device()


# -- gate window state ----------------------------------------------------------

class GateWindow:
    """Device-resident RecentSpaceWindow (profiler.py:138-153) carried across
    batches, as the ``rs_window`` struct."""

    def __init__(self, device, spaces=()):
        rec = np.zeros(1, dtype=WINDOW_DTYPE)
        spaces = list(spaces)[-_lib.WINDOW_CAPACITY:]
        if spaces:
            rec["spaces"][0, :len(spaces)] = pack_spaces(spaces)
        rec["len"] = len(spaces)
        self.tensor = to_device(rec, device).reshape(-1)

    def records(self) -> np.ndarray:
        rec = from_device(self.tensor, WINDOW_DTYPE)[0]
        return rec["spaces"][: int(rec["len"])]


# -- kernels ----------------------------------------------------------------------

def prune_gate(profiles: torch.Tensor, window: GateWindow, *, threshold: float = GATE_THRESHOLD,
               default_space=None, max_chunks: int = DEFAULT_MAX_CHUNKS, out: torch.Tensor | None = None,
               workspace: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """gate_profile for a device batch of rs_profile (uint8 [n,16]) in order.
    Returns device rs_space records (uint8 [n,16]); ``window`` is updated."""
    n = profiles.shape[0]
    dev = _dev_index(profiles)
    lib = _lib.lib_for_device(dev)
    if out is None:
        out = torch.empty((n, 16), dtype=torch.uint8, device=profiles.device)
    ws_bytes = int(lib.rs_prune_gate_workspace_size(n))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=profiles.device)
    if default_space is None:
        ds = (2, 1, 5, 0, 0)  # DEFAULT_FALLBACK_SPACE = stuff [1,5] (profiler.py:40-42)
    else:
        ds = space_record(default_space) if hasattr(default_space, "synthesis_methods") else tuple(default_space)
    gp = _lib.GateParamsC(float(threshold), _lib.SpaceC(ds[0], ds[1], ds[2], ds[3], ds[4], 1, 0), int(max_chunks), 0)
    _lib.check(lib.rs_prune_gate(_lib.ptr(profiles), n, ctypes.byref(gp), _lib.ptr(window.tensor), _lib.ptr(out),
                                 _lib.ptr(workspace), workspace.numel(), _lib.stream_ptr(stream)), "rs_prune_gate")
    return out


def select(spaces: torch.Tensor, profiles: torch.Tensor | None, qlen: torch.Tensor, free_bytes: torch.Tensor,
           params: SelectParams, *, cost: CostModel | None = None, running_before: torch.Tensor | None = None,
           out: torch.Tensor | None = None, delay: torch.Tensor | None = None, stream=None):
    """best_fit_select -> fallback_config for each query of a device batch.
    Returns (configs uint8 [n,16] of rs_config, delay float64 [n] or None)."""
    n = spaces.shape[0]
    dev = _dev_index(spaces)
    lib = _lib.lib_for_device(dev)
    if qlen.dtype != torch.int32 or free_bytes.dtype != torch.int64:
        raise TypeError("qlen must be int32 and free_bytes int64 device tensors")
    if out is None:
        out = torch.empty((n, 16), dtype=torch.uint8, device=spaces.device)
    cp = None
    if cost is not None:
        cp = ctypes.byref(cost.c())
        if delay is None:
            delay = torch.empty(n, dtype=torch.float64, device=spaces.device)
    pc = params.c()
    _lib.check(lib.rs_select(_lib.ptr(spaces), _lib.ptr(profiles), _lib.ptr(qlen), _lib.ptr(free_bytes), n,
                             ctypes.byref(pc), cp, _lib.ptr(running_before), _lib.ptr(delay) if cost else 0,
                             _lib.ptr(out), _lib.stream_ptr(stream)), "rs_select")
    return out, (delay if cost is not None else None)


def plan_calls(configs: torch.Tensor, qlen: torch.Tensor, params: SelectParams, max_context_tokens: int,
               stream=None):
    """memory.plan_calls (memory.py:89-150) for a device batch of chosen
    rs_config records.  Returns (offsets int64 [n+1], calls uint8 [total,24]
    of rs_call, total_bytes int64 [n], status uint8 [n]) on the device;
    query i's calls are calls[offsets[i]:offsets[i+1]]."""
    n = configs.shape[0]
    lib = _lib.lib_for_device(_dev_index(configs))
    dev = configs.device
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    totals = torch.empty(n, dtype=torch.int64, device=dev)
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    ws_bytes = int(lib.rs_plan_calls_workspace_size(n))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    pc = params.c()
    s = _lib.stream_ptr(stream)
    _lib.check(lib.rs_plan_calls(_lib.ptr(configs), _lib.ptr(qlen), n, ctypes.byref(pc), int(max_context_tokens),
                                 _lib.ptr(offsets), 0, 0, _lib.ptr(status), _lib.ptr(ws), ws.numel(), s),
               "rs_plan_calls(count)")
    total_calls = int(offsets[n].item())  # one host read to size the CSR
    calls = torch.empty((max(total_calls, 1), 24), dtype=torch.uint8, device=dev)
    _lib.check(lib.rs_plan_calls(_lib.ptr(configs), _lib.ptr(qlen), n, ctypes.byref(pc), int(max_context_tokens),
                                 _lib.ptr(offsets), _lib.ptr(calls), _lib.ptr(totals), 0, _lib.ptr(ws), ws.numel(),
                                 s), "rs_plan_calls(fill)")
    return offsets, calls[:total_calls], totals, status


def admit_fifo(spaces: torch.Tensor, profiles: torch.Tensor | None, qlen: torch.Tensor, params: SelectParams, *,
               capacity_bytes: int, used_bytes: int, max_context_tokens: int,
               has_profile: torch.Tensor | None = None, stream=None):
    """The FIFO new-query admission loop of Scheduler.step (scheduler.py
    :397-410) over a device batch of waiting entries in queue order.
    Returns device tensors (configs uint8 [n,16] rs_config, info uint8 [n,16]
    rs_admit_info, result uint8 [24] rs_admit_result); entries
    [0, result.admitted) were admitted, and ``result.stop`` says why the loop
    ended (rs_admit_stop)."""
    n = spaces.shape[0]
    dev = spaces.device
    lib = _lib.lib_for_device(_dev_index(spaces))
    configs = torch.empty((max(n, 1), 16), dtype=torch.uint8, device=dev)
    info = torch.empty((max(n, 1), 16), dtype=torch.uint8, device=dev)
    result = torch.empty(24, dtype=torch.uint8, device=dev)
    pc = params.c()
    ap = _lib.AdmitParamsC(int(capacity_bytes), int(used_bytes), int(max_context_tokens))
    _lib.check(lib.rs_admit_fifo(_lib.ptr(spaces), _lib.ptr(profiles), _lib.ptr(has_profile), _lib.ptr(qlen), n,
                                 ctypes.byref(pc), ctypes.byref(ap), _lib.ptr(configs), _lib.ptr(info),
                                 _lib.ptr(result), _lib.stream_ptr(stream)), "rs_admit_fifo")
    return configs[:n], info[:n], result


def candidate_costs(spaces: torch.Tensor, qlen: torch.Tensor, params: SelectParams, *, cost: CostModel | None = None,
                    running_before: torch.Tensor | None = None, stream=None):
    """Every candidate of every query's pruned space (enumerate_candidates
    order, mapping.py:129-156) with its plan_bytes and, given a cost model,
    its plan's critical-path delay.  Returns device (offsets int64 [n+1],
    records uint8 [total, 24] of rs_candidate); query i's candidates are
    records[offsets[i]:offsets[i+1]]."""
    n = spaces.shape[0]
    dev = spaces.device
    lib = _lib.lib_for_device(_dev_index(spaces))
    offsets = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ws = torch.empty(max(int(lib.rs_candidate_costs_workspace_size(n)), 4), dtype=torch.uint8, device=dev)
    pc = params.c()
    cp = ctypes.byref(cost.c()) if cost is not None else None
    s = _lib.stream_ptr(stream)
    _lib.check(lib.rs_candidate_costs(_lib.ptr(spaces), _lib.ptr(qlen), _lib.ptr(running_before), n, ctypes.byref(pc),
                                      cp, _lib.ptr(offsets), 0, _lib.ptr(ws), ws.numel(), s),
               "rs_candidate_costs(count)")
    total = int(offsets[n].item())  # one host read to size the table
    out = torch.empty((max(total, 1), 24), dtype=torch.uint8, device=dev)
    _lib.check(lib.rs_candidate_costs(_lib.ptr(spaces), _lib.ptr(qlen), _lib.ptr(running_before), n, ctypes.byref(pc),
                                      cp, _lib.ptr(offsets), _lib.ptr(out), _lib.ptr(ws), ws.numel(), s),
               "rs_candidate_costs(fill)")
    return offsets, out[:total]


def call_latency_batch(prompt_tokens: torch.Tensor, max_output_tokens: torch.Tensor, concurrent: torch.Tensor,
                       cost: CostModel, stream=None) -> torch.Tensor:
    n = prompt_tokens.shape[0]
    lib = _lib.lib_for_device(_dev_index(prompt_tokens))
    out = torch.empty(n, dtype=torch.float64, device=prompt_tokens.device)
    c = cost.c()
    _lib.check(lib.rs_call_latency(_lib.ptr(prompt_tokens), _lib.ptr(max_output_tokens), _lib.ptr(concurrent), n,
                                   ctypes.byref(c), _lib.ptr(out), _lib.stream_ptr(stream)), "rs_call_latency")
    return out


def plan_bytes_batch(method: torch.Tensor, num_chunks: torch.Tensor, interlen: torch.Tensor, qlen: torch.Tensor,
                     params: SelectParams, stream=None) -> torch.Tensor:
    n = method.shape[0]
    lib = _lib.lib_for_device(_dev_index(method))
    out = torch.empty(n, dtype=torch.int64, device=method.device)
    pc = params.c()
    _lib.check(lib.rs_plan_bytes(_lib.ptr(method), _lib.ptr(num_chunks), _lib.ptr(interlen), _lib.ptr(qlen), n,
                                 ctypes.byref(pc), _lib.ptr(out), _lib.stream_ptr(stream)), "rs_plan_bytes")
    return out


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.LibraryUnavailable("no CUDA device: paper_2412_10543_b200 runs only on a B200 (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())
