"""Best-fit + fallback selection (reference ``scheduler.py:127-191``) and the
stateful FIFO ``Scheduler`` (``scheduler.py:194-469``), on the GPU.  Scalar
drop-ins with the reference signatures; the batched fast paths are
:func:`paper_2412_10543_b200.batch.select` and ``batch.admit_fifo``.
"""

from __future__ import annotations

import itertools
from collections import deque
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np
import torch

from . import _lib
from . import batch as _b
from . import scalar as _scalar
from . import memory as _mem
from ._lib import SPACE_DTYPE
from .mapping import EnumGranularity
from .types import (
    DEFAULT_MAX_CHUNKS,
    DEFAULT_TEMPLATE_TOKENS,
    ContextOverflow,
    InvalidChunkCount,
    RagConfig,
    SynthesisMethod,
)


class SchedulingImpossible(RuntimeError):
    """scheduler.py:41."""


def _run_select(space, profile, q, free_bytes, params, config_cls, method_enum):
    """One query through ``rs_select`` (scalar fast path: pinned, device-mapped
    arguments; see scalar.py)."""
    rec = _scalar.select_one(_b.space_record(space) if space is not None else None,
                             _b.profile_tuple(profile) if profile is not None else None,
                             int(q.query_token_len), int(free_bytes), _b.params_c(params))
    return _b.unpack_config(rec, config_cls=config_cls, method_enum=method_enum)


def best_fit_select(space, q, free_bytes: int, *, model, meta, out_budget: int,
                    template_tokens: int = DEFAULT_TEMPLATE_TOKENS, granularity=EnumGranularity(),
                    config_cls=RagConfig, method_enum=SynthesisMethod):
    """scheduler.py:127-156 — the candidate with the largest whole-plan bytes
    that fits ``free_bytes`` (byte ties -> latest grid position); None if none
    fits."""
    params = _b.SelectParams.from_model(model, meta, out_budget, template_tokens, DEFAULT_MAX_CHUNKS, granularity,
                                        allow_fallback=False)
    return _run_select(space, None, q, free_bytes, params, config_cls, method_enum)


def fallback_config(profile, q, free_bytes: int, *, model, meta, out_budget: int,
                    template_tokens: int = DEFAULT_TEMPLATE_TOKENS, max_chunks: int = DEFAULT_MAX_CHUNKS,
                    config_cls=RagConfig, method_enum=SynthesisMethod):
    """scheduler.py:159-191 — rerank with as many chunks as fit (non-joint) or
    the largest fitting stuff (joint); never map_reduce; None = MustQueue."""
    params = _b.SelectParams.from_model(model, meta, out_budget, template_tokens, max_chunks, None,
                                        allow_fallback=True)
    # no candidates: the kernel goes straight to the fallback
    return _run_select(None, profile, q, free_bytes, params, config_cls, method_enum)


# -- the stateful scheduler (scheduler.py:33-469) -------------------------------
#
# Scheduler mirrors the reference class (same attributes, methods, trace
# events and exceptions).  Its new-query admission loop — the serial FIFO
# chain of best-fit / fallback / memory accounting that Scheduler.step runs
# over the waiting queue — is ONE kernel launch (rs_admit_fifo) over the
# packed queue, followed by one rs_plan_calls launch that expands the
# admitted configs into their calls.  The host applies those decisions to the
# per-call state (active runs, backlog, trace), which the reference keeps in
# Python objects too; completions and the backlog pass are pure bookkeeping.


class UnknownCall(KeyError):
    """A completion names a query or call that is not running."""


class MemorySafetyViolation(RuntimeError):
    """The KV accounting left [0, capacity] (a bug, never an input error)."""


@dataclass(frozen=True)
class SchedulerParams:
    """Model, corpus, output budget, template tokens, chunk cap, grid steps;
    ``allow_fallback`` off = the fixed-config baseline (scheduler.py:45-56)."""

    model: object
    meta: object
    out_budget: int
    template_tokens: int = DEFAULT_TEMPLATE_TOKENS
    max_chunks: int = DEFAULT_MAX_CHUNKS
    granularity: EnumGranularity = EnumGranularity()
    allow_fallback: bool = True


@dataclass
class PendingQuery:
    """A waiting-queue entry: the query, its pruned space and the gate
    metadata the caller reports later."""

    query: object
    space: object
    arrival_time: float
    profile: object = None
    truth: object = None
    gate_fallback: bool = False
    confidence: float = 1.0
    profiler_latency: float = 0.0


@dataclass(frozen=True)
class Admission:
    """What step() decided for one query."""

    query_id: str
    chosen_config: RagConfig
    admitted_calls: tuple
    deferred_calls: tuple
    is_fallback: bool


@dataclass(frozen=True)
class AdmittedCall:
    """One LLM call that entered the running batch."""

    query_id: str
    call_index: int
    prompt_tokens: int
    max_output_tokens: int
    kv_bytes: int


@dataclass(frozen=True)
class CompletionInfo:
    """What complete() reports back."""

    query_done: bool
    config: RagConfig
    is_fallback: bool
    newly_ready: tuple
    winning_rerank: int | None = None


@dataclass
class QueryRun:
    """Per-query call state: which plan calls are admitted / completed."""

    pending: PendingQuery
    config: RagConfig
    plan: object
    is_fallback: bool
    admission_time: float
    admitted: set = field(default_factory=set)
    completed: set = field(default_factory=set)
    rerank_confidences: dict = field(default_factory=dict)

    def deferred(self) -> list[int]:
        return sorted(set(range(len(self.plan.calls))).difference(self.admitted))

    def ready(self, idx: int) -> bool:
        return self.plan.calls[idx].depends_on.issubset(self.completed)

    def fully_admitted(self) -> bool:
        return not self.deferred()

    def done(self) -> bool:
        return len(self.completed) == len(self.plan.calls)


def own_classes() -> SimpleNamespace:
    """The value/exception classes a Scheduler builds (this package's
    mirrors; ``dropin`` substitutes the reference's own)."""
    return SimpleNamespace(
        Admission=Admission, AdmittedCall=AdmittedCall, CompletionInfo=CompletionInfo, QueryRun=QueryRun,
        UnknownCall=UnknownCall, MemorySafetyViolation=MemorySafetyViolation,
        SchedulingImpossible=SchedulingImpossible, InvalidChunkCount=InvalidChunkCount,
        ContextOverflow=ContextOverflow, RagConfig=RagConfig, SynthesisMethod=SynthesisMethod,
        LlmCall=_mem.LlmCall, CallPlan=_mem.CallPlan, CallKind=_mem.CallKind)


class Scheduler:
    """scheduler.py:194-469: the FIFO waiting queue, the running batch and the
    KV memory accounting, with the admission chain on the GPU."""

    classes = None  # SimpleNamespace of the classes to build (own_classes() when None)
    FIRST_CHUNK = 32  # queue entries packed for the first admission launch of a step (doubles)

    def __init__(self, capacity_bytes: int, params) -> None:
        if capacity_bytes <= 0:
            raise ValueError("capacity_bytes must be positive")
        self.capacity_bytes = capacity_bytes
        self.params = params
        self.used_bytes = 0
        self.waiting: deque = deque()
        self.active: dict = {}
        self.backlog_order: list[str] = []
        self.trace: list[dict] = []
        self._k = self.classes or own_classes()
        self._packed: dict[int, tuple] = {}
        g = params.granularity
        self._sel = _b.SelectParams.from_model(params.model, params.meta, params.out_budget, params.template_tokens,
                                               params.max_chunks, g, allow_fallback=params.allow_fallback)
        self._dev = None
        self._arena_obj = None
        self._inflight = 0  # calls admitted by step() and not yet completed (the sim's `running`, sim.py:224-281)

    @property
    def free_bytes(self) -> int:
        return self.capacity_bytes - self.used_bytes

    def submit(self, pending) -> None:
        self.waiting.append(pending)

    # -- admission ---------------------------------------------------------

    def _check_accounting(self) -> None:
        if self.used_bytes < 0 or self.used_bytes > self.capacity_bytes:
            raise self._k.MemorySafetyViolation(f"used {self.used_bytes} outside [0, {self.capacity_bytes}]")

    def _log(self, event: str, now: float, query: str, **fields) -> None:
        # trace records keep the reference's key order (event, t, query, ...)
        self.trace.append({"event": event, "t": now, "query": query, **fields})

    def _take(self, run, idx: int, now: float, sink: list, from_backlog: bool) -> None:
        """Admit one call: account its KV bytes and report it."""
        c = run.plan.calls[idx]
        qid = run.pending.query.id
        self.used_bytes += c.kv_bytes
        self._check_accounting()
        run.admitted.add(idx)
        sink.append(self._k.AdmittedCall(query_id=qid, call_index=idx, prompt_tokens=c.prompt_tokens,
                                         max_output_tokens=c.max_output_tokens, kv_bytes=c.kv_bytes))
        if from_backlog:
            self._log("admit_deferred", now, qid, call=idx, kv_bytes=c.kv_bytes)

    def _admit_backlog(self, now: float, sink: list) -> bool:
        """Deferred work first, in admission order (scheduler.py:257-270): a
        ready call that does not fit blocks everything behind it (returns
        True)."""
        for qid in tuple(self.backlog_order):
            run = self.active[qid]
            for idx in (i for i in run.deferred() if run.ready(i)):
                if run.plan.calls[idx].kv_bytes > self.free_bytes:
                    return True
                self._take(run, idx, now, sink, from_backlog=True)
            if run.fully_admitted():
                self.backlog_order.remove(qid)
        return False

    def _start_run(self, pending, cfg, plan, is_fallback: bool, now: float, sink: list, *,
                   admit_all_independent: bool):
        """Open the query's run and admit its independent calls
        (scheduler.py:281-333); the plan is rs_plan_calls' expansion."""
        qid = pending.query.id
        run = self._k.QueryRun(pending=pending, config=cfg, plan=plan, is_fallback=is_fallback, admission_time=now)
        self.active[qid] = run
        for idx in plan.independent_calls():
            if plan.calls[idx].kv_bytes <= self.free_bytes:
                self._take(run, idx, now, sink, from_backlog=False)
            elif admit_all_independent:
                raise self._k.MemorySafetyViolation(f"call {idx} of {qid} should fit after best-fit selection")
        later = tuple(run.deferred())
        if later:
            self.backlog_order.append(qid)
        now_in = tuple(sorted(run.admitted))
        self._log("admission", now, qid, config=cfg.describe(), admitted=list(now_in), deferred=list(later),
                  fallback=is_fallback)
        return self._k.Admission(query_id=qid, chosen_config=cfg, admitted_calls=now_in, deferred_calls=later,
                                 is_fallback=is_fallback)

    def _pack(self, pending) -> tuple:
        key = id(pending)
        rec = self._packed.get(key)
        if rec is None or rec[0] is not pending:
            sp = np.zeros(1, dtype=SPACE_DTYPE)
            sp[0] = (*_b.space_record(pending.space), 0, 0)
            prof = pending.profile
            pr = _b.pack_profiles([prof]) if prof is not None else np.zeros(1, dtype=_lib.PROFILE_DTYPE)
            rec = (pending, sp.tobytes(), pr.tobytes(), prof is not None, int(pending.query.query_token_len))
            self._packed[key] = rec
        return rec

    def _device(self):
        if self._dev is None:
            self._dev = _b.default_device()
        return self._dev

    def _arena(self):
        if self._arena_obj is None:
            self._arena_obj = _scalar.AdmitArena(self.FIRST_CHUNK, self.params.max_chunks + 1)
        return self._arena_obj

    def _admit_new(self, now: float, admissions: list, admitted: list) -> None:
        """The loop of scheduler.py:404-409 over _try_admit_new (:335-395),
        as rs_admit_fifo launches over chunks of the waiting queue (packed
        into a pinned, device-mapped arena: no copies, one round trip per
        chunk — the plan expansion follows the chain in stream order).  An entry the C records cannot hold (e.g. a map_reduce range
        starting at 0, memory.py:186-188) cuts the chunk before it; its error
        is raised only once it reaches the head of the queue, as the
        reference raises only for the entry it is admitting."""
        k, p = self._k, self.params
        arena = self._arena()
        chunk = self.FIRST_CHUNK
        while self.waiting:
            entries, pack_error = [], None
            for pq in itertools.islice(self.waiting, 0, chunk):
                try:
                    entries.append(self._pack(pq))
                except (ValueError, OverflowError) as e:
                    pack_error = e
                    break
            n = len(entries)
            if n == 0:
                raise pack_error
            arena.ensure(n)
            arena.spaces[:n] = np.frombuffer(b"".join(e[1] for e in entries), dtype=np.uint8).reshape(n, 16)
            arena.profiles[:n] = np.frombuffer(b"".join(e[2] for e in entries), dtype=np.uint8).reshape(n, 16)
            arena.hasprof[:n] = [e[3] for e in entries]
            arena.qlen[:n] = [e[4] for e in entries]
            m, stop, planned = arena.admit_and_plan(n, _b.params_c(self._sel), self.capacity_bytes, self.used_bytes,
                                                    p.model.max_context_tokens)
            cfg_all = arena.configs[: min(m + 1, n)].copy()
            if m:
                plans = _mem.plans_from_host(*planned, call_cls=k.LlmCall, plan_cls=k.CallPlan,
                                             kind_enum=k.CallKind)
                infos = arena.info[:m].copy()
            for j in range(m):
                pending = self.waiting[0]
                rec = cfg_all[j]
                cfg = _b.unpack_config(rec, config_cls=k.RagConfig, method_enum=k.SynthesisMethod)
                plan = plans[j]
                if isinstance(plan, int):  # the kernel checked the plan; a mismatch is a bug
                    raise _lib.RagschedError(f"rs_plan_calls rejected an admitted config (status {plan})")
                used0 = self.used_bytes
                adm = self._start_run(pending, cfg, plan, int(rec["status"]) == _lib.RS_SELECT_FALLBACK, now,
                                      admitted, admit_all_independent=not int(infos[j]["fixed_path"]))
                if self.used_bytes - used0 != int(infos[j]["admitted_bytes"]):
                    raise _lib.RagschedError("admission accounting diverged from rs_admit_fifo")
                self.waiting.popleft()
                self._packed.pop(id(pending), None)
                admissions.append(adm)
            if stop == _lib.RS_ADMIT_DRAINED:
                if pack_error is not None:
                    continue  # the unpackable entry is now the head: the next pass raises its error
                chunk *= 2
                continue
            if stop == _lib.RS_ADMIT_BLOCKED:
                return
            self._raise_stop(stop, self.waiting[0], cfg_all[m] if m < len(cfg_all) else None)

    def _raise_stop(self, stop: int, pending, rec) -> None:
        k, p = self._k, self.params
        q = pending.query
        cfg = None
        if rec is not None and int(rec["method"]) in (1, 2, 4):
            m = int(rec["method"])
            cfg = k.RagConfig(k.SynthesisMethod({1: "map_rerank", 2: "stuff", 4: "map_reduce"}[m]),
                              int(rec["num_chunks"]), int(rec["interlen"]) if m == 4 else None)
        if stop == _lib.RS_ADMIT_NO_PROFILE:
            raise k.SchedulingImpossible(f"query {q.id} needs the fallback path but carries no profile")
        if stop == _lib.RS_ADMIT_IMPOSSIBLE:
            if p.allow_fallback:
                raise k.SchedulingImpossible(f"query {q.id} cannot fit even with all memory free")
            raise k.SchedulingImpossible(f"fixed config {cfg.describe()} can never fit capacity for query {q.id}")
        if stop == _lib.RS_ADMIT_FIXED_SPACE:
            raise k.SchedulingImpossible("fallback is disabled but the space is not a single fixed config")
        if stop == _lib.RS_ADMIT_INVALID_CHUNKS:
            raise k.InvalidChunkCount(f"num_chunks {cfg.num_chunks} outside [1, {p.max_chunks}]")
        if stop == _lib.RS_ADMIT_BAD_INTERLEN:
            raise ValueError("map_reduce config requires a positive intermediate_length")
        if stop == _lib.RS_ADMIT_CONTEXT_OVERFLOW:
            raise k.ContextOverflow(self._overflow_message(q.query_token_len, cfg))
        raise OverflowError(f"KV byte arithmetic exceeds int64 for query {q.id}")

    def _overflow_message(self, qlen: int, cfg) -> str:
        p = self.params
        return _mem.context_overflow_message(qlen, cfg, p.meta.chunk_size, p.template_tokens, p.out_budget,
                                             p.model.max_context_tokens)

    def step(self, now: float):
        """One admission round (scheduler.py:397-410): the backlog, then — if
        it did not block — new queries in FIFO order."""
        decided, started = [], []
        if not self._admit_backlog(now, started) and self.waiting:
            self._admit_new(now, decided, started)
        if started:
            # the caller usually asks each started call's latency next, the
            # i-th at concurrency (calls running before) + i (sim.py:223-229):
            # evaluate them in one batch now (sim.precompute_latencies)
            from .sim import precompute_latencies

            precompute_latencies(started, self._inflight)
            self._inflight += len(started)
        return decided, started

    # -- completion --------------------------------------------------------

    def complete(self, query_id: str, call_index: int, now: float, rerank_confidence: float | None = None):
        """Release a finished call's KV bytes; settle the query after its last
        call (map_rerank: the highest-confidence call wins, lowest index on
        ties) — scheduler.py:414-466."""
        k = self._k
        run = self.active.get(query_id)
        if run is None:
            raise k.UnknownCall(f"no active query {query_id}")
        if call_index in run.completed or call_index not in run.admitted:
            raise k.UnknownCall(f"call {call_index} of {query_id} is not running")
        done_before = set(run.completed)
        self._inflight -= 1
        self.used_bytes -= run.plan.calls[call_index].kv_bytes
        self._check_accounting()
        run.completed.add(call_index)
        if rerank_confidence is not None:
            run.rerank_confidences[call_index] = rerank_confidence
        self._log("completion", now, query_id, call=call_index)
        # deferred calls this completion made ready (they were not before)
        newly_ready = tuple(i for i in run.deferred()
                            if run.ready(i) and not run.plan.calls[i].depends_on.issubset(done_before))
        info = dict(config=run.config, is_fallback=run.is_fallback, newly_ready=newly_ready)
        if not run.done():
            return k.CompletionInfo(query_done=False, **info)
        conf = run.rerank_confidences
        winner = None
        if conf and run.config.synthesis_method.value == "map_rerank":
            best = max(conf.values())
            winner = min(i for i, v in conf.items() if v == best)
        del self.active[query_id]
        if query_id in self.backlog_order:
            self.backlog_order.remove(query_id)
        self._log("query_done", now, query_id, winning_rerank=winner)
        return k.CompletionInfo(query_done=True, winning_rerank=winner, **info)

    def idle(self) -> bool:
        return not self.waiting and not self.active
