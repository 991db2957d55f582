"""Pure-Python restatement of the reference config path — TEST INFRASTRUCTURE.

Every function cites the reference ``file:line`` (paths relative to
``/root/reference/pkg/src/ragsched/``) whose behaviour it restates.  Values
are plain ints / floats / tuples so the oracle has no dependency on the
reference package (which does not exist on the GPU box).

Encodings shared with the CUDA path and the golden fixtures:

* method bits, in the reference grid order ``METHOD_ORDER`` (mapping.py:24):
  ``RERANK = 1`` (map_rerank), ``STUFF = 2``, ``REDUCE = 4`` (map_reduce).
* a space is ``(methods, n_lo, n_hi, il_lo, il_hi)``; ``il_lo = il_hi = 0``
  when map_reduce is absent (the reference's ``None`` range).
* a config is ``(method, num_chunks, interlen)`` with ``interlen = 0`` for the
  non-map_reduce methods (reference ``None``).
* selection status: ``0`` best fit inside the space, ``1`` fallback config,
  ``2`` MustQueue (the reference returns ``None`` from both functions).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass

RERANK, STUFF, REDUCE = 1, 2, 4
METHOD_ORDER = (RERANK, STUFF, REDUCE)          # mapping.py:24
SUMMARY_DOMAIN = (30, 200)                      # types.py:16
CHUNK_RANGE_FACTOR = 3                          # mapping.py:20
BUF_NUM, BUF_DEN = 102, 100                     # memory.py:25-26
GATE_THRESHOLD = 0.90                           # profiler.py:30
WINDOW_CAPACITY = 10                            # profiler.py:31
DEFAULT_FALLBACK_SPACE = (STUFF, 1, 5, 0, 0)    # profiler.py:40-42

ST_BEST_FIT, ST_FALLBACK, ST_MUST_QUEUE = 0, 1, 2


@dataclass(frozen=True)
class SelectParams:
    """Scalar parameters of best_fit_select / fallback_config
    (scheduler.py:127-191; defaults from config.py:36-47, types.py:12-13,
    mapping.py:90-91)."""

    per_token_bytes: int = 131072
    chunk_size: int = 1000
    out_budget: int = 10
    template_tokens: int = 64
    max_chunks: int = 35
    chunk_step: int = 1
    interlen_step: int = 10


def bytes_per_kv_token(num_layers, num_kv_heads, head_dim, bytes_per_element) -> int:
    """memory.py:70-73 — int(2 * L * H * D * width)."""
    return int(2 * num_layers * num_kv_heads * head_dim * bytes_per_element)


# -- Algorithm 1 pruning ------------------------------------------------------

def clamp_range(lo: int, hi: int, a: int, b: int) -> tuple[int, int]:
    """types.py:53-54 — IntRange.clamp_to."""
    return min(max(lo, a), b), min(max(hi, a), b)


def map_profile(complexity_high, joint, pieces, s_lo, s_hi, max_chunks=35):
    """mapping.py:106-126 — rule table: no joint -> {rerank}; joint & low
    complexity -> {stuff}; joint & high -> {stuff, reduce}.  Chunks
    [p, 3p] clamped to [1, max_chunks]; interlen = summary range iff reduce."""
    if not joint:
        methods = RERANK
    elif not complexity_high:
        methods = STUFF
    else:
        methods = STUFF | REDUCE
    n_lo, n_hi = clamp_range(pieces, CHUNK_RANGE_FACTOR * pieces, 1, max_chunks)
    if methods & REDUCE:
        return (methods, n_lo, n_hi, s_lo, s_hi)
    return (methods, n_lo, n_hi, 0, 0)


def hull_of_spaces(spaces):
    """mapping.py:180-200 — union of method sets, interval hulls; the
    interlen hull only over spaces carrying one, [30,200] when reduce is in
    the union but no space carried a range, dropped without reduce."""
    if not spaces:
        raise ValueError("hull of zero spaces")
    methods = 0
    n_lo, n_hi = spaces[0][1], spaces[0][2]
    il = None
    for m, lo, hi, a, b in spaces:
        methods |= m
        n_lo, n_hi = min(n_lo, lo), max(n_hi, hi)
        if m & REDUCE:
            il = (a, b) if il is None else (min(il[0], a), max(il[1], b))
    if methods & REDUCE:
        if il is None:
            il = SUMMARY_DOMAIN
        return (methods, n_lo, n_hi, il[0], il[1])
    return (methods, n_lo, n_hi, 0, 0)


def gate_sequence(profiles, threshold=GATE_THRESHOLD, default_space=DEFAULT_FALLBACK_SPACE,
                  max_chunks=35, window=None):
    """profiler.py:467-486 + RecentSpaceWindow :138-153, applied in order.

    ``profiles`` is a sequence of (cx, joint, pieces, s_lo, s_hi, conf).
    Returns (list of (space, used_fallback), window as a list, oldest first).
    """
    if not 0.0 < threshold <= 1.0:
        raise ValueError(f"threshold must be in (0, 1], got {threshold}")
    win = deque(window or (), maxlen=WINDOW_CAPACITY)
    out = []
    for cx, joint, pieces, s_lo, s_hi, conf in profiles:
        if conf >= threshold:
            space = map_profile(cx, joint, pieces, s_lo, s_hi, max_chunks)
            win.append(space)
            out.append((space, False))
        else:
            out.append((hull_of_spaces(list(win)) if win else default_space, True))
    return out, list(win)


# -- enumeration + KV memory model --------------------------------------------

def enumerate_grid(space, chunk_step=1, interlen_step=10):
    """mapping.py:129-156 (unsorted) — method-major, then n ascending (from
    lo by chunk_step, hi only when on-step), then interlen ascending."""
    methods, n_lo, n_hi, il_lo, il_hi = space
    chunks = range(n_lo, n_hi + 1, chunk_step)
    out = []
    for m in METHOD_ORDER:
        if not methods & m:
            continue
        if m == REDUCE:
            for n in chunks:
                for il in range(il_lo, il_hi + 1, interlen_step):
                    out.append((m, n, il))
        else:
            for n in chunks:
                out.append((m, n, 0))
    return out


def buffered_bytes(tokens: int, per_token_bytes: int) -> int:
    """memory.py:76-78 — integer ceil of the 2% buffer."""
    return (BUF_NUM * tokens * per_token_bytes + BUF_DEN - 1) // BUF_DEN


def plan_bytes(qlen, cfg, p: SelectParams) -> int:
    """memory.py:164-195 — whole-admission bytes in closed form."""
    m, n, il = cfg
    q, c, t, o, pt = qlen, p.chunk_size, p.template_tokens, p.out_budget, p.per_token_bytes
    if m == STUFF:
        return buffered_bytes(q + n * c + t + o, pt)
    if m == RERANK:
        return n * buffered_bytes(q + c + t + o, pt)
    if il <= 0:
        raise ValueError("map_reduce config requires a positive intermediate_length")
    return n * buffered_bytes(q + c + t + il, pt) + buffered_bytes(q + n * il + t + o, pt)


def best_fit_select(space, qlen, free_bytes, p: SelectParams):
    """scheduler.py:127-156 — stable ascending sort of the grid by bytes,
    reverse scan, first fit wins (so byte ties go to the latest grid slot).
    Returns (cfg, bytes) or None."""
    grid = enumerate_grid(space, p.chunk_step, p.interlen_step)
    keyed = sorted(((plan_bytes(qlen, c, p), i) for i, c in enumerate(grid)),
                   key=lambda t: t[0])
    for b, i in reversed(keyed):
        if b <= free_bytes:
            return grid[i], b
    return None


def fallback_config(joint, qlen, free_bytes, p: SelectParams):
    """scheduler.py:159-191 — rerank with as many chunks as fit (capped at
    max_chunks) for non-joint profiles, else the largest fitting stuff;
    never map_reduce.  Returns (cfg, bytes) or None (MustQueue)."""
    if not joint:
        call = buffered_bytes(qlen + p.chunk_size + p.template_tokens + p.out_budget,
                              p.per_token_bytes)
        k = min(free_bytes // call, p.max_chunks)
        if k < 1:
            return None
        return (RERANK, int(k), 0), int(k) * call
    for k in range(p.max_chunks, 0, -1):
        b = plan_bytes(qlen, (STUFF, k, 0), p)
        if b <= free_bytes:
            return (STUFF, k, 0), b
    return None


def select(space, joint, qlen, free_bytes, p: SelectParams, allow_fallback=True):
    """Decision order of Scheduler._try_admit_new (scheduler.py:335-378) for
    one query evaluated independently: best fit, else fallback, else
    MustQueue.  Returns (method, n, il, bytes, status); (0,0,0,0,2) queues."""
    r = best_fit_select(space, qlen, free_bytes, p)
    if r is not None:
        (m, n, il), b = r
        return (m, n, il, b, ST_BEST_FIT)
    if allow_fallback:
        r = fallback_config(joint, qlen, free_bytes, p)
        if r is not None:
            (m, n, il), b = r
            return (m, n, il, b, ST_FALLBACK)
    return (0, 0, 0, 0, ST_MUST_QUEUE)


# -- prefill / decode delay model ----------------------------------------------

@dataclass(frozen=True)
class CostModel:
    """sim.py:42-57 defaults."""

    prefill_secs_per_token: float = 1.0e-4
    decode_secs_per_token_base: float = 4.0e-3
    batch_slowdown_per_seq: float = 0.01


def call_latency(prompt_tokens, max_output_tokens, concurrent_seqs, cost: CostModel) -> float:
    """sim.py:84-92, evaluated in the same IEEE-double order."""
    prefill = cost.prefill_secs_per_token * prompt_tokens
    decode = (max_output_tokens * cost.decode_secs_per_token_base
              * (1.0 + cost.batch_slowdown_per_seq * concurrent_seqs))
    return prefill + decode


def plan_call_shapes(qlen, cfg, p: SelectParams):
    """memory.py:117-148 — per-call (prompt_tokens, max_output_tokens,
    independent) in plan order, without the context-window checks."""
    m, n, il = cfg
    q, c, t, o = qlen, p.chunk_size, p.template_tokens, p.out_budget
    if m == STUFF:
        return [(q + n * c + t, o, True)]
    if m == RERANK:
        return [(q + c + t, o, True)] * n
    return [(q + c + t, il, True)] * n + [(q + n * il + t, o, False)]


PLAN_OK, PLAN_NONE, PLAN_INVALID_CHUNKS, PLAN_CONTEXT_OVERFLOW, PLAN_BAD_INTERLEN = range(5)
KIND_SINGLE, KIND_MAPPER, KIND_REDUCER, KIND_RERANK = range(4)  # CallKind order (memory.py:29-33)


def plan_calls(qlen, cfg, p: SelectParams, max_context_tokens: int):
    """memory.py:89-150 — (status, calls, total_bytes); calls are
    (kind, prompt_tokens, max_output_tokens, kv_bytes, index).  The reference's
    exceptions map to statuses, checked in its order: InvalidChunkCount
    (:108-109), non-positive interlen (:531-532), then each call's context
    window (:81-86)."""
    m, n, il = cfg
    if not 1 <= n <= p.max_chunks:
        return PLAN_INVALID_CHUNKS, [], 0
    q, c, t, o, pt = qlen, p.chunk_size, p.template_tokens, p.out_budget, p.per_token_bytes
    if m == STUFF:
        prompt = q + n * c + t
        if prompt + o > max_context_tokens:
            return PLAN_CONTEXT_OVERFLOW, [], 0
        calls = [(KIND_SINGLE, prompt, o, buffered_bytes(prompt + o, pt), 0)]
    elif m == RERANK:
        prompt = q + c + t
        if prompt + o > max_context_tokens:
            return PLAN_CONTEXT_OVERFLOW, [], 0
        kv = buffered_bytes(prompt + o, pt)
        calls = [(KIND_RERANK, prompt, o, kv, i) for i in range(n)]
    else:
        if il <= 0:
            return PLAN_BAD_INTERLEN, [], 0
        mp = q + c + t
        if mp + il > max_context_tokens:
            return PLAN_CONTEXT_OVERFLOW, [], 0
        mkv = buffered_bytes(mp + il, pt)
        calls = [(KIND_MAPPER, mp, il, mkv, i) for i in range(n)]
        rp = q + n * il + t
        if rp + o > max_context_tokens:
            return PLAN_CONTEXT_OVERFLOW, [], 0
        calls.append((KIND_REDUCER, rp, o, buffered_bytes(rp + o, pt), 0))
    return PLAN_OK, calls, sum(x[3] for x in calls)


def plan_delay(qlen, cfg, p: SelectParams, cost: CostModel, running_before: int) -> float:
    """Critical-path delay of one admitted plan under the sim's dispatch rule
    (sim.py:223-229): the j-th independent call starts with
    ``running_before + j`` sequences already running; a map_reduce reducer is
    admitted once its mappers finished, i.e. with ``running_before``
    running.  Delay = max over independent calls + reducer latency."""
    calls = plan_call_shapes(qlen, cfg, p)
    indep = [c for c in calls if c[2]]
    worst = 0.0
    for j, (pr, out, _) in enumerate(indep):
        worst = max(worst, call_latency(pr, out, running_before + j, cost))
    for pr, out, ind in calls:
        if not ind:
            worst = worst + call_latency(pr, out, running_before, cost)
    return worst


# -- FIFO admission chain (Scheduler.step, scheduler.py:335-410) ---------------

(ADMIT_DRAINED, ADMIT_BLOCKED, ADMIT_NO_PROFILE, ADMIT_IMPOSSIBLE, ADMIT_FIXED_SPACE, ADMIT_INVALID_CHUNKS,
 ADMIT_CONTEXT_OVERFLOW, ADMIT_BAD_INTERLEN) = range(8)
_PLAN_TO_ADMIT = {PLAN_INVALID_CHUNKS: ADMIT_INVALID_CHUNKS, PLAN_CONTEXT_OVERFLOW: ADMIT_CONTEXT_OVERFLOW,
                  PLAN_BAD_INTERLEN: ADMIT_BAD_INTERLEN}


def admit_chain(entries, p: SelectParams, capacity: int, used: int, max_context_tokens: int,
                allow_fallback: bool = True):
    """The new-query loop of Scheduler.step over _try_admit_new
    (scheduler.py:335-410) with the accounting of _start_run (:281-333).
    ``entries``: (space, joint, has_profile, qlen) in queue order.  Returns
    (admitted, used_after, stop, stop_cfg): admitted = [(cfg, bytes, status,
    admitted_bytes, admitted_calls, fixed_path)], stop_cfg = the config of the
    entry that raised (plan errors and the fixed path's capacity check)."""
    out = []
    for space, joint, hasp, q in entries:
        free = capacity - used
        fixed = False
        r = best_fit_select(space, q, free, p)
        if r is not None:
            cfg, b = r
            status = ST_BEST_FIT
        elif allow_fallback:
            if not hasp:
                return out, used, ADMIT_NO_PROFILE, None          # :356-359
            r = fallback_config(joint, q, free, p)
            if r is None:
                return out, used, (ADMIT_IMPOSSIBLE if used == 0 else ADMIT_BLOCKED), None  # :370-378
            cfg, b = r
            status = ST_FALLBACK
        else:                                                    # fixed-config baseline :380-395
            grid = enumerate_grid(space, p.chunk_step, p.interlen_step)
            if len(grid) != 1:
                return out, used, ADMIT_FIXED_SPACE, None
            cfg, b, status, fixed = grid[0], None, ST_BEST_FIT, True
        st, calls, total = plan_calls(q, cfg, p, max_context_tokens)
        if st != PLAN_OK:
            return out, used, _PLAN_TO_ADMIT[st], cfg
        indep = [c for c in calls if c[0] != KIND_REDUCER]
        if fixed:
            smallest = min(c[3] for c in indep)
            if smallest > capacity:
                return out, used, ADMIT_IMPOSSIBLE, cfg
            if smallest > free:
                return out, used, ADMIT_BLOCKED, cfg
            adm, n_adm = 0, 0
            for c in indep:                                      # each call against the free bytes left
                if c[3] <= free - adm:
                    adm += c[3]
                    n_adm += 1
            b = total
        else:
            adm, n_adm = sum(c[3] for c in indep), len(indep)
        used += adm
        out.append((cfg, b, status, adm, n_adm, fixed))
    return out, used, ADMIT_DRAINED, None
