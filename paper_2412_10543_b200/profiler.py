"""Confidence gate (reference ``profiler.py:467-486``) on the GPU.

``gate_profile`` keeps the reference signature and semantics; the decision
(accept → Algorithm-1 space, reject → hull of the last <= 10 accepted spaces
or the default space) is computed by the ``rs_prune_gate`` kernel with the
caller's window contents as carry-in state.  For streams of queries use
:func:`paper_2412_10543_b200.batch.prune_gate`, which gates a whole batch in
one launch sequence.
"""

from __future__ import annotations

import functools
from collections import deque
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import batch as _b
from . import scalar as _scalar
from .mapping import PrunedConfigSpace, hull_of_spaces
from .types import DEFAULT_MAX_CHUNKS, IntRange, SynthesisMethod

GATE_THRESHOLD = 0.90                 # profiler.py:30
WINDOW_CAPACITY = 10                  # profiler.py:31
DEFAULT_FALLBACK_SPACE = PrunedConfigSpace(frozenset({SynthesisMethod.STUFF}), IntRange(1, 5))  # :40-42


class RecentSpaceWindow:
    """Ring buffer of the most recently accepted spaces (profiler.py:138-153)."""

    def __init__(self, capacity: int = WINDOW_CAPACITY) -> None:
        self._spaces: deque = deque(maxlen=capacity)

    def push(self, space) -> None:
        self._spaces.append(space)

    def hull(self):
        return hull_of_spaces(list(self._spaces)) if self._spaces else None

    def spaces(self) -> list:
        return list(self._spaces)

    def __len__(self) -> int:
        return len(self._spaces)


@dataclass(frozen=True)
class GateDecision:
    """profiler.py:156-163."""

    space: PrunedConfigSpace
    used_fallback: bool
    confidence: float


def _window_spaces(window) -> list:
    if window is None:
        return []
    if hasattr(window, "spaces") and callable(window.spaces):
        return window.spaces()
    return list(getattr(window, "_spaces", ()))  # the reference's RecentSpaceWindow


def _gate_one(profile, window_spaces, *, threshold, default_space, max_chunks, space_cls=None,
              method_enum=None, range_cls=None):
    """Run the gate kernel on one profile (scalar fast path, scalar.py).
    threshold=None means "always accept" (plain map_profile).  Returns
    (space, used_fallback)."""
    space_cls = space_cls or PrunedConfigSpace
    method_enum = method_enum or SynthesisMethod
    range_cls = range_cls or IntRange
    prof = _b.profile_tuple(profile)
    if threshold is None:
        prof = prof[:5] + (1.0,)
    ds = _space_rec(default_space if default_space is not None else DEFAULT_FALLBACK_SPACE)
    gp = _gate_params(float(threshold) if threshold is not None else 1.0, ds, int(max_chunks))
    r = _scalar.gate_one(prof, [_space_rec(s) for s in window_spaces], gp)
    if r[5] and default_space is not None and not window_spaces:
        return default_space, True  # `window.hull() or default_space` returns the object itself
    return _space_obj(r[:5], space_cls, method_enum, range_cls), bool(r[5])


def _space_rec(space) -> tuple:
    """space_record, memoised for hashable (frozen) spaces: a gate call
    re-encodes the default space and up to 10 window spaces."""
    try:
        return _space_rec_cached(space)
    except TypeError:  # unhashable space object
        return _b.space_record(space)


@functools.lru_cache(maxsize=4096)
def _space_rec_cached(space) -> tuple:
    return _b.space_record(space)


@functools.lru_cache(maxsize=4096)
def _space_obj(rec: tuple, space_cls, method_enum, range_cls):
    """A gate result record -> the (frozen, immutable) space object, memoised."""
    m, nlo, nhi, illo, ilhi = rec
    return _b.unpack_space({"methods": m, "num_chunks_lo": nlo, "num_chunks_hi": nhi, "interlen_lo": illo,
                            "interlen_hi": ilhi}, space_cls=space_cls, method_enum=method_enum, range_cls=range_cls)


@functools.lru_cache(maxsize=64)
def _gate_params(threshold: float, ds: tuple, max_chunks: int):
    return _lib.GateParamsC(threshold, _lib.SpaceC(ds[0], ds[1], ds[2], ds[3], ds[4], 1, 0), max_chunks, 0)


def gate_profile(out, window, threshold: float = GATE_THRESHOLD, *, default_space=DEFAULT_FALLBACK_SPACE,
                 max_chunks: int = DEFAULT_MAX_CHUNKS, decision_cls=GateDecision, space_cls=None,
                 method_enum=None, range_cls=None):
    """profiler.py:467-486 — accept the profile's space when confident, else
    the window hull (or ``default_space`` when nothing was accepted yet).
    Accepted spaces are pushed into ``window``."""
    if not 0.0 < threshold <= 1.0:
        raise ValueError(f"threshold must be in (0, 1], got {threshold}")
    profile = out.profile
    space, fb = _gate_one(profile, _window_spaces(window), threshold=threshold, default_space=default_space,
                          max_chunks=max_chunks, space_cls=space_cls, method_enum=method_enum,
                          range_cls=range_cls)
    if not fb:
        window.push(space)
    return decision_cls(space=space, used_fallback=fb, confidence=profile.confidence)


def window_records(window) -> np.ndarray:
    return _b.pack_spaces(_window_spaces(window))


# -- answer ingestion (profiler.py:191-254) -------------------------------------

PROFILE_FIELDS = ("complexity", "joint_reasoning", "pieces", "summary_range")  # profiler.py:51


class UnparseableAnswer(ValueError):
    """profiler.py:84-85."""


def parse_profile_text(text: str, confidence: float = 1.0, *, profile_cls=None, range_cls=IntRange,
                       exc_cls=UnparseableAnswer):
    """profiler.py:203-254 through the native batch parser (``rs_parse_profiles``):
    (profile, clamped field names, field line numbers); raises
    UnparseableAnswer when a field is missing."""
    recs, clamped, status, lines = _b.parse_profiles([text], [confidence], nthreads=1)
    if status[0] != _b.RS_PARSE_OK:
        raise exc_cls(f"missing fields {[PROFILE_FIELDS[i] for i in range(4) if lines[0, i] < 0]} "
                      f"in estimator answer: {text!r}")
    return (_b.unpack_profile(recs[0], profile_cls=profile_cls, range_cls=range_cls),
            _b.clamped_names(clamped[0]), {f: int(lines[0, i]) for i, f in enumerate(PROFILE_FIELDS)})


def per_field_confidences(content: str, tokens: list[dict] | None) -> dict[str, float]:
    """_per_field_confidences (profiler.py:427-464) through the native
    ``rs_field_confidences``: each answer token falls on the line its
    starting character lies in; a field's confidence is the exponentiated
    mean log-prob of its line's tokens, 1.0 without any (or without tokens,
    or when the answer does not parse)."""
    if not tokens:
        return {name: 1.0 for name in PROFILE_FIELDS}
    row = _b.field_confidences([content], [tokens], nthreads=1)[0]
    return {name: float(row[i]) for i, name in enumerate(PROFILE_FIELDS)}
