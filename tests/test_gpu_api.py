"""The reference-named scalar API on the GPU, mirroring the reference's own
unit tests (test_scheduler.py, test_profiler.py, test_memory.py, test_sim.py)
with this package's types."""

import random

import pytest

from oracle import config_oracle as co
from paper_2412_10543_b200 import (
    DEFAULT_FALLBACK_SPACE,
    DatasetMeta,
    EnumGranularity,
    GateDecision,
    IntRange,
    ModelSpec,
    PrunedConfigSpace,
    QueryProfile,
    QueryRecord,
    RagConfig,
    RecentSpaceWindow,
    SynthesisMethod,
    best_fit_select,
    call_latency,
    enumerate_candidates,
    fallback_config,
    gate_profile,
    map_profile,
    plan_bytes,
)
from paper_2412_10543_b200.sim import CostModel

pytestmark = pytest.mark.gpu

RR, ST, MR = SynthesisMethod.MAP_RERANK, SynthesisMethod.STUFF, SynthesisMethod.MAP_REDUCE
MODEL = ModelSpec(32, 8, 128, 2, max_context_tokens=131072)
META = DatasetMeta(description="corpus", chunk_size=1000)
OUT = 40
KW = dict(model=MODEL, meta=META, out_budget=OUT)
P = co.SelectParams(chunk_size=1000, out_budget=OUT)


def q(tokens=100):
    return QueryRecord(id="q", text="t", query_token_len=tokens)


def whole(query, cfg):
    bit = {RR: 1, ST: 2, MR: 4}[cfg.synthesis_method]
    return co.plan_bytes(query.query_token_len, (bit, cfg.num_chunks, cfg.intermediate_length or 0), P)


def prof(joint, complex_=False, pieces=2, conf=0.95, lo=60, hi=120):
    return QueryProfile(complex_, joint, pieces, IntRange(lo, hi), conf)


def test_best_fit_picks_six_when_seven_does_not_fit():
    space = PrunedConfigSpace(frozenset({ST}), IntRange(5, 10))
    free = whole(q(), RagConfig(ST, 6))
    assert best_fit_select(space, q(), free, **KW) == RagConfig(ST, 6)


def test_best_fit_top_of_range_and_none():
    space = PrunedConfigSpace(frozenset({ST}), IntRange(5, 10))
    assert best_fit_select(space, q(), 10**15, **KW) == RagConfig(ST, 10)
    assert best_fit_select(space, q(), whole(q(), RagConfig(ST, 5)) - 1, **KW) is None


def test_best_fit_matches_exhaustive_oracle():
    rng = random.Random(2024)
    for trial in range(60):
        p = prof(rng.random() < 0.5, rng.random() < 0.5, rng.randint(1, 10),
                 lo=min(a := rng.randint(30, 200), b := rng.randint(30, 200)), hi=max(a, b))
        space = map_profile(p)
        query = q(rng.randint(10, 3000))
        sizes = [whole(query, c) for c in enumerate_candidates(space)]
        free = rng.choice([rng.randint(0, min(sizes)), rng.randint(min(sizes), max(sizes))])
        want = None
        for i, c in enumerate(enumerate_candidates(space)):
            b = whole(query, c)
            if b <= free and (want is None or (b, i) > want[0]):
                want = ((b, i), c)
        assert best_fit_select(space, query, free, **KW) == (want[1] if want else None)


def test_best_fit_respects_granularity():
    space = PrunedConfigSpace(frozenset({ST, MR}), IntRange(3, 9), IntRange(40, 110))
    g = EnumGranularity(2, 25)
    got = best_fit_select(space, q(), 10**15, granularity=g, **KW)
    cands = enumerate_candidates(space, g)
    best = max(range(len(cands)), key=lambda i: (whole(q(), cands[i]), i))
    assert got == cands[best]


def test_fallback_cases():
    one = whole(q(), RagConfig(RR, 1))
    assert fallback_config(prof(False), q(), 2 * one + one // 2, **KW) == RagConfig(RR, 2)
    st3 = whole(q(), RagConfig(ST, 3))
    assert fallback_config(prof(True), q(), st3, **KW) == RagConfig(ST, 3)
    assert fallback_config(prof(False), q(), 0, **KW) is None
    assert fallback_config(prof(True), q(), 0, **KW) is None
    assert fallback_config(prof(False), q(), 10**15, max_chunks=20, **KW) == RagConfig(RR, 20)


def test_map_profile_rule_table():
    assert map_profile(prof(False, True, 4)) == PrunedConfigSpace(frozenset({RR}), IntRange(4, 12))
    assert map_profile(prof(True, False, 4)) == PrunedConfigSpace(frozenset({ST}), IntRange(4, 12))
    assert map_profile(prof(True, True, 9)) == PrunedConfigSpace(frozenset({ST, MR}), IntRange(9, 27),
                                                                 IntRange(60, 120))
    assert map_profile(prof(True, True, 10), max_chunks=20).num_chunks_range == IntRange(10, 20)
    assert map_profile(prof(True, False, 10, conf=0.0)).num_chunks_range == IntRange(10, 30)


class Out:
    def __init__(self, p):
        self.profile = p


def test_gate_accept_reject_and_window():
    w = RecentSpaceWindow()
    d = gate_profile(Out(prof(True, False, 2, conf=0.95)), w, threshold=0.90)
    assert isinstance(d, GateDecision) and not d.used_fallback and len(w) == 1
    w2 = RecentSpaceWindow()
    w2.push(PrunedConfigSpace(frozenset({ST}), IntRange(2, 6)))
    w2.push(PrunedConfigSpace(frozenset({ST}), IntRange(4, 9)))
    d = gate_profile(Out(prof(True, conf=0.80)), w2, threshold=0.90)
    assert d.used_fallback and d.space.num_chunks_range == IntRange(2, 9) and len(w2) == 2
    d = gate_profile(Out(prof(True, conf=0.80)), RecentSpaceWindow(), threshold=0.90)
    assert d.used_fallback and d.space == DEFAULT_FALLBACK_SPACE
    with pytest.raises(ValueError):
        gate_profile(Out(prof(True)), RecentSpaceWindow(), threshold=0.0)


def test_window_is_bounded_at_ten_through_gate():
    w = RecentSpaceWindow()
    for i in range(25):
        w.push(PrunedConfigSpace(frozenset({ST}), IntRange(1, i + 1)))
    d = gate_profile(Out(prof(True, conf=0.5)), w)
    assert d.space.num_chunks_range == IntRange(1, 25)


def test_plan_bytes_and_latency_scalars():
    assert plan_bytes(100, RagConfig(ST, 3), 1000, 131072, 40) == whole(q(), RagConfig(ST, 3))
    with pytest.raises(ValueError):
        plan_bytes(100, RagConfig(MR, 3, None), 1000, 131072, 40)

    class Call:
        prompt_tokens, max_output_tokens = 6564, 10

    assert call_latency(Call, 0, CostModel()) == 0.6564 + 0.04 or abs(call_latency(Call, 0, CostModel()) - 0.6964) < 1e-12
    assert call_latency(Call, 10, CostModel()) == co.call_latency(6564, 10, 10, co.CostModel())
