"""§8(f1): the stateful FIFO Scheduler (scheduler.py:194-469) with its
admission chain on the GPU (rs_admit_fifo + rs_plan_calls), replayed against
traces recorded from the reference Scheduler (tests/golden/
make_sched_golden.py): every admission, admitted call, completion info,
exception and the full ``trace`` must be identical."""

import pytest

from tests.golden_data import PARAM_SETS, scheduler_traces
from paper_2412_10543_b200 import scheduler as S
from paper_2412_10543_b200.mapping import EnumGranularity, PrunedConfigSpace, QueryProfile
from paper_2412_10543_b200.types import DatasetMeta, IntRange, ModelSpec, QueryRecord, SynthesisMethod

pytestmark = pytest.mark.gpu

TRACES = scheduler_traces()
FROM_BIT = {1: SynthesisMethod.MAP_RERANK, 2: SynthesisMethod.STUFF, 4: SynthesisMethod.MAP_REDUCE}


def dec_space(t):
    m, lo, hi, a, b = t
    return PrunedConfigSpace(frozenset(FROM_BIT[x] for x in (1, 2, 4) if m & x), IntRange(lo, hi),
                             IntRange(a, b) if m & 4 else None)


def make_scheduler(sc):
    L, H, D, w, cs, out, tmpl, mc, cstep, istep = PARAM_SETS[sc["ps"]]
    model = ModelSpec(L, H, D, w, max_context_tokens=sc.get("ctx", 131072))
    params = S.SchedulerParams(model=model, meta=DatasetMeta("golden", cs), out_budget=out, template_tokens=tmpl,
                               max_chunks=sc.get("max_chunks", mc), granularity=EnumGranularity(cstep, istep),
                               allow_fallback=sc.get("allow_fallback", True))
    return S.Scheduler(sc["capacity"], params)


def enc_adm(a):
    return [a.query_id, a.chosen_config.describe(), list(a.admitted_calls), list(a.deferred_calls), a.is_fallback]


def enc_call(c):
    return [c.query_id, c.call_index, c.prompt_tokens, c.max_output_tokens, c.kv_bytes]


def enc_info(i):
    return [i.query_done, i.config.describe(), i.is_fallback, list(i.newly_ready), i.winning_rerank]


@pytest.mark.parametrize("rec", TRACES, ids=[r["name"] for r in TRACES])
def test_scheduler_replays_reference_trace(rec):
    sched = make_scheduler(rec["scenario"])
    for k, op in enumerate(rec["ops"]):
        if op[0] == "submit":
            _, qid, qlen, space, prof = op
            p = None if prof is None else QueryProfile(bool(prof[0]), bool(prof[1]), prof[2],
                                                       IntRange(prof[3], prof[4]), prof[5])
            sched.submit(S.PendingQuery(query=QueryRecord(id=qid, text="t", query_token_len=qlen),
                                        space=dec_space(space), arrival_time=0.0, profile=p))
        elif op[0] == "step":
            _, now, want = op
            if "raise" in want:
                with pytest.raises(Exception) as ei:
                    sched.step(now)
                assert [type(ei.value).__name__, str(ei.value)] == want["raise"], k
                continue
            adms, admitted = sched.step(now)
            assert [enc_adm(a) for a in adms] == want["admissions"], k
            assert [enc_call(c) for c in admitted] == want["admitted"], k
            assert sched.used_bytes == want["used"], k
        else:
            _, qid, idx, now, conf, want = op
            if "raise" in want:
                with pytest.raises(S.UnknownCall):
                    sched.complete(qid, idx, now)
                continue
            info = sched.complete(qid, idx, now, rerank_confidence=conf)
            assert enc_info(info) == want["info"], k
            assert sched.used_bytes == want["used"], k
    assert sched.trace == rec["trace"]


def test_admit_chain_single_launch_for_a_burst():
    """A burst of waiting queries is admitted by one rs_admit_fifo launch per
    chunk (plus the plan expansion), not one launch per query."""
    from paper_2412_10543_b200 import _lib
    from paper_2412_10543_b200 import sim as SIM

    SIM._LAST_COST[0] = None  # no latency batch yet (test_dispatch_latencies_are_batch_evaluated)
    sc = dict(ps=0, capacity=64 * 1024**3)
    sched = make_scheduler(sc)
    prof = QueryProfile(False, True, 2, IntRange(30, 60), 0.95)
    for i in range(30):
        sched.submit(S.PendingQuery(query=QueryRecord(id=f"q{i}", text="t", query_token_len=500),
                                    space=PrunedConfigSpace(frozenset({SynthesisMethod.STUFF}), IntRange(2, 6)),
                                    arrival_time=0.0, profile=prof))
    l0 = _lib.launch_count()
    adms, admitted = sched.step(0.0)
    assert len(adms) == 30 and len(admitted) == 30
    assert _lib.launch_count() - l0 <= 4


def test_dispatch_latencies_are_batch_evaluated():
    """Scheduler.step evaluates the started calls' latencies in one launch at
    concurrency (running before) + i, as the reference's dispatch asks for
    them (sim.py:223-229); call_latency then returns those values — bit-equal
    to the scalar path — and takes the scalar path for anything else."""
    from paper_2412_10543_b200 import _lib
    from paper_2412_10543_b200 import sim as SIM
    from paper_2412_10543_b200.batch import CostModel

    cost = CostModel()
    sched = make_scheduler(dict(ps=0, capacity=64 * 1024**3))
    prof = QueryProfile(False, True, 2, IntRange(30, 60), 0.95)
    for i in range(12):
        sched.submit(S.PendingQuery(query=QueryRecord(id=f"q{i}", text="t", query_token_len=300 + 37 * i),
                                    space=PrunedConfigSpace(frozenset({SynthesisMethod.MAP_RERANK}), IntRange(2, 6)),
                                    arrival_time=0.0, profile=prof))
    SIM._LAST_COST[0] = None
    SIM._PRE.clear()
    _, first = sched.step(0.0)  # no cost model seen yet: nothing precomputed
    assert len(first) > 2 and not SIM._PRE
    scalar = [SIM.call_latency(ac, i, cost) for i, ac in enumerate(first)]  # learns the cost model
    for ac in first:
        sched.complete(ac.query_id, ac.call_index, 1.0, rerank_confidence=0.5)
    for i in range(12, 20):
        sched.submit(S.PendingQuery(query=QueryRecord(id=f"q{i}", text="t", query_token_len=300 + 37 * i),
                                    space=PrunedConfigSpace(frozenset({SynthesisMethod.MAP_RERANK}), IntRange(2, 6)),
                                    arrival_time=1.0, profile=prof))
    l0 = _lib.launch_count()
    _, started = sched.step(1.0)
    assert len(started) > 2 and len(SIM._PRE) == len(started)
    launches = _lib.launch_count() - l0
    running = 0  # every first-step call completed
    got = [SIM.call_latency(ac, running + i, cost) for i, ac in enumerate(started)]
    assert _lib.launch_count() - l0 == launches  # served from the batch, no scalar launch
    SIM._PRE.clear()
    want = [SIM.call_latency(ac, running + i, cost) for i, ac in enumerate(started)]  # scalar path
    assert got == want and all(isinstance(x, float) for x in got)
    # a different concurrency or cost model is never served from the batch
    sched2 = make_scheduler(dict(ps=0, capacity=64 * 1024**3))
    sched2.submit(S.PendingQuery(query=QueryRecord(id="z", text="t", query_token_len=500),
                                 space=PrunedConfigSpace(frozenset({SynthesisMethod.MAP_RERANK}), IntRange(4, 4)),
                                 arrival_time=0.0, profile=prof))
    _, st2 = sched2.step(0.0)
    v_wrong = SIM.call_latency(st2[0], 7, cost)
    SIM._PRE.clear()
    assert v_wrong == SIM.call_latency(st2[0], 7, cost)
    assert scalar and all(isinstance(x, float) for x in scalar)


SIM_GATES = [r for r in TRACES if r.get("gates")]


@pytest.mark.parametrize("rec", SIM_GATES, ids=[r["name"] for r in SIM_GATES])
def test_gate_replays_reference_sim(rec):
    """The confidence gate as the reference's sim.run drove it (QueryProfiler.gate
    -> gate_profile, profiler.py:534-541): the same profiles in order through this
    package's GPU gate_profile with its own window give the same decisions."""
    from types import SimpleNamespace

    from paper_2412_10543_b200 import profiler as G

    window = G.RecentSpaceWindow()
    for k, (prof, want, (thr, default_space, max_chunks)) in enumerate(rec["gates"]):
        p = QueryProfile(bool(prof[0]), bool(prof[1]), prof[2], IntRange(prof[3], prof[4]), prof[5])
        d = G.gate_profile(SimpleNamespace(profile=p), window, thr, default_space=dec_space(default_space),
                           max_chunks=max_chunks)
        m = 0
        for x in d.space.synthesis_methods:
            m |= {"map_rerank": 1, "stuff": 2, "map_reduce": 4}[x.value]
        il = d.space.intermediate_length_range
        got = [[m, d.space.num_chunks_range.low, d.space.num_chunks_range.high, il.low if il else 0,
                il.high if il else 0], d.used_fallback, d.confidence]
        assert got == want, (k, got, want)
