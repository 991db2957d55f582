"""Generate the golden fixtures by RUNNING THE REFERENCE (``ragsched``).

Run in the dev container only (``/root/reference`` does not exist on the GPU
box):  ``python tests/golden/make_golden.py``.  The outputs are committed
(``tests/golden/*.npz``) and are the parity pins for the oracle and the CUDA
path.  Every case is produced by calling the reference's own public functions:
``map_profile`` / ``gate_profile`` / ``mock_estimate`` (profiler.py,
mapping.py), ``plan_bytes`` / ``plan_calls`` / ``buffered_bytes``
(memory.py), ``best_fit_select`` / ``fallback_config`` (scheduler.py) and
``call_latency`` (sim.py).  The random streams replay the reference tests'
own seeds where they exist (A1 seed 42, A2 seed 43 — test_acceptance.py:132,
:173; best-fit oracle seed 2024 — test_scheduler.py:122; zero-noise gate seed
17 — test_profiler.py:219).
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from ragsched.config import DEFAULT_META, DEFAULT_MODEL  # noqa: E402
from ragsched.mapping import (  # noqa: E402
    EnumGranularity,
    PrunedConfigSpace,
    QueryProfile,
    enumerate_candidates,
    map_profile,
)
from ragsched.memory import (  # noqa: E402
    buffered_bytes,
    bytes_per_kv_token,
    plan_bytes,
    plan_calls,
)
from ragsched.profiler import (  # noqa: E402
    DEFAULT_FALLBACK_SPACE,
    NoiseParams,
    RecentSpaceWindow,
    ZERO_NOISE,
    gate_profile,
    mock_estimate,
    profile_from_truth,
)
from ragsched.scheduler import best_fit_select, fallback_config  # noqa: E402
from ragsched.sim import CostModel, call_latency  # noqa: E402
from ragsched.types import (  # noqa: E402
    DatasetMeta,
    IntRange,
    ModelSpec,
    QueryRecord,
    RagConfig,
    SynthesisMethod,
    TrueProfile,
)
from ragsched.workload import DATASET_PROFILES, TruthDistribution  # noqa: E402

OUT_DIR = os.path.dirname(os.path.abspath(__file__))
BIT = {SynthesisMethod.MAP_RERANK: 1, SynthesisMethod.STUFF: 2, SynthesisMethod.MAP_REDUCE: 4}
FROM_BIT = {v: k for k, v in BIT.items()}


def enc_space(s: PrunedConfigSpace):
    m = 0
    for x in s.synthesis_methods:
        m |= BIT[x]
    il = s.intermediate_length_range
    return (m, s.num_chunks_range.low, s.num_chunks_range.high,
            il.low if il else 0, il.high if il else 0)


def dec_space(t) -> PrunedConfigSpace:
    m, lo, hi, a, b = (int(x) for x in t)
    methods = frozenset(FROM_BIT[bit] for bit in (1, 2, 4) if m & bit)
    return PrunedConfigSpace(methods, IntRange(lo, hi), IntRange(a, b) if m & 4 else None)


def enc_cfg(c: RagConfig | None):
    if c is None:
        return (0, 0, 0)
    return (BIT[c.synthesis_method], c.num_chunks, c.intermediate_length or 0)


def profile(cx, joint, pieces, lo, hi, conf=0.95):
    return QueryProfile(complexity_high=bool(cx), needs_joint_reasoning=bool(joint),
                        pieces_required=int(pieces), summary_len_range=IntRange(int(lo), int(hi)),
                        confidence=float(conf))


# -- G1: Algorithm-1 mapping (A1 replay, seed 42) ----------------------------

def gen_mapping():
    rng = random.Random(42)
    rows, spaces = [], []
    for _ in range(10_000):
        joint = rng.random() < 0.5
        cx = rng.random() < 0.5
        pieces = rng.randint(1, 10)
        lo = rng.randint(30, 200)
        hi = rng.randint(lo, 200)
        for mc in (35, 12):
            rows.append((int(cx), int(joint), pieces, lo, hi, mc))
            spaces.append(enc_space(map_profile(profile(cx, joint, pieces, lo, hi), max_chunks=mc)))
    np.savez_compressed(os.path.join(OUT_DIR, "mapping.npz"),
                        profiles=np.array(rows, dtype=np.int32),
                        spaces=np.array(spaces, dtype=np.int32))
    print("mapping:", len(rows))


# -- G2: best-fit + fallback selection ---------------------------------------

PARAM_SETS = [
    # (layers, heads, head_dim, width, chunk_size, out_budget, template, max_chunks, chunk_step, interlen_step)
    (32, 8, 128, 2, 1000, 10, 64, 35, 1, 10),    # DEFAULT_MODEL / DEFAULT_META, out 10 (A2)
    (32, 8, 128, 2, 1000, 40, 64, 35, 1, 10),    # test_scheduler.py MODEL/META/OUT
    (32, 8, 128, 2, 1024, 40, 64, 35, 1, 10),    # doc_level_qa, FinSec chunk 1024
    (32, 8, 128, 2, 1024, 60, 64, 35, 1, 10),    # summarization_qa
    (32, 8, 128, 2, 1000, 20, 64, 35, 1, 10),    # multihop_qa
    (80, 8, 128, 1, 512, 10, 0, 20, 2, 5),       # fp8 70B-ish, coarse grid
    (28, 4, 128, 0.5, 1000, 60, 100, 50, 1, 1),  # packed 4-bit, fine interlen grid
    (16, 16, 64, 4, 700, 7, 33, 35, 3, 7),       # fp32 cache, odd steps
]


def params_kw(ps):
    L, H, D, w, cs, out, tmpl, mc, cstep, istep = ps
    model = ModelSpec(L, H, D, w, max_context_tokens=131072)
    meta = DatasetMeta(description="golden", chunk_size=cs)
    return model, meta, out, tmpl, mc, EnumGranularity(cstep, istep)


def whole(q, cfg, model, meta, out, tmpl):
    return plan_bytes(q.query_token_len, cfg, meta.chunk_size, bytes_per_kv_token(model), out, tmpl)


def ref_select(space, prof, q, free, ps):
    model, meta, out, tmpl, mc, gran = params_kw(ps)
    cfg = best_fit_select(space, q, free, model=model, meta=meta, out_budget=out,
                          template_tokens=tmpl, granularity=gran)
    status = 0
    if cfg is None:
        cfg = fallback_config(prof, q, free, model=model, meta=meta, out_budget=out,
                              template_tokens=tmpl, max_chunks=mc)
        status = 1 if cfg is not None else 2
    b = whole(q, cfg, model, meta, out, tmpl) if cfg is not None else 0
    return enc_cfg(cfg), b, status


def random_profile(rng):
    return profile(rng.random() < 0.5, rng.random() < 0.5, rng.randint(1, 10),
                   *sorted((rng.randint(30, 200), rng.randint(30, 200))))


def random_arbitrary_space(rng, mc):
    m = rng.randint(1, 7)
    lo = rng.randint(1, mc)
    hi = rng.randint(lo, mc)
    methods = frozenset(FROM_BIT[b] for b in (1, 2, 4) if m & b)
    il = None
    if m & 4:
        a = rng.randint(1, 300)
        il = IntRange(a, rng.randint(a, 320))
    return PrunedConfigSpace(methods, IntRange(lo, hi), il)


FULL_SPACE = PrunedConfigSpace(frozenset(SynthesisMethod), IntRange(1, 35), IntRange(30, 200))


def gen_select():
    rows = []  # ps, methods, n_lo, n_hi, il_lo, il_hi, joint, qlen, free, m, n, il, bytes, status, tie

    def add(ps_i, space, prof, q, free):
        ps = PARAM_SETS[ps_i]
        (m, n, il), b, st = ref_select(space, prof, q, free, ps)
        model, meta, out, tmpl, mc, gran = params_kw(ps)
        sizes = [whole(q, c, model, meta, out, tmpl) for c in enumerate_candidates(space, gran)]
        tie = int(len(sizes) != len(set(sizes)))
        rows.append((ps_i, *enc_space(space), int(prof.needs_joint_reasoning),
                     q.query_token_len, free, m, n, il, b, st, tie))

    # A2 replay (test_acceptance.py:172-208), seed 43, DEFAULT_MODEL/META, out 10
    rng = random.Random(43)
    for trial in range(1000):
        prof = random_profile(rng)
        space = map_profile(prof)
        q = QueryRecord(id=f"a2-{trial}", text="t", query_token_len=rng.randint(10, 3000))
        sizes = [whole(q, c, DEFAULT_MODEL, DEFAULT_META, 10, 64) for c in enumerate_candidates(space)]
        lo, hi = min(sizes), max(sizes)
        free = rng.choice([rng.randint(0, max(lo - 1, 0)), rng.randint(lo, hi), rng.randint(hi, 2 * hi)])
        add(0, space, prof, q, free)

    # best-fit exhaustive-oracle replay (test_scheduler.py:121-136), seed 2024, out 40
    rng = random.Random(2024)
    for trial in range(300):
        prof = random_profile(rng)
        space = map_profile(prof)
        q = QueryRecord(id=f"q{trial}", text="t", query_token_len=rng.randint(10, 3000))
        model, meta, out, tmpl, _, gran = params_kw(PARAM_SETS[1])
        sizes = [whole(q, c, model, meta, out, tmpl) for c in enumerate_candidates(space)]
        lo, hi = min(sizes), max(sizes)
        free = rng.choice([rng.randint(0, lo), rng.randint(lo, hi), rng.randint(hi, 2 * hi)])
        add(1, space, prof, q, free)

    # wide random: every parameter set, mapped / hull / full / arbitrary spaces
    rng = random.Random(20241217)
    ties = 0
    for ps_i in range(len(PARAM_SETS)):
        model, meta, out, tmpl, mc, gran = params_kw(PARAM_SETS[ps_i])
        for trial in range(600):
            prof = random_profile(rng)
            kind = trial % 4
            if kind == 0:
                space = map_profile(prof, max_chunks=mc)
            elif kind == 1:
                space = FULL_SPACE if mc >= 35 else PrunedConfigSpace(
                    frozenset(SynthesisMethod), IntRange(1, mc), IntRange(30, 200))
            else:
                space = random_arbitrary_space(rng, mc)
            q = QueryRecord(id=f"w{trial}", text="t", query_token_len=rng.randint(1, 12000))
            sizes = [whole(q, c, model, meta, out, tmpl) for c in enumerate_candidates(space, gran)]
            lo, hi = min(sizes), max(sizes)
            free = rng.choice([
                rng.randint(0, max(lo - 1, 0)), rng.randint(lo, hi), rng.randint(hi, 2 * hi),
                16 * 1024**3 - rng.randint(0, 16 * 1024**3), rng.choice(sizes), 0,
            ])
            add(ps_i, space, prof, q, free)
            ties += rows[-1][-1]

    # byte-tie hunt: keep cases whose candidate grid has equal byte counts and
    # whose free budget lands exactly on a tied size (the latest-grid rule)
    rng = random.Random(77)
    found = 0
    while found < 400:
        ps_i = rng.choice((0, 1, 2, 4))
        model, meta, out, tmpl, mc, gran = params_kw(PARAM_SETS[ps_i])
        prof = profile(1, 1, rng.randint(1, 10), *sorted((rng.randint(30, 200), rng.randint(30, 200))))
        space = map_profile(prof, max_chunks=mc) if rng.random() < 0.7 else FULL_SPACE
        q = QueryRecord(id="tie", text="t", query_token_len=rng.randint(1, 5000))
        sizes = [whole(q, c, model, meta, out, tmpl) for c in enumerate_candidates(space, gran)]
        dup = sorted({s for s in sizes if sizes.count(s) > 1})
        if not dup:
            continue
        free = rng.choice(dup) + rng.choice((0, 0, 1))
        add(ps_i, space, prof, q, free)
        found += 1

    arr = np.array(rows, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT_DIR, "select.npz"), rows=arr,
                        param_sets=np.array(PARAM_SETS, dtype=np.float64))
    print("select:", len(rows), "rows; with byte ties:", int(arr[:, -1].sum()),
          "status counts:", np.bincount(arr[:, 13], minlength=3).tolist())


# -- G3: confidence gate sequences --------------------------------------------

def gen_gate():
    seqs = []  # list of dicts of arrays
    dist = TruthDistribution()

    def run(name, profiles, threshold=0.90, default_space=DEFAULT_FALLBACK_SPACE, max_chunks=35,
            prefill=()):
        window = RecentSpaceWindow()
        for s in prefill:
            window.push(s)
        outs = []
        for p in profiles:
            class _Out:  # gate_profile only reads .profile
                pass
            o = _Out()
            o.profile = p
            d = gate_profile(o, window, threshold, default_space=default_space, max_chunks=max_chunks)
            outs.append((*enc_space(d.space), int(d.used_fallback)))
        seqs.append(dict(
            name=name,
            profiles=np.array([(int(p.complexity_high), int(p.needs_joint_reasoning), p.pieces_required,
                                p.summary_len_range.low, p.summary_len_range.high) for p in profiles],
                              dtype=np.int32),
            conf=np.array([p.confidence for p in profiles], dtype=np.float64),
            expected=np.array(outs, dtype=np.int32),
            threshold=threshold, default_space=np.array(enc_space(default_space), dtype=np.int32),
            max_chunks=max_chunks,
            prefill=np.array([enc_space(s) for s in prefill], dtype=np.int32).reshape(-1, 5),
        ))

    def mock_stream(seed, n, noise, truthdist=dist):
        rng = random.Random(seed)
        return [mock_estimate(truthdist.sample(rng), noise, seed=i).profile for i in range(n)]

    run("default_noise", mock_stream(1, 3000, NoiseParams()))
    run("a6_noise", mock_stream(2, 2000, NoiseParams(0.1, 0.0, 0.0, 0.0)))
    run("heavy_noise", mock_stream(3, 2000, NoiseParams(0.3, 0.3, 0.3, 0.3)))
    run("very_heavy_noise", mock_stream(4, 1500, NoiseParams(0.9, 0.9, 0.9, 0.9)))
    run("threshold_0.5", mock_stream(5, 1000, NoiseParams(0.3, 0.3, 0.3, 0.3)), threshold=0.5)
    run("threshold_1.0", mock_stream(6, 500, NoiseParams()), threshold=1.0)
    run("threshold_0.99", mock_stream(7, 500, NoiseParams(0.2, 0.2, 0.2, 0.2)), threshold=0.99)
    run("custom_default", mock_stream(8, 800, NoiseParams(0.5, 0.5, 0.5, 0.5)),
        default_space=PrunedConfigSpace(frozenset({SynthesisMethod.MAP_RERANK}), IntRange(2, 4)),
        max_chunks=20)
    run("prefilled_window", mock_stream(9, 800, NoiseParams(0.4, 0.4, 0.4, 0.4)),
        prefill=[map_profile(profile(1, 1, 3, 40, 90)), map_profile(profile(0, 0, 7, 30, 30)),
                 PrunedConfigSpace(frozenset({SynthesisMethod.STUFF}), IntRange(1, 2))])
    # zero-noise replay (test_profiler.py:219-234), seed 17
    rng = random.Random(17)
    zs = []
    for i in range(300):
        t = TrueProfile(needs_joint_reasoning=rng.random() < 0.5, complexity_high=rng.random() < 0.5,
                        pieces_required=rng.randint(1, 10), required_summary_len=rng.randint(30, 200))
        zs.append(mock_estimate(t, ZERO_NOISE, seed=i).profile)
    run("zero_noise_seed17", zs)
    # all rejected -> default space throughout; all accepted
    run("all_rejected", [profile(1, 1, 5, 50, 60, 0.1)] * 50)
    run("doc_level_truths", [profile_from_truth(TruthDistribution(p_joint=0.9).sample(random.Random(i)),
                                                confidence=(0.5 if i % 7 == 0 else 0.99))
                             for i in range(600)])

    out = {}
    for i, s in enumerate(seqs):
        for k, v in s.items():
            out[f"{i}_{k}"] = np.asarray(v)
    out["count"] = np.array(len(seqs))
    np.savez_compressed(os.path.join(OUT_DIR, "gate.npz"), **out)
    print("gate:", len(seqs), "sequences,", sum(len(s["conf"]) for s in seqs), "profiles")


# -- G4: latency model (sim.call_latency over reference plan_calls) ------------

def gen_latency():
    rng = random.Random(123)
    costs = [CostModel(), CostModel(1e-4, 1e-2, 0.0, 0.0), CostModel(3.3e-5, 7.1e-3, 0.037, 0.0)]
    rows, lat = [], []
    plan_rows, plan_delay = [], []
    for ci, cost in enumerate(costs):
        for trial in range(400):
            ps_i = rng.randrange(len(PARAM_SETS))
            model, meta, out, tmpl, mc, gran = params_kw(PARAM_SETS[ps_i])
            m = rng.choice((1, 2, 4))
            n = rng.randint(1, mc)
            il = rng.randint(30, 300) if m == 4 else 0
            cfg = RagConfig(FROM_BIT[m], n, il if m == 4 else None)
            q = QueryRecord(id="l", text="t", query_token_len=rng.randint(1, 12000))
            plan = plan_calls(q, cfg, meta, model, out, template_tokens=tmpl, max_chunks=mc)
            c0 = rng.randint(0, 200)
            # per-call latency exactly as sim.dispatch issues it (sim.py:226-228)
            worst = 0.0
            j = 0
            for call in plan.calls:
                conc = c0 + j if not call.depends_on else c0
                v = call_latency(call, conc, cost)
                rows.append((ci, call.prompt_tokens, call.max_output_tokens, conc))
                lat.append(v)
                if not call.depends_on:
                    worst = max(worst, v)
                    j += 1
            for call in plan.calls:
                if call.depends_on:
                    worst = worst + call_latency(call, c0, cost)
            plan_rows.append((ci, ps_i, m, n, il, q.query_token_len, c0))
            plan_delay.append(worst)
    np.savez_compressed(
        os.path.join(OUT_DIR, "latency.npz"),
        calls=np.array(rows, dtype=np.int64), latency=np.array(lat, dtype=np.float64),
        plans=np.array(plan_rows, dtype=np.int64), plan_delay=np.array(plan_delay, dtype=np.float64),
        costs=np.array([(c.prefill_secs_per_token, c.decode_secs_per_token_base,
                         c.batch_slowdown_per_seq) for c in costs], dtype=np.float64))
    print("latency:", len(rows), "calls,", len(plan_rows), "plans")


# -- G6: per-call expansion (memory.plan_calls) --------------------------------

def gen_plan_calls():
    from ragsched.memory import CallKind
    from ragsched.types import ContextOverflow, InvalidChunkCount

    kinds = {CallKind.SINGLE: 0, CallKind.MAPPER: 1, CallKind.REDUCER: 2, CallKind.RERANK: 3}
    rng = random.Random(31)
    rows, calls = [], []
    for trial in range(3000):
        ps_i = rng.randrange(len(PARAM_SETS))
        model0, meta, out, tmpl, mc, _ = params_kw(PARAM_SETS[ps_i])
        max_ctx = rng.choice([131072, 32768, 16000, 8192])
        model = ModelSpec(model0.num_layers, model0.num_kv_heads, model0.head_dim, model0.bytes_per_element,
                          max_context_tokens=max_ctx)
        m = rng.choice((1, 2, 4))
        n = rng.choice([rng.randint(1, mc), rng.randint(1, mc), rng.randint(1, mc), 0, mc + 1])
        il = rng.choice([rng.randint(1, 400), rng.randint(1, 400), 0]) if m == 4 else 0
        q = QueryRecord(id="p", text="t", query_token_len=rng.randint(1, 12000))
        cfg = RagConfig(FROM_BIT[m], n, il if m == 4 else None)
        status, total = 0, 0
        try:
            plan = plan_calls(q, cfg, meta, model, out, template_tokens=tmpl, max_chunks=mc)
            first = len(calls)
            for c in plan.calls:
                assert (not c.depends_on) or c.depends_on == frozenset(range(n))
                calls.append((trial, kinds[c.kind], c.prompt_tokens, c.max_output_tokens, c.kv_bytes, c.index))
            total = plan.total_bytes
            assert len(calls) - first == len(plan.calls)
        except InvalidChunkCount:
            status = 2
        except ContextOverflow:
            status = 3
        except ValueError:
            status = 4
        rows.append((trial, ps_i, max_ctx, m, n, il, q.query_token_len, status, total))
    np.savez_compressed(os.path.join(OUT_DIR, "plan_calls.npz"), rows=np.array(rows, dtype=np.int64),
                        calls=np.array(calls, dtype=np.int64))
    print("plan_calls:", len(rows), "plans,", len(calls), "calls, statuses",
          np.bincount(np.array(rows)[:, 7], minlength=5).tolist())


# -- G5: known answers from the reference's own tests --------------------------

def gen_known():
    per_tok = bytes_per_kv_token(DEFAULT_MODEL)
    q = QueryRecord(id="k", text="t", query_token_len=100)
    known = {
        "bytes_per_kv_token_default": per_tok,                                      # test_memory.py:33-34
        "bytes_per_kv_token_unit": bytes_per_kv_token(ModelSpec(1, 1, 1, 1, 100)),  # :37-38
        "bytes_per_kv_token_4bit": bytes_per_kv_token(ModelSpec(3, 5, 7, 0.5, 100)),  # :47-48
        "buffered_100_131072": buffered_bytes(100, 131072),                         # :104-106
        "buffered_7_3": buffered_bytes(7, 3),                                       # :107-108
        "stuff3_prompt": plan_calls(q, RagConfig(SynthesisMethod.STUFF, 3),
                                    DatasetMeta("corpus", 1000), DEFAULT_MODEL, 40).calls[0].prompt_tokens,
        "max_whole_plan_cfg4": max(
            plan_bytes(12000, c, 1024, per_tok, 60, 64)
            for c in enumerate_candidates(FULL_SPACE)),
        "single_hop_out_budget": DATASET_PROFILES["single_hop_qa"].out_budget,
    }
    np.savez(os.path.join(OUT_DIR, "known.npz"), **{k: np.array(v) for k, v in known.items()})
    print("known:", known)


# -- G7: estimator answer parsing (profiler.parse_profile_text) -----------------

def gen_parse():
    """Random answers around the four-line grammar (profiler.py:191-200):
    case, spacing (incl. Unicode spaces), line separators, out-of-domain and
    huge numbers, reversed ranges, duplicate / missing / garbled fields,
    word-boundary and folding edge cases.  ASCII digits only."""
    import gzip
    import json

    from ragsched.profiler import UnparseableAnswer, parse_profile_text

    rng = random.Random(7)
    spaces = [" ", "  ", "\t", "", "\u00a0", "\u3000", " \t ", "\x1f"]
    seps = ["\n", "\r\n", "\r", "\n\n", "\x0b", "\x0c", "\u2028", "\x1c", "\x85"]

    def case(w):
        r = rng.random()
        if r < 0.5:
            return w
        if r < 0.7:
            return w.upper()
        if r < 0.85:
            return w.lower()
        return "".join(c.upper() if rng.random() < 0.5 else c.lower() for c in w)

    def sp():
        return rng.choice(spaces) if rng.random() < 0.4 else rng.choice([" ", ""])

    def num():
        r = rng.random()
        if r < 0.6:
            return str(rng.randint(-5, 260))
        if r < 0.7:
            return "0" + str(rng.randint(0, 99))
        if r < 0.8:
            return str(rng.randint(10 ** 18, 10 ** 30)) * rng.choice([1, 2])
        if r < 0.9:
            return "-" + str(rng.randint(10 ** 18, 10 ** 25))
        return str(rng.randint(1, 12))

    def tail():
        if rng.random() < 0.8:
            return ""
        return rng.choice([".", " ", "x", "_", "1", "é", "—", "!", " extra", "\u00a0"])

    def field(kind):
        if kind == 0:
            word = rng.choice(["High", "Low"]) if rng.random() < 0.9 else rng.choice(["Hıgh", "Medium", "Lo"])
            return f"{sp()}{case('Complexity')}{sp()}:{sp()}{case(word) if word.isascii() else word}{tail()}"
        if kind == 1:
            word = rng.choice(["Yes", "No"]) if rng.random() < 0.9 else rng.choice(["Maybe", "Yeſ", "Ye"])
            key = "Joint Reasoning needed" if rng.random() < 0.9 else rng.choice(
                ["Joint  Reasoning needed", "Joint reaſoning needed", "Joint Reasoning"])
            return f"{sp()}{case(key) if key.isascii() else key}{sp()}:{sp()}{word}{tail()}"
        if kind == 2:
            key = "Pieces" if rng.random() < 0.93 else rng.choice(["Piece", "Pİeces"])
            return f"{sp()}{case(key) if key.isascii() else key}{sp()}:{sp()}{num()}{tail()}"
        a, b = num(), num()
        dash = rng.choice(["-", " - ", "--"]) if rng.random() < 0.93 else rng.choice(["–", "to"])
        key = "Summary range" if rng.random() < 0.93 else rng.choice(["summary  range", "Summary"])
        return f"{sp()}{case(key)}{sp()}:{sp()}{a}{sp()}{dash}{sp()}{b}{tail()}"

    rows = []
    for i in range(4000):
        kinds = [0, 1, 2, 3]
        rng.shuffle(kinds) if rng.random() < 0.3 else None
        lines = []
        for k in kinds:
            if rng.random() < 0.03:
                continue  # missing field
            lines.append(field(k))
            if rng.random() < 0.15:
                lines.append(field(k))  # duplicate: the first match wins
            if rng.random() < 0.1:
                lines.append(rng.choice(["", "Note: none", "Answer:", "   ", "Complexity", "Pieces:"]))
        if rng.random() < 0.2:
            lines.insert(0, rng.choice(["Here is the profile:", "", "Profile"]))
        text = ""
        for j, ln in enumerate(lines):
            text += ln + (rng.choice(seps) if j + 1 < len(lines) or rng.random() < 0.3 else "")
        conf = rng.random()
        try:
            prof, clamped, lnums = parse_profile_text(text, confidence=conf)
            res = [int(prof.complexity_high), int(prof.needs_joint_reasoning), prof.pieces_required,
                   prof.summary_len_range.low, prof.summary_len_range.high, sorted(clamped),
                   [lnums.get(f, -1) for f in ("complexity", "joint_reasoning", "pieces", "summary_range")]]
        except UnparseableAnswer:
            res = None
        rows.append([text, conf, res])
    with gzip.open(os.path.join(OUT_DIR, "parse.json.gz"), "wt", encoding="utf-8") as f:
        json.dump(rows, f, ensure_ascii=False)
    print("parse:", len(rows), "answers,", sum(r[2] is None for r in rows), "unparseable,",
          sum(bool(r[2] and r[2][5]) for r in rows), "clamped")


# -- G8: cost table of every pruned candidate ----------------------------------

def gen_costs():
    """Per candidate of random spaces: plan_bytes and the plan's critical-path
    delay (the definition of gen_latency: independent calls dispatched with
    concurrency c0 + j, the reducer after its mappers, sim.py:223-229)."""
    rng = random.Random(77)
    costs = [CostModel(), CostModel(1e-4, 1e-2, 0.0, 0.0), CostModel(3.3e-5, 7.1e-3, 0.037, 0.0)]
    queries, cands = [], []
    for trial in range(600):
        ps_i = rng.randrange(len(PARAM_SETS))
        model0, meta, out, tmpl, mc, gran = params_kw(PARAM_SETS[ps_i])
        model = ModelSpec(model0.num_layers, model0.num_kv_heads, model0.head_dim, model0.bytes_per_element,
                          max_context_tokens=10 ** 9)  # delays need no context check
        space = FULL_SPACE if rng.random() < 0.05 else random_arbitrary_space(rng, mc)
        qlen = rng.randint(1, 12000)
        c0 = rng.randint(0, 200)
        ci = rng.randrange(len(costs))
        q = QueryRecord(id="c", text="t", query_token_len=qlen)
        queries.append((trial, ps_i, *enc_space(space), qlen, c0, ci))
        for cfg in enumerate_candidates(space, gran):
            b = plan_bytes(qlen, cfg, meta.chunk_size, bytes_per_kv_token(model), out, tmpl)
            plan = plan_calls(q, cfg, meta, model, out, template_tokens=tmpl, max_chunks=max(mc, cfg.num_chunks))
            worst, j = 0.0, 0
            for call in plan.calls:
                if not call.depends_on:
                    worst = max(worst, call_latency(call, c0 + j, costs[ci]))
                    j += 1
            for call in plan.calls:
                if call.depends_on:
                    worst = worst + call_latency(call, c0, costs[ci])
            m, n, il = enc_cfg(cfg)
            cands.append((trial, m, n, il, b, worst))
    np.savez_compressed(os.path.join(OUT_DIR, "costs.npz"), queries=np.array(queries, dtype=np.int64),
                        cand=np.array([c[:5] for c in cands], dtype=np.int64),
                        delay=np.array([c[5] for c in cands], dtype=np.float64),
                        costs=np.array([(c.prefill_secs_per_token, c.decode_secs_per_token_base,
                                         c.batch_slowdown_per_seq) for c in costs], dtype=np.float64))
    print("costs:", len(queries), "queries,", len(cands), "candidates")


if __name__ == "__main__":
    gen_mapping()
    gen_select()
    gen_gate()
    gen_latency()
    gen_plan_calls()
    gen_known()
    gen_parse()
    gen_costs()
