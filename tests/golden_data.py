"""Loaders for the committed golden fixtures (generated from the reference by
``tests/golden/make_golden.py``)."""

from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLDEN, name))


def param_sets():
    """List of dicts: model-derived per_token_bytes + selection scalars."""
    z = _load("select.npz")
    out = []
    for L, H, D, w, cs, ob, tmpl, mc, cstep, istep in z["param_sets"]:
        out.append(dict(per_token_bytes=int(2 * int(L) * int(H) * int(D) * float(w)),
                        chunk_size=int(cs), out_budget=int(ob), template_tokens=int(tmpl),
                        max_chunks=int(mc), chunk_step=int(cstep), interlen_step=int(istep)))
    return out


def select_rows():
    """int64 [n, 16]: ps, methods, n_lo, n_hi, il_lo, il_hi, joint, qlen, free,
    m, n, il, bytes, status, tie."""
    return _load("select.npz")["rows"]


def mapping():
    z = _load("mapping.npz")
    return z["profiles"], z["spaces"]


def gate_sequences():
    z = _load("gate.npz")
    seqs = []
    for i in range(int(z["count"])):
        g = lambda k: z[f"{i}_{k}"]  # noqa: E731
        seqs.append(dict(name=str(g("name")), profiles=g("profiles"), conf=g("conf"),
                         expected=g("expected"), threshold=float(g("threshold")),
                         default_space=tuple(int(x) for x in g("default_space")),
                         max_chunks=int(g("max_chunks")),
                         prefill=[tuple(int(x) for x in r) for r in g("prefill")]))
    return seqs


def latency():
    z = _load("latency.npz")
    return {k: z[k] for k in z.files}


def known():
    z = _load("known.npz")
    return {k: z[k].item() for k in z.files}


def plan_calls():
    """rows int64 [n, 9]: trial, ps, max_ctx, m, n, il, qlen, status, total;
    calls int64 [c, 6]: trial, kind, prompt, out, kv_bytes, index."""
    z = _load("plan_calls.npz")
    return z["rows"], z["calls"]


# PARAM_SETS of make_golden.py (layers, heads, head_dim, width, chunk, out, template, max_chunks, cstep, istep)
PARAM_SETS = [
    (32, 8, 128, 2, 1000, 10, 64, 35, 1, 10),
    (32, 8, 128, 2, 1000, 40, 64, 35, 1, 10),
    (32, 8, 128, 2, 1024, 40, 64, 35, 1, 10),
    (32, 8, 128, 2, 1024, 60, 64, 35, 1, 10),
    (32, 8, 128, 2, 1000, 20, 64, 35, 1, 10),
    (80, 8, 128, 1, 512, 10, 0, 20, 2, 5),
    (28, 4, 128, 0.5, 1000, 60, 100, 50, 1, 1),
    (16, 16, 64, 4, 700, 7, 33, 35, 3, 7),
]


def scheduler_traces():
    """Reference Scheduler runs (tests/golden/make_sched_golden.py)."""
    import gzip
    import json

    with gzip.open(os.path.join(GOLDEN, "scheduler_traces.json.gz"), "rt") as f:
        return json.load(f)


def parse_answers():
    """[text, confidence, result | None] from the reference's parse_profile_text
    (tests/golden/make_golden.py gen_parse)."""
    import gzip
    import json

    with gzip.open(os.path.join(GOLDEN, "parse.json.gz"), "rt", encoding="utf-8") as f:
        return json.load(f)


def candidate_costs():
    """Per-candidate plan bytes and plan delays from the reference
    (tests/golden/make_golden.py gen_costs)."""
    return _load("costs.npz")


def field_conf_rows():
    """[text, tokens, [float.hex x 4]] from the reference's _per_field_confidences
    (tests/golden/make_field_conf.py)."""
    import gzip
    import json

    with gzip.open(os.path.join(GOLDEN, "field_conf.json.gz"), "rt", encoding="utf-8") as f:
        return json.load(f)
