"""Golden vectors for the per-field answer confidences (§8 f3), made by RUNNING
THE REFERENCE: ``ragsched.profiler._per_field_confidences`` (profiler.py:427-464)
on estimator answers with token streams.

Run in the dev container only (``/root/reference`` is not on the GPU box):
``python tests/golden/make_field_conf.py`` -> ``tests/golden/field_conf.json.gz``.

The answers are the 4,000 texts of ``parse.json.gz`` (the parser fixtures:
every line separator, Unicode spaces, missing / duplicate fields, about half
of them unparseable).  Each gets a token stream drawn from one of these
families:
* a faithful tokenization (the text cut into 1-8 character pieces), which is
  what an endpoint returns;
* whole lines (``tests/test_remote_profiler.py:21-22``);
* unrelated tokens whose lengths run short of or past the text, including
  multi-byte characters;
* empty or None streams.
Log-probs are mostly in [-4, 0], with exact 0.0 / -0.0, None entries, huge and
tiny magnitudes and long same-line runs, which exercise CPython 3.12's
compensated ``sum``.  Expected values are stored as ``float.hex`` strings, so
the comparison is bit-exact.
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from ragsched.profiler import PROFILE_FIELDS, _per_field_confidences  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def logprob(rng: random.Random):
    r = rng.random()
    if r < 0.08:
        return None
    if r < 0.12:
        return rng.choice([0.0, -0.0])
    if r < 0.16:
        return -rng.choice([1e-300, 1e-17, 3e-9, 1e10, 1e16, 7.5e300])
    if r < 0.2:
        return -rng.randint(0, 5)  # ints pass through float()
    return -rng.random() * 4.0


def tokens_for(text: str, rng: random.Random):
    r = rng.random()
    if r < 0.05:
        return None
    if r < 0.1:
        return []
    toks = []
    if r < 0.6:  # faithful tokenization
        i = 0
        while i < len(text):
            n = rng.randint(1, 8)
            toks.append({"token": text[i:i + n], "logprob": logprob(rng)})
            i += n
    elif r < 0.75:  # whole lines (the reference test's tokenizer)
        lp = logprob(rng)
        toks = [{"token": piece, "logprob": lp if rng.random() < 0.5 else logprob(rng)}
                for piece in text.splitlines(keepends=True)]
    elif r < 0.9:  # unrelated pieces, total length short of or past the text
        alphabet = "abc \né 中\U0001f600:-0123"
        for _ in range(rng.randint(1, 60)):
            tok = {"token": "".join(rng.choice(alphabet) for _ in range(rng.randint(0, 6)))}
            if rng.random() < 0.9:
                tok["logprob"] = logprob(rng)
            if rng.random() < 0.03:
                del tok["token"]  # tok.get("token", "")
            toks.append(tok)
    else:  # long runs on the field lines: many terms per sum
        i = 0
        while i < len(text):
            toks.append({"token": text[i:i + 1], "logprob": -rng.random() * rng.choice([1e-3, 1.0, 1e3])})
            i += 1
    return toks


def main():
    with gzip.open(os.path.join(HERE, "parse.json.gz"), "rt") as f:
        answers = [row[0] for row in json.load(f)]
    rng = random.Random(11)
    rows = []
    for text in answers:
        toks = tokens_for(text, rng)
        got = _per_field_confidences(text, toks)
        rows.append([text, toks, [float(got[name]).hex() for name in PROFILE_FIELDS]])
    # the reference test's own case (test_remote_profiler.py:74-93)
    answer = "Complexity: High\nJoint Reasoning needed: Yes\nPieces: 4\nSummary range: 50-120"
    toks = ([{"token": "Complexity: High\n", "logprob": -0.05}]
            + [{"token": "Joint Reasoning needed: Yes\n", "logprob": -0.2}]
            + [{"token": "Pieces:", "logprob": -0.4}, {"token": " 4\n", "logprob": -0.6}]
            + [{"token": "Summary range: 50-120", "logprob": -0.01}])
    got = _per_field_confidences(answer, toks)
    rows.append([answer, toks, [float(got[name]).hex() for name in PROFILE_FIELDS]])
    out = os.path.join(HERE, "field_conf.json.gz")
    with gzip.open(out, "wt") as f:
        json.dump(rows, f)
    nontrivial = sum(any(h != (1.0).hex() for h in r[2]) for r in rows)
    print(f"wrote {len(rows)} cases ({nontrivial} with a confidence != 1.0) to {out}")


if __name__ == "__main__":
    main()
