"""§8(f3): estimator answer ingestion (profiler.py:191-254, :427-464) — the
native batch parser ``rs_parse_profiles`` and the per-field confidences
``rs_field_confidences`` (host code in libragsched_b200.so, no GPU needed)
against 4,000 answers run through the reference's own parse_profile_text
(tests/golden/make_golden.py gen_parse) and _per_field_confidences
(tests/golden/make_field_conf.py), plus the reference tests' known answers
(test_profiler.py:95-123, test_remote_profiler.py:74-100)."""

import os

import numpy as np
import pytest

from paper_2412_10543_b200 import _lib, batch
from paper_2412_10543_b200 import profiler as P
from paper_2412_10543_b200.types import IntRange
from tests.golden_data import field_conf_rows, parse_answers

pytestmark = pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="library not built")


def test_batch_parser_matches_reference_answers():
    rows = parse_answers()
    texts = [r[0] for r in rows]
    recs, clamped, status, lines = batch.parse_profiles(texts, [r[1] for r in rows], nthreads=4)
    bad = []
    for i, (text, conf, want) in enumerate(rows):
        if want is None:
            if status[i] != batch.RS_PARSE_UNPARSEABLE:
                bad.append((i, "should be unparseable"))
            continue
        r = recs[i]
        got = [int(r["complexity_high"]), int(r["needs_joint_reasoning"]), int(r["pieces_required"]),
               int(r["summary_lo"]), int(r["summary_hi"]), sorted(batch.clamped_names(clamped[i])),
               [int(x) for x in lines[i]]]
        if status[i] != batch.RS_PARSE_OK or got != want or r["confidence"] != conf:
            bad.append((i, text, got, want))
    assert not bad, bad[:5]
    assert (status == batch.RS_PARSE_OK).sum() > 1000 and (status != batch.RS_PARSE_OK).sum() > 1000


def test_thread_count_does_not_change_results():
    texts = [r[0] for r in parse_answers()[:1500]]
    a = batch.parse_profiles(texts, nthreads=1)
    b = batch.parse_profiles(texts, nthreads=7)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_reference_known_answers():
    # test_profiler.py:95-103
    prof, clamped, lines = P.parse_profile_text(
        "Complexity: High\nJoint Reasoning needed: Yes\nPieces: 4\nSummary range: 50-120", confidence=0.97)
    assert prof.complexity_high and prof.needs_joint_reasoning and prof.pieces_required == 4
    assert prof.summary_len_range == IntRange(50, 120) and prof.confidence == 0.97 and not clamped
    assert lines == {"complexity": 0, "joint_reasoning": 1, "pieces": 2, "summary_range": 3}
    # :106-110
    prof, clamped, _ = P.parse_profile_text("Complexity: Low\nJoint Reasoning needed: No\nPieces: 15\nSummary range: 50-120")
    assert prof.pieces_required == 10 and "pieces" in clamped
    # :113-117
    prof, clamped, _ = P.parse_profile_text("Complexity: Low\nJoint Reasoning needed: No\nPieces: 2\nSummary range: 250-10")
    assert prof.summary_len_range == IntRange(30, 200) and "summary_range" in clamped
    # :120-123
    with pytest.raises(P.UnparseableAnswer):
        P.parse_profile_text("Complexity: High\nPieces: 3")


def test_empty_batch_and_empty_text():
    recs, clamped, status, lines = batch.parse_profiles([])
    assert len(recs) == 0
    recs, clamped, status, lines = batch.parse_profiles(["", "\n\n"])
    assert list(status) == [batch.RS_PARSE_UNPARSEABLE] * 2 and (lines == -1).all()



def test_field_confidences_match_reference_bit_exact():
    """Every answer's four confidences equal the reference's bit for bit
    (float.hex): the token -> line mapping over Unicode line breaks, the
    CPython 3.12 compensated sum, the mean and exp."""
    rows = field_conf_rows()
    got = batch.field_confidences([r[0] for r in rows], [r[1] for r in rows], nthreads=4)
    bad = [(i, [float(x).hex() for x in got[i]], r[2]) for i, r in enumerate(rows)
           if [float(x).hex() for x in got[i]] != r[2]]
    assert not bad, bad[:5]
    assert sum(any(h != (1.0).hex() for h in r[2]) for r in rows) > 1000


def test_field_confidences_thread_count_invariant():
    rows = field_conf_rows()[:1500]
    a = batch.field_confidences([r[0] for r in rows], [r[1] for r in rows], nthreads=1)
    b = batch.field_confidences([r[0] for r in rows], [r[1] for r in rows], nthreads=0)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_per_field_confidences_known_answers():
    """test_remote_profiler.py:74-100: per-line log-probs -> exp(mean) per
    field; no tokens -> pass-through 1.0."""
    import math

    answer = "Complexity: High\nJoint Reasoning needed: Yes\nPieces: 4\nSummary range: 50-120"
    toks = ([{"token": "Complexity: High\n", "logprob": -0.05}]
            + [{"token": "Joint Reasoning needed: Yes\n", "logprob": -0.2}]
            + [{"token": "Pieces:", "logprob": -0.4}, {"token": " 4\n", "logprob": -0.6}]
            + [{"token": "Summary range: 50-120", "logprob": -0.01}])
    c = P.per_field_confidences(answer, toks)
    assert c["complexity"] == pytest.approx(math.exp(-0.05))
    assert c["joint_reasoning"] == pytest.approx(math.exp(-0.2))
    assert c["pieces"] == pytest.approx(math.exp(-0.5))
    assert c["summary_range"] == pytest.approx(math.exp(-0.01))
    assert min(c.values()) == pytest.approx(math.exp(-0.5))  # the remote estimator's gate confidence
    for none in (None, []):
        assert all(v == 1.0 for v in P.per_field_confidences(answer, none).values())
    assert all(v == 1.0 for v in P.per_field_confidences("no fields here", toks).values())  # unparseable
    with pytest.raises(TypeError):
        P.per_field_confidences(answer, [{"token": None, "logprob": -1.0}])
