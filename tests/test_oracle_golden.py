"""Pin the CPU oracle to the reference: every golden vector (produced by
running ``ragsched`` itself) must be reproduced exactly by the restatement in
``oracle/config_oracle.py``.  CPU only."""

import numpy as np
import pytest

from oracle import config_oracle as co
from tests import golden_data as gd


def test_known_answers():
    k = gd.known()
    assert co.bytes_per_kv_token(32, 8, 128, 2) == k["bytes_per_kv_token_default"] == 131072
    assert co.bytes_per_kv_token(1, 1, 1, 1) == k["bytes_per_kv_token_unit"] == 2
    assert co.bytes_per_kv_token(3, 5, 7, 0.5) == k["bytes_per_kv_token_4bit"] == 105
    assert co.buffered_bytes(100, 131072) == k["buffered_100_131072"] == 13369344
    assert co.buffered_bytes(7, 3) == k["buffered_7_3"] == 22
    p = co.SelectParams(chunk_size=1000, out_budget=40)
    assert co.plan_call_shapes(100, (co.STUFF, 3, 0), p)[0][0] == k["stuff3_prompt"] == 3164
    p4 = co.SelectParams(chunk_size=1024, out_budget=60)
    full = (7, 1, 35, 30, 200)
    assert max(co.plan_bytes(12000, c, p4) for c in co.enumerate_grid(full)) == k["max_whole_plan_cfg4"]


def test_buffer_exactness_property():
    rng = np.random.default_rng(0)
    for raw_tokens, per_tok in rng.integers(1, 10**6, size=(2000, 2)):
        kv = co.buffered_bytes(int(raw_tokens), int(per_tok))
        raw = int(raw_tokens) * int(per_tok)
        assert 0 <= kv * 100 - 102 * raw < 100


def test_mapping_matches_reference():
    profiles, spaces = gd.mapping()
    for (cx, joint, pieces, lo, hi, mc), want in zip(profiles, spaces):
        got = co.map_profile(bool(cx), bool(joint), int(pieces), int(lo), int(hi), int(mc))
        assert got == tuple(int(x) for x in want)


def test_full_space_grid_size():
    assert len(co.enumerate_grid((7, 1, 35, 30, 200))) == 700
    # test_mapping.py:163-171 counts 9 + 72 = 81 for stuff+reduce [3,11] il [40,110]
    assert len(co.enumerate_grid((6, 3, 11, 40, 110))) == 9 + 72


def test_select_matches_reference():
    psets = [co.SelectParams(**p) for p in gd.param_sets()]
    rows = gd.select_rows()
    for r in rows:
        ps, m, lo, hi, a, b, joint, qlen, free, em, en, eil, eb, est, _ = (int(x) for x in r)
        got = co.select((m, lo, hi, a, b), bool(joint), qlen, free, psets[ps])
        assert got == (em, en, eil, eb, est), r


def test_select_covers_ties_and_all_statuses():
    rows = gd.select_rows()
    assert rows[:, 14].sum() > 100
    assert set(np.unique(rows[:, 13]).tolist()) == {0, 1, 2}


@pytest.mark.parametrize("seq", gd.gate_sequences(), ids=lambda s: s["name"])
def test_gate_matches_reference(seq):
    profs = [(bool(p[0]), bool(p[1]), int(p[2]), int(p[3]), int(p[4]), float(c))
             for p, c in zip(seq["profiles"], seq["conf"])]
    out, _ = co.gate_sequence(profs, seq["threshold"], seq["default_space"], seq["max_chunks"],
                              window=seq["prefill"])
    got = np.array([(*s, int(fb)) for s, fb in out], dtype=np.int32)
    np.testing.assert_array_equal(got, seq["expected"])


def test_latency_bit_exact():
    z = gd.latency()
    costs = [co.CostModel(*c) for c in z["costs"]]
    for (ci, pr, out, conc), want in zip(z["calls"], z["latency"]):
        got = co.call_latency(int(pr), int(out), int(conc), costs[int(ci)])
        assert got == float(want)  # bit-exact, not approx


def test_plan_delay_bit_exact():
    z = gd.latency()
    costs = [co.CostModel(*c) for c in z["costs"]]
    psets = [co.SelectParams(**p) for p in gd.param_sets()]
    for (ci, ps, m, n, il, qlen, c0), want in zip(z["plans"], z["plan_delay"]):
        got = co.plan_delay(int(qlen), (int(m), int(n), int(il)), psets[int(ps)],
                            costs[int(ci)], int(c0))
        assert got == float(want)


# -- the C restatement (CPU baseline / large-size checker) ----------------------

def test_c_oracle_select_matches_reference():
    from oracle import c_oracle

    psets = [co.SelectParams(**p) for p in gd.param_sets()]
    rows = gd.select_rows()
    for ps in range(len(psets)):
        sub = rows[rows[:, 0] == ps]
        cfg, b, st = c_oracle.select_batch(sub[:, 1:6], sub[:, 6], sub[:, 7], sub[:, 8], psets[ps])
        np.testing.assert_array_equal(cfg, sub[:, 9:12])
        np.testing.assert_array_equal(b, sub[:, 12])
        np.testing.assert_array_equal(st, sub[:, 13])


@pytest.mark.parametrize("seq", gd.gate_sequences(), ids=lambda s: s["name"])
def test_c_oracle_gate_matches_reference(seq):
    from oracle import c_oracle

    out, fb, _ = c_oracle.gate_batch(seq["profiles"], seq["conf"], seq["threshold"],
                                     seq["default_space"], seq["max_chunks"], seq["prefill"])
    np.testing.assert_array_equal(np.concatenate([out, fb[:, None]], axis=1), seq["expected"])


def test_plan_calls_matches_reference():
    psets = [co.SelectParams(**p) for p in gd.param_sets()]
    rows, calls = gd.plan_calls()
    by_trial = {}
    for c in calls:
        by_trial.setdefault(int(c[0]), []).append(tuple(int(x) for x in c[1:]))
    for trial, ps, max_ctx, m, n, il, qlen, status, total in (tuple(int(x) for x in r) for r in rows):
        st, got, tot = co.plan_calls(qlen, (m, n, il), psets[ps], max_ctx)
        assert st == status, (trial, st, status)
        assert got == by_trial.get(trial, [])
        assert tot == total
