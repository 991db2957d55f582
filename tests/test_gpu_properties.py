"""Property-based checks in the style of the reference's own hypothesis tests
(test_memory.py:111-116, :150-180; test_scheduler.py:99-136): hypothesis
draws whole parameter sets and query batches, the GPU kernels run them, and
the results must equal the pure-Python restatement of the reference rules
(oracle/config_oracle.py) and satisfy the reference's invariants:

* select: best fit is the arg-max of (bytes, grid position) over the
  candidates that fit; else the fallback; else MustQueue;
* plan_bytes == the sum of the admitted calls' kv bytes (memory.py:169-180);
* plan_bytes is monotone in num_chunks and intermediate_length.
"""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import config_oracle as co
from paper_2412_10543_b200 import _lib, batch
from tests.test_gpu_config import select_dev

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow])

KV_WIDTHS = (0.5, 1, 2, 4)


@st.composite
def select_params(draw):
    layers, heads, dim = draw(st.integers(1, 80)), draw(st.integers(1, 16)), draw(st.sampled_from([64, 96, 128]))
    width = draw(st.sampled_from(KV_WIDTHS))
    return co.SelectParams(per_token_bytes=int(2 * layers * heads * dim * width),
                           chunk_size=draw(st.integers(1, 4096)), out_budget=draw(st.integers(1, 200)),
                           template_tokens=draw(st.integers(0, 256)), max_chunks=draw(st.integers(1, 35)),
                           chunk_step=draw(st.integers(1, 5)), interlen_step=draw(st.integers(1, 20)))


@st.composite
def select_batch(draw, p):
    n = draw(st.integers(1, 48))
    rows = []
    for _ in range(n):
        m = draw(st.integers(1, 7))
        lo = draw(st.integers(1, p.max_chunks))
        hi = draw(st.integers(lo, p.max_chunks))
        a = draw(st.integers(30, 200)) if m & 4 else 0
        b = draw(st.integers(a, 200)) if m & 4 else 0
        joint = draw(st.integers(0, 1))
        qlen = draw(st.integers(1, 20000))
        free = draw(st.one_of(st.integers(0, 2**34), st.integers(0, 2**44)))
        rows.append((m, lo, hi, a, b, joint, qlen, free))
    return np.array(rows, dtype=np.int64)


@SETTINGS
@given(data=st.data())
def test_select_equals_reference_rules(data):
    p = data.draw(select_params())
    rows = data.draw(select_batch(p))
    spaces, joint, qlen, free = rows[:, :5].astype(np.int32), rows[:, 5], rows[:, 6], rows[:, 7]
    cfg, _ = select_dev(spaces, joint, qlen, free, p)
    for i in range(len(rows)):
        m, n_, il, b, status = co.select(tuple(int(x) for x in spaces[i]), bool(joint[i]), int(qlen[i]),
                                         int(free[i]), p)
        got = (int(cfg["method"][i]), int(cfg["num_chunks"][i]), int(cfg["interlen"][i]),
               int(cfg["kv_bytes"][i]), int(cfg["status"][i]))
        assert got == (m, n_, il, b, status), (i, rows[i].tolist())
        if status != co.ST_MUST_QUEUE:
            assert b <= free[i]  # never over-admits (MemorySafetyViolation can't follow)


@SETTINGS
@given(data=st.data())
def test_plan_bytes_is_the_sum_of_the_calls_and_monotone(data):
    p = data.draw(select_params())
    p = co.SelectParams(**{**p.__dict__, "max_chunks": 35})  # room for the +1 chunk below
    n = data.draw(st.integers(1, 32))
    ints = lambda lo, hi: np.array(data.draw(st.lists(st.integers(lo, hi), min_size=n, max_size=n)))  # noqa: E731
    method = np.array(data.draw(st.lists(st.sampled_from([1, 2, 4]), min_size=n, max_size=n)), dtype=np.uint8)
    chunks = ints(1, 34).astype(np.int32)
    il = np.where(method == 4, ints(1, 400), 0).astype(np.int32)
    qlen = ints(1, 20000).astype(np.int32)
    dev = torch.device("cuda", 0)
    params = batch.SelectParams(p.per_token_bytes, p.chunk_size, p.out_budget, p.template_tokens, p.max_chunks,
                                p.chunk_step, p.interlen_step)

    def plan_bytes(ch, ilv):
        t = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
        return batch.plan_bytes_batch(t(method), t(ch), t(ilv), t(qlen), params).cpu().numpy()

    got = plan_bytes(chunks, il)
    want = [co.plan_bytes(int(qlen[i]), (int(method[i]), int(chunks[i]), int(il[i])), p) for i in range(n)]
    np.testing.assert_array_equal(got, want)
    # plan_bytes == the whole plan's kv bytes (rs_plan_calls totals; memory.py:169-180)
    cfg = np.zeros(n, dtype=_lib.CONFIG_DTYPE)
    cfg["method"], cfg["num_chunks"], cfg["interlen"] = method, chunks, il
    cfg["status"], cfg["kv_bytes"] = _lib.RS_SELECT_BEST_FIT, got
    _, _, totals, status = batch.plan_calls(batch.to_device(cfg, dev), torch.as_tensor(qlen, device=dev), params,
                                            max_context_tokens=10**9)
    assert (status.cpu().numpy() == _lib.RS_PLAN_OK).all()
    np.testing.assert_array_equal(totals.cpu().numpy(), got)
    # monotone in num_chunks and (map_reduce) intermediate length (memory.py:150-164)
    assert (plan_bytes(chunks + 1, il) > got).all()
    longer = plan_bytes(chunks, np.where(method == 4, il + 1, 0).astype(np.int32))
    assert (longer[method == 4] > got[method == 4]).all() and (longer[method != 4] == got[method != 4]).all()
