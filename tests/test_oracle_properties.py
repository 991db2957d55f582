"""The reference's own property tests restated against the oracle (CPU):
buffered_bytes is the exact ceiling of the 2% buffer (test_memory.py:111-116)
and the admission rules' invariants hold for any parameters
(test_scheduler.py:99-136)."""

from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import config_oracle as co


@settings(max_examples=300, deadline=None)
@given(tokens=st.integers(0, 10**7), per_tok=st.integers(1, 10**7))
def test_buffered_bytes_is_the_exact_ceiling(tokens, per_tok):
    raw = tokens * per_tok
    kv = co.buffered_bytes(tokens, per_tok)
    assert 0 <= kv * 100 - 102 * raw < 100


@settings(max_examples=200, deadline=None)
@given(m=st.integers(1, 7), lo=st.integers(1, 35), span=st.integers(0, 34), a=st.integers(30, 200),
       span_il=st.integers(0, 170), qlen=st.integers(1, 20000), free=st.integers(0, 2**40), joint=st.booleans(),
       chunk=st.integers(1, 4096), step=st.integers(1, 5), istep=st.integers(1, 20))
def test_best_fit_is_the_largest_fitting_candidate(m, lo, span, a, span_il, qlen, free, joint, chunk, step, istep):
    p = co.SelectParams(chunk_size=chunk, chunk_step=step, interlen_step=istep)
    hi = min(lo + span, 35)
    space = (m, lo, hi, a if m & 4 else 0, min(a + span_il, 200) if m & 4 else 0)
    grid = co.enumerate_grid(space, p.chunk_step, p.interlen_step)
    fits = [(co.plan_bytes(qlen, c, p), i) for i, c in enumerate(grid) if co.plan_bytes(qlen, c, p) <= free]
    got = co.best_fit_select(space, qlen, free, p)
    if not fits:
        assert got is None
    else:
        b, i = max(fits)  # (bytes, grid position): byte ties go to the latest slot
        assert got == (grid[i], b)
    m_, n_, il_, b_, status = co.select(space, joint, qlen, free, p)
    if status != co.ST_MUST_QUEUE:
        assert b_ <= free
    if status == co.ST_FALLBACK:  # never map_reduce; rerank exactly when the profile is not joint
        assert m_ == (co.STUFF if joint else co.RERANK)
