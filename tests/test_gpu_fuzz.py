"""A fixed-seed slice of tools/fuzz_retrieval.py: 40 random retrieval cases
(dtypes, shapes, k, duplicate / zero / non-normalised rows, id bases, ragged
adds, wrap-around walks, every algorithm) against the float64 oracle.  The
round's long run (2,142 cases, 420 s) is recorded in DESIGN.md."""

import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(900)
def test_fuzz_fixed_seed():
    import fuzz_retrieval

    assert fuzz_retrieval.main(seconds=600, seed=7, max_cases=40) == 0
