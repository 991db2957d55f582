"""The float64 retrieval oracle pinned against INDEPENDENT third-party exact
k-NN (scikit-learn brute force + scipy cdist, tests/golden/make_retrieval_golden.py):
FAISS itself is not available, so these are the retrieval path's golden
vectors.  CPU only."""

import numpy as np

from oracle import retrieval_oracle as ro
from tests import retrieval_golden as rg


def test_oracle_equals_sklearn_brute_force_knn():
    seen = 0
    for name, q, c, k, D, I, _ in rg.cases():
        Do, Io = ro.search_exact(q, c, k)
        np.testing.assert_array_equal(Io, I, err_msg=name)
        np.testing.assert_allclose(Do, D, rtol=1e-12, atol=1e-12, err_msg=name)
        seen += 1
    assert seen == 6
