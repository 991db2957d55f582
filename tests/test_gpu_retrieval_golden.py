"""The GPU search against the third-party golden vectors (scikit-learn /
scipy exact k-NN, tests/golden/retrieval_sklearn.npz) within the north-star
tolerance relative to the distance (1e-3 bf16, 1e-5 fp32)."""

import pytest
import torch

from oracle import retrieval_oracle as ro
from paper_2412_10543_b200 import IndexFlatL2
from tests import retrieval_golden as rg

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["auto", "simt"])
def test_gpu_search_matches_sklearn_golden(algo):
    for name, q, c, k, D, I, bf in rg.cases():
        ix = IndexFlatL2(c.shape[1], dtype=c.dtype, capacity=c.shape[0])
        ix.set_algo(algo)
        ix.add(c.cuda())
        Dg, Ig = ix.search(q.cuda(), k)
        ix.close()
        res = ro.check_topk_rel(Dg.cpu().numpy(), Ig.cpu().numpy(), q, c, D, I, 1e-3 if bf else 1e-5)
        assert not res["violations"], (name, res["violations"][:3])
        assert res["exact_rows"] >= 0.95 * res["rows"], (name, res)
