"""fp32 edge cases of the 3xTF32 tensor-core search:

* k up to 40 keeps its 8 spare candidates for the exact re-rank: a corpus
  whose ranks k-8 .. k+8 are spaced 3e-6 apart in distance (below the tf32
  pass's ~1e-5 error, far above the exact fp32 re-rank's ~3e-7) must come back
  as the exact top-k, ids and order, for k = 32, 35, 40;
* an fp32 index whose dim is not a multiple of 4 (no tensor-core path: no
  tf32 residuals are built) adds rows and searches on the CUDA-core kernel.
"""

import numpy as np
import pytest
import torch

from oracle import retrieval_oracle as ro
from paper_2412_10543_b200 import IndexFlatL2

pytestmark = pytest.mark.gpu


def _near_tie_corpus(d=768, n_close=80, n_far=20000, step=1.5e-6, seed=3):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(d, generator=g, dtype=torch.float64)
    q /= q.norm()
    r = torch.randn(n_close, d, generator=g, dtype=torch.float64)
    r -= (r @ q)[:, None] * q[None, :]
    r /= r.norm(dim=1, keepdim=True)
    alpha = 0.5 - step * torch.arange(n_close, dtype=torch.float64)  # D = 2 - 2 alpha: +3e-6 per rank
    close = alpha[:, None] * q[None, :] + torch.sqrt(1 - alpha ** 2)[:, None] * r
    far = torch.randn(n_far, d, generator=g, dtype=torch.float64)
    far /= far.norm(dim=1, keepdim=True)
    # scatter the close rows through the corpus (not in id order of their distance)
    perm = torch.randperm(n_close + n_far, generator=g)
    c = torch.empty(n_close + n_far, d, dtype=torch.float64)
    c[perm[:n_close]] = close
    c[perm[n_close:]] = far
    return q[None].float(), c.float(), perm[:n_close].numpy()


@pytest.mark.parametrize("k", [32, 35, 40])
def test_tf32_near_ties_at_rank_k_exact(k):
    q, c, close_ids = _near_tie_corpus()
    ix = IndexFlatL2(c.shape[1], dtype=torch.float32, capacity=c.shape[0])
    ix.add(c.cuda())
    D, I = ix.search(q.cuda(), k)
    assert ix.last_plan()["algo"] == "tcgen05"
    ix.close()
    # exact fp64 order of the close rows = their construction order
    d64 = ((c.double()[close_ids] - q.double()) ** 2).sum(1).numpy()
    assert (np.diff(d64) > 2e-6).all()
    np.testing.assert_array_equal(I.cpu().numpy()[0], close_ids[:k])
    assert np.abs(D.cpu().numpy()[0] - d64[:k]).max() < 1e-6


@pytest.mark.parametrize("d", [130, 77, 3])
def test_fp32_dim_not_multiple_of_4_add_and_search(d):
    g = torch.Generator().manual_seed(d)
    c = torch.nn.functional.normalize(torch.randn(3000, d, generator=g), dim=1)
    q = torch.nn.functional.normalize(c[:50] + 0.3 * torch.randn(50, d, generator=g), dim=1)
    ix = IndexFlatL2(d, dtype=torch.float32, capacity=3000)
    ix.add(c[:1000].cuda())
    ix.add(c[1000:].cuda())  # incremental adds
    D, I = ix.search(q.cuda(), 35)
    assert ix.last_plan()["algo"] == "simt"
    ix.close()
    res = ro.check_topk(D.cpu().numpy(), I.cpu().numpy(), q, c, 35, 1e-5)
    assert not res["violations"], res["violations"][:3]
