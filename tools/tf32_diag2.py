import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.test_gpu_retrieval import make_data, run_search  # noqa: E402

for (nq, n, d, k) in [(129, 257, 768, 35), (128, 256, 768, 35), (129, 256, 768, 35), (128, 257, 768, 35), (64, 257, 768, 35), (129, 257, 128, 35)]:
    q, c = make_data(nq, n, d, torch.float32, seed=9 + nq)
    D, I, plan = run_search(q, c, k)
    q64, c64 = q.double(), c.double()
    exact = ((q64 ** 2).sum(1, keepdim=True) + (c64 ** 2).sum(1)[None] - 2 * q64 @ c64.T).numpy()
    g = np.take_along_axis(exact, np.maximum(I, 0), 1)
    err = np.abs(D - g)
    bad = np.argwhere(err > 2e-5)
    print((nq, n, d, k), plan, "max err", err.max(), "bad", len(bad), bad[:6].tolist(), "I ok",
          (np.sort(I, 1) == np.sort(np.argsort(exact, 1)[:, :k], 1)).mean())
