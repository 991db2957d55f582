"""The bench's synthetic corpus generator is the same on every side: the C
copy the CPU arms use (oracle/csrc/synth.c) equals tools/synth.py (torch)
bit for bit; queries are deterministic and have the SURVEY §8(d) shape."""

import numpy as np
import torch

from oracle import synth_host
from tools import synth


def test_c_generator_equals_torch_cpu():
    for r0, n, d, seed, dt in ((0, 300, 768, 0, torch.bfloat16), (9_999_000, 257, 1024, 0, torch.bfloat16),
                               (123_456, 200, 768, 7, torch.float32), (5, 3, 64, 2**31 + 5, torch.bfloat16)):
        a = synth_host.corpus_rows(r0, r0 + n, d, seed, dt == torch.bfloat16)
        b = synth.corpus_rows(r0, r0 + n, d, seed, dt, "cpu").float().numpy()
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (r0, d, seed)


def test_rows_are_unit_norm_and_independent():
    x = synth.corpus_rows(0, 2048, 1024, 0, torch.float32, "cpu").double()
    assert torch.allclose(x.norm(dim=1), torch.ones(2048, dtype=torch.float64), atol=1e-6)
    g = x @ x.T - torch.eye(2048, dtype=torch.float64)
    assert g.abs().max() < 0.2  # random unit vectors in d = 1024: |cos| ~ 0.03 typical
    assert abs(x.mean().item()) < 1e-3


def test_queries_noisy_neighbours_and_random():
    n, d = 50_000, 256
    q = synth.make_queries(64, n, d, 0, torch.bfloat16).double()
    q2 = synth.make_queries(64, n, d, 0, torch.bfloat16).double()
    assert torch.equal(q, q2)
    src = synth.query_sources(64, n, 0)
    c = synth.rows_by_id(torch.as_tensor(src), d, 0, torch.bfloat16).double()
    dist = ((q - c) ** 2).sum(1)
    assert (dist[0::2] < 0.35).all() and (dist[0::2] > 0.1).all()   # neighbours at ~0.2
    assert (dist[1::2] > 1.5).all()                                   # random queries at ~2


def test_mixture_families_shape():
    for data in ("clustered", "doc_contiguous"):
        x = synth.corpus_rows(0, 256, 128, 0, torch.float32, "cpu", data=data).double()
        assert torch.allclose(x.norm(dim=1), torch.ones(256, dtype=torch.float64), atol=1e-5)
    x = synth.corpus_rows(0, 64, 128, 0, torch.float32, "cpu", data="doc_contiguous").double()
    same_doc = ((x[0] - x[1]) ** 2).sum()
    other_doc = ((x[0] - x[40]) ** 2).sum()
    assert same_doc < 0.3 < other_doc
