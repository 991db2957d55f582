"""The pair kernel's probe pass (rs_index_set_probe) and drift limiter.

Before the main launch the same kernel scans the corpus's first rows (one
256-row tile per segment) and folds the kCas-th smallest of those lists'
rank-ceil(k/kCas) distances into every query's shared admission bound
(fold_probe_bounds_kernel).  That bound is backed by >= k real rows, so the
main launch must return exactly what it returns without a probe: these tests
pin bit-identical (D, I) with the probe on and off (the default), against
the float64 oracle too, including exact-duplicate rows inside the
probed rows (ties at the bound itself) and the wrap-around walk."""

import numpy as np
import pytest
import torch

from oracle import retrieval_oracle as ro
from paper_2412_10543_b200 import IndexFlatL2
from tools import synth

pytestmark = pytest.mark.gpu

RTOL = {torch.bfloat16: 1e-3, torch.float32: 1e-5}


def search(q, c, k, probe, bias=0):
    ix = IndexFlatL2(c.shape[1], dtype=c.dtype, capacity=c.shape[0])
    ix.set_algo("tcgen05")
    if probe is not None:
        ix.set_probe(probe)
    if bias:
        ix.set_walk_bias(bias)
    ix.add(c.cuda())
    D, I = ix.search(q.cuda(), k)
    torch.cuda.synchronize()
    rows = ix.last_probe_rows()
    ix.close()
    return D.cpu().numpy(), I.cpu().numpy(), rows


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("data", ["iso", "clustered", "doc_contiguous"])
def test_probe_bit_identical_and_matches_oracle(dtype, data):
    n, d, k, nq = 100_000, 768 if dtype == torch.float32 else 512, 35, 1000
    c = synth.corpus_rows(0, n, d, 11, dtype, "cuda", data).cpu()
    q = synth.make_queries(nq, n, d, 11, dtype, data)
    D1, I1, rows_on = search(q, c, k, "on")
    D0, I0, rows_off = search(q, c, k, "off")
    Dd, Id, rows_default = search(q, c, k, None)
    assert rows_on > 0 and rows_off == 0 and rows_default == 0  # off by default
    np.testing.assert_array_equal(I1, I0)
    np.testing.assert_array_equal(D1, D0)
    np.testing.assert_array_equal(Id, I0)
    res = ro.check_topk(D1[:200], I1[:200], q[:200], c, k, RTOL[dtype])
    assert not res["violations"], res["violations"][:5]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("bias", [0, 2])
def test_probe_ties_inside_probed_rows(dtype, bias):
    """Every query equals a block of 40 identical rows, some inside the probed
    prefix: the probe's bound is then exactly the tied distance, and the main
    launch must still return the block's lowest ids first."""
    n, d, k, nq, block = 60_000, 128, 35, 600, 40
    g = torch.Generator().manual_seed(5 + bias)
    c = torch.nn.functional.normalize(torch.randn(n, d, generator=g), dim=1)
    starts = torch.randint(0, n // block - 1, (nq,), generator=g) * block
    starts[: nq // 4] = torch.randint(0, 4096 // block - 1, (nq // 4,), generator=g) * block  # in the probe rows
    for s in starts.tolist():
        c[s:s + block] = c[s]
    c = c.to(dtype)
    q = c[starts].clone()
    D1, I1, rows = search(q, c, k, "on", bias)
    D0, I0, _ = search(q, c, k, "off", bias)
    assert rows > 0
    np.testing.assert_array_equal(I1, I0)
    np.testing.assert_array_equal(D1, D0)
    for r, s in enumerate(starts.tolist()):
        np.testing.assert_array_equal(I1[r], s + np.arange(k), err_msg=f"row {r}")


@pytest.mark.parametrize("bias", [0, 3])
def test_drift_limiter_shapes_match_oracle(bias):
    """2 query tiles whose units are exactly one round of pairs: make_plan turns the
    drift limiter on (a unit waits, bounded, while it runs ahead of its
    segment's slowest unit).  With a walk bias the units of a segment run at
    permanently different positions, so every wait times out: the results
    must still equal the unbiased search and the oracle."""
    n, d, k, nq = 1_000_000, 128, 35, 512
    c = synth.corpus_rows(0, n, d, 13, torch.bfloat16, "cuda")
    q = synth.make_queries(nq, n, d, 13, torch.bfloat16)
    ix = IndexFlatL2(d, dtype=torch.bfloat16, capacity=n)
    ix.add(c)
    D0, I0 = ix.search(q.cuda(), k)
    if bias:
        ix.set_walk_bias(bias)
    D1, I1 = ix.search(q.cuda(), k)
    torch.cuda.synchronize()
    plan = ix.last_plan()
    ix.close()
    pairs = torch.cuda.get_device_properties(0).multi_processor_count // 2
    assert plan["qtiles"] == 2 and plan["qtiles"] * plan["segments"] == pairs, plan
    np.testing.assert_array_equal(I1.cpu().numpy(), I0.cpu().numpy())
    np.testing.assert_array_equal(D1.cpu().numpy(), D0.cpu().numpy())
    res = ro.check_topk(D1[:64].cpu().numpy(), I1[:64].cpu().numpy(), q[:64], c.cpu(), k, 1e-3)
    assert not res["violations"], res["violations"][:5]
