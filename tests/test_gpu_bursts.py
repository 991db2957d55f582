"""Candidate bursts in the pair kernel's register top-k.

When a corpus stores a document's chunks under consecutive ids, a query's
candidates arrive as a burst in ONE lane of an epilogue warp (its document's
chunks fill a 32-column chunk), and the flush merges that lane's list
cooperatively (the whole warp sorts it with the lane's buffered candidates,
RegTopK::coop_merge / coop_sort64) whenever the lane holds
RS_TOPK_COOP_GAIN more candidates than every other lane; the rest goes
through the lockstep insert.  These tests pin both paths against the float64
oracle and the lower-id tie rule, with exact-duplicate documents (every
burst member ties), forced wrap-around walks (bursts that straddle the
walk's phase change) and mixed burst sizes inside one warp (the greedy
fullest-lane-first loop, then lockstep for the remainder)."""

import numpy as np
import pytest
import torch

from oracle import retrieval_oracle as ro
from paper_2412_10543_b200 import IndexFlatL2
from tools import synth

pytestmark = pytest.mark.gpu

RTOL = {torch.bfloat16: 1e-3, torch.float32: 1e-5}


def search(q, c, k, bias=0):
    ix = IndexFlatL2(c.shape[1], dtype=c.dtype, capacity=c.shape[0])
    ix.set_algo("tcgen05")
    if bias:
        ix.set_walk_bias(bias)
    ix.add(c.cuda())
    D, I = ix.search(q.cuda(), k)
    torch.cuda.synchronize()
    plan = ix.last_plan()
    ix.close()
    return D.cpu().numpy(), I.cpu().numpy(), plan


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("nq", [64, 1000])
def test_doc_contiguous_corpus_matches_oracle(nq, dtype):
    n, d, k = 120_000, 256, 35
    c = synth.corpus_rows(0, n, d, 7, dtype, "cuda", "doc_contiguous").cpu()
    q = synth.make_queries(nq, n, d, 7, dtype, "doc_contiguous")
    D, I, plan = search(q, c, k)
    assert plan["segments"] > 1
    res = ro.check_topk(D, I, q, c, k, RTOL[dtype])
    assert not res["violations"], res["violations"][:5]
    assert res["exact_rows"] >= 0.9 * nq, res


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("bias", [0, 3])
@pytest.mark.parametrize("block", [32, 12])
def test_duplicate_document_bursts_keep_lower_ids(block, bias, dtype):
    """Documents of `block` identical rows at consecutive ids: a query equal to
    a document's vector ties with all of its rows, which must come back first
    and in ascending id order, then the nearest other rows."""
    n, d, k, nq = 150_000, 128, 35, 512
    g = torch.Generator().manual_seed(block * 10 + bias)
    c = torch.nn.functional.normalize(torch.randn(n, d, generator=g), dim=1)
    starts = torch.randint(0, n // block - 1, (nq,), generator=g) * block
    for s in starts.tolist():
        c[s:s + block] = c[s]
    c = c.to(dtype)
    q = c[starts].clone()
    D, I, plan = search(q, c, k, bias)
    assert plan["segments"] > 1 and plan["qtiles"] > 1
    m = min(block, k)
    for r, s in enumerate(starts.tolist()):
        np.testing.assert_array_equal(I[r, :m], s + np.arange(m), err_msg=f"row {r}")
        assert np.all(D[r, :m] == D[r, 0])
    res = ro.check_topk(D[:128], I[:128], q[:128], c, k, RTOL[dtype])
    assert not res["violations"], res["violations"][:5]
    # the production walk (no bias) returns the same lists
    if bias:
        D0, I0, _ = search(q, c, k)
        np.testing.assert_array_equal(I0, I)
        np.testing.assert_array_equal(D0, D)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("bias", [0, 5])
def test_mixed_burst_sizes_in_one_warp(bias, dtype):
    """Each 32-row corpus chunk of a group holds duplicate documents of sizes
    16, 8, 3 and 5; four consecutive queries (lanes of one epilogue warp) equal
    those four documents, so one flush sees bursts of different sizes in
    several lanes: the fullest lane is merged cooperatively while it leads the
    others by the gain threshold, the rest in lockstep.  Every query must get
    its document's rows first, in ascending id order, then the oracle's."""
    n, d, k = 160_000, 128, 35
    sizes = [16, 8, 3, 5]
    g = torch.Generator().manual_seed(99 + bias)
    c = torch.nn.functional.normalize(torch.randn(n, d, generator=g), dim=1)
    groups = torch.randperm(n // 32 - 1, generator=g)[:192].tolist()
    starts = []
    for grp in groups:
        b = grp * 32
        for sz in sizes:
            c[b:b + sz] = torch.nn.functional.normalize(torch.randn(d, generator=g), dim=0)
            starts.append((b, sz))
            b += sz
    c = c.to(dtype)
    q = torch.stack([c[s] for s, _ in starts]).clone()
    D, I, plan = search(q, c, k, bias)
    assert plan["segments"] > 1 and plan["qtiles"] > 1
    for r, (s, sz) in enumerate(starts):
        np.testing.assert_array_equal(I[r, :sz], s + np.arange(sz), err_msg=f"row {r}")
        assert np.all(D[r, :sz] == D[r, 0])
    res = ro.check_topk(D, I, q, c, k, RTOL[dtype])
    assert not res["violations"], res["violations"][:5]


def _index(c, mode):
    ix = IndexFlatL2(c.shape[1], dtype=c.dtype, capacity=c.shape[0])
    ix.set_algo("tcgen05")
    ix.set_burst_merge(mode)
    ix.add(c.cuda())
    return ix


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("data", ["doc_contiguous", "iso"])
def test_lean_and_cooperative_variants_are_bit_identical(data, dtype):
    """The lean kernel (no cooperative merge) and the cooperative one return
    the same keys bit for bit, and the automatic mode equals both."""
    n, d, k, nq = 200_000, 256, 35, 700
    c = synth.corpus_rows(0, n, d, 3, dtype, "cuda", data).cpu()
    q = synth.make_queries(nq, n, d, 3, dtype, data).cuda()
    out = {}
    for mode in ("off", "on", "auto"):
        ix = _index(c, mode)
        keys = [ix.search_keys(q, k).cpu() for _ in range(3)]  # auto may switch variants between searches
        torch.cuda.synchronize()
        ix.close()
        for t in keys[1:]:
            assert torch.equal(t, keys[0]), mode
        out[mode] = keys[0]
    assert torch.equal(out["off"], out["on"]) and torch.equal(out["auto"], out["on"])


def test_auto_mode_switches_on_bursty_corpora_only():
    """Automatic choice: a doc-contiguous corpus turns the cooperative variant
    on after one search; an isotropic one keeps the lean variant."""
    n, d, k, nq = 400_000, 256, 35, 2048
    for data, want in (("doc_contiguous", True), ("iso", False)):
        c = synth.corpus_rows(0, n, d, 5, torch.bfloat16, "cuda", data).cpu()
        q = synth.make_queries(nq, n, d, 5, torch.bfloat16, data).cuda()
        ix = _index(c, "auto")
        assert not ix.burst_merge_active()  # lean until a search reports bursts
        ix.search_keys(q, k)
        torch.cuda.synchronize()
        assert ix.burst_merge_active() == want, data
        ix.set_burst_merge("on")
        assert ix.burst_merge_active()
        ix.set_burst_merge("off")
        assert not ix.burst_merge_active()
        ix.close()
