"""GPU parity of dense retrieval (fused score + top-k, k-way merge, join)
against the float64 FAISS-semantics oracle (oracle/retrieval_oracle.py).

Tolerances (north star): distances within 1e-3 relative for bf16 and 1e-5
for fp32, measured against ||q||^2 + ||c||^2; ids identical except where the
oracle's k-th / (k+1)-th distances tie within that tolerance."""

import numpy as np
import pytest
import torch

from oracle import retrieval_oracle as ro
from paper_2412_10543_b200 import IndexFlatL2, _lib, batch, merge_topk
from paper_2412_10543_b200.retriever import keys_to_dist_ids

pytestmark = pytest.mark.gpu

RTOL = {torch.bfloat16: 1e-3, torch.float32: 1e-5}


def make_data(nq, n, d, dtype, seed=0, dup_every=0):
    g = torch.Generator().manual_seed(seed)
    c = torch.randn(n, d, generator=g)
    c = c / c.norm(dim=1, keepdim=True)
    if dup_every:
        c[dup_every::dup_every] = c[0]
    src = torch.randint(0, max(n, 1), (nq,), generator=g)
    qv = torch.randn(nq, d, generator=g)
    half = nq // 2
    if n:
        qv[:half] = c[src[:half]] + 0.5 * qv[:half] / np.sqrt(d)
    qv = qv / qv.norm(dim=1, keepdim=True)
    return qv.to(dtype), c.to(dtype)


def run_search(q, c, k, algo="auto", id_base=0):
    ix = IndexFlatL2(c.shape[1], dtype=c.dtype, capacity=max(c.shape[0], 1), id_base=id_base)
    ix.set_algo(algo)
    if c.shape[0]:
        ix.add(c.cuda())
    D, I = ix.search(q.cuda(), k)
    torch.cuda.synchronize()
    plan = ix.last_plan()
    ix.close()
    return D.cpu().numpy(), I.cpu().numpy(), plan


def assert_parity(q, c, k, D, I, dtype, id_base=0, min_exact=0.9):
    I0 = np.where(I >= 0, I - id_base, -1)
    res = ro.check_topk(D, I0, q, c, k, RTOL[dtype])
    assert not res["violations"], res["violations"][:5]
    assert res["exact_rows"] >= min_exact * res["rows"], res


SHAPES = [  # nq, n, d, k
    (1, 1, 64, 1),
    (5, 34, 64, 35),
    (128, 256, 128, 10),
    (129, 257, 768, 35),
    (300, 5000, 1024, 35),
    (64, 70000, 768, 40),
    (200, 3000, 72, 17),      # dim not a multiple of the 64-element k-block
    (1000, 20000, 256, 35),
    (300, 6000, 4096, 35),    # long rows: 64 k-blocks per tile
    (40, 9000, 1536, 7),
    (33, 1000, 8, 5),         # one 16-byte row: a single partial k-block
    (77, 3001, 16, 35),
]


@pytest.mark.parametrize("algo", ["tcgen05", "tcgen05_1sm"])
@pytest.mark.parametrize("nq,n,d,k", SHAPES)
def test_tcgen05_bf16_matches_oracle(nq, n, d, k, algo):
    q, c = make_data(nq, n, d, torch.bfloat16, seed=nq + n)
    D, I, plan = run_search(q, c, k, algo=algo)
    assert plan["algo"] == algo
    assert_parity(q, c, k, D, I, torch.bfloat16)


def test_pair_and_single_cta_kernels_agree():
    q, c = make_data(700, 50_000, 1024, torch.bfloat16, seed=77)
    D2, I2, _ = run_search(q, c, 35, algo="tcgen05")
    D1, I1, _ = run_search(q, c, 35, algo="tcgen05_1sm")
    # identical fp32 products, possibly different accumulation order inside the MMA
    assert (I1 == I2).mean() > 0.99
    np.testing.assert_allclose(D1, D2, rtol=0, atol=1e-5)


@pytest.mark.parametrize("nq,n,d,k", SHAPES[:6])
def test_simt_fp32_matches_oracle(nq, n, d, k):
    q, c = make_data(nq, n, d, torch.float32, seed=7 + nq)
    D, I, plan = run_search(q, c, k, algo="simt")
    assert plan["algo"] == "simt"
    assert_parity(q, c, k, D, I, torch.float32)


@pytest.mark.parametrize("nq,n,d,k", SHAPES + [(1000, 100_000, 768, 35)])
def test_tf32x3_fp32_matches_oracle(nq, n, d, k):
    """fp32 corpus on the tensor cores (3xTF32 split, CTA-pair kernel) within
    the north star's fp32 tolerance (1e-5 relative)."""
    q, c = make_data(nq, n, d, torch.float32, seed=9 + nq)
    D, I, plan = run_search(q, c, k)
    assert plan["algo"] == "tcgen05"
    assert_parity(q, c, k, D, I, torch.float32)


def test_tf32x3_ties_and_wrapped_walk():
    nq, n, d, k, base = 600, 120_000, 128, 35, 60_001
    q, c = make_data(nq, n, d, torch.float32, seed=4)
    c[base::97] = c[base]
    q[:8] = c[base]
    ix = IndexFlatL2(d, dtype=torch.float32, capacity=n)
    ix.set_walk_bias(3)
    ix.add(c.cuda())
    D, I = ix.search(q.cuda(), k)
    torch.cuda.synchronize()
    ix.close()
    D, I = D.cpu().numpy(), I.cpu().numpy()
    for r in range(8):
        np.testing.assert_array_equal(I[r], base + 97 * np.arange(k))
    assert_parity(q[:100], c, k, D[:100], I[:100], torch.float32)


def test_simt_bf16_and_large_k():
    q, c = make_data(50, 3000, 128, torch.bfloat16, seed=3)
    D, I, _ = run_search(q, c, 100, algo="simt")
    assert_parity(q, c, 100, D, I, torch.bfloat16)


def test_ties_go_to_lower_chunk_id():
    # exact duplicate rows: identical distances must be ordered by chunk id
    q, c = make_data(64, 4096, 256, torch.bfloat16, seed=11, dup_every=97)
    q[:8] = c[0]
    for algo in ("tcgen05", "tcgen05_1sm", "simt"):
        D, I, _ = run_search(q, c, 35, algo=algo)
        dups = np.arange(0, 4096, 97)
        np.testing.assert_array_equal(I[0, :len(dups[:35])], dups[:35])
        assert np.all(D[0, :35] == D[0, 0])
        assert_parity(q, c, 35, D, I, torch.bfloat16)


def test_k_larger_than_corpus_pads_with_minus_one():
    q, c = make_data(10, 7, 64, torch.bfloat16)
    D, I, _ = run_search(q, c, 20)
    assert (I[:, 7:] == -1).all() and np.isinf(D[:, 7:]).all()
    assert_parity(q, c, 20, D, I, torch.bfloat16, min_exact=1.0)


def test_empty_index_and_empty_batch():
    ix = IndexFlatL2(64, dtype=torch.bfloat16, capacity=16)
    D, I = ix.search(torch.zeros(3, 64, dtype=torch.bfloat16, device="cuda"), 5)
    assert (I.cpu() == -1).all() and torch.isinf(D.cpu()).all()
    D, I = ix.search(torch.zeros(0, 64, dtype=torch.bfloat16, device="cuda"), 5)
    assert D.shape == (0, 5)
    with pytest.raises(ValueError):
        ix.add(torch.zeros(17, 64, dtype=torch.bfloat16))
    ix.close()


def test_numpy_in_numpy_out_faiss_convention():
    q, c = make_data(20, 500, 128, torch.float32)
    ix = IndexFlatL2(128, dtype=torch.float32, capacity=500)
    ix.add(c.numpy())
    D, I = ix.search(q.numpy(), 5)
    assert isinstance(D, np.ndarray) and D.dtype == np.float32 and I.dtype == np.int64
    assert_parity(q, c, 5, D, I, torch.float32)


def test_virtual_shards_merge_equals_single_index():
    """Corpus split into P shards with global id offsets, per-shard keys,
    k-way merge (the multi-GPU exchange path on one device)."""
    nq, n, d, k, P = 300, 40000, 512, 35, 4
    q, c = make_data(nq, n, d, torch.bfloat16, seed=21)
    D1, I1, _ = run_search(q, c, k)
    keys = []
    for r in range(P):
        lo, hi = r * n // P, (r + 1) * n // P
        ix = IndexFlatL2(d, dtype=torch.bfloat16, capacity=hi - lo, id_base=lo)
        ix.add(c[lo:hi].cuda())
        keys.append(ix.search_keys(q.cuda(), k))
        torch.cuda.synchronize()
        ix.close()
    gathered = torch.stack(keys)  # [P, nq, k] — the all_gather_into_tensor layout
    D, I = merge_topk(gathered, P, k, nq * k, k, nq=nq)
    np.testing.assert_array_equal(I.cpu().numpy(), I1)
    np.testing.assert_array_equal(D.cpu().numpy(), D1)
    # per-shard key lists are themselves sorted and carry global ids
    d0, i0 = keys_to_dist_ids(keys[1])
    assert (i0 >= n // P).all() and (i0 < 2 * n // P).all()
    assert np.all(np.diff(d0, axis=1) >= 0)


def test_join_keep_truncates_to_num_chunks():
    nq, n, d, k = 40, 2000, 128, 35
    q, c = make_data(nq, n, d, torch.bfloat16, seed=5)
    ix = IndexFlatL2(d, dtype=torch.bfloat16, capacity=n)
    ix.add(c.cuda())
    full_D, full_I = ix.search(q.cuda(), k)
    cfg = np.zeros(nq, dtype=_lib.CONFIG_DTYPE)
    cfg["status"] = np.where(np.arange(nq) % 5 == 0, 2, np.arange(nq) % 2)
    cfg["num_chunks"] = np.arange(nq) % 36
    keep = batch.to_device(cfg, torch.device("cuda"))
    D, I = ix.search(q.cuda(), k, keep=keep)
    I, fI = I.cpu().numpy(), full_I.cpu().numpy()
    for r in range(nq):
        m = 0 if cfg["status"][r] == 2 else min(int(cfg["num_chunks"][r]), k)
        np.testing.assert_array_equal(I[r, :m], fI[r, :m])
        assert (I[r, m:] == -1).all()
    ix.close()


@pytest.mark.parametrize("nq", [64, 2048])
def test_plan_shapes_multi_segment(nq):
    """Many segments x query tiles (the persistent segment-major schedule)."""
    q, c = make_data(nq, 300_000, 256, torch.bfloat16, seed=nq)
    D, I, plan = run_search(q, c, 35, algo="tcgen05")
    assert plan["segments"] > 1
    sub = slice(0, 64)
    assert_parity(q[sub], c, 35, D[sub], I[sub], torch.bfloat16)


@pytest.mark.parametrize("bias", [1, 7])
def test_wrapped_segment_walk_keeps_lower_id_ties(bias):
    """The pair kernel joins a corpus segment at its frontier and wraps around,
    so ids reach a row's top-k out of order; exact-duplicate rows must still
    resolve to the lowest ids (the walk bias forces a wrap in every unit)."""
    nq, n, d, k, base = 1024, 300_000, 256, 35, 150_001
    q, c = make_data(nq, n, d, torch.bfloat16, seed=bias)
    c[base::97] = c[base]
    q[:8] = c[base]
    q[8:16] = c[base] + 1e-3  # near-tie neighbours of the duplicate cluster
    ix = IndexFlatL2(d, dtype=torch.bfloat16, capacity=n)
    ix.set_algo("tcgen05")
    ix.set_walk_bias(bias)
    ix.add(c.cuda())
    D, I = ix.search(q.cuda(), k)
    torch.cuda.synchronize()
    plan = ix.last_plan()
    ix.close()
    D, I = D.cpu().numpy(), I.cpu().numpy()
    assert plan["segments"] > 1 and plan["qtiles"] > 1
    want = base + 97 * np.arange(k)
    for r in range(8):
        np.testing.assert_array_equal(I[r], want)
        assert np.all(D[r] == D[r, 0])
    assert_parity(q[:64], c, k, D[:64], I[:64], torch.bfloat16)
    assert_parity(q[-64:], c, k, D[-64:], I[-64:], torch.bfloat16)
    # the same search with the production walk agrees bit for bit
    D0, I0, _ = run_search(q, c, k, algo="tcgen05")
    np.testing.assert_array_equal(I0, I)
    np.testing.assert_array_equal(D0, D)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("nq", [1, 37, 128])
def test_small_batch_m128_tile(nq, dtype):
    """nq <= 128 runs the CTA pair's M = 128 tile (two top-k lists per row and
    segment, one per column half); duplicates + a forced wrap-around walk."""
    n, d, k, base = 200_000, 256, 35, 100_003
    q, c = make_data(nq, n, d, dtype, seed=nq)
    c[base::89] = c[base]
    q[0] = c[base]
    ix = IndexFlatL2(d, dtype=dtype, capacity=n)
    ix.set_walk_bias(5)
    ix.add(c.cuda())
    D, I = ix.search(q.cuda(), k)
    torch.cuda.synchronize()
    plan = ix.last_plan()
    ix.close()
    D, I = D.cpu().numpy(), I.cpu().numpy()
    assert plan["algo"] == "tcgen05" and plan["qtiles"] == 1 and plan["segments"] > 1
    np.testing.assert_array_equal(I[0], base + 89 * np.arange(k))
    assert_parity(q, c, k, D, I, dtype)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_incremental_adds_and_reset(dtype):
    """Rows appended in ragged pieces (partial 32-row norm chunks, the
    epilogue's dot bound must be recomputed for them) search exactly like one
    add; reset() empties the index for reuse."""
    nq, n, d, k = 300, 20_011, 128, 35
    q, c = make_data(nq, n, d, dtype, seed=13)
    # make the late rows the near neighbours, with norms below the early chunk minima
    c[n - 500:] *= 0.5
    q[: nq // 2] = c[n - 500: n - 500 + nq // 2] * 1.01
    ix = IndexFlatL2(d, dtype=dtype, capacity=n)
    for lo, hi in ((0, 1000), (1000, 1001), (1001, 7777), (7777, n - 500), (n - 500, n - 37), (n - 37, n)):
        ix.add(c[lo:hi].cuda())
    D, I = ix.search(q.cuda(), k)
    D, I = D.cpu().numpy(), I.cpu().numpy()
    assert_parity(q, c, k, D, I, dtype)
    D1, I1, _ = run_search(q, c, k)
    np.testing.assert_array_equal(I, I1)
    ix.reset()
    ix.add(c[:5000].cuda())
    D2, I2 = ix.search(q.cuda(), k)
    assert_parity(q, c[:5000], k, D2.cpu().numpy(), I2.cpu().numpy(), dtype)
    ix.close()


def test_ids_near_the_uint32_limit():
    nq, n, d, k = 64, 3000, 64, 20
    q, c = make_data(nq, n, d, torch.bfloat16, seed=2)
    base = (1 << 32) - 2 - n
    D, I, _ = run_search(q, c, k, id_base=base)
    assert I.max() < (1 << 32) - 1 and I.min() >= base
    assert_parity(q, c, k, D, I, torch.bfloat16, id_base=base)
