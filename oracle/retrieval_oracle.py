"""Exact squared-L2 k-NN oracle (FAISS ``IndexFlatL2.search`` semantics) —
TEST INFRASTRUCTURE.

The reference package has no retriever (SPEC.md:15 puts "real embedding models
and vector databases" out of scope); the paper retrieves with FAISS
``IndexFlatL2`` + ``index.search(query_embedding, top_k)`` (PAPER.md:653,
PAPER.md:709).  FAISS is a third-party dependency that is NOT vendored under
/root/reference, has NO pinned version (pkg/pyproject.toml:10-12 lists only
``requests``) and is not installed here, so parity is UNPINNED against the
reference.  This module restates FAISS's published flat-L2 algorithm:

* ``D[i, j] = ||q_i||^2 + ||c_I[i,j]||^2 - 2 <q_i, c_I[i,j]>`` (the BLAS
  decomposition of ``exhaustive_L2sqr_blas``), negative round-off clamped to 0;
* results ascending by distance; when fewer than k vectors exist the tail is
  ``I = -1``, ``D = +inf``;
* ties broken by the LOWER chunk index (the north star's deterministic rule;
  FAISS's heap order on ties is unspecified).

``search_exact`` computes in float64 from the exact input values (bf16 and
fp32 both widen to float64 exactly) and is the parity checker.
``search_blas_fp32`` is the fast FAISS-style CPU implementation (fp32 sgemm on
all host cores + partial selection) timed as the CPU baseline.
"""

from __future__ import annotations

import numpy as np


def _as_f64(x) -> np.ndarray:
    """Widen fp32 / bf16 (given as a torch tensor or numpy array) to float64."""
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().to("cpu", torch.float64).numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x, dtype=np.float64)


def topk_lex(dist: np.ndarray, k: int, base: int = 0):
    """Row-wise k smallest of ``dist`` [nq, n] ordered by (distance, index)."""
    nq, n = dist.shape
    kk = min(k, n)
    D = np.full((nq, k), np.inf, dtype=np.float64)
    I = np.full((nq, k), -1, dtype=np.int64)
    if kk == 0:
        return D, I
    idx = np.arange(n, dtype=np.int64)
    for r in range(nq):
        row = dist[r]
        if kk < n:
            # candidates: everything <= the kk-th smallest value (keeps ties)
            thr = np.partition(row, kk - 1)[kk - 1]
            cand = np.nonzero(row <= thr)[0]
        else:
            cand = idx
        order = np.lexsort((cand, row[cand]))[:kk]
        sel = cand[order]
        D[r, :kk] = row[sel]
        I[r, :kk] = sel + base
    return D, I


def search_exact(queries, corpus, k: int, *, block: int = 65536):
    """Float64 exact search.  Returns (D float64 [nq,k], I int64 [nq,k])."""
    q = _as_f64(queries)
    nq = q.shape[0]
    qn = np.einsum("ij,ij->i", q, q)
    bestD = np.full((nq, k), np.inf)
    bestI = np.full((nq, k), -1, dtype=np.int64)
    c_all = corpus
    n = c_all.shape[0]
    for s in range(0, n, block):
        c = _as_f64(c_all[s:s + block])
        cn = np.einsum("ij,ij->i", c, c)
        d = qn[:, None] + cn[None, :] - 2.0 * (q @ c.T)
        np.maximum(d, 0.0, out=d)
        D, I = topk_lex(d, k, base=s)
        bestD, bestI = merge_lists([bestD, D], [bestI, I], k)
    return bestD, bestI


def merge_lists(Ds, Is, k: int):
    """k-way merge of sorted per-shard lists by (distance, global index) — the
    restatement of the multi-GPU merge (``-1`` entries sort last)."""
    D = np.concatenate(Ds, axis=1)
    I = np.concatenate(Is, axis=1)
    nq = D.shape[0]
    outD = np.full((nq, k), np.inf)
    outI = np.full((nq, k), -1, dtype=np.int64)
    for r in range(nq):
        ids = np.where(I[r] < 0, np.iinfo(np.int64).max, I[r])
        order = np.lexsort((ids, D[r]))
        keep = order[:k]
        outD[r, :len(keep)] = D[r, keep]
        outI[r, :len(keep)] = I[r, keep]
    return outD, outI


def search_blas_fp32(queries: np.ndarray, corpus: np.ndarray, k: int, *,
                     corpus_norms: np.ndarray | None = None, block: int = 262144):
    """FAISS-style flat-L2 on the CPU: fp32 sgemm (numpy BLAS, all host
    threads) over corpus blocks + running top-k selection.  The timed CPU
    baseline; not bit-identical to ``search_exact`` (fp32 accumulation)."""
    q = np.ascontiguousarray(queries, dtype=np.float32)
    nq = q.shape[0]
    qn = np.einsum("ij,ij->i", q, q)
    bestD = np.full((nq, k), np.inf, dtype=np.float32)
    bestI = np.full((nq, k), -1, dtype=np.int64)
    n = corpus.shape[0]
    for s in range(0, n, block):
        c = np.ascontiguousarray(corpus[s:s + block], dtype=np.float32)
        cn = corpus_norms[s:s + block] if corpus_norms is not None else np.einsum("ij,ij->i", c, c)
        d = q @ c.T
        d *= -2.0
        d += qn[:, None]
        d += cn[None, :]
        np.maximum(d, 0.0, out=d)
        kk = min(k, d.shape[1])
        part = np.argpartition(d, kk - 1, axis=1)[:, :kk]
        pd = np.take_along_axis(d, part, axis=1)
        D = np.concatenate([bestD, pd], axis=1)
        I = np.concatenate([bestI, part.astype(np.int64) + s], axis=1)
        o = np.argsort(D, axis=1, kind="stable")[:, :k]
        bestD = np.take_along_axis(D, o, axis=1)
        bestI = np.take_along_axis(I, o, axis=1)
    return bestD, bestI


def check_topk(D_gpu, I_gpu, queries, corpus, k, rtol, *, D_ref=None, I_ref=None):
    """Parity check of a GPU result against the float64 oracle.

    Tolerance is relative to ``||q||^2 + ||c||^2`` (the scale the distance is
    computed at; a raw relative error is meaningless near 0 for
    near-duplicates).  Rules (north star): (1) every returned distance within
    tolerance of the true float64 distance of the returned id; (2) rank-wise
    distance within tolerance of the oracle's; (3) ids identical except
    where the oracle's distances are tied within tolerance.

    Returns a dict with the number of exact-id rows and any violations.
    """
    q = _as_f64(queries)
    if D_ref is None:
        D_ref, I_ref = search_exact(queries, corpus, k)
    D_gpu = np.asarray(D_gpu, dtype=np.float64)
    I_gpu = np.asarray(I_gpu, dtype=np.int64)
    qn = np.einsum("ij,ij->i", q, q)
    viol = []
    exact_rows = 0
    for r in range(q.shape[0]):
        if np.array_equal(I_gpu[r], I_ref[r]):
            exact_rows += 1
        valid = I_ref[r] >= 0
        if not np.array_equal(I_gpu[r] >= 0, valid):
            viol.append((r, "padding mismatch"))
            continue
        ids = I_gpu[r][valid]
        if len(set(ids.tolist())) != len(ids):
            viol.append((r, "duplicate ids"))
            continue
        c = _as_f64(corpus[ids]) if len(ids) else np.zeros((0, q.shape[1]))
        cn = np.einsum("ij,ij->i", c, c)
        true_d = np.maximum(qn[r] + cn - 2.0 * (c @ q[r]), 0.0)
        scale = qn[r] + cn + 1e-30
        tol = rtol * scale
        if np.any(np.abs(D_gpu[r][valid] - true_d) > tol):
            viol.append((r, "distance off"))
            continue
        if np.any(np.abs(true_d - D_ref[r][valid]) > tol):
            viol.append((r, "rank distance off"))
            continue
        # id mismatches are allowed only inside tolerance-ties of the oracle
        mism = np.nonzero(I_gpu[r][valid] != I_ref[r][valid])[0]
        for j in mism:
            if abs(true_d[j] - D_ref[r][j]) > tol[j]:
                viol.append((r, f"id mismatch at {j} outside tie tolerance"))
                break
    return {"rows": q.shape[0], "exact_rows": exact_rows, "violations": viol}


def search_torch_cpu(queries: np.ndarray, corpus: np.ndarray, corpus_norms: np.ndarray, k: int, *,
                     block: int = 16384):
    """FAISS-style flat-L2 on the CPU with torch's BLAS on all host threads
    (the ``exhaustive_L2sqr_blas`` decomposition: ``|q|^2 + |c|^2 - 2 q.c`` per
    corpus block, then a running per-query top-k).  The timed CPU baseline /
    reference-arm retrieval; fp32 arithmetic, so ties and near-ties come back
    in arbitrary order (``exact_topk`` re-ranks the candidates in float64).
    The corpus norms are precomputed (as the GPU index does at ``add``)."""
    import torch

    q = torch.from_numpy(np.ascontiguousarray(queries, dtype=np.float32))
    qn = (q * q).sum(1, keepdim=True)
    n = corpus.shape[0]
    kk = min(k, n)
    bestD = torch.full((q.shape[0], 0), float("inf"))
    bestI = torch.zeros((q.shape[0], 0), dtype=torch.int64)
    for s in range(0, n, block):
        c = torch.from_numpy(corpus[s:s + block])
        base = qn + torch.from_numpy(corpus_norms[s:s + block])[None, :]
        d = torch.addmm(base, q, c.T, beta=1.0, alpha=-2.0).clamp_(min=0.0)
        dd, ii = torch.topk(d, min(kk, d.shape[1]), dim=1, largest=False, sorted=False)
        bestD = torch.cat([bestD, dd], 1)
        bestI = torch.cat([bestI, ii + s], 1)
        if bestD.shape[1] > 4 * kk:
            bestD, sel = torch.topk(bestD, kk, dim=1, largest=False, sorted=False)
            bestI = torch.gather(bestI, 1, sel)
    bestD, sel = torch.topk(bestD, kk, dim=1, largest=False, sorted=True)
    bestI = torch.gather(bestI, 1, sel)
    return bestD.numpy(), bestI.numpy()


def exact_topk(queries, corpus, cand_ids: np.ndarray, k: int):
    """Float64 re-score of candidate ids per query, ordered by (distance, id):
    the exact top-k whenever the true top-k is among the candidates (a
    fp32 scan with a margin of extra candidates guarantees that outside
    near-ties far below the tolerance)."""
    q = _as_f64(queries)
    nq = q.shape[0]
    D = np.full((nq, k), np.inf)
    I = np.full((nq, k), -1, dtype=np.int64)
    for r in range(nq):
        ids = np.unique(cand_ids[r][cand_ids[r] >= 0])
        c = _as_f64(corpus[ids])
        d = ((c - q[r]) ** 2).sum(1)
        o = np.lexsort((ids, d))[:k]
        D[r, :len(o)] = d[o]
        I[r, :len(o)] = ids[o]
    return D, I


def check_topk_rel(D_gpu, I_gpu, queries, corpus, D_ref, I_ref, rtol: float, atol_scale: float = 1e-6):
    """Parity of a GPU result against the exact (float64) top-k, tolerance
    RELATIVE TO THE DISTANCE (north star: 1e-3 for bf16, 1e-5 for fp32):
    ``|D - D_true| <= rtol * D_true + atol_scale * (|q|^2 + |c|^2)``; the
    second term is the cancellation floor of the ``|q|^2 + |c|^2 - 2 q.c``
    form (FAISS's too) and only matters for (near-)duplicates, D ~ 0.

    Rules: (1) each returned distance within tolerance of the float64
    distance of the returned id; (2) rank by rank within tolerance of the
    exact distance; (3) so ids may differ only inside tolerance-ties.
    Returns rows, exact-id rows, violations, and the max relative error
    ``|D - D_true| / D_true`` over entries with D_true >= 1e-3."""
    q = _as_f64(queries)
    D_gpu = np.asarray(D_gpu, dtype=np.float64)
    I_gpu = np.asarray(I_gpu, dtype=np.int64)
    qn = np.einsum("ij,ij->i", q, q)
    viol, exact_rows, max_rel, max_abs = [], 0, 0.0, 0.0
    for r in range(q.shape[0]):
        exact_rows += int(np.array_equal(I_gpu[r], I_ref[r]))
        valid = I_ref[r] >= 0
        if not np.array_equal(I_gpu[r] >= 0, valid):
            viol.append((r, "padding mismatch"))
            continue
        ids = I_gpu[r][valid]
        if len(np.unique(ids)) != len(ids):
            viol.append((r, "duplicate ids"))
            continue
        c = _as_f64(corpus[ids]) if len(ids) else np.zeros((0, q.shape[1]))
        true_d = ((c - q[r]) ** 2).sum(1)
        tol = rtol * true_d + atol_scale * (qn[r] + np.einsum("ij,ij->i", c, c))
        err = np.abs(D_gpu[r][valid] - true_d)
        big = true_d >= 1e-3
        if big.any():
            max_rel = max(max_rel, float((err[big] / true_d[big]).max()))
        if len(err):
            max_abs = max(max_abs, float(err.max()))
        if np.any(err > tol):
            viol.append((r, "distance off"))
            continue
        tol_ref = rtol * D_ref[r][valid] + atol_scale * (qn[r] + np.einsum("ij,ij->i", c, c))
        if np.any(np.abs(true_d - D_ref[r][valid]) > np.maximum(tol, tol_ref)):
            viol.append((r, "rank distance off"))
    return {"rows": int(q.shape[0]), "exact_rows": exact_rows, "violations": viol,
            "max_rel_err": max_rel, "max_abs_err": max_abs}
