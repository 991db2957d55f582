"""Synthetic embeddings for bench.py and the parity tests.

One generator, bit-identical on the GPU (torch CUDA), on the host (torch CPU)
and in C (``oracle/csrc/synth.c``, the CPU arms' copy), so that the GPU arm,
its CPU baseline and the ``--impl reference`` arm search the SAME corpus with
the SAME queries.  Every value is built from exact integer arithmetic plus
correctly rounded IEEE operations:

* ``mix32`` — a 32-bit bijective integer hash (xor-shift / multiply; the
  multiply is split into 16-bit halves so every int64 product stays < 2^63);
* element (row r, column j): ``h_t = mix32(hrow(r) ^ hcol(2j + t))`` for
  t = 0, 1, and ``v = (sum of the four 16-bit halves of h_0, h_1) - 131070``,
  an Irwin-Hall(4) integer (approximately Gaussian);
* row normalisation: ``S = sum_j v_j^2`` exactly in int64 (< 2^45), then
  ``x_j = float32(double(v_j) / sqrt(double(S)))`` — IEEE division and square
  root are correctly rounded on the CPU and the GPU alike — and, for a bf16
  corpus, round-to-nearest-even to bf16.

Queries (``make_queries``) are built on the host in float64 numpy (pairwise
summation: deterministic): even queries are noisy neighbours
``normalize(c_src + 0.5 u)`` of a hashed corpus row (u a unit vector, so the
source row sits at squared distance ~0.2 while random rows sit at ~2), odd
queries random unit vectors.

Data families (``data=``, the robustness workloads; generated on one device
per run, so they are not bit-pinned across CPU and GPU like ``iso``):
* ``iso``            — isotropic unit rows (the default);
* ``clustered``      — a Gaussian mixture of ``N_CLUSTERS`` unit centers; row r
  belongs to cluster ``mix32(r ^ key) % N_CLUSTERS`` (ids of a cluster are
  scattered) and is ``normalize(center + NOISE * unit noise)``;
* ``doc_contiguous`` — documents of ``DOC_CHUNKS`` consecutive chunk ids share
  a center (id order correlates with similarity).
For both, odd queries sit near a center: ``normalize(center + 0.3 g)``.
"""

from __future__ import annotations

import numpy as np
import torch

M32 = 0xFFFFFFFF
DOC_CHUNKS = 32          # doc_contiguous: chunks per document
N_CLUSTERS = 100_000     # clustered: mixture components (~100 rows each at 10M)
NOISE = 0.25             # mixture families: noise norm relative to the unit center
_ROW_KEY = 0xA5A5A5A5
_COL_KEY = 0x5BD1E995
_CLUSTER_KEY = 0x27D4EB2F
_CENTER_KEY = 0x3C6EF372
_NOISE_KEY = 0x1B873593
_SRC_KEY = 0x68E31DA4
_QU_KEY = 0x7F4A7C15
_QG_KEY = 0x94D049BB
DATA = ("iso", "clustered", "doc_contiguous")


def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for int64 x in [0, 2^32) without int64 overflow."""
    return (x * (c & 0xFFFF) + (((x * (c >> 16)) & 0xFFFF) << 16)) & M32


def mix32(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    return x ^ (x >> 16)


def mix32_int(x: int) -> int:
    x &= M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & M32
    return x ^ (x >> 16)


def row_key(seed: int) -> int:
    return mix32_int((seed & M32) ^ _ROW_KEY)


def int_rows(rows: torch.Tensor, d: int, seed: int) -> torch.Tensor:
    """Irwin-Hall integers v [len(rows), d] (int64) of the given row ids."""
    hr = mix32((rows.to(torch.int64) & M32) ^ row_key(seed))[:, None]
    j = torch.arange(2 * d, dtype=torch.int64, device=rows.device)
    hc = mix32(j ^ _COL_KEY)[None, :]
    h = mix32(hr ^ hc)                                   # [R, 2d]: column j, draw t at 2j + t
    v = (h & 0xFFFF) + (h >> 16)
    return v.view(-1, d, 2).sum(-1) - 131070


def normalize_int_rows(v: torch.Tensor, dtype) -> torch.Tensor:
    """float32(double(v) / sqrt(double(sum v^2))), then ``dtype`` (RNE)."""
    s = (v * v).sum(1, keepdim=True).double().sqrt()
    x = (v.double() / s).float()
    return x if dtype == torch.float32 else x.to(dtype)


def _unit(x: torch.Tensor) -> torch.Tensor:
    return x / (x * x).sum(1, keepdim=True).sqrt()


def cluster_of(rows: torch.Tensor, data: str) -> torch.Tensor:
    rows = rows.to(torch.int64)
    if data == "clustered":
        return mix32((rows & M32) ^ _CLUSTER_KEY) % N_CLUSTERS
    return rows // DOC_CHUNKS


def centers(cid: torch.Tensor, d: int, seed: int) -> torch.Tensor:
    return _unit(int_rows(cid, d, seed ^ _CENTER_KEY).double())


def corpus_rows(r0: int, r1: int, d: int, seed: int, dtype, device, data: str = "iso",
                chunk: int = 65536) -> torch.Tensor:
    """Corpus rows [r0, r1) in ``dtype`` on ``device``."""
    if data not in DATA:
        raise ValueError(f"data must be one of {DATA}")
    out = torch.empty(r1 - r0, d, dtype=dtype, device=device)
    for a in range(r0, r1, chunk):
        b = min(r1, a + chunk)
        out[a - r0:b - r0] = rows_by_id(torch.arange(a, b, dtype=torch.int64, device=device), d, seed, dtype, data)
    return out


def rows_by_id(rows: torch.Tensor, d: int, seed: int, dtype, data: str = "iso") -> torch.Tensor:
    """Corpus rows with the given ids (any order), on ``rows.device``."""
    if data == "iso":
        return normalize_int_rows(int_rows(rows, d, seed), dtype)
    c = centers(cluster_of(rows, data), d, seed)
    z = _unit(int_rows(rows, d, seed ^ _NOISE_KEY).double())
    return _unit(c + NOISE * z).float().to(dtype)


def query_sources(nq: int, n: int, seed: int) -> np.ndarray:
    """The corpus row each even query is a noisy neighbour of."""
    h = mix32(torch.arange(nq, dtype=torch.int64) ^ mix32_int(seed ^ _SRC_KEY))
    return ((h * n) >> 32).numpy()


def _unit_np(v: np.ndarray) -> np.ndarray:
    v = np.asarray(v, dtype=np.float64)
    return v / np.sqrt((v * v).sum(1, keepdims=True))


def make_queries(nq: int, n: int, d: int, seed: int, dtype, data: str = "iso") -> torch.Tensor:
    """[nq, d] host queries in ``dtype`` over the corpus of seed ``seed``."""
    src = query_sources(nq, n, seed)
    rows = torch.arange(nq, dtype=torch.int64)
    u = _unit_np(int_rows(rows, d, seed ^ _QU_KEY).numpy())
    g = _unit_np(int_rows(rows, d, seed ^ _QG_KEY).numpy())
    srct = torch.as_tensor(src, dtype=torch.int64)
    c = rows_by_id(srct, d, seed, dtype, data).double().numpy()
    if data == "iso":
        far = g
    else:
        far = _unit_np(centers(cluster_of(srct, data), d, seed).numpy() + 0.3 * g)
    near = _unit_np(c + 0.5 * u)
    q = np.where((np.arange(nq) % 2 == 0)[:, None], near, far)
    return torch.from_numpy(q.astype(np.float32)).to(dtype)
