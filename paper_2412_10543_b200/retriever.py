"""Dense chunk retrieval: a B200 ``IndexFlatL2`` (FAISS semantics).

The reference abstracts retrieval away; the paper retrieves with
FAISS ``IndexFlatL2`` + ``index.search(query_embedding, top_k)``
(PAPER.md:653, :709).  This class keeps that surface — ``add``, ``search``,
``ntotal``, ``reset`` — over one HBM-resident corpus shard owned by the
``rs_index`` handle of ``libragsched_b200.so``.  bf16 corpora run the fused
tcgen05/TMA/TMEM score + top-k kernel; fp32 corpora the CUDA-core kernel.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_DTYPES = {torch.bfloat16: _lib.RS_BF16, torch.float32: _lib.RS_F32}
ALGOS = {"auto": _lib.RS_ALGO_AUTO, "simt": _lib.RS_ALGO_SIMT, "tcgen05": _lib.RS_ALGO_TCGEN05,
         "tcgen05_1sm": _lib.RS_ALGO_TCGEN05_1SM}


class IndexFlatL2:
    """Exact squared-L2 index over one corpus shard.

    Args:
        d: embedding dimension.
        dtype: ``torch.bfloat16`` (tensor-core path) or ``torch.float32``.
        capacity: rows to preallocate in HBM (``add`` beyond it raises).
        device: CUDA device (default: current).
        id_base: global chunk id of this shard's row 0 (corpus sharding).
    """

    def __init__(self, d: int, dtype=torch.bfloat16, capacity: int = 1 << 20, device=None, id_base: int = 0):
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be torch.bfloat16 or torch.float32, got {dtype}")
        if not torch.cuda.is_available():
            raise _lib.LibraryUnavailable("IndexFlatL2 needs a CUDA (B200) device; there is no CPU fallback")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self._lib = _lib.lib_for_device(dev)
        self.d = int(d)
        self.dtype = dtype
        self.capacity = int(capacity)
        self.id_base = int(id_base)
        h = ctypes.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(self._lib.rs_index_create(self.d, _DTYPES[dtype], self.capacity, dev, ctypes.byref(h)),
                       "rs_index_create")
        self._h = h

    # -- FAISS-like surface ---------------------------------------------------
    @property
    def ntotal(self) -> int:
        v = ctypes.c_int64()
        _lib.check(self._lib.rs_index_ntotal(self._h, ctypes.byref(v)))
        return int(v.value)

    def _dev_tensor(self, x) -> torch.Tensor:
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        if x.dim() != 2 or x.shape[1] != self.d:
            raise ValueError(f"expected [n, {self.d}] embeddings, got {tuple(x.shape)}")
        return x.to(self.device, self.dtype).contiguous()

    def add(self, x, stream=None) -> None:
        """Append embeddings (copied into the index's HBM; norms on device)."""
        t = self._dev_tensor(x)
        _lib.check(self._lib.rs_index_add(self._h, _lib.ptr(t), t.shape[0], _lib.stream_ptr(stream)), "rs_index_add")
        # keep the source alive until the stream-ordered copy ran
        (stream or torch.cuda.current_stream()).synchronize()

    def reset(self) -> None:
        _lib.check(self._lib.rs_index_reset(self._h))

    def reserve(self, nq_max: int, k: int) -> None:
        _lib.check(self._lib.rs_index_reserve(self._h, int(nq_max), int(k)), "rs_index_reserve")

    def set_algo(self, algo: str) -> None:
        _lib.check(self._lib.rs_index_set_algo(self._h, ALGOS[algo]))

    def set_segment_rows(self, rows: int) -> None:
        """Tuning knob: corpus rows per segment of the CTA-pair schedule (0 = auto)."""
        _lib.check(self._lib.rs_index_set_segment_rows(self._h, int(rows)))

    def set_burst_merge(self, mode: str | int) -> None:
        """The pair kernel's cooperative burst merge: "auto" (default; the lean
        variant until searches report bursts — a document's consecutive chunks
        landing in one epilogue lane — then the cooperative one), "off"/0 or
        "on"/1.  Results are bit-identical in every mode."""
        m = {"auto": -1, "off": 0, "on": 1}.get(mode, mode)
        _lib.check(self._lib.rs_index_set_burst_merge(self._h, int(m)))

    def set_probe(self, mode: str | int) -> None:
        """The pair kernel's probe pass (a first launch over the corpus's first
        rows that seeds every query's admission bound; an experiment measured
        slower at cfg1): "off"/0 (default) or "on"/1.  Results are
        bit-identical either way."""
        m = {"off": 0, "on": 1}.get(mode, mode)
        _lib.check(self._lib.rs_index_set_probe(self._h, int(m)))

    def last_probe_rows(self) -> int:
        """Corpus rows the last search's probe pass scanned (0 = no probe)."""
        v = ctypes.c_int32(0)
        _lib.check(self._lib.rs_index_last_probe_rows(self._h, ctypes.byref(v)))
        return int(v.value)

    def burst_merge_active(self) -> bool:
        """Whether the next search runs the cooperative variant."""
        v = ctypes.c_int32(0)
        _lib.check(self._lib.rs_index_burst_merge_active(self._h, ctypes.byref(v)))
        return bool(v.value)

    def set_walk_bias(self, bias: int) -> None:
        """Test hook: start every pair-kernel unit past its segment frontier
        (exercises the wrap-around, out-of-id-order top-k path)."""
        _lib.check(self._lib.rs_index_set_walk_bias(self._h, int(bias)))

    def search(self, x, k: int, *, keep: torch.Tensor | None = None, out=None, stream=None):
        """k nearest chunks per query: (D float32 [nq,k], I int64 [nq,k]).

        Device tensors in -> device tensors out (stream-ordered, no sync);
        a numpy array in -> numpy arrays out (FAISS convention).  ``keep`` is an
        optional device rs_config batch: only the first ``num_chunks`` results
        of each selected query are returned (the retrieve-after-select join)."""
        host = isinstance(x, np.ndarray)
        q = self._dev_tensor(x)
        nq = q.shape[0]
        if out is None:
            D = torch.empty((nq, k), dtype=torch.float32, device=self.device)
            I = torch.empty((nq, k), dtype=torch.int64, device=self.device)
        else:
            D, I = out
        _lib.check(self._lib.rs_index_search(self._h, _lib.ptr(q), nq, int(k), self.id_base, _lib.ptr(keep),
                                             _lib.ptr(D), _lib.ptr(I), _lib.stream_ptr(stream)), "rs_index_search")
        if host:
            return D.cpu().numpy(), I.cpu().numpy()
        return D, I

    def search_keys(self, x: torch.Tensor, k: int, *, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """Sorted per-query top-k as packed uint64 keys (int64 tensor view):
        fp32 distance bits << 32 | global chunk id; all-ones = missing."""
        q = self._dev_tensor(x)
        keys = out if out is not None else torch.empty((q.shape[0], k), dtype=torch.int64, device=self.device)
        _lib.check(self._lib.rs_index_search_keys(self._h, _lib.ptr(q), q.shape[0], int(k), self.id_base,
                                                  _lib.ptr(keys), _lib.stream_ptr(stream)), "rs_index_search_keys")
        return keys

    def search_scatter(self, x: torch.Tensor, k: int, peer, epoch: int, *, stream=None) -> None:
        """``search_keys`` whose final merge stores each query's key row into
        its slice owner's peer region and signals ``epoch`` (``dist.PeerExchange``);
        the owners collect with ``PeerExchange.merge_slice``."""
        q = self._dev_tensor(x)
        _lib.check(self._lib.rs_index_search_scatter(self._h, _lib.ptr(q), q.shape[0], int(k), self.id_base,
                                                     ctypes.byref(peer.exchange_struct), int(epoch),
                                                     _lib.stream_ptr(stream)), "rs_index_search_scatter")

    def last_plan(self) -> dict:
        s, q, c, a = (ctypes.c_int32() for _ in range(4))
        _lib.check(self._lib.rs_index_last_plan(self._h, ctypes.byref(s), ctypes.byref(q), ctypes.byref(c),
                                                ctypes.byref(a)))
        return {"segments": s.value, "qtiles": q.value, "ctas": c.value,
                "algo": {v: k for k, v in ALGOS.items()}.get(a.value, "none")}

    def enable_timing(self, enable: bool = True) -> None:
        """Bracket the fused score kernel of every search with CUDA events."""
        _lib.check(self._lib.rs_index_enable_timing(self._h, int(enable)))

    def kernel_times_ms(self) -> list[float]:
        """Durations of the score kernels since the last call (streams synced)."""
        buf = (ctypes.c_float * 512)()
        cnt = ctypes.c_int32()
        _lib.check(self._lib.rs_index_kernel_times(self._h, buf, 512, ctypes.byref(cnt)), "rs_index_kernel_times")
        return [float(buf[i]) for i in range(cnt.value)]

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.rs_index_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def merge_topk(keys: torch.Tensor, nlists: int, k_in: int, list_stride: int, k: int, *,
               keep: torch.Tensor | None = None, nq: int | None = None, stream=None):
    """K2: k-way merge of sorted key lists (list l of query q at
    ``keys[l * list_stride + q * k_in]``) -> (D, I), optional join with ``keep``."""
    lib = _lib.lib_for_device(keys.device.index if keys.device.index is not None else torch.cuda.current_device())
    nq = nq if nq is not None else keys.shape[-2] if keys.dim() >= 2 else keys.numel() // (nlists * k_in)
    D = torch.empty((nq, k), dtype=torch.float32, device=keys.device)
    I = torch.empty((nq, k), dtype=torch.int64, device=keys.device)
    _lib.check(lib.rs_merge_topk(_lib.ptr(keys), nq, nlists, k_in, list_stride, k, _lib.ptr(keep), _lib.ptr(D),
                                 _lib.ptr(I), _lib.stream_ptr(stream)), "rs_merge_topk")
    return D, I


def keys_to_dist_ids(keys: torch.Tensor):
    """Decode packed keys (debug / tests)."""
    u = keys.to("cpu").numpy().view(np.uint64)
    d = (u >> np.uint64(32)).astype(np.uint32).view(np.float32)
    i = (u & np.uint64(0xFFFFFFFF)).astype(np.int64)
    empty = u == np.uint64(0xFFFFFFFFFFFFFFFF)
    d = np.where(empty, np.inf, d)
    i = np.where(empty, -1, i)
    return d, i
