"""The per-query hot path end to end on one GPU: confidence gate + pruning,
best-fit / fallback selection with the cost models, dense retrieval, and the
join "retrieve the selected number of chunks".

Selection never looks at chunk content (it needs only the profile, the query
length and the free KV bytes; scheduler.py:127-191), and top-``num_chunks`` of
a sorted top-``k_max`` list is its prefix, so the config path runs on a side
stream concurrently with the retrieval GEMM and the two meet in a last merge
pass that truncates each query's list to its chosen ``num_chunks``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import batch as _b
from ._lib import CONFIG_DTYPE, SPACE_DTYPE
from .retriever import IndexFlatL2, merge_topk


@dataclass
class BatchResult:
    configs: torch.Tensor        # uint8 [n,16] rs_config
    spaces: torch.Tensor         # uint8 [n,16] rs_space (gate output)
    distances: torch.Tensor      # float32 [n,k]; +inf past num_chunks
    chunk_ids: torch.Tensor      # int64 [n,k];  -1 past num_chunks
    delay: torch.Tensor | None   # float64 [n] plan delay (if a cost model is set)

    def configs_np(self) -> np.ndarray:
        return _b.from_device(self.configs, CONFIG_DTYPE)

    def spaces_np(self) -> np.ndarray:
        return _b.from_device(self.spaces, SPACE_DTYPE)


class RetrieveSelect:
    """Batched retrieve + config-select over one corpus shard.

    Args:
        index: the corpus (``IndexFlatL2``).
        params: selection scalars (``batch.SelectParams``).
        k: results retrieved per query (default ``params.max_chunks``, the
           largest chunk count any selected config can ask for).
        threshold / default_space: gate parameters (profiler.py:467-477).
        cost: optional ``batch.CostModel``; adds the plan delay per query.
    """

    def __init__(self, index: IndexFlatL2, params: _b.SelectParams, *, k: int | None = None,
                 threshold: float = _b.GATE_THRESHOLD, default_space=None, cost: _b.CostModel | None = None):
        self.index = index
        self.params = params
        self.k = int(k or params.max_chunks)
        self.threshold = threshold
        self.default_space = default_space
        self.cost = cost
        self.device = index.device
        self.window = _b.GateWindow(self.device)
        self.side = torch.cuda.Stream(device=self.device)
        self._ws = None

    def run(self, queries: torch.Tensor, profiles: torch.Tensor, qlen: torch.Tensor, free_bytes: torch.Tensor,
            running_before: torch.Tensor | None = None) -> BatchResult:
        """Device-resident batch in, device results out (stream-ordered on the
        current stream; nothing synchronises the host)."""
        main = torch.cuda.current_stream(self.device)
        ready = main.record_event()
        self.side.wait_event(ready)
        n = profiles.shape[0]
        with torch.cuda.stream(self.side):
            ws_need = int(_b._lib.load().rs_prune_gate_workspace_size(n))
            if self._ws is None or self._ws.numel() < ws_need:
                self._ws = torch.empty(max(ws_need, 1), dtype=torch.uint8, device=self.device)
            spaces = _b.prune_gate(profiles, self.window, threshold=self.threshold,
                                   default_space=self.default_space, max_chunks=self.params.max_chunks,
                                   workspace=self._ws, stream=self.side)
            configs, delay = _b.select(spaces, profiles, qlen, free_bytes, self.params, cost=self.cost,
                                       running_before=running_before, stream=self.side)
        selected = self.side.record_event()
        keys = self.index.search_keys(queries, self.k, stream=main)
        main.wait_event(selected)
        D, I = merge_topk(keys, 1, self.k, n * self.k, self.k, keep=configs, nq=n, stream=main)
        for t in (spaces, configs, delay):
            if t is not None:
                t.record_stream(main)
        return BatchResult(configs, spaces, D, I, delay)

    def run_host(self, queries: torch.Tensor, profiles: np.ndarray | torch.Tensor, qlen: torch.Tensor,
                 free_bytes: torch.Tensor, *, pinned_out: dict | None = None) -> dict:
        """End-to-end call with HOST inputs (ideally pinned): H2D copies, the
        device pipeline, and D2H of the configs and the joined chunk ids."""
        dev = self.device
        if isinstance(profiles, np.ndarray):
            profiles = torch.from_numpy(profiles.view(np.uint8).reshape(len(profiles), 16))
        q = queries.to(dev, non_blocking=True)
        p = profiles.to(dev, non_blocking=True)
        ql = qlen.to(dev, non_blocking=True)
        fr = free_bytes.to(dev, non_blocking=True)
        res = self.run(q, p, ql, fr)
        out = pinned_out or {}
        for name, t in (("configs", res.configs), ("chunk_ids", res.chunk_ids)):
            dst = out.get(name)
            if dst is None or dst.shape != t.shape:
                dst = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                out[name] = dst
            dst.copy_(t, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        return out
