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
        self._host = None

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

    def submit_host(self, queries: torch.Tensor, profiles: np.ndarray | torch.Tensor, qlen: torch.Tensor,
                    free_bytes: torch.Tensor) -> "HostTicket":
        """Asynchronous end-to-end call with HOST inputs (pinned for overlap).

        The H2D copies run on a copy stream, the pipeline on the current stream
        and the D2H copies of the configs and joined chunk ids on a second copy
        stream, through a ring of ``HOST_DEPTH`` slots: while batch i computes,
        batch i+1's inputs upload and batch i-1's results download.  Returns a
        ticket; ``ticket.wait()`` gives the pinned host outputs, valid until the
        slot is reused ``HOST_DEPTH`` submits later (submit blocks on that)."""
        if self._host is None:
            self._host = _HostRing(self.device, HOST_DEPTH)
        if isinstance(profiles, np.ndarray):
            profiles = torch.from_numpy(profiles.view(np.uint8).reshape(len(profiles), 16))
        ring = self._host
        slot = ring.acquire()
        q, p, ql, fr = slot.upload(ring.h2d, (queries, profiles, qlen, free_bytes))
        main = torch.cuda.current_stream(self.device)
        main.wait_event(slot.uploaded)
        res = self.run(q, p, ql, fr)
        return slot.download(ring.d2h, main, {"configs": res.configs, "chunk_ids": res.chunk_ids})

    def run_host(self, queries: torch.Tensor, profiles: np.ndarray | torch.Tensor, qlen: torch.Tensor,
                 free_bytes: torch.Tensor) -> dict:
        """Synchronous end-to-end call with HOST inputs: H2D copies, the
        device pipeline, and D2H of the configs and the joined chunk ids."""
        return self.submit_host(queries, profiles, qlen, free_bytes).wait()

    def host_stream(self, queries, profiles, qlen, free_bytes) -> "HostStream":
        """A repeated host batch through ``submit_host`` (the e2e benchmark)."""
        return HostStream(lambda: self.submit_host(queries, profiles, qlen, free_bytes))


HOST_DEPTH = 2


class HostTicket:
    """One submitted host batch: ``wait()`` blocks until its outputs are on the host."""

    def __init__(self, event: torch.cuda.Event, out: dict):
        self.event, self.out = event, out

    def wait(self) -> dict:
        self.event.synchronize()
        return self.out


class _Slot:
    def __init__(self):
        self.inputs, self.outputs, self.ticket, self.uploaded = None, {}, None, None

    def upload(self, h2d: torch.cuda.Stream, host: tuple) -> tuple:
        dev = h2d.device
        if self.inputs is None or any(a.shape != b.shape or a.dtype != b.dtype for a, b in zip(self.inputs, host)):
            self.inputs = tuple(torch.empty(t.shape, dtype=t.dtype, device=dev) for t in host)
        with torch.cuda.stream(h2d):
            for dst, src in zip(self.inputs, host):
                dst.copy_(src, non_blocking=True)
            self.uploaded = h2d.record_event()
        return self.inputs

    def download(self, d2h: torch.cuda.Stream, producer: torch.cuda.Stream, results: dict) -> HostTicket:
        d2h.wait_event(producer.record_event())
        with torch.cuda.stream(d2h):
            for name, t in results.items():
                dst = self.outputs.get(name)
                if dst is None or dst.shape != t.shape or dst.dtype != t.dtype:
                    dst = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                    self.outputs[name] = dst
                t.record_stream(d2h)
                dst.copy_(t, non_blocking=True)
            self.ticket = HostTicket(d2h.record_event(), dict(self.outputs))
        return self.ticket


class _HostRing:
    """Slots of device input buffers + pinned output buffers, and the two copy streams."""

    def __init__(self, device, depth: int):
        self.h2d = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self.slots = [_Slot() for _ in range(depth)]
        self.next = 0

    def acquire(self) -> _Slot:
        slot = self.slots[self.next]
        self.next = (self.next + 1) % len(self.slots)
        if slot.ticket is not None:
            # its D2H finished => the compute that read its device inputs finished too
            slot.ticket.event.synchronize()
        return slot


class HostStream:
    """``run(steps)``: submit the same host batch ``steps`` times, wait for the last."""

    def __init__(self, submit):
        self.submit = submit

    def run(self, steps: int) -> dict | None:
        t = None
        for _ in range(steps):
            t = self.submit()
        return t.wait() if t is not None else None


class SelectHostStream(HostStream):
    """The config path alone (cfg5) end to end with host inputs: H2D of
    (spaces, profiles, qlen, free), ``batch.select`` with delays, D2H of the
    configs and delays, pipelined like ``RetrieveSelect.submit_host``."""

    def __init__(self, host_inputs, params: _b.SelectParams, *, cost: _b.CostModel | None = None, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ring = _HostRing(self.device, HOST_DEPTH)
        self.host_inputs, self.params, self.cost = tuple(host_inputs), params, cost
        super().__init__(self._submit)

    def _submit(self) -> HostTicket:
        slot = self.ring.acquire()
        sp, pr, ql, fr = slot.upload(self.ring.h2d, self.host_inputs)
        main = torch.cuda.current_stream(self.device)
        main.wait_event(slot.uploaded)
        cfg, delay = _b.select(sp, pr, ql, fr, self.params, cost=self.cost)
        res = {"configs": cfg}
        if delay is not None:
            res["delay"] = delay
        return slot.download(self.ring.d2h, main, res)


class FnHostStream(HostStream):
    """Any device pipeline end to end with host inputs, pipelined like
    ``RetrieveSelect.submit_host``: ``fn(*device_inputs)`` runs on the current
    stream and returns a dict of device outputs, which are copied back to
    pinned host buffers.  The sharded multi-GPU pipeline (``dist``) uses it
    for its end-to-end numbers."""

    def __init__(self, fn, host_inputs, *, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ring = _HostRing(self.device, HOST_DEPTH)
        self.fn, self.host_inputs = fn, tuple(host_inputs)
        super().__init__(self._submit)

    def _submit(self) -> HostTicket:
        slot = self.ring.acquire()
        ins = slot.upload(self.ring.h2d, self.host_inputs)
        main = torch.cuda.current_stream(self.device)
        main.wait_event(slot.uploaded)
        return slot.download(self.ring.d2h, main, self.fn(*ins))
