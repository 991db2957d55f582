"""One-query calls of the C ABI at the lowest latency the GPU allows.

The reference-facing scalar functions (``best_fit_select``,
``fallback_config``, ``gate_profile`` / ``map_profile``, ``plan_bytes``,
``call_latency``) get one query per call.  A batch API round trip (allocate
device tensors, copy each argument H2D, launch, copy D2H) costs several
synchronous copies per call; here the arguments and results live in ONE
pinned host block that the kernels read and write directly (pinned host
memory is device-accessible under unified addressing), so a call is: fill
the block from Python, one launch on a private stream, one stream
synchronize, read the block.  Same kernels, same results as the batch path.
"""

from __future__ import annotations

import ctypes
import struct
import threading

import numpy as np
import torch

from . import _lib
from ._lib import CONFIG_DTYPE, PROFILE_DTYPE, SPACE_DTYPE, WINDOW_DTYPE

# byte offsets inside the pinned block
_SPACE, _PROFILE, _QLEN, _FREE, _CONFIG, _WINDOW, _OUTSPACE = 0, 16, 32, 40, 48, 64, 240
_LAT_IN, _LAT_OUT, _PB_IN, _PB_OUT = 256, 280, 288, 312
_BLOCK = 512
# struct layouts of the records written per call (PROFILE_DTYPE, SPACE_DTYPE, WINDOW_DTYPE in _lib)
_PROFILE_FMT, _SPACE_FMT = "<BBHHHd", "<HHHHHHI"
_SPACE_BYTES = struct.calcsize(_SPACE_FMT)
_WINDOW_LEN = WINDOW_DTYPE.fields["len"][1]
assert struct.calcsize(_PROFILE_FMT) == PROFILE_DTYPE.itemsize and _SPACE_BYTES == SPACE_DTYPE.itemsize


class _Ctx:
    def __init__(self, device: int):
        self.device = device
        self.lib = _lib.lib_for_device(device)
        with torch.cuda.device(device):
            self.stream = torch.cuda.Stream(device=device)
            self.block = torch.zeros(_BLOCK, dtype=torch.uint8, pin_memory=True)
            self.ws = torch.empty(max(int(self.lib.rs_prune_gate_workspace_size(1)), 1), dtype=torch.uint8,
                                  device=torch.device("cuda", device))
        self.base = int(self.block.data_ptr())
        self.buf = self.block.numpy()
        v = lambda off, dt, n=1: self.buf[off:off + dt.itemsize * n].view(dt)  # noqa: E731
        self.space = v(_SPACE, SPACE_DTYPE)
        self.profile = v(_PROFILE, PROFILE_DTYPE)
        self.qlen = v(_QLEN, np.dtype("<i4"))
        self.free = v(_FREE, np.dtype("<i8"))
        self.config = v(_CONFIG, CONFIG_DTYPE)
        self.window = v(_WINDOW, WINDOW_DTYPE)
        self.outspace = v(_OUTSPACE, SPACE_DTYPE)
        self.lat_in = v(_LAT_IN, np.dtype("<i8"), 3)
        self.lat_out = v(_LAT_OUT, np.dtype("<f8"))
        self.pb_in = v(_PB_IN, np.dtype("<i4"), 4)   # method, num_chunks, interlen, qlen
        self.pb_out = v(_PB_OUT, np.dtype("<i8"))
        self.sptr = int(self.stream.cuda_stream)
        self.mv = memoryview(self.buf)  # struct.pack_into / unpack_from: cheaper than numpy setitem per call
        self.many, self.many_np, self.many_cap = None, None, 0  # call_latency_many's pinned arrays
        self._lat_fn = self.lib.rs_call_latency
        self._lat_args = (self.p(_LAT_IN), self.p(_LAT_IN + 8), self.p(_LAT_IN + 16), 1)
        self._pb_fn = self.lib.rs_plan_bytes
        self._pb_args = (self.p(_PB_IN), self.p(_PB_IN + 4), self.p(_PB_IN + 8), self.p(_PB_IN + 12), 1)

    def p(self, off: int) -> int:
        return self.base + off

    def sync(self):
        self.stream.synchronize()


_ctx: dict[int, _Ctx] = {}
_lock = threading.Lock()


def ctx() -> _Ctx:
    dev = torch.cuda.current_device() if _ctx else None  # no context yet: check the device first
    c = _ctx.get(dev) if dev is not None else None
    if c is None:
        # (torch.cuda.is_available() costs ~4 us: checked once per device context, not per call)
        if not torch.cuda.is_available():
            raise _lib.LibraryUnavailable("no CUDA device: paper_2412_10543_b200 runs only on a B200 (no CPU fallback)")
        dev = torch.cuda.current_device()
        with _lock:
            c = _ctx.get(dev) or _Ctx(dev)
            _ctx[dev] = c
    return c


def select_one(space: tuple | None, profile: tuple | None, qlen: int, free_bytes: int,
               params: _lib.SelectParamsC) -> np.void:
    """rs_select for one query.  ``space`` = (methods, n_lo, n_hi, il_lo,
    il_hi) or None (no candidates: straight to the fallback); ``profile`` =
    an rs_profile tuple or None.  Returns the rs_config record (a copy)."""
    c = ctx()
    with _lock:
        c.space[0] = (*space, 0, 0) if space is not None else (0, 0, 0, 0, 0, 0, 0)
        if profile is not None:
            c.profile[0] = profile
        c.qlen[0] = qlen
        c.free[0] = free_bytes
        _lib.check(c.lib.rs_select(c.p(_SPACE), c.p(_PROFILE) if profile is not None else 0, c.p(_QLEN),
                                   c.p(_FREE), 1, ctypes.byref(params), None, 0, 0, c.p(_CONFIG), c.sptr),
                   "rs_select")
        c.sync()
        return c.config[0].copy()


def gate_one(profile: tuple, window_spaces: list, gate_params: _lib.GateParamsC) -> np.void:
    """rs_prune_gate for one profile against a window of <= 10 space tuples.
    Returns the rs_space record as a tuple (methods, num_chunks_lo,
    num_chunks_hi, interlen_lo, interlen_hi, gate_fallback)."""
    c = ctx()
    with _lock:
        struct.pack_into(_PROFILE_FMT, c.mv, _PROFILE, *profile)
        n = len(window_spaces)
        for i, s in enumerate(window_spaces):
            struct.pack_into(_SPACE_FMT, c.mv, _WINDOW + i * _SPACE_BYTES, *s, 0, 0)
        struct.pack_into("<i", c.mv, _WINDOW + _WINDOW_LEN, n)
        _lib.check(c.lib.rs_prune_gate(c.p(_PROFILE), 1, ctypes.byref(gate_params), c.p(_WINDOW), c.p(_OUTSPACE),
                                       int(c.ws.data_ptr()), c.ws.numel(), c.sptr), "rs_prune_gate")
        c.stream.synchronize()
        return struct.unpack_from(_SPACE_FMT, c.mv, _OUTSPACE)[:6]


def call_latency_one(prompt_tokens: int, max_output_tokens: int, concurrent: int, cost: _lib.CostModelC) -> float:
    c = ctx()
    with _lock:
        struct.pack_into("<qqq", c.mv, _LAT_IN, prompt_tokens, max_output_tokens, concurrent)
        rc = c._lat_fn(*c._lat_args, ctypes.byref(cost), c.p(_LAT_OUT), c.sptr)
        if rc:
            _lib.check(rc, "rs_call_latency")
        c.stream.synchronize()
        return struct.unpack_from("<d", c.mv, _LAT_OUT)[0]


def call_latency_many(prompt_tokens: list, max_output_tokens: list, concurrent: list,
                      cost: _lib.CostModelC) -> list:
    """rs_call_latency over a small batch through pinned, device-mapped
    arrays: one launch + one synchronize for all of them."""
    c = ctx()
    n = len(prompt_tokens)
    with _lock:
        if c.many_cap < n:
            cap = max(n, 2 * c.many_cap, 64)
            c.many = torch.zeros((4, cap), dtype=torch.int64, pin_memory=True)  # prompt, out, concurrency, latency
            c.many_np = c.many.numpy()
            c.many_cap = cap
        a = c.many_np
        a[0, :n] = prompt_tokens
        a[1, :n] = max_output_tokens
        a[2, :n] = concurrent
        base, row = int(c.many.data_ptr()), 8 * c.many_cap
        rc = c._lat_fn(base, base + row, base + 2 * row, n, ctypes.byref(cost), base + 3 * row, c.sptr)
        if rc:
            _lib.check(rc, "rs_call_latency")
        c.stream.synchronize()
        return a[3, :n].view(np.float64).tolist()


def plan_bytes_one(method: int, num_chunks: int, interlen: int, qlen: int, params: _lib.SelectParamsC) -> int:
    c = ctx()
    with _lock:
        struct.pack_into("<iiii", c.mv, _PB_IN, method, num_chunks, interlen, qlen)
        rc = c._pb_fn(*c._pb_args, ctypes.byref(params), c.p(_PB_OUT), c.sptr)
        if rc:
            _lib.check(rc, "rs_plan_bytes")
        c.stream.synchronize()
        return struct.unpack_from("<q", c.mv, _PB_OUT)[0]


class AdmitArena:
    """Pinned, device-mapped buffers of one Scheduler's admission launches
    (``rs_admit_fifo`` over a chunk of the waiting queue, then
    ``rs_plan_calls`` over the admitted configs): the kernels read the packed
    queue entries and write their results straight into host memory, so a
    chunk costs two launch + synchronize round trips and no copies."""

    def __init__(self, cap: int = 32, calls_per_plan: int = 36):
        self.c = ctx()
        self.cap = 0
        self.calls_per_plan = calls_per_plan  # map_reduce: num_chunks + 1 calls
        self._grow(cap)

    def _grow(self, cap: int):
        dev = torch.device("cuda", self.c.device)
        pin = lambda shape, dt: torch.zeros(shape, dtype=dt, pin_memory=True)  # noqa: E731
        self.cap = cap
        self.t_spaces, self.t_profiles = pin((cap, 16), torch.uint8), pin((cap, 16), torch.uint8)
        self.t_hasprof, self.t_qlen = pin(cap, torch.uint8), pin(cap, torch.int32)
        self.t_configs, self.t_info, self.t_result = pin((cap, 16), torch.uint8), pin((cap, 16), torch.uint8), \
            pin(24, torch.uint8)
        self.t_offsets, self.t_totals, self.t_status = pin(cap + 1, torch.int64), pin(cap, torch.int64), \
            pin(cap, torch.uint8)
        self._grow_calls(cap * self.calls_per_plan)
        self.ws = torch.empty(max(int(self.c.lib.rs_plan_calls_workspace_size(cap)), 1), dtype=torch.uint8,
                              device=dev)
        self.spaces = self.t_spaces.numpy()
        self.profiles = self.t_profiles.numpy()
        self.hasprof = self.t_hasprof.numpy()
        self.qlen = self.t_qlen.numpy()
        self.configs = self.t_configs.numpy().reshape(-1).view(CONFIG_DTYPE)
        self.info = self.t_info.numpy().reshape(-1).view(_lib.ADMIT_INFO_DTYPE)
        self.result = self.t_result.numpy().view(_lib.ADMIT_RESULT_DTYPE)
        self.offsets = self.t_offsets.numpy()
        self.totals = self.t_totals.numpy()
        self.status = self.t_status.numpy()

    def _grow_calls(self, n: int):
        self.calls_cap = n
        self.t_calls = torch.zeros((n, 24), dtype=torch.uint8, pin_memory=True)
        self.calls = self.t_calls.numpy().reshape(-1).view(_lib.CALL_DTYPE)

    def ensure(self, n: int):
        if n > self.cap:
            self._grow(max(n, 2 * self.cap))

    def admit(self, n: int, params: _lib.SelectParamsC, capacity: int, used: int, max_ctx: int) -> tuple[int, int]:
        """rs_admit_fifo over entries [0, n) (filled by the caller).  Returns
        (admitted, stop)."""
        c = self.c
        ap = _lib.AdmitParamsC(int(capacity), int(used), int(max_ctx))
        p = lambda t: int(t.data_ptr())  # noqa: E731
        _lib.check(c.lib.rs_admit_fifo(p(self.t_spaces), p(self.t_profiles), p(self.t_hasprof), p(self.t_qlen), n,
                                       ctypes.byref(params), ctypes.byref(ap), p(self.t_configs), p(self.t_info),
                                       p(self.t_result), c.sptr), "rs_admit_fifo")
        c.sync()
        r = self.result[0]
        return int(r["admitted"]), int(r["stop"])

    def admit_and_plan(self, n: int, params: _lib.SelectParamsC, capacity: int, used: int, max_ctx: int):
        """rs_admit_fifo over entries [0, n), then rs_plan_calls (count and
        fill) over all n configs, in stream order with ONE synchronize: the
        entries the chain did not reach are pre-marked MustQueue (no calls),
        and the calls buffer holds max_chunks + 1 calls per entry.  Returns
        (admitted, stop, (offsets [m+1], calls, totals [m], status [m]))."""
        c = self.c
        need = n * (int(params.max_chunks) + 1)
        if need > self.calls_cap:
            self._grow_calls(need)
        self.configs[:n] = np.zeros(1, dtype=CONFIG_DTYPE)
        self.configs["status"][:n] = _lib.RS_SELECT_MUST_QUEUE
        ap = _lib.AdmitParamsC(int(capacity), int(used), int(max_ctx))
        p = lambda t: int(t.data_ptr())  # noqa: E731
        pp = ctypes.byref(params)
        _lib.check(c.lib.rs_admit_fifo(p(self.t_spaces), p(self.t_profiles), p(self.t_hasprof), p(self.t_qlen), n,
                                       pp, ctypes.byref(ap), p(self.t_configs), p(self.t_info), p(self.t_result),
                                       c.sptr), "rs_admit_fifo")
        args = (p(self.t_configs), p(self.t_qlen), n, pp, int(max_ctx), p(self.t_offsets))
        ws = (int(self.ws.data_ptr()), self.ws.numel(), c.sptr)
        _lib.check(c.lib.rs_plan_calls(*args, 0, 0, p(self.t_status), *ws), "rs_plan_calls(count)")
        _lib.check(c.lib.rs_plan_calls(*args, p(self.t_calls), p(self.t_totals), 0, *ws), "rs_plan_calls(fill)")
        c.stream.synchronize()
        r = self.result[0]
        m = int(r["admitted"])
        return m, int(r["stop"]), (self.offsets[:m + 1], self.calls, self.totals[:m], self.status[:m])

    def plan_calls(self, m: int, params: _lib.SelectParamsC, max_ctx: int):
        """rs_plan_calls over the first m configs: the count pass, then (after
        sizing) the fill pass.  Returns numpy views (offsets [m+1], calls,
        totals [m], status [m])."""
        c = self.c
        p = lambda t: int(t.data_ptr())  # noqa: E731
        args = (p(self.t_configs), p(self.t_qlen), m, ctypes.byref(params), int(max_ctx), p(self.t_offsets))
        _lib.check(c.lib.rs_plan_calls(*args, 0, 0, p(self.t_status), int(self.ws.data_ptr()), self.ws.numel(),
                                       c.sptr), "rs_plan_calls(count)")
        # a plan has at most max_chunks + 1 calls (map_reduce): when the buffer
        # holds that for every config, the fill follows the count in stream
        # order with no round trip in between
        if m * (int(params.max_chunks) + 1) > self.calls_cap:
            c.sync()
            if int(self.offsets[m]) > self.calls_cap:
                self._grow_calls(int(self.offsets[m]))
        _lib.check(c.lib.rs_plan_calls(*args, p(self.t_calls), p(self.t_totals), 0, int(self.ws.data_ptr()),
                                       self.ws.numel(), c.sptr), "rs_plan_calls(fill)")
        c.sync()
        return self.offsets[:m + 1], self.calls, self.totals[:m], self.status[:m]
