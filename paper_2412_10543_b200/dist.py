"""Multi-GPU hot path: one process per GPU, ``torch.distributed`` (NCCL over
NVLink/NVSwitch) for the single exchange step.

* Corpus sharding: rank r owns rows [r*N/P, (r+1)*N/P) with global ids
  starting at ``id_base = r*N/P``; every rank scores ALL queries against its
  shard (fused score + top-k) -> sorted top-k keys [nq, k] with global ids.
* Exchange: rank r receives every shard's list for its own query slice only
  (nq*k*8/P bytes from each peer; 2.3 MB out per rank at 8,192 x 35) — the
  only collective of the path.  ``exchange="peer"``: ``PeerExchange``, the
  library's own NVLink exchange (``rs_peer_*``: a scatter kernel stores the
  key rows straight into the owners' CUDA-IPC-mapped regions and raises epoch
  flags; the owner's merge kernel waits on them in-kernel).
  ``"all_to_all"``: NCCL ``all_to_all_single``; ``"all_gather"``: every rank
  receives every full key matrix (P x more traffic).
* Query sharding of the config stage: rank r gates the whole batch (the gate
  is order-dependent and O(nq)), selects its own query slice [q0, q1) and
  runs the k-way merge (K2) of the P shard lists for that slice, joined with
  its configs.  Results stay sharded by query; ``gather_results`` collects them.

The per-rank kernels are injectable (``ShardOps``) so the distributed
plumbing is tested with world_size 2 over gloo on CPU against the oracle.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Callable

import ctypes

import torch
import torch.distributed as dist

from . import _lib


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced split: rank r gets [r*n//P, (r+1)*n//P)."""
    return (rank * n) // world, ((rank + 1) * n) // world


@dataclass
class ShardOps:
    """Per-rank compute steps (defaults: the CUDA library)."""

    search_keys: Callable      # (queries, k) -> int64 [nq, k] packed keys (global ids)
    gate: Callable             # (profiles) -> spaces (whole batch, in order)
    select: Callable           # (spaces, profiles, qlen, free) -> configs (query slice)
    merge: Callable            # (gathered_slice, nlists, k, list_stride, nq_slice, configs) -> (D, I)
    # (queries, k, peer, epoch) -> None: search whose final merge stores the key rows to the slice owners
    search_scatter: Callable | None = None


def gpu_ops(index, pipeline_params, window, *, threshold=0.90, default_space=None, cost=None) -> ShardOps:
    from . import batch as _b
    from .retriever import merge_topk

    def search_keys(q, k):
        return index.search_keys(q, k)

    def gate(profiles):
        return _b.prune_gate(profiles, window, threshold=threshold, default_space=default_space,
                             max_chunks=pipeline_params.max_chunks)

    def select(spaces, profiles, qlen, free):
        cfg, _ = _b.select(spaces, profiles, qlen, free, pipeline_params, cost=cost)
        return cfg

    def merge(keys_slice, nlists, k, list_stride, nq, configs):
        return merge_topk(keys_slice, nlists, k, list_stride, k, keep=configs, nq=nq)

    def search_scatter(q, k, peer, epoch):
        index.search_scatter(q, k, peer, epoch)

    return ShardOps(search_keys, gate, select, merge, search_scatter)


class PeerExchange:
    """Peer-memory exchange of the sharded search's key lists over NVLink
    (``rs_peer_*``, csrc/peer.cu).  Every rank allocates one region, shares its
    CUDA IPC handle through ``torch.distributed`` (plumbing only) and maps the
    others'.  ``merge(keys, nq, k, keep)`` scatters this rank's [nq, k_in] keys
    to the slice owners and returns the merged (D, I) of this rank's slice;
    both kernels run on the current stream, with no host synchronisation."""

    def __init__(self, nq_max: int, k_in: int, *, group=None, device=None, timeout_ms: int = 0):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.lib = _lib.lib_for_device(self.device.index)
        self.k_in, self.timeout_ms, self.epoch = int(k_in), int(timeout_ms), 0
        if self.world > _lib.PEER_MAX:
            raise ValueError(f"peer exchange supports at most {_lib.PEER_MAX} ranks")
        self.slice_cap = max(1, -(-int(nq_max) // self.world))
        nbytes = ctypes.c_uint64()
        _lib.check(self.lib.rs_peer_region_bytes(self.world, self.slice_cap, self.k_in, ctypes.byref(nbytes)))
        own = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(_lib.PEER_HANDLE_BYTES)
        _lib.check(self.lib.rs_peer_alloc(nbytes.value, self.device.index, ctypes.byref(own), handle),
                   "rs_peer_alloc")
        self._own = own.value
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=group)
        self._opened = []
        self._ex = _lib.PeerExchangeC(self.rank, self.world, self.k_in, 0, self.slice_cap)
        err = None
        try:
            for r, h in enumerate(handles):
                if r == self.rank:
                    self._ex.region[r] = self._own
                    continue
                p = ctypes.c_void_p()
                buf = ctypes.create_string_buffer(h, _lib.PEER_HANDLE_BYTES)
                _lib.check(self.lib.rs_peer_open(buf, self.device.index, ctypes.byref(p)), "rs_peer_open")
                self._opened.append(p.value)
                self._ex.region[r] = p.value
        except Exception as e:  # noqa: BLE001 - reported collectively below
            err = f"rank {self.rank}: {e}"
        # doubles as the barrier: every rank has mapped every region before the first store
        errs = [None] * self.world
        dist.all_gather_object(errs, err, group=group)
        errs = [e for e in errs if e]
        if errs:
            self.close()
            raise RuntimeError("peer exchange setup failed: " + "; ".join(errs))

    def slice(self, nq: int) -> tuple[int, int]:
        return shard_range(nq, self.rank, self.world)

    @property
    def exchange_struct(self) -> _lib.PeerExchangeC:
        return self._ex

    def begin(self) -> int:
        """Next epoch (one per exchanged batch)."""
        self.epoch = (self.epoch + 1) & 0xFFFFFFFF or 2  # skip 0 (initial flags), keep parity alternating
        return self.epoch

    def scatter(self, keys: torch.Tensor, nq: int, epoch: int, stream=None) -> None:
        """Store ``keys`` [nq, k_in] (this rank's shard, global ids) into the
        slice owners' regions and signal ``epoch``."""
        if keys.dtype != torch.int64 or keys.shape != (nq, self.k_in) or not keys.is_contiguous():
            raise ValueError(f"keys must be a contiguous int64 [{nq}, {self.k_in}] tensor")
        _lib.check(self.lib.rs_peer_scatter_keys(ctypes.byref(self._ex), _lib.ptr(keys), nq, epoch,
                                                 _lib.stream_ptr(stream)), "rs_peer_scatter_keys")

    def merge_slice(self, nq: int, k: int, epoch: int, keep: torch.Tensor | None = None, stream=None):
        """Wait for every source's rows of ``epoch`` and merge this rank's slice
        of the nq batch -> (D [slice, k] fp32, I [slice, k] int64)."""
        q0, q1 = self.slice(nq)
        D = torch.empty((q1 - q0, k), dtype=torch.float32, device=self.device)
        I = torch.empty((q1 - q0, k), dtype=torch.int64, device=self.device)
        _lib.check(self.lib.rs_peer_merge_topk(ctypes.byref(self._ex), nq, epoch, k, _lib.ptr(keep), _lib.ptr(D),
                                               _lib.ptr(I), self.timeout_ms, _lib.stream_ptr(stream)),
                   "rs_peer_merge_topk")
        return D, I

    def merge(self, keys: torch.Tensor, nq: int, k: int, keep: torch.Tensor | None = None, stream=None):
        """``scatter`` + ``merge_slice`` of one batch."""
        epoch = self.begin()
        self.scatter(keys, nq, epoch, stream)
        return self.merge_slice(nq, k, epoch, keep, stream)

    def check(self) -> None:
        """Raise if some merge of this exchange timed out waiting for a peer
        (then its rows were merged from a stale buffer).  Synchronous: call it
        at batch boundaries, or pass ``validate=True`` to
        ``sharded_retrieve_select``."""
        if self.error():
            raise RuntimeError(f"peer exchange rank {self.rank}: a merge timed out after {self.timeout_ms} ms "
                               "waiting for a peer's rows (results of that batch are invalid)")

    def error(self, clear: bool = False) -> int:
        """1 if some merge timed out waiting for a peer (synchronous read)."""
        out = ctypes.c_int32()
        _lib.check(self.lib.rs_peer_error(ctypes.byref(self._ex), int(clear), ctypes.byref(out)))
        return out.value

    def close(self, barrier: bool = True) -> None:
        if self._own is None:
            return
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            self.lib.rs_peer_close(p)
        self._opened = []
        if barrier:  # no peer may still store into our region
            dist.barrier(group=self.group)
        self.lib.rs_peer_free(self._own)
        self._own = None


def sharded_retrieve_select(ops: ShardOps, queries, profiles, qlen, free_bytes, k: int, *, group=None,
                            exchange: str = "all_to_all", peer: PeerExchange | None = None,
                            validate: bool = False):
    """One batch through the sharded path on this rank.  All inputs are the
    full batch (replicated); returns (q0, q1, configs, D, I) for this rank's
    query slice.

    ``exchange="all_to_all"`` (default): each rank sends the keys of query
    slice r to rank r only (``all_to_all_single``, nq*k*8 bytes out per rank,
    and in: the P lists of its own slice).  ``"all_gather"``: every rank
    receives every rank's full key matrix (P x more traffic).  ``"peer"``:
    the same traffic as all_to_all through ``peer`` (a ``PeerExchange``),
    stored by the library's kernels over NVLink, merged in the waiting
    kernel.  ``validate=True`` (peer only) synchronises after the merge and
    raises if it timed out waiting for a peer (``PeerExchange.check``); else
    check ``peer.error()`` at batch boundaries."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nq = queries.shape[0]
    q0, q1 = shard_range(nq, rank, world)
    if exchange == "peer":
        if peer is None:
            raise ValueError('exchange="peer" needs a PeerExchange')
        epoch = peer.begin()
        if ops.search_scatter is not None:   # the search's final merge stores to the owners
            ops.search_scatter(queries, k, peer, epoch)
        else:
            peer.scatter(ops.search_keys(queries, k).contiguous(), nq, epoch)
        spaces = ops.gate(profiles)
        configs = ops.select(spaces[q0:q1], profiles[q0:q1], qlen[q0:q1], free_bytes[q0:q1])
        D, I = peer.merge_slice(nq, k, epoch, keep=configs)
        if validate:
            peer.check()
        return q0, q1, configs, D, I
    keys = ops.search_keys(queries, k).contiguous()                     # [nq, k] local shard
    if exchange == "all_to_all":
        sizes = [shard_range(nq, r, world)[1] - shard_range(nq, r, world)[0] for r in range(world)]
        recv = torch.empty(((q1 - q0) * world, k), dtype=keys.dtype, device=keys.device)  # source-rank-major
        dist.all_to_all_single(recv, keys, output_split_sizes=[q1 - q0] * world, input_split_sizes=sizes,
                               group=group)
        flat, stride = recv.reshape(-1), (q1 - q0) * k                  # list l of query q at l*nq_slice*k + (q-q0)*k
    elif exchange == "all_gather":
        gathered = torch.empty((world * nq, k), dtype=keys.dtype, device=keys.device)  # rank-major
        dist.all_gather_into_tensor(gathered, keys, group=group)
        flat, stride = gathered.reshape(-1)[q0 * k:], nq * k            # list l of query q at l*nq*k + (q-q0)*k
    else:
        raise ValueError(f"unknown exchange {exchange!r}")
    spaces = ops.gate(profiles)                                         # full batch, in order
    configs = ops.select(spaces[q0:q1], profiles[q0:q1], qlen[q0:q1], free_bytes[q0:q1])
    D, I = ops.merge(flat, world, k, stride, q1 - q0, configs)
    return q0, q1, configs, D, I


def init_from_env(backend: str | None = None):
    """torchrun-style init (RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT)."""
    if dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world == 1:
        return 0, 1
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("RS_BENCH_DEVICE", os.environ.get("LOCAL_RANK", rank))))
    dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world
