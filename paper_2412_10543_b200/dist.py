"""Multi-GPU hot path: one process per GPU, ``torch.distributed`` (NCCL over
NVLink/NVSwitch) for the single exchange step.

* Corpus sharding: rank r owns rows [r*N/P, (r+1)*N/P) with global ids
  starting at ``id_base = r*N/P``; every rank scores ALL queries against its
  shard (fused score + top-k) -> sorted top-k keys [nq, k] with global ids.
* Exchange: ``all_to_all_single`` of the keys — rank r receives every
  shard's list for its own query slice only (nq*k*8/P bytes from each peer;
  2.3 MB out per rank at 8,192 x 35) — the only collective of the path
  (``all_gather_into_tensor`` of the full key matrices is kept as an option).
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

import torch
import torch.distributed as dist


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

    return ShardOps(search_keys, gate, select, merge)


def sharded_retrieve_select(ops: ShardOps, queries, profiles, qlen, free_bytes, k: int, *, group=None,
                            exchange: str = "all_to_all"):
    """One batch through the sharded path on this rank.  All inputs are the
    full batch (replicated); returns (q0, q1, configs, D, I) for this rank's
    query slice.

    ``exchange="all_to_all"`` (default): each rank sends the keys of query
    slice r to rank r only (``all_to_all_single``, nq*k*8 bytes out per rank,
    and in: the P lists of its own slice).  ``"all_gather"``: every rank
    receives every rank's full key matrix (P x more traffic)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nq = queries.shape[0]
    keys = ops.search_keys(queries, k).contiguous()                     # [nq, k] local shard
    q0, q1 = shard_range(nq, rank, world)
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
