"""Multi-process (world_size 2, gloo, CPU) test of the sharded hot path's
plumbing: corpus sharding with global id offsets, the all-gather of per-shard
top-k keys, the query-sharded config stage and the per-slice k-way merge +
join.  The per-rank compute steps are injected as oracle functions (the CUDA
kernels need a B200); the result must equal the single-process oracle."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import config_oracle as co
from oracle import retrieval_oracle as ro
from paper_2412_10543_b200 import dist as rdist

K = 6
NQ, N, D = 37, 503, 16


def pack_keys(Dm, Im):
    d = np.asarray(Dm, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (d << np.uint64(32)) | np.asarray(Im, dtype=np.int64).astype(np.uint64)
    u[np.asarray(Im) < 0] = np.uint64(0xFFFFFFFFFFFFFFFF)
    return torch.from_numpy(u.view(np.int64).copy())


def unpack_keys(t):
    u = t.numpy().view(np.uint64)
    d = (u >> np.uint64(32)).astype(np.uint32).view(np.float32)
    i = (u & np.uint64(0xFFFFFFFF)).astype(np.int64)
    empty = u == np.uint64(0xFFFFFFFFFFFFFFFF)
    return np.where(empty, np.inf, d), np.where(empty, -1, i)


def data():
    rng = np.random.default_rng(0)
    corpus = rng.standard_normal((N, D)).astype(np.float32)
    queries = rng.standard_normal((NQ, D)).astype(np.float32)
    prof = np.stack([rng.integers(0, 2, NQ), rng.integers(0, 2, NQ), rng.integers(1, 11, NQ),
                     rng.integers(30, 100, NQ), rng.integers(100, 201, NQ)], 1)
    conf = np.where(rng.random(NQ) < 0.3, 0.6, 0.99)
    qlen = rng.integers(400, 2001, NQ)
    free = rng.integers(0, 4 * 10**9, NQ)
    return corpus, queries, prof, conf, qlen, free


P = co.SelectParams(chunk_size=1000, out_budget=10, max_chunks=K)


def oracle_ops(rank, world, corpus):
    r0, r1 = rdist.shard_range(N, rank, world)

    def search_keys(q, k):
        Dm, Im = ro.search_exact(q.numpy(), corpus[r0:r1], k)
        Im = np.where(Im >= 0, Im + r0, -1)
        return pack_keys(Dm.astype(np.float32), Im)

    def gate(profiles):
        pr, conf = profiles
        out, _ = co.gate_sequence([(bool(a), bool(b), int(c), int(d), int(e), float(f))
                                   for (a, b, c, d, e), f in zip(pr, conf)], max_chunks=K)
        return np.array([(*s, int(fb)) for s, fb in out])

    def select(spaces, profiles, qlen, free):
        pr, _ = profiles
        return np.array([co.select(tuple(int(x) for x in s[:5]), bool(p[1]), int(q), int(f), P)
                         for s, p, q, f in zip(spaces, pr, qlen, free)])

    def merge(flat_keys, nlists, k, list_stride, nq, configs):
        Ds, Is = [], []
        for l in range(nlists):
            chunk = flat_keys[l * list_stride: l * list_stride + nq * k].reshape(nq, k)
            d, i = unpack_keys(chunk)
            Ds.append(d)
            Is.append(i)
        Dm, Im = ro.merge_lists(Ds, Is, k)
        keep = np.where(configs[:, 4] < 2, configs[:, 1], 0)
        for r in range(nq):
            Im[r, keep[r]:] = -1
            Dm[r, keep[r]:] = np.inf
        return Dm, Im

    return rdist.ShardOps(search_keys, gate, select, merge)


class Sliceable:
    """(profiles, conf) pair that slices together (the ops see profile rows)."""

    def __init__(self, pr, conf):
        self.pr, self.conf = pr, conf

    def __getitem__(self, s):
        return (self.pr[s], self.conf[s])


class GlooPeer:
    """The PeerExchange protocol (begin / scatter / merge_slice) over gloo on
    CPU: the scatter's row routing is an all-to-all of the query slices, the
    owner's merge the oracle merge.  Exercises dist.py's "peer" branch, with
    and without a fused search_scatter op."""

    def __init__(self, world, k, merge):
        self.world, self.k, self.merge, self.epoch, self.pending = world, k, merge, 0, {}

    def begin(self):
        self.epoch += 1
        return self.epoch

    def scatter(self, keys, nq, epoch):
        sizes = [rdist.shard_range(nq, r, self.world)[1] - rdist.shard_range(nq, r, self.world)[0]
                 for r in range(self.world)]
        mine = sizes[dist.get_rank()]
        recv = torch.empty((mine * self.world, self.k), dtype=torch.int64)
        dist.all_to_all_single(recv, keys, output_split_sizes=[mine] * self.world, input_split_sizes=sizes)
        self.pending[epoch] = (recv.reshape(-1), mine)

    def merge_slice(self, nq, k, epoch, keep=None):
        flat, mine = self.pending.pop(epoch)
        return self.merge(flat, self.world, k, mine * k, mine, keep)


def worker(rank, world, port, out_q, exchange="all_to_all"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    corpus, queries, prof, conf, qlen, free = data()
    ops = oracle_ops(rank, world, corpus)
    # gate takes the whole batch; select/merge take the rank's slice
    ops_gate = ops.gate
    fused = None
    if exchange == "peer_fused":
        def fused(q, k, peer, epoch):
            peer.scatter(ops.search_keys(q, k), q.shape[0], epoch)
    ops = rdist.ShardOps(ops.search_keys, lambda p: ops_gate((p.pr, p.conf)), ops.select, ops.merge, fused)
    profiles = Sliceable(prof, conf)
    peer = GlooPeer(world, K, ops.merge) if exchange.startswith("peer") else None
    q0, q1, cfg, Dm, Im = rdist.sharded_retrieve_select(ops, torch.from_numpy(queries), profiles, qlen, free, K,
                                                        exchange="peer" if peer else exchange, peer=peer)
    out_q.put((rank, q0, q1, cfg, Dm, Im))
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 10_000_000):
        for w in (1, 2, 3, 8):
            ranges = [rdist.shard_range(n, r, w) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


@pytest.mark.timeout(300)
@pytest.mark.parametrize("exchange", ["all_to_all", "all_gather", "peer", "peer_fused"])
def test_two_rank_gloo_matches_single_process(exchange):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, q, exchange)) for r in range(2)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=240) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    corpus, queries, prof, conf, qlen, free = data()
    # single-process oracle pipeline over the whole corpus
    gated, _ = co.gate_sequence([(bool(a), bool(b), int(c), int(d), int(e), float(f))
                                 for (a, b, c, d, e), f in zip(prof, conf)], max_chunks=K)
    want_cfg = np.array([co.select(s, bool(p[1]), int(ql), int(fr), P)
                         for (s, _), p, ql, fr in zip(gated, prof, qlen, free)])
    Dfull, Ifull = ro.search_exact(queries, corpus, K)
    cfg = np.concatenate([r[3] for r in results])
    Im = np.concatenate([r[5] for r in results])
    assert [r[1:3] for r in results] == [rdist.shard_range(NQ, 0, 2), rdist.shard_range(NQ, 1, 2)]
    np.testing.assert_array_equal(cfg, want_cfg)
    for i in range(NQ):
        m = int(want_cfg[i, 1]) if want_cfg[i, 4] < 2 else 0
        np.testing.assert_array_equal(Im[i, :m], Ifull[i, :m])
        assert (Im[i, m:] == -1).all()
