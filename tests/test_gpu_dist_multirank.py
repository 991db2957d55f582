"""The sharded path with REAL ranks on the GPU: world_size 2 (and 3, uneven
slices) processes share cuda:0 over gloo (the pool gives one GPU per call;
the measured configuration is NCCL, one GPU per rank, same code).  Each rank
owns a corpus shard with global ids, runs the fused kernel, exchanges keys
(all-to-all, all-gather, or the library's peer-memory exchange through CUDA
IPC mappings — here of the same device), gates the batch, selects and merges
its query slice; the concatenated result must equal the single-index
pipeline, for three consecutive batches with the peer exchange (both of its
buffers and the epoch flags)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

NQ, N, D, K = 301, 40_003, 256, 35


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(nq=None):
    out = _all_inputs()
    return out if nq is None else (out[0], out[1][:nq], out[2][:nq], out[3][:nq], out[4][:nq])


def _all_inputs():
    g = torch.Generator().manual_seed(9)
    corpus = torch.nn.functional.normalize(torch.randn(N, D, generator=g), dim=1).bfloat16()
    queries = torch.nn.functional.normalize(torch.randn(NQ, D, generator=g), dim=1).bfloat16()
    rng = np.random.default_rng(3)
    from paper_2412_10543_b200 import batch

    prof = batch.profiles_from_arrays(rng.integers(0, 2, NQ), rng.integers(0, 2, NQ), rng.integers(1, 11, NQ),
                                      np.full(NQ, 40), np.full(NQ, 120), np.where(rng.random(NQ) < 0.2, 0.5, 0.99))
    qlen = rng.integers(400, 2001, NQ).astype(np.int32)
    free = rng.integers(0, 10**10, NQ).astype(np.int64)
    return corpus, queries, prof, qlen, free


def _worker(rank, world, port, exchange, q, nq, multi_device=False):
    import torch.distributed as dist

    from paper_2412_10543_b200 import IndexFlatL2, batch
    from paper_2412_10543_b200 import dist as rdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    # multi_device: the measured configuration — one GPU per rank over NCCL
    # (the peer exchange then stores over NVLink into the other GPUs' regions)
    devi = rank if multi_device else 0
    torch.cuda.set_device(devi)
    dist.init_process_group("nccl" if multi_device else "gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", devi)
    corpus, queries, prof, qlen, free = _inputs(nq)
    r0, r1 = rdist.shard_range(N, rank, world)
    ix = IndexFlatL2(D, capacity=r1 - r0, id_base=r0)
    ix.add(corpus[r0:r1].to(dev))
    params = batch.SelectParams(per_token_bytes=131072, chunk_size=1000, out_budget=10)
    peer = rdist.PeerExchange(nq, K, device=dev) if exchange == "peer" else None
    out = []
    for it in range(_iters(exchange)):  # the peer exchange alternates its two buffers
        ops = rdist.gpu_ops(ix, params, batch.GateWindow(dev))
        q0, q1, cfg, Dm, Im = rdist.sharded_retrieve_select(
            ops, queries.roll(it, 0).to(dev), batch.to_device(prof, dev), torch.as_tensor(qlen, device=dev),
            torch.as_tensor(free, device=dev), K, exchange=exchange, peer=peer)
        out.append((cfg.cpu().numpy(), Im.cpu().numpy()))
    torch.cuda.synchronize()
    if peer is not None:
        assert peer.error() == 0
        peer.close()
    q.put((rank, q0, q1, out))
    ix.close()
    dist.destroy_process_group()


def _iters(exchange):
    return 3 if exchange == "peer" else 1


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,exchange,nq", [(2, "all_to_all", NQ), (3, "all_to_all", NQ), (2, "all_gather", NQ),
                                               (2, "peer", NQ), (3, "peer", NQ), (3, "peer", 2)])
def test_multirank_sharded_path_equals_single_index(world, exchange, nq):
    _run_and_check(world, exchange, nq, multi_device=False)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("world,exchange", [(2, "peer"), (2, "all_to_all"), (2, "all_gather"), (4, "peer"),
                                            (8, "peer"), (8, "all_gather")])
def test_multidevice_nccl_sharded_path_equals_single_index(world, exchange):
    """Runs by itself on the first box with >= world GPUs: one rank per GPU
    over NCCL, the peer exchange's stores crossing NVLink/NVSwitch."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    _run_and_check(world, exchange, NQ, multi_device=True)


def _run_and_check(world, exchange, nq, multi_device):
    from paper_2412_10543_b200 import IndexFlatL2, batch
    from paper_2412_10543_b200.pipeline import RetrieveSelect

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, exchange, q, nq, multi_device)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=500) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    corpus, queries, prof, qlen, free = _inputs(nq)
    dev = torch.device("cuda", 0)
    ix = IndexFlatL2(D, capacity=N)
    ix.add(corpus.to(dev))
    params = batch.SelectParams(per_token_bytes=131072, chunk_size=1000, out_budget=10)
    assert [(r[1], r[2]) for r in res] == [(nq * i // world, nq * (i + 1) // world) for i in range(world)]
    for it in range(_iters(exchange)):
        ref = RetrieveSelect(ix, params).run(queries.roll(it, 0).to(dev), batch.to_device(prof, dev),
                                             torch.as_tensor(qlen, device=dev), torch.as_tensor(free, device=dev))
        torch.cuda.synchronize()
        cfg = np.concatenate([r[3][it][0] for r in res])
        Im = np.concatenate([r[3][it][1] for r in res])
        np.testing.assert_array_equal(batch.from_device(torch.from_numpy(cfg), batch.CONFIG_DTYPE),
                                      ref.configs_np())
        np.testing.assert_array_equal(Im, ref.chunk_ids.cpu().numpy())
    ix.close()
