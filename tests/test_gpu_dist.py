"""The sharded path's GPU ops (fused search on a shard with global ids, the
NCCL all-to-all (or all-gather) exchange, query-slice select, k-way merge + join) on one B200: a
single-rank NCCL group runs the exact code bench.py runs per rank under
torchrun, and must equal the single-index pipeline."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2412_10543_b200 import IndexFlatL2, batch
from paper_2412_10543_b200 import dist as rdist
from paper_2412_10543_b200.pipeline import RetrieveSelect

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    if not dist.is_initialized():
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(_port())
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("exchange", ["all_to_all", "all_gather"])
def test_sharded_path_equals_single_index(nccl_group, exchange):
    dev = torch.device("cuda", 0)
    nq, n, d, k = 500, 30_000, 256, 35
    g = torch.Generator().manual_seed(4)
    corpus = torch.nn.functional.normalize(torch.randn(n, d, generator=g), dim=1).bfloat16()
    queries = torch.nn.functional.normalize(torch.randn(nq, d, generator=g), dim=1).bfloat16().to(dev)
    rng = np.random.default_rng(1)
    prof = batch.profiles_from_arrays(rng.integers(0, 2, nq), rng.integers(0, 2, nq), rng.integers(1, 11, nq),
                                      np.full(nq, 40), np.full(nq, 120), np.where(rng.random(nq) < 0.2, 0.5, 0.99))
    profiles = batch.to_device(prof, dev)
    qlen = torch.as_tensor(rng.integers(400, 2001, nq).astype(np.int32), device=dev)
    free = torch.as_tensor(rng.integers(0, 10**10, nq).astype(np.int64), device=dev)
    params = batch.SelectParams(per_token_bytes=131072, chunk_size=1000, out_budget=10)

    # shard = the whole corpus, offset ids (rank 0 of 1 with a non-zero base)
    base = 1_000_000
    ix = IndexFlatL2(d, capacity=n, id_base=base)
    ix.add(corpus.to(dev))
    ops = rdist.gpu_ops(ix, params, batch.GateWindow(dev))
    q0, q1, cfg, D, I = rdist.sharded_retrieve_select(ops, queries, profiles, qlen, free, k, exchange=exchange)
    torch.cuda.synchronize()
    assert (q0, q1) == (0, nq)

    ix2 = IndexFlatL2(d, capacity=n)
    ix2.add(corpus.to(dev))
    res = RetrieveSelect(ix2, params).run(queries, profiles, qlen, free)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(batch.from_device(cfg, batch.CONFIG_DTYPE), res.configs_np())
    Ig = I.cpu().numpy()
    Ir = res.chunk_ids.cpu().numpy()
    np.testing.assert_array_equal(np.where(Ig >= 0, Ig - base, -1), Ir)
    ix.close()
    ix2.close()
