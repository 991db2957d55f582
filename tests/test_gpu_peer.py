"""The peer-memory exchange (csrc/peer.cu) in one process: a world-1 group
maps only its own region, so scatter + waiting merge is a copy of the
sorted lists with the join applied; a merge whose epoch never arrives must
time out, raise the error word and return (never hang)."""

import ctypes

import numpy as np
import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


def _sorted_keys(nq, k, seed):
    rng = np.random.default_rng(seed)
    d = np.sort(rng.random((nq, k), dtype=np.float32) * 4, axis=1)
    ids = rng.integers(0, 2**31, (nq, k), dtype=np.int64)
    keys = (d.view(np.uint32).astype(np.uint64) << np.uint64(32)) | ids.astype(np.uint64)
    return torch.from_numpy(keys.view(np.int64)), d, ids


@pytest.fixture
def group(tmp_path):
    dist.init_process_group("gloo", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


def test_world1_exchange_is_a_copy_and_timeout_is_reported(group):
    from paper_2412_10543_b200 import _lib, batch
    from paper_2412_10543_b200 import dist as rdist

    dev = torch.device("cuda", 0)
    px = rdist.PeerExchange(100, 35, device=dev, timeout_ms=50)
    for it, nq in enumerate((100, 37, 1)):  # three epochs: both parities
        keys, d, ids = _sorted_keys(nq, 35, it)
        D, I = px.merge(keys.to(dev), nq, 35)
        np.testing.assert_array_equal(I.cpu().numpy(), ids)
        np.testing.assert_array_equal(D.cpu().numpy(), d)
    # fewer outputs than list entries: the k smallest
    keys, d, ids = _sorted_keys(50, 35, 5)
    D, I = px.merge(keys.to(dev), 50, 10)
    np.testing.assert_array_equal(I.cpu().numpy(), ids[:, :10])
    # the join: only the first num_chunks of selected queries survive
    keys, d, ids = _sorted_keys(4, 35, 7)
    cfg = np.zeros(4, dtype=_lib.CONFIG_DTYPE)
    cfg["status"] = [_lib.RS_SELECT_BEST_FIT, _lib.RS_SELECT_FALLBACK, _lib.RS_SELECT_MUST_QUEUE,
                     _lib.RS_SELECT_BEST_FIT]
    cfg["num_chunks"] = [3, 35, 5, 40]
    D, I = px.merge(keys.to(dev), 4, 35, keep=batch.to_device(cfg, dev))
    I = I.cpu().numpy()
    assert (I[0, :3] == ids[0, :3]).all() and (I[0, 3:] == -1).all()
    assert (I[1] == ids[1]).all() and (I[2] == -1).all() and (I[3] == ids[3]).all()
    torch.cuda.synchronize()
    assert px.error() == 0
    # an epoch no source ever raised: bounded wait, error word set
    D = torch.empty((8, 35), dtype=torch.float32, device=dev)
    I = torch.empty((8, 35), dtype=torch.int64, device=dev)
    _lib.check(px.lib.rs_peer_merge_topk(ctypes.byref(px._ex), 8, px.epoch + 5, 35, None, _lib.ptr(D), _lib.ptr(I),
                                         50, _lib.stream_ptr()))
    torch.cuda.synchronize()
    assert px.error(clear=True) == 1 and px.error() == 0
    with pytest.raises(ValueError):
        px.merge(keys.to(dev), 300, 35)  # exceeds the region's slice capacity
    px.close()


@pytest.mark.parametrize("dtype,n", [(torch.bfloat16, 20_000), (torch.bfloat16, 200), (torch.float32, 5_000),
                                     (torch.bfloat16, 0)])
def test_world1_search_scatter_equals_search(group, dtype, n):
    """rs_index_search_scatter: the fused merge-to-peers (bf16, one or many
    segments), the local-rows-then-scatter path (3xTF32 re-rank, empty index)
    and the owner's merge give the plain search's result."""
    from paper_2412_10543_b200 import IndexFlatL2
    from paper_2412_10543_b200 import dist as rdist

    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(n)
    c = torch.nn.functional.normalize(torch.randn(n, 256, generator=g), dim=1).to(dtype)
    q = torch.nn.functional.normalize(torch.randn(77, 256, generator=g), dim=1).to(dtype).to(dev)
    ix = IndexFlatL2(256, dtype=dtype, capacity=max(n, 1), id_base=1000)
    if n:
        ix.add(c.to(dev))
    px = rdist.PeerExchange(77, 35, device=dev)
    for _ in range(3):
        epoch = px.begin()
        ix.search_scatter(q, 35, px, epoch)
        D, I = px.merge_slice(77, 35, epoch)
        D0, I0 = ix.search(q, 35)
        torch.cuda.synchronize()
        assert torch.equal(I, I0) and torch.equal(D, D0)
    assert px.error() == 0
    px.close()
    ix.close()
