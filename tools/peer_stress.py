"""Stress of the peer-memory exchange: P processes (sharing one GPU here, one
GPU each on a multi-GPU box) run many consecutive exchanges of varying batch
sizes through ``rs_index_search_scatter`` + ``PeerExchange.merge_slice`` with
no host synchronisation between batches, and every batch's merged slices must
equal the single-index search.

    python tools/peer_stress.py [world] [iters]
"""

import os
import socket
import sys

import numpy as np
import torch
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

N, D, K, NQ_MAX = 60_000, 256, 35, 700


def _data():
    g = torch.Generator().manual_seed(5)
    c = torch.nn.functional.normalize(torch.randn(N, D, generator=g), dim=1).bfloat16()
    q = torch.nn.functional.normalize(torch.randn(NQ_MAX, D, generator=g), dim=1).bfloat16()
    return c, q


def _sizes(iters):
    g = torch.Generator().manual_seed(11)
    return torch.randint(0, NQ_MAX + 1, (iters,), generator=g).tolist()


def _worker(rank, world, port, iters, out):
    import torch.distributed as dist

    from paper_2412_10543_b200 import IndexFlatL2
    from paper_2412_10543_b200 import dist as rdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    c, q = _data()
    r0, r1 = rdist.shard_range(N, rank, world)
    ix = IndexFlatL2(D, capacity=r1 - r0, id_base=r0)
    ix.add(c[r0:r1].to(dev))
    qd = q.to(dev)
    peer = rdist.PeerExchange(NQ_MAX, K, device=dev, timeout_ms=20000)
    results = []
    for it, nq in enumerate(_sizes(iters)):
        epoch = peer.begin()
        ix.search_scatter(qd[:nq].roll(it, 0) if nq else qd[:0], K, peer, epoch)
        _, I = peer.merge_slice(nq, K, epoch)
        results.append(I)  # no synchronisation: the next batch overwrites the other parity buffer
    torch.cuda.synchronize()
    err = peer.error()
    out.put((rank, err, [I.cpu().numpy() for I in results]))  # by value: the worker exits right after
    peer.close()
    ix.close()
    dist.destroy_process_group()


def main(world=4, iters=200):
    from paper_2412_10543_b200 import IndexFlatL2
    from paper_2412_10543_b200 import dist as rdist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, iters, out)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([out.get(timeout=1800) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
    c, q = _data()
    dev = torch.device("cuda", 0)
    ix = IndexFlatL2(D, capacity=N)
    ix.add(c.to(dev))
    qd = q.to(dev)
    bad = 0
    for it, nq in enumerate(_sizes(iters)):
        _, I0 = ix.search(qd[:nq].roll(it, 0) if nq else qd[:0], K)
        got = np.concatenate([r[2][it] for r in res])
        if not np.array_equal(got, I0.cpu().numpy()):
            bad += 1
    errs = [r[1] for r in res]
    print(f"peer stress: world {world}, {iters} batches (0..{NQ_MAX} queries), mismatched batches {bad}, "
          f"timeouts {errs}, exit codes {[p.exitcode for p in procs]}")
    ix.close()
    return bad == 0 and not any(errs)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:3]]
    sys.exit(0 if main(*a) else 1)
