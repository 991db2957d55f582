"""One rank's view of the sharded cfg4 step at N = 8 on a single GPU (world-1
group, so the peer regions are local): a 1.25M x 1024 bf16 shard, 8,192
queries, the search whose final merge stores to the owners
(merge_topk64_kernel<kMergeScatter>), then the owner's waiting merge
(merge_topk64_kernel<kMergeWait>).  Run under ncu for the launch list:

    ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --csv \\
        python tools/peer_launches.py
"""

import os
import sys
import tempfile

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2412_10543_b200 import IndexFlatL2  # noqa: E402
from paper_2412_10543_b200 import dist as rdist  # noqa: E402


def main(n=1_250_000, nq=8192, d=1024, k=35, steps=2):
    with tempfile.TemporaryDirectory() as tmp:
        dist.init_process_group("gloo", init_method=f"file://{tmp}/pg", rank=0, world_size=1)
        dev = torch.device("cuda", 0)
        g = torch.Generator(device=dev).manual_seed(0)
        c = torch.nn.functional.normalize(torch.randn(n, d, generator=g, device=dev), dim=1).bfloat16()
        q = torch.nn.functional.normalize(torch.randn(nq, d, generator=g, device=dev), dim=1).bfloat16()
        ix = IndexFlatL2(d, capacity=n)
        ix.add(c)
        del c
        peer = rdist.PeerExchange(nq, k, device=dev)
        for _ in range(2):  # warm-up
            e = peer.begin()
            ix.search_scatter(q, k, peer, e)
            peer.merge_slice(nq, k, e)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("timed")
        for _ in range(steps):
            e = peer.begin()
            ix.search_scatter(q, k, peer, e)
            peer.merge_slice(nq, k, e)
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        print("plan", ix.last_plan(), "peer error", peer.error())
        peer.close()
        ix.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
