"""Diagnose the 3xTF32 path: kernel distances vs float64, and vs emulated
1xTF32 / 3xTF32 (truncation) references."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_10543_b200 import IndexFlatL2  # noqa: E402


def trunc(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


for d in (64, 128, 256, 512, 768, 1024):
    g = torch.Generator().manual_seed(d)
    nq, n = 64, 512
    c = torch.nn.functional.normalize(torch.randn(n, d, generator=g), dim=1)
    q = torch.nn.functional.normalize(torch.randn(nq, d, generator=g), dim=1)
    ix = IndexFlatL2(d, dtype=torch.float32, capacity=n)
    ix.add(c.cuda())
    D, I = ix.search(q.cuda(), 10)
    torch.cuda.synchronize()
    D, I = D.cpu().double(), I.cpu()
    q64, c64 = q.double(), c.double()
    exact = (q64 ** 2).sum(1, keepdim=True) + (c64 ** 2).sum(1)[None] - 2 * q64 @ c64.T
    got_exact = torch.gather(exact, 1, I)
    qh, ch = trunc(q).double(), trunc(c).double()
    ql, cl = (q - trunc(q)).double(), (c - trunc(c)).double()
    one = (q64 ** 2).sum(1, keepdim=True) + (c64 ** 2).sum(1)[None] - 2 * qh @ ch.T
    three = (q64 ** 2).sum(1, keepdim=True) + (c64 ** 2).sum(1)[None] - 2 * (qh @ ch.T + qh @ trunc(c - trunc(c)).double().T + trunc(q - trunc(q)).double() @ ch.T)
    e_exact = (D - got_exact).abs().max().item()
    e_one = (D - torch.gather(one, 1, I)).abs().max().item()
    e_three = (D - torch.gather(three, 1, I)).abs().max().item()
    print(f"d={d:5d} max|D-exact|={e_exact:.3e}  |D-1xtf32|={e_one:.3e}  |D-3xtf32|={e_three:.3e}  plan={ix.last_plan()}")
    ix.close()
