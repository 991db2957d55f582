"""Loader of tests/golden/retrieval_sklearn.npz (tests/golden/make_retrieval_golden.py)."""

import os

import numpy as np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "retrieval_sklearn.npz")
KINDS = ["iso", "clustered", "doc_contiguous"]


def cases():
    import torch

    from tools import synth

    z = np.load(PATH)
    names = sorted({k.split("__")[0] for k in z.files})
    for name in names:
        nq, n, d, bf, k, seed, kind = (int(x) for x in z[f"{name}__params"])
        dt = torch.bfloat16 if bf else torch.float32
        c = synth.corpus_rows(0, n, d, seed, dt, "cpu", data=KINDS[kind])
        q = synth.make_queries(nq, n, d, seed, dt, data=KINDS[kind])
        yield name, q, c, k, z[f"{name}__D"], z[f"{name}__I"], bool(bf)
