"""A1 on the GPU: the 20,000 reference mapping vectors (tests/golden/mapping.npz,
seed 42 as test_acceptance.py:120-167, both max_chunks 35 and 12) through the
gate kernel with every profile accepted (Algorithm 1, mapping.py:106-126),
bit-exact; and through the scalar drop-in ``map_profile``."""

import numpy as np
import pytest
import torch

from paper_2412_10543_b200 import _lib, batch
from paper_2412_10543_b200.mapping import QueryProfile, map_profile
from paper_2412_10543_b200.types import IntRange
from tests import golden_data as gd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("max_chunks", [35, 12])
def test_a1_vectors_batch_kernel(max_chunks):
    profiles, spaces = gd.mapping()
    sel = profiles[:, 5] == max_chunks
    p, want = profiles[sel], spaces[sel]
    assert len(p) == 10_000
    dev = torch.device("cuda", 0)
    rec = batch.profiles_from_arrays(p[:, 0], p[:, 1], p[:, 2], p[:, 3], p[:, 4], np.ones(len(p)))
    out = batch.prune_gate(batch.to_device(rec, dev), batch.GateWindow(dev), threshold=0.9, max_chunks=max_chunks)
    got = batch.from_device(out, _lib.SPACE_DTYPE)
    assert not got["gate_fallback"].any()
    for i, f in enumerate(("methods", "num_chunks_lo", "num_chunks_hi", "interlen_lo", "interlen_hi")):
        np.testing.assert_array_equal(got[f], want[:, i], err_msg=f)


def test_a1_vectors_scalar_map_profile():
    profiles, spaces = gd.mapping()
    for (cx, joint, pieces, lo, hi, mc), want in zip(profiles[:2000], spaces[:2000]):
        s = map_profile(QueryProfile(bool(cx), bool(joint), int(pieces), IntRange(int(lo), int(hi)), 0.99), int(mc))
        assert batch.space_record(s) == tuple(int(x) for x in want)
