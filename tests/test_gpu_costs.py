"""Cost table of every pruned candidate (rs_candidate_costs): enumerate_candidates
order, plan_bytes and the plan's critical-path delay, bit-exact against
~120k candidates of 600 random spaces evaluated by the reference
(tests/golden/make_golden.py gen_costs)."""

import numpy as np
import pytest
import torch

from paper_2412_10543_b200 import _lib, batch
from tests.golden_data import PARAM_SETS, candidate_costs

pytestmark = pytest.mark.gpu


def test_cost_table_matches_reference():
    z = candidate_costs()
    qs, cand, delay, costs = z["queries"], z["cand"], z["delay"], z["costs"]
    dev = torch.device("cuda", 0)
    for ps_i in np.unique(qs[:, 1]):
        L, H, D, w, cs, out, tmpl, mc, cstep, istep = PARAM_SETS[int(ps_i)]
        params = batch.SelectParams(int(2 * L * H * D * w), cs, out, tmpl, mc, cstep, istep)
        for ci, (a, b, s) in enumerate(costs):
            sel = np.where((qs[:, 1] == ps_i) & (qs[:, 9] == ci))[0]
            if len(sel) == 0:
                continue
            rows = qs[sel]
            spaces = batch.to_device(batch.spaces_from_arrays(rows[:, 2], rows[:, 3], rows[:, 4], rows[:, 5],
                                                              rows[:, 6]), dev)
            qlen = torch.as_tensor(rows[:, 7].astype(np.int32), device=dev)
            run = torch.as_tensor(rows[:, 8].astype(np.int32), device=dev)
            off, recs = batch.candidate_costs(spaces, qlen, params, cost=batch.CostModel(a, b, s), running_before=run)
            off = off.cpu().numpy()
            got = batch.from_device(recs, _lib.CANDIDATE_DTYPE) if recs.numel() else np.zeros(0, _lib.CANDIDATE_DTYPE)
            lo = np.searchsorted(cand[:, 0], rows[:, 0], side="left")   # candidates are grouped by trial
            hi = np.searchsorted(cand[:, 0], rows[:, 0], side="right")
            idx = np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)])
            np.testing.assert_array_equal(np.diff(off), hi - lo)
            want = cand[idx]
            np.testing.assert_array_equal(got["method"], want[:, 1])
            np.testing.assert_array_equal(got["num_chunks"], want[:, 2])
            np.testing.assert_array_equal(got["interlen"], want[:, 3])
            np.testing.assert_array_equal(got["kv_bytes"], want[:, 4])
            np.testing.assert_array_equal(got["delay"], delay[idx])


def test_cost_table_without_cost_model_and_empty():
    dev = torch.device("cuda", 0)
    params = batch.SelectParams(131072, 1000, 10)
    sp = batch.to_device(batch.spaces_from_arrays([7, 2], [1, 3], [35, 3], [30, 0], [200, 0]), dev)
    off, recs = batch.candidate_costs(sp, torch.tensor([500, 900], dtype=torch.int32, device=dev), params)
    off = off.cpu().numpy()
    assert list(off) == [0, 700, 701]
    got = batch.from_device(recs, _lib.CANDIDATE_DTYPE)
    assert (got["delay"] == 0).all() and got["kv_bytes"].min() > 0
    off, recs = batch.candidate_costs(sp[:0], torch.zeros(0, dtype=torch.int32, device=dev), params)
    assert off.cpu().tolist() == [0] and recs.shape[0] == 0
