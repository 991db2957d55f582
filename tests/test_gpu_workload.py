"""GPU config path on the committed bench workloads (tests/golden/workload_cfg*.npz:
profiles from the reference's TruthDistribution + mock_estimate, decisions
from the reference's own gate_profile / best_fit_select / fallback_config):
the gate kernels and the select kernel must reproduce every gated space and
every decision bit for bit."""

import numpy as np
import pytest
import torch

from paper_2412_10543_b200 import _lib, batch
from tools import workload as wl

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_gpu_workload_decisions_match_reference(name):
    dev = torch.device("cuda", 0)
    w = wl.load(name)
    n = len(w["qlen"])
    prof = batch.to_device(batch.profiles_from_arrays(w["cx"], w["joint"], w["pieces"], w["s_lo"], w["s_hi"],
                                                      w["conf"]), dev)
    if wl.full_space(w):
        sp = batch.spaces_from_arrays(*(np.full(n, int(x)) for x in w["fixed_space"]))
        spaces = batch.to_device(sp, dev)
    else:
        spaces = batch.prune_gate(prof, batch.GateWindow(dev))
        got = batch.from_device(spaces, _lib.SPACE_DTYPE)
        for i, f in enumerate(("methods", "num_chunks_lo", "num_chunks_hi", "interlen_lo", "interlen_hi")):
            np.testing.assert_array_equal(got[f], w["exp_space"][:, i], err_msg=f)
        np.testing.assert_array_equal(got["gate_fallback"], w["exp_gate_fb"])
    params = batch.SelectParams(per_token_bytes=131072, chunk_size=w["chunk_size"], out_budget=w["out_budget"])
    out, _ = batch.select(spaces, prof, torch.as_tensor(w["qlen"], device=dev), torch.as_tensor(w["free"], device=dev),
                          params)
    cfg = batch.from_device(out, _lib.CONFIG_DTYPE)
    e = w["exp_select"]
    np.testing.assert_array_equal(cfg["status"], e[:, 3])
    np.testing.assert_array_equal(cfg["method"], e[:, 0])
    np.testing.assert_array_equal(cfg["num_chunks"], e[:, 1])
    np.testing.assert_array_equal(cfg["interlen"], e[:, 2])
    np.testing.assert_array_equal(cfg["kv_bytes"], e[:, 4])
