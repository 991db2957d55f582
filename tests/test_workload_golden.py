"""The committed bench workloads (tests/golden/workload_cfg*.npz, made by
running the reference's TruthDistribution / mock_estimate / gate_profile /
best_fit_select / fallback_config) against the C restatement of the config
path: every gated space and every decision bit-exact.  CPU only."""

import numpy as np
import pytest

from oracle import c_oracle
from oracle import config_oracle as co
from tools import workload as wl


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_workload_decisions_match_reference(name):
    w = wl.load(name)
    n = len(w["qlen"])
    if wl.full_space(w):
        spaces = np.tile(w["fixed_space"].astype(np.int32), (n, 1))
        assert np.array_equal(w["exp_space"], spaces)
    else:
        spaces, fb, _ = c_oracle.gate_batch(wl.profiles_int5(w), w["conf"])
        np.testing.assert_array_equal(spaces, w["exp_space"])
        np.testing.assert_array_equal(fb, w["exp_gate_fb"])
    p = co.SelectParams(chunk_size=w["chunk_size"], out_budget=w["out_budget"])
    cfg, b, st = c_oracle.select_batch(spaces, w["joint"], w["qlen"], w["free"], p, nthreads=0)
    e = w["exp_select"]
    np.testing.assert_array_equal(st, e[:, 3])
    np.testing.assert_array_equal(cfg, e[:, :3])
    np.testing.assert_array_equal(b, e[:, 4])


def test_workloads_cover_the_survey_mix():
    """~4.9% noisy profiles through the gate hull (cfg1/2/4),
    every decision kind present, cfg5 full space (700 candidates)."""
    for name in ("cfg1", "cfg2", "cfg4"):
        w = wl.load(name)
        frac = float(w["exp_gate_fb"].mean())
        assert 0.02 < frac < 0.08, (name, frac)
        assert set(np.unique(w["exp_select"][:, 3]).tolist()) == {0, 1, 2}
    w3 = wl.load("cfg3")
    assert (w3["exp_space"][:, 0] == 6).all() and (w3["exp_space"][:, 3:] == [30, 200]).all()
    w5 = wl.load("cfg5")
    assert len(co.enumerate_grid(tuple(int(x) for x in w5["fixed_space"]))) == 700
