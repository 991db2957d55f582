"""The drop-in rebinds exactly the reference's hot-path attributes (CPU check;
needs the reference package, present only in the dev container)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.fixture()
def ragsched():
    if not os.path.isdir(REF):
        pytest.skip("reference package not available here")
    sys.path.insert(0, REF)
    import ragsched as pkg

    yield pkg
    sys.path.remove(REF)


def test_install_and_uninstall(ragsched):
    import ragsched.mapping as mapping
    import ragsched.memory as memory
    import ragsched.profiler as profiler
    import ragsched.scheduler as scheduler
    import ragsched.sim as sim

    from paper_2412_10543_b200 import dropin

    names = lambda: (scheduler.best_fit_select, scheduler.fallback_config, profiler.gate_profile,  # noqa: E731
                     mapping.map_profile, memory.plan_bytes, sim.call_latency, scheduler.Scheduler, sim.Scheduler,
                     memory.plan_calls, scheduler.plan_calls, profiler.parse_profile_text)
    before = names()
    originals = dropin.install(ragsched)
    after = names()
    assert all(a is not b for a, b in zip(before, after))
    # wrappers produce the reference's own classes
    assert scheduler.best_fit_select.keywords["config_cls"] is ragsched.types.RagConfig
    assert profiler.gate_profile.keywords["decision_cls"] is profiler.GateDecision
    # the GPU Scheduler builds the reference's own value classes
    assert scheduler.Scheduler.classes.Admission is ragsched.scheduler.Admission
    assert scheduler.Scheduler.classes.CallKind is ragsched.memory.CallKind
    assert sim.Scheduler is scheduler.Scheduler
    # the native parser returns the reference's own QueryProfile (host code: runs without a GPU)
    p, clamped, lines = profiler.parse_profile_text("Complexity: High\nJoint Reasoning needed: Yes\nPieces: 4\n"
                                                    "Summary range: 50-120", 0.97)
    assert isinstance(p, ragsched.mapping.QueryProfile) and p.summary_len_range == ragsched.types.IntRange(50, 120)
    dropin.uninstall(originals)
    restored = names()
    assert all(a is b for a, b in zip(before, restored))
