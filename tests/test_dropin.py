"""The drop-in rebinds exactly the reference's hot-path attributes (CPU check;
needs the reference package, present only in the dev container)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture()
def ragsched():
    if not os.path.isdir(REF):
        pytest.skip("reference package not available here")
    sys.path.insert(0, REF)
    import ragsched as pkg

    yield pkg
    sys.path.remove(REF)


def test_install_and_uninstall(ragsched):
    from tests.golden_data import field_conf_rows

    import ragsched.mapping as mapping
    import ragsched.memory as memory
    import ragsched.profiler as profiler
    import ragsched.scheduler as scheduler
    import ragsched.sim as sim

    from paper_2412_10543_b200 import dropin

    names = lambda: (scheduler.best_fit_select, scheduler.fallback_config, profiler.gate_profile,  # noqa: E731
                     mapping.map_profile, memory.plan_bytes, sim.call_latency, scheduler.Scheduler, sim.Scheduler,
                     memory.plan_calls, scheduler.plan_calls, profiler.parse_profile_text,
                     profiler._per_field_confidences)
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
    # the remote estimator's per-field confidences (profiler.py:417) go through the native routine, bit-exact
    ref_conf = originals[(profiler, "_per_field_confidences")]
    for text, toks, _ in field_conf_rows()[::40]:
        assert profiler._per_field_confidences(text, toks) == ref_conf(text, toks)
    dropin.uninstall(originals)
    restored = names()
    assert all(a is b for a, b in zip(before, restored))


REF_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")


@pytest.mark.skipif(not os.path.exists(os.path.join(REF_TESTS, "test_remote_profiler.py")),
                    reason="reference tests not installed (tools/install_reference.sh)")
def test_reference_remote_profiler_suite_with_dropin():
    """The reference's own RemoteEstimator tests (a stub HTTP endpoint with
    token log-probs) pass with the drop-in active: profile_query's answer
    parsing and per-field confidences run through the native routines (host
    code, no GPU)."""
    import subprocess

    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(REF_TESTS, "test_remote_profiler.py"), "-p",
                        "tests.dropin_plugin", "-q", "-p", "no:cacheprovider"], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "passed" in r.stdout and "GPU drop-in active" in r.stdout
