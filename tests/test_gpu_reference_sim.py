"""f4: the reference's own pipeline with the GPU drop-in.

* ``ragsched.sim.run`` (sim.py:150-325), the unmodified reference installed
  in ``baseline/_ref``, run stock and with ``dropin.install(ragsched)`` on the
  same seeds: the report, summary and trace files (metrics.py:151-214, the A9
  writers) must be byte-identical — adaptive Poisson / sequential zero-noise /
  A6 noise / 2 GiB / fixed-config baselines / 1,000 doc-level queries;
* the reference's own acceptance suite (``baseline/_ref_tests``, a copy of
  pkg/tests made by tools/install_reference.sh) run with the drop-in active
  (tests/dropin_plugin.py): A2, A5, A6, A9 and A10 must pass.
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = os.path.join(ROOT, "baseline", "_ref_tests")


@pytest.fixture(scope="module")
def rs():
    from oracle import refpath

    try:
        return refpath.import_ragsched(refpath.REF_INSTALL)
    except ImportError as e:
        pytest.skip(f"reference not installed in baseline/_ref: {e}")


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("scenario", list(range(7)))
def test_sim_run_byte_identical_with_dropin(rs, scenario):
    from tools import dropin_sim

    res = dropin_sim.compare(rs, dropin_sim.SCENARIOS[scenario])
    print(res)
    assert res["identical"], res


@pytest.mark.timeout(1800)
def test_reference_acceptance_suite_with_dropin():
    if not os.path.isdir(REF_TESTS):
        pytest.skip("reference tests not installed (tools/install_reference.sh)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "baseline", "_ref")]))
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(REF_TESTS, "test_acceptance.py"), "-p",
                        "tests.dropin_plugin", "-q", "-rA", "-p", "no:cacheprovider"],
                       capture_output=True, text=True, timeout=1700, cwd=ROOT, env=env)
    out = r.stdout
    print(out[-6000:])
    assert "GPU drop-in active" in out
    passed = set(re.findall(r"PASSED \S*::test_(a\d+)_", out))
    for crit in ("a2", "a5", "a6", "a9", "a10"):
        assert crit in passed, (crit, sorted(passed))


def test_plan_calls_exceptions_match_reference(rs):
    """memory.plan_calls (memory.py:89-150) through the drop-in raises the
    reference's exception types WITH the reference's messages, in the
    reference's check order (InvalidChunkCount before the out_budget check)."""
    import random

    from paper_2412_10543_b200 import dropin

    T, C, Mem = rs.types, rs.config, rs.memory
    rng = random.Random(5)
    model = T.ModelSpec(num_layers=32, num_kv_heads=8, head_dim=128, bytes_per_element=2, max_context_tokens=8192)
    meta = T.DatasetMeta(description="d", chunk_size=1000)
    cases = []
    for i in range(400):
        m = rng.choice(list(T.SynthesisMethod))
        n = rng.choice([0, -1, 1, 5, 9, 35, 36, 40])
        il = rng.choice([None, 0, -5, 30, 200, 900]) if m is T.SynthesisMethod.MAP_REDUCE else None
        try:
            cfg = T.RagConfig(m, n, il) if il is not None else T.RagConfig(m, n)
        except Exception:
            continue
        q = T.QueryRecord(id=f"q{i}", text="t", query_token_len=rng.choice([10, 2000, 7000]))
        cases.append((q, cfg, rng.choice([-1, 0, 10, 60])))

    def outcome(fn):
        out = []
        for q, cfg, ob in cases:
            try:
                plan = fn(q, cfg, meta, model, ob)
                out.append(("ok", tuple((c.kind.value, c.prompt_tokens, c.max_output_tokens, c.kv_bytes)
                                        for c in plan.calls), plan.total_bytes))
            except Exception as e:  # noqa: BLE001
                out.append((type(e).__name__, str(e)))
        return out

    stock = outcome(Mem.plan_calls)
    originals = dropin.install(rs)
    try:
        gpu = outcome(Mem.plan_calls)
    finally:
        dropin.uninstall(originals)
    kinds = {s[0] for s in stock}
    assert {"ok", "InvalidChunkCount", "ContextOverflow", "ValueError"} <= kinds, kinds
    for a, b, case in zip(stock, gpu, cases):
        assert a == b, (case, a, b)
