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
