"""pytest plugin: install this package's GPU drop-in into the reference
package BEFORE the reference's own tests import it, so that
``from ragsched.scheduler import best_fit_select`` (etc.) in those test
modules binds the GPU functions.  Used by tests/test_gpu_reference_sim.py:

    python -m pytest baseline/_ref_tests/test_acceptance.py -p tests.dropin_plugin
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INSTALLED = {}


def pytest_configure(config):
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    sys.path.insert(0, ROOT)
    import ragsched

    from paper_2412_10543_b200 import dropin

    INSTALLED["originals"] = dropin.install(ragsched)
    print(f"GPU drop-in active: ragsched from {os.path.dirname(ragsched.__file__)}", flush=True)


def pytest_report_header(config):
    import ragsched

    return [f"GPU drop-in active: ragsched from {os.path.dirname(ragsched.__file__)}"]
