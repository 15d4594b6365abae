"""The reference's OWN test suites, run against the B200 engine (drop-in proof).

The unmodified reference (wedgegraph 0.1.0) is installed, with its tests, in
the git-ignored baseline/_ref by baseline/install_ref.sh; it travels to the GPU
box with the repo snapshot.  tests/refsuite_plugin.py injects the B200 backend
through the reference's own seam (kernels.py:128-163):

* tier 1 -- ``B200Backend`` as the reference's "native" and default backend:
  backend equivalence (pkg/tests/test_kernels_backends.py:24-112) then compares
  the reference's numpy kernels with the sm_100a kernels bit for bit, and the
  stock engine's known-answer / convergence tests (test_engine.py:58-310) and
  the 200-graph acceptance corpus (test_acceptance.py:97-355) run their
  transforms and pulls on the GPU;
* tier 2 -- the whole loop: ``run_until_convergence`` (engine.py:330-388) is
  the B200 device loop for min-plus programs, so acceptance C1 (values and
  per-iteration frontiers identical to the push oracle across W in {1,2,4} and
  vpg in {1..16}) checks the device-resident loop.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
SUITES = ["test_kernels_backends.py", "test_engine.py", "test_acceptance.py"]

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "tests" / "conftest.py").exists(),
                                 reason="baseline/_ref not installed (baseline/install_ref.sh)")]


def _run(tier: str, suites, extra=()):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT / "tests"), str(ROOT)])
    env["WG_REFSUITE_TIER"] = tier
    env.pop("WEDGE_BACKEND", None)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "refsuite_plugin", "-p", "no:cacheprovider",
           "--rootdir", str(REF / "tests"), *extra, *suites]
    r = subprocess.run(cmd, cwd=REF / "tests", env=env, capture_output=True, text=True, timeout=1800)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
    return r.stdout


def test_plugin_injects_b200_into_the_reference():
    code = ("import wedgegraph.kernels as k, wedgegraph.engine as e; "
            "from paper_1903_07754_b200.backend import B200Backend; "
            "assert isinstance(k.get_backend('native'), B200Backend); "
            "assert isinstance(k.get_backend(None), B200Backend); "
            "import wedgegraph; assert wedgegraph.__file__.startswith(%r)" % str(REF))
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT / "tests"), str(ROOT)])
    env["WG_REFSUITE_TIER"] = "1"
    r = subprocess.run([sys.executable, "-c", "import refsuite_plugin; " + code], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]


def test_reference_suites_tier1_kernel_protocol():
    out = _run("1", SUITES)
    print(out[-2000:])


def test_reference_suites_tier2_device_loop():
    out = _run("2", ["test_engine.py", "test_acceptance.py"])
    print(out[-2000:])
