"""The reference's own tests, run against the GPU engine.

``baseline/_ref/pkg/tests`` is the reference's test suite as shipped
(tools/install_reference.sh copies /root/reference/pkg there; it travels to
the GPU box with the reference install).  tests/refshim.py points
``robench.initialize`` at this package, so every ``initialize(...)`` /
``engine.evaluate(fn, PointBatch(...))`` in those tests runs on the device,
with the reference's own config, batch and exception classes.

Run: all of test_engine.py (/root/reference/pkg/tests/test_engine.py) and
test_acceptance.py criteria 1-8 (:61-283).  Not run: criterion 9 (landscape
grids through the CLI's scalar evaluator, no engine involved; a documented
red in the reference itself, pkg/README.md:36-40).

Criterion 6 also starts two subprocesses with a replaced environment
(PYTHONPATH = the reference sources only): those legs check the reference's
own CPU path across processes; its in-process thread-count leg runs here.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

from tests.conftest import cuda_available

ROOT = Path(__file__).resolve().parent.parent
REF_PKG = ROOT / "baseline" / "_ref" / "pkg"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not cuda_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not (REF_PKG / "tests" / "test_engine.py").exists(),
                                 reason="reference not installed (tools/install_reference.sh)")]

CRITERIA = " or ".join("test_criterion_%d_" % k for k in range(1, 9))


def _run(targets):
    env = dict(os.environ, PYTHONPATH=f"{REF_PKG / 'src'}{os.pathsep}{ROOT}")
    cmd = [sys.executable, "-m", "pytest", "-p", "tests.refshim", "-p", "no:cacheprovider",
           "-q", "-rA", *targets]
    proc = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = proc.stdout + proc.stderr
    print(out[-6000:])
    return proc.returncode, out


def _launches(out):
    for line in out.splitlines():
        if line.startswith("refshim:"):
            return int(line.split()[1])
    return 0


def test_reference_engine_tests_pass_on_the_gpu_engine():
    rc, out = _run([str(REF_PKG / "tests" / "test_engine.py")])
    assert rc == 0, out[-3000:]
    assert _launches(out) > 100, "the reference tests did not reach the device engine"


def test_reference_acceptance_criteria_pass_on_the_gpu_engine():
    acc = REF_PKG / "tests" / "test_acceptance.py"
    rc, out = _run([str(acc), "-k", CRITERIA])
    assert rc == 0, out[-3000:]
    assert _launches(out) > 1000, "the reference tests did not reach the device engine"
