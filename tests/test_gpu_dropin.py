"""GPU: the reference's OWN acceptance criteria c3 (optimize_plan + execute_plan
of a 2-MPF net vs oracle::sliding_window_ref, fp32 tolerance 1e-6) and c10
(hand-built ExecutionPlan with plain pooling + measure_throughput), compiled
from the unmodified reference test text (oracle/build_refcompat.py):

* refcompat_acceptance -- against this repo's drop-in include/voxin/*.hpp;
* refpatched_acceptance -- against the reference library itself, its executor
  (PlanRunner) dispatching every conv / pool to libvxg.so through the three
  one-line hooks of INTEGRATION.md §1.
"""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BINS = ["refcompat_acceptance", "refpatched_acceptance"]


@pytest.mark.parametrize("name", BINS)
def test_reference_acceptance_criteria_on_b200(name, ctx):
    exe = ROOT / "oracle" / "_ref" / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (oracle/build_refcompat.py needs the reference checkout)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS") == 2, r.stdout
