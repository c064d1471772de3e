"""The reference's own test suite (/root/reference/proj/tests/*.cpp: the unit
tests and the acceptance criteria C01-C10), compiled UNCHANGED against this
repository's drop-in headers (include/ttsvd/*.hpp, the reference's file
names) and run on the B200 — VERDICT r01 "next" #2, row a12.

Baseline: tests/golden/ref_suite_cpu.json, the same files built against the
reference's headers and run on the CPU (made by
tests/golden/make_ref_suite_cpu.py).  Every test the reference passes must pass
on the device, except the documented exclusions below; for C01 (which the
reference itself fails on its thick-bounds and two-sided cells) the device
must match the reference's own cell counts.

Excluded, with the reason:
  ReduceBlock.HandHouseholderStep   expects R = [-5]; R is unique up to the signs
                                    of its rows and the device pivots on the
                                    stacked R(j,j), giving +5 (DESIGN.md §4 (1)).
  Tsqr.AuxiliaryMemoryIndependentOfN  TsqrStats::scratch_bytes is a CPU blocking
  Tsqr.ReflectorNormInstrumentation   / reflector instrumentation; the device
                                    kernels are not instrumented (the fields stay
                                    as the caller set them).
"""
import json
import os
import subprocess

import pytest

from refsuite_parse import parse

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "refsuite", "_build", "ref_suite")
GOLDEN = os.path.join(ROOT, "tests", "golden", "ref_suite_cpu.json")
EXCLUDED = ["ReduceBlock.HandHouseholderStep", "Tsqr.AuxiliaryMemoryIndependentOfN",
            "Tsqr.ReflectorNormInstrumentation"]
# suites that never touch the device (storage, shapes, TT helpers, cost model, report)
HOST_ONLY = ["PaddedStride.*", "Shape.*", "DenseTensor.*", "ReshapeView.*", "FrobeniusNorm.*", "RandomTensor.*",
             "DumpLoad.*", "TensorTrain.*", "TtReconstruct.RankOneIsOuterProduct",
             "TtReconstruct.MatchesNaiveSummation", "TtError.*", "TtSaveLoad.*", "Roofline.*", "TsqrCost.*",
             "TsmmCost.*", "VolumeEstimate.*", "FlopsEstimate.*", "PerStepModel.*", "ProfileFile.*", "Report.*",
             "SelectRank.*", "DeriveDelta.*", "BlockParams.*", "ChooseCombinedDims.*"]


def run(filter_: str, timeout: int = 1200):
    if not os.path.exists(EXE):
        pytest.skip("tests/refsuite/_build/ref_suite not built (make -C tests/refsuite)")
    env = dict(os.environ, LD_LIBRARY_PATH=os.path.join(ROOT, "paper_2102_00104_b200"))
    r = subprocess.run([EXE, f"--gtest_filter={filter_}"], capture_output=True, text=True, timeout=timeout,
                       cwd="/tmp", env=env)
    return r, parse(r.stdout)


def test_host_only_reference_tests_pass_on_cpu():
    """No device needed: shapes, storage, TT helpers, the cost model, the report."""
    r, res = run(":".join(HOST_ONLY))
    assert len(res["passed"]) >= 35, r.stdout[-3000:]
    assert not res["failed"], (res["failed"], r.stdout[-3000:])


@pytest.mark.gpu
def test_reference_suite_on_device():
    golden = json.load(open(GOLDEN))
    r, res = run("*-" + ":".join(EXCLUDED), timeout=3000)
    print(r.stdout[-6000:])
    expected = set(golden["passed"]) - set(EXCLUDED)
    missing = sorted(expected - set(res["passed"]))
    assert not missing, (missing, r.stdout[-6000:])
    # C01: the reference itself fails it on thick / two-sided cells; the device
    # variants must reproduce the reference's own outcome cell for cell
    c01_ref, c01 = golden["acceptance"]["C01"], res["acceptance"]["C01"]
    assert (c01["ranks_ok"], c01["errors_ok"]) == (c01_ref["ranks_ok"], c01_ref["errors_ok"]), (c01, c01_ref)
    assert c01["failing_cells"] == c01_ref["failing_cells"]
    for k in ("C02", "C03", "C04", "C05", "C06", "C07", "C08", "C10"):
        assert res["acceptance"][k]["status"] == "PASS", res["acceptance"][k]
