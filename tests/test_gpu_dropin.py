"""The drop-in claim, tested with the reference's OWN code (SURVEY §4 strategy (1)):

* every unmodified reference test module but the acceptance suite (pkg/tests/test_hdm.py,
  test_filtering.py, test_rom.py, test_trustregion.py, test_problems.py, test_fem.py, test_mma.py,
  test_cli.py, test_report.py; 192 tests, staged under baseline/_ref/romtopt_tests by
  tools/stage_reference.sh) runs with
  HdmSolver / HelmholtzFilter / RomModel / ReducedBasis / gram_schmidt / pod swapped for the B200
  classes (tests/dropin_plugin.py);
* the reference's TrustRegionDriver.run (trustregion.py:383-513) on its built-in mbb-small
  problem gives the same J history and accept/reject decisions with the drop-in classes as
  the pure-CPU reference run.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "romtopt_tests")

# reference tests whose assertion is about the reference's own solver internals, not about the
# results the drop-in must reproduce (each with the reason)
EXPECTED_DIFFERENT = {
    # counts calls of romtopt.fem.PatternAssembler.factorize (SuperLU); the drop-in has no
    # factorisation (matrix-free pCG) -- its hdm_solves / factorizations counters
    # are asserted equal to the solve count in test_dropin_counters below
    "TestSolve::test_solve_counter_audit",
}


def _need_ref():
    if not os.path.isdir(os.path.join(REF, "romtopt")) or not os.path.isdir(REF_TESTS):
        pytest.skip("baseline/_ref not staged (tools/stage_reference.sh needs /root/reference)")


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([HERE, REF, REPO, env.get("PYTHONPATH", "")])
    return env



def test_reference_acceptance_on_dropin(cuda):
    """The reference's own acceptance suite (pkg/tests/test_acceptance.py) on
    the drop-in: criteria 1-5 (dense oracles, finite differences, centre consistency, error
    bounds, Galerkin optimality), 8 (trust-region mechanics on mbb-small, with the driver's
    runtime centre checks) and 9.  Criteria 6-7 run 2000-iteration MMA references on the full
    benchmarks (~100 s); measured separately."""
    _need_ref()
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "dropin_plugin", "-p", "no:cacheprovider",
                        "--rootdir", REF_TESTS, "-o", "addopts=", os.path.join(REF_TESTS, "test_acceptance.py"),
                        "-k", "not criterion_6 and not criterion_7", "-rf"],
                       cwd=REF_TESTS, env=_env(), capture_output=True, text=True, timeout=900)
    tail = r.stdout[-4000:]
    assert r.returncode == 0, tail
    assert "7 passed" in tail, tail

@pytest.mark.parametrize("module", ["test_hdm.py", "test_filtering.py", "test_rom.py", "test_trustregion.py",
                                    "test_problems.py", "test_fem.py", "test_mma.py", "test_cli.py",
                                    "test_report.py"])
def test_reference_suite_on_dropin(cuda, module):
    _need_ref()
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "dropin_plugin", "-p", "no:cacheprovider",
                        "--rootdir", REF_TESTS, "-o", "addopts=", os.path.join(REF_TESTS, module), "-rf"],
                       cwd=REF_TESTS, env=_env(), capture_output=True, text=True, timeout=900)
    tail = r.stdout[-4000:]
    failed = [ln.split(" ")[1].split("::", 1)[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED ")]
    unexpected = [f for f in failed if f.split(" - ")[0] not in EXPECTED_DIFFERENT]
    assert not unexpected, tail
    assert r.returncode in (0, 1), tail
    assert " passed" in tail, tail


def test_dropin_counters(cuda):
    """The audit of test_solve_counter_audit without its SuperLU hook: the reference's
    hdm_mma_driver (mma.py:180-225) on the drop-in solver counts one hdm solve and one
    'factorization' per design, 6 for 5 MMA iterations."""
    _need_ref()
    code = (
        "import numpy as np, dropin_plugin\n"
        "from conftest import make_cantilever\n"
        "from romtopt.hdm import ComplianceObjective\n"
        "from romtopt.mma import hdm_mma_driver\n"
        "s = make_cantilever(6, 3)\n"
        "assert type(s).__module__.startswith('paper_2004_05756_b200')\n"
        "n = s.mesh.n_elems; w = np.full(n, s.mesh.elem_volume)\n"
        "hdm_mma_driver(s, ComplianceObjective(s.f), np.full(n, 0.4), w, 0.45 * w.sum(), max_iters=5)\n"
        "print(s.stats.hdm_solves, s.stats.factorizations, s.stats.filter_solves)\n")
    env = _env()
    env["PYTHONPATH"] = os.pathsep.join([REF_TESTS, env["PYTHONPATH"]])
    r = subprocess.run([sys.executable, "-c", "import pytest\n" + code], cwd=REF_TESTS, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    h, f, fl = (int(v) for v in r.stdout.split()[-3:])
    assert h == f == 6 and fl >= 6


def _tr(mode, iters):
    r = subprocess.run([sys.executable, os.path.join(HERE, "dropin_tr.py"), mode, str(iters)], env=_env(),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_trust_region_driver_matches_reference(cuda):
    _need_ref()
    ref = _tr("ref", 6)
    gpu = _tr("gpu", 6)
    assert ref["solver"] == "romtopt.hdm" and gpu["solver"].startswith("paper_2004_05756_b200")
    assert len(ref["records"]) == len(gpu["records"])
    for a, b in zip(ref["records"], gpu["records"]):
        assert a["accepted"] == b["accepted"] and a["basis_size"] == b["basis_size"], (a, b)
        assert abs(a["j_center"] - b["j_center"]) <= 1e-8 * abs(a["j_center"]), (a, b)
        assert abs(a["j_candidate"] - b["j_candidate"]) <= 1e-6 * abs(a["j_candidate"]), (a, b)
    assert ref["hdm_solves"] == gpu["hdm_solves"] and ref["rom_solves"] == gpu["rom_solves"]
