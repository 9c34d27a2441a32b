"""Drop-in check: the reference's OWN unit tests,
validation suite and acceptance criteria, compiled unmodified against the
B200-backed metagrad/{moment2,meta,adam}.hpp (include/metagrad_gpu), pass
on the GPU.  Built by tests/cpp/dropin/Makefile (needs the reference
sources, so it is built in the development container by
__graft_entry__.build(); the binaries travel with the repo snapshot)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BUILD = os.path.join(os.path.dirname(__file__), "cpp", "_build", "dropin")


def _run(args, timeout=900):
    exe = os.path.join(BUILD, args[0])
    if not os.path.exists(exe):
        pytest.skip("drop-in binaries not built (tests/cpp/dropin needs the reference sources)")
    p = subprocess.run([exe] + args[1:], capture_output=True, text=True, timeout=timeout)
    return p.returncode, p.stdout + p.stderr


@pytest.mark.parametrize("suite", ["test_moment2", "test_meta", "test_adam", "test_problems",
                                   "test_harness"])
def test_reference_unit_tests_on_gpu_estimators(suite):
    # CLI cases need CLI11, absent from the reference checkout (excluded as
    # in oracle/ref/Makefile `check`)
    rc, out = _run([suite, "--exclude=cli"])
    assert rc == 0, out[-3000:]
    assert "0 failed" in out, out[-3000:]


def test_reference_validation_suite_on_gpu_estimators():
    rc, out = _run(["validate"])
    assert rc == 0, out[-3000:]


@pytest.mark.parametrize("criterion", [str(i) for i in range(1, 10)])
def test_reference_acceptance_on_gpu_estimators(criterion):
    rc, out = _run(["acceptance", criterion], timeout=1500)
    assert rc == 0, out[-3000:]


def test_gpu_problem_adapters_match_reference_samplers():
    """metagrad_gpu::{MiniRenderProblem, ExpRateProblem, MultNoiseQuadratic}
    (device sample_pair behind the reference's Problem interface) vs the
    reference's CPU samplers on twin Rngs (tests/cpp/dropin/test_gpu_problems.cpp)."""
    rc, out = _run(["test_gpu_problems"])
    assert rc == 0, out[-3000:]
    assert "0 failed" in out, out[-3000:]
