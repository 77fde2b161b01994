"""The reference's OWN test-suite (pkg/tests, 178 tests) on the GPU.

SURVEY.md §8(b)2: rebinding the reference's kernel seam to the C-ABI moves its
whole orchestration onto this repository's f64 parity kernels
(``lfmmi_{forward,backward,posterior}_kernel``) with no test edits.  The suite
is copied next to the reference install (``scripts/install_reference.sh`` ->
``baseline/_ref/tests_ref``, git-ignored, shipped to the GPU box) and run in a
subprocess with ``tests/seam_plugin.py`` installing the seam first.

Bitwise assertions: the parity kernels follow the reference's
operation order with no FMA contraction, so none needs relaxing — every
reference test, including the bit-exact comparison with the sequential
transliteration (tests/test_forward_backward.py:75), must pass as written.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "tests_ref")


def test_reference_suite_through_gpu_seam(cuda, tmp_path):
    if not os.path.isdir(SUITE):
        pytest.skip("reference suite not installed (scripts/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, SUITE, ROOT, os.path.join(ROOT, "tests")])
    env.setdefault("NUMBA_CACHE_DIR", str(tmp_path / "numba"))
    log = tmp_path / "suite.log"
    report = tmp_path / "seam_calls.json"
    env["LFMMI_SEAM_REPORT"] = str(report)
    cmd = [sys.executable, "-m", "pytest", SUITE, "-q", "-p", "seam_plugin", "-p",
           "no:cacheprovider", "-x", "--tb=short"]
    r = subprocess.run(cmd, env=env, cwd=str(tmp_path), capture_output=True, text=True,
                       timeout=1800)
    log.write_text(r.stdout + r.stderr)
    tail = "\n".join((r.stdout + r.stderr).splitlines()[-30:])
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and " failed" not in r.stdout, tail
    import json

    calls = json.loads(report.read_text())  # the reference's kernels ran on the GPU
    assert calls["forward_kernel"] > 100 and calls["backward_kernel"] > 50, calls
    assert calls["posterior_kernel"] > 50, calls
