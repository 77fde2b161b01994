"""compute-sanitizer over the hot-path kernels.

The kernels rely on intra-CTA protocols that determinism tests cannot prove
race-free: cp.async rings, double-buffered posterior slot buffers, one block
barrier per frame with deferred normalisation, chore warps, the split
kernel's __threadfence + cluster-barrier handoff, the stream kernel's DSMEM
exchange, the linear kernel's warp-synchronous histogram.  Each case
(scripts/sanitize_case.py) runs one short chain_loss under racecheck,
synccheck and memcheck, restricted to this library's kernels.
"""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
CASES = ["split", "tile", "tile1x", "tilep", "stream2", "stream1", "ring", "ssplit", "ssplit0",
         "hmm", "numtile", "lin16"]


@pytest.mark.parametrize("tool", ["racecheck", "synccheck", "memcheck"])
@pytest.mark.parametrize("case", CASES)
def test_sanitizer_clean(cuda, tool, case):
    if not os.path.exists(SAN):
        pytest.skip("compute-sanitizer not found")
    # this library's kernels only (fb_* and the combine kernel), not torch's
    # (the stream kernel's TMA ring holds up to 128 mbarriers per CTA)
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--num-cuda-barriers", "256",
           "--kernel-name", "kns=fb_",
           "--kernel-name", "kns=combine_kernel",
           sys.executable, os.path.join(ROOT, "scripts", "sanitize_case.py"), case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    tail = "\n".join(out.splitlines()[-25:])
    assert r.returncode == 0, tail
    assert f"case {case}:" in out, tail
    assert "ERROR SUMMARY: 0 errors" in out or "0 hazards" in out, tail
