"""Resource budgets of the hot kernels, read from the built library's SASS
(cuobjdump, no GPU needed).  The two-pass chain loss depends on them: the
split denominator kernel takes 128 SMs and the numerator pass must keep all
128 WSJ-mono numerators resident on the 20 SMs left (7 CTAs of 128 threads
per SM -> <= 72 registers; at 75 the step went from 1.09 to 1.17 ms)."""

import os
import re
import shutil
import subprocess

import pytest

from paper_2005_09824_b200 import _backend

CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"


def _usage():
    path = _backend.core_library_path()
    if not os.path.exists(path) or not os.path.exists(CUOBJDUMP):
        pytest.skip("built library or cuobjdump not available")
    out = subprocess.run([CUOBJDUMP, "-res-usage", path], capture_output=True, text=True,
                         check=True).stdout
    res, name = {}, None
    for line in out.splitlines():
        m = re.match(r"\s*Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", line)
        if m and name:
            res[name] = tuple(int(x) for x in m.groups())
    return res


def _find(res, pattern):
    hits = {k: v for k, v in res.items() if re.search(pattern, k)}
    assert hits, f"no kernel matching {pattern}"
    return hits


def test_numerator_kernel_fits_seven_per_sm():
    for name, (reg, stack, local) in _find(_usage(), r"fb_tile_kernelIfLi128ELi1ELb1E").items():
        assert reg <= 72, f"{name}: {reg} registers (> 72: fewer than 7 numerators per SM)"
        assert stack == 0 and local == 0, f"{name}: spills"


def test_split_and_tile_den_kernels_do_not_spill():
    res = _usage()
    for pat in (r"fb_split_kernel", r"fb_tile_kernelIfLi512ELi1ELb1ELb0ELb1E"):
        for name, (reg, stack, local) in _find(res, pat).items():
            assert reg <= 128 and stack == 0 and local == 0, (name, reg, stack, local)
