#!/bin/bash
# Reference arm + reference test-suite (both git-ignored under baseline/_ref,
# both travel to the GPU box with the gpurun snapshot):
#   baseline/_ref/chainloss   the unmodified reference package (bench.py --impl reference)
#   baseline/_ref/tests_ref   its own pkg/tests, run on the GPU through the kernel seam
#                             (tests/test_reference_suite_seam.py)
set -e
cd "$(dirname "$0")/.."
python -m pip install --no-index --no-build-isolation --no-deps --target baseline/_ref /root/reference/pkg
rm -rf baseline/_ref/tests_ref
cp -r /root/reference/pkg/tests baseline/_ref/tests_ref
