#!/bin/bash
# Build in-tree (nvcc cross-compile) and refuse to ship a stale build; then run
# a command on the GPU box.   usage: scripts/gpurun.sh <timeout_s> '<command>'
set -e
cd /root/repo
python paper_2005_09824_b200/_build.py > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head -20; exit 1; }
make -s -C oracle
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
