#!/bin/bash
# Build in-tree (nvcc cross-compile), then run a command on the GPU box.
# usage: scripts/gpurun.sh <timeout_s> '<command>'
set -e
cd /root/repo
python paper_2005_09824_b200/_build.py > /tmp/build.log 2>&1 || { tail -30 /tmp/build.log; exit 1; }
make -s -C oracle
/usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
