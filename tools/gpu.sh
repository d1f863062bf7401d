#!/bin/bash
# Build in-tree, then run a command on the B200 box:  tools/gpu.sh <timeout_s> '<command>'
set -e
cd /root/repo
python -m paper_1905_07439_b200.build > /dev/null
T=${1:-900}; shift
exec /usr/local/graft/bin/gpurun --timeout "$T" -- "$@"
