#!/bin/bash
# Lane overlap and host-buffer pipeline experiments (GPU box):
#   step time under the lane priority modes, serial lanes, and truth tile
#   variants; e2e call times under RBC_E2E_SLOTS.
mkdir -p gpurun_out
CONFIG=c2 bash tools/sweep_env.sh "RBC_LANE_PRIO=0" "RBC_LANE_PRIO=1" "RBC_LANE_PRIO=2" \
  "RBC_SERIAL_LANES=1" "RBC_LEAF_TILE=305" "RBC_LANE_PRIO=2 RBC_LEAF_TILE=305" "RBC_SUBTREE_SUB=2" "RBC_SUBTREE_SUB=3"
for s in 3 5 7; do
  echo "RBC_E2E_SLOTS=$s"; RBC_E2E_SLOTS=$s python tools/e2e_probe.py c2 2>&1 | tail -2
done
