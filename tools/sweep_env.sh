#!/bin/bash
# Time the c2 fused-subtree stage under several env settings (run on the GPU box):
#   tools/sweep_env.sh "RBC_A=1 RBC_B=2" "RBC_A=0" ...
for cfg in "$@"; do
  env $cfg python bench.py --no-cpu --no-e2e --steps 5 > gpurun_out/sweep.json 2>gpurun_out/sweep.err || { echo "$cfg FAILED"; tail -3 gpurun_out/sweep.err; continue; }
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/sweep.json"))
r = d["roofline"]
print(f"{sys.argv[1]:40s} step {d['ms_per_step']:.3f} ms  subtree {r['avg_launch_ms']:.3f} ms/launch")
PY
done
