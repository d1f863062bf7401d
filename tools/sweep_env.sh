#!/bin/bash
# Time one config's stages under several env settings (run on the GPU box):
#   CONFIG=c2 tools/sweep_env.sh "RBC_A=1 RBC_B=2" "RBC_A=0" ...
# Prints step time and ms per launch of every profiled stage.
for cfg in "$@"; do
  env $cfg python bench.py --config ${CONFIG:-c2} --no-cpu --no-e2e --steps 5 > gpurun_out/sweep.json 2>gpurun_out/sweep.err || { echo "$cfg FAILED"; tail -3 gpurun_out/sweep.err; continue; }
  python - "$cfg" <<'PY'
import json, sys
d = json.load(open("gpurun_out/sweep.json"))
r = d["roofline"]
st = " ".join(f"{k} {v['ms'] / v['count']:.3f}" for k, v in r["stages"].items())
print(f"{sys.argv[1]:40s} step {d['ms_per_step']:.3f} ms | ms/launch: {st}")
PY
done
