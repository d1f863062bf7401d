#!/bin/bash
# Every BASELINE config's bench line (+ the reference arm on c2) into gpurun_out/ (GPU box)
mkdir -p gpurun_out
for c in c2 c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err || echo "bench $c failed"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
python tools/matgen_bench.py > gpurun_out/matgen_bench.jsonl 2>&1
