#!/bin/bash
# ncu launch list of the default bench command and one full capture per top
# kernel (GPU box; each only after the plain bench exited 0)
mkdir -p gpurun_out
NCU="ncu --clock-control none"
timeout 600 $NCU --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launch.log 2>&1
cap() {  # name config kernel-regex skip   (summaries only: reports stay on the box)
  timeout 900 $NCU --set full --import-source on -k regex:"$3" -s $4 -c 1 -o /tmp/ncu_$1 \
    python bench.py --config $2 --steps 1 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_$1.log 2>&1
  { python tools/ncu_summary.py /tmp/ncu_$1.ncu-rep; python tools/sass_hist.py /tmp/ncu_$1.ncu-rep 16; } \
    > gpurun_out/ncu_$1_summary.txt 2>&1
  rm -f /tmp/ncu_$1.ncu-rep
}
cap c2_subtree c2 subtree 2
cap c2_expand2 c2 expand2 2
cap c2_contract2 c2 contract2 2
cap c2_truth c2 truth_tiled 1
cap c5_truth c5 truth_bulk 1
cap c5_leaf c5 leaf_f32v 1
cap c4_leaf c4 h2dup 1
cap c3_contract c3 contract_dense 10
cap c3_leaf c3 leaf_smem 4
exit 0
