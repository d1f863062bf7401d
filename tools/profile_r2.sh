#!/bin/bash
# Round-2 profiles (GPU box): launch list of the default bench command (c5)
# and full ncu captures of its top kernels.  Each runs only after the plain
# bench has exited 0.   usage: tools/profile_r2.sh [tag] [captures...]
mkdir -p gpurun_out
TAG=${1:-r02}; shift
NCU="ncu --clock-control none"
BENCH="python bench.py --no-cpu --no-e2e --no-tts --no-dropin"
if [ "$#" -eq 0 ]; then set -- launches c5_truth c5_leaf c5_expand; fi
cap() {  # name config kernel-regex skip
  timeout 900 $NCU --set full --import-source on -k regex:"$3" -s $4 -c 1 -o /tmp/ncu_$1 \
    $BENCH --config $2 --steps 1 --warmup 2 > gpurun_out/ncu_${TAG}_$1.log 2>&1
  { python tools/ncu_summary.py /tmp/ncu_$1.ncu-rep; python tools/sass_hist.py /tmp/ncu_$1.ncu-rep 16; } \
    > gpurun_out/ncu_${TAG}_$1_summary.txt 2>&1
  ncu -i /tmp/ncu_$1.ncu-rep --page details > gpurun_out/ncu_${TAG}_$1_details.txt 2>&1
  # reports stay on the box (gpurun copies back at most 64 MiB)
  rm -f /tmp/ncu_$1.ncu-rep
}
for c in "$@"; do
  case $c in
    launches) timeout 900 $NCU --metrics gpu__time_duration.sum --csv \
                --log-file gpurun_out/launches_${TAG}_c5.csv $BENCH --steps 2 --warmup 3 \
                > gpurun_out/ncu_${TAG}_launch.log 2>&1 ;;
    c5_truth) cap c5_truth c5 truth_bulk 1 ;;
    c5_leaf) cap c5_leaf c5 leaf_f32v 1 ;;
    c5_expand) cap c5_expand c5 "expand_plan" 1 ;;
    c2_subtree) cap c2_subtree c2 subtree 2 ;;
    # per pair: the deterministic product (1 product) then the 32 randomized ones
    c3_leaf) cap c3_leaf c3 leaf_ring 5 ;;
    c3_expand) cap c3_expand c3 expand_dense 8 ;;
    c3_contract) cap c3_contract c3 contract_dense 3 ;;
    c4_leaf) cap c4_leaf c4 h2dup 1 ;;
    c2_truth) cap c2_truth c2 truth_tiled 1 ;;
  esac
done
exit 0
