mkdir -p gpurun_out
CONFIG=c2 bash tools/sweep_env.sh "RBC_SUBTREE_ROT=2" "RBC_SUBTREE_ROT=2 RBC_SUBTREE_SUB=2" > gpurun_out/sw2.txt 2>&1
RBC_NVCC_EXTRA="-DRBC_SUBTREE_ROT2_DROP=0" python -m paper_1905_07439_b200.build > gpurun_out/build_drop0.log 2>&1
CONFIG=c2 bash tools/sweep_env.sh "RBC_SUBTREE_ROT=2 RBC_TAG=drop0" >> gpurun_out/sw2.txt 2>&1
cat gpurun_out/sw2.txt
