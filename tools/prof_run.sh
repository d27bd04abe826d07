#!/bin/bash
# Profiling session: ALU microbench, launch list of one c4 pass, ncu --set full of the top kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-prof}; mkdir -p $out
NCU="ncu --clock-control none"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_alu.cu && /tmp/ub > $out/ubench.txt 2>&1
for c in c4 c3; do
  python tools/profile_step.py $c > $out/plain_$c.log 2>&1 && \
  $NCU --metrics gpu__time_duration.sum --csv --log-file $out/launches_$c.csv python tools/profile_step.py $c > $out/ncu_$c.log 2>&1
done
$NCU --set full --import-source on -k regex:k_sketch_srht -c 1 -o $out/srht_c4 python tools/profile_step.py c4 --warm 0 > $out/ncufull_srht.log 2>&1
$NCU --set full --import-source on -k regex:k_sketch_gauss -c 1 -o $out/gauss_c3 python tools/profile_step.py c3 --warm 0 > $out/ncufull_gauss.log 2>&1
$NCU --set full --import-source on -k regex:"k_leaf_factor|k_leaf_applyq|k_tree_factor|k_tree_applyq" -s 40 -c 4 -o $out/tsqr_c4 python tools/profile_step.py c4 --warm 0 > $out/ncufull_tsqr.log 2>&1
ls -la $out
