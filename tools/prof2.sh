#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-prof2}; mkdir -p $out
echo "== gauss 2cta precision" > $out/log.txt
timeout 180 python tools/gauss_precision.py 2048 8192 65536 >> $out/log.txt 2>&1; echo "exit=$?" >> $out/log.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c3 or gauss or omega or randomness" >> $out/log.txt 2>&1; echo "exit=$?" >> $out/log.txt
timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $out/bench_c3.log 2>&1
KS_GAUSS_1CTA=1 timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $out/bench_c3_1cta.log 2>&1
NCU="ncu --clock-control none --set full --import-source on"
python tools/profile_step.py c4 > /dev/null 2>&1 && \
$NCU -k regex:k_sketch_srht -c 1 -o $out/srht_c4 python tools/profile_step.py c4 --warm 0 > $out/ncu1.log 2>&1
$NCU -k regex:"k_leaf_factor|k_leaf_applyq|k_tree_qr|k_tree_apply" -s 8 -c 4 -o $out/tsqr_c4 python tools/profile_step.py c4 --warm 0 > $out/ncu2.log 2>&1
$NCU -k regex:k_sketch_gauss -c 1 -o $out/gauss2_c3 python tools/profile_step.py c3 --warm 0 > $out/ncu3.log 2>&1
ls -la $out >> $out/log.txt
