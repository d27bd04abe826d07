#!/bin/bash
# ncu --set full of the SRHT sketch kernel (c4 and c5) on one warm pass of the hot path.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-srhtprof}; mkdir -p $out
for c in ${CONFIGS:-c4}; do
  timeout 900 ncu --clock-control none --set full --import-source on -k regex:k_sketch_srht -c 1 -o $out/srht_$c \
    python tools/profile_step.py $c --warm 0 > $out/ncu_$c.log 2>&1
done
ls $out
