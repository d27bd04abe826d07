#!/bin/bash
# Timing study of the staged apply: phases switched off by KS_APPLY_DEBUG bits (results wrong, timing only).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-applystudy}; mkdir -p $out
for b in 0 1 2 3 4 7; do echo "dbg=$b $(KS_APPLY_DEBUG=$b python tools/tsqr_one.py 512 262144 8 3 | tail -1)"; done > $out/study.txt 2>&1
cat $out/study.txt
