#!/bin/bash
# Timing study of the staged apply: phases compiled out by -DKS_APPLY_DEBUG bits (results wrong, timing only):
# bit 0 skips W1 = V^T X, bit 1 skips X -= V W2, bit 2 skips the tile write-back.  Rebuilds the library per case.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-applystudy}; mkdir -p $out
for b in 0 1 2 3 4 7; do
  NVCC_APPEND_FLAGS="-DKS_APPLY_DEBUG=$b" python -m paper_1312_1869_b200.build --force > /dev/null 2>&1
  echo "dbg=$b $(python tools/tsqr_one.py 512 262144 8 3 | tail -1)"
done > $out/study.txt 2>&1
python -m paper_1312_1869_b200.build --force > /dev/null 2>&1
cat $out/study.txt
