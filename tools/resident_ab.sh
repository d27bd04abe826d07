#!/bin/bash
# TSQR parity tests, then factor+Q timing with the resident node levels (default) and without (KS_TSQR_RESIDENT=0).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/$1; mkdir -p $out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py tests/test_gpu_gp.py -x -q -k "tsqr or lowrank or solve or inplace or host or full or repeat or world2 or merge or nystrom or qform" > $out/tests.txt 2>&1
echo "tests rc=$?" >> $out/tests.txt
for env in "KS_TSQR_RESIDENT=1" "KS_TSQR_RESIDENT=0"; do
  for cfg in "512 262144 8" "256 65536 16" "128 16384 8" "64 2048 4"; do
    echo "== $env $cfg" >> $out/timing.txt
    env $env timeout 60 python tools/tsqr_one.py $cfg 6 2>&1 | tail -1 >> $out/timing.txt
  done
done
