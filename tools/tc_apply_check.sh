#!/bin/bash
# TSQR with the tcgen05 leaf apply (default) vs the SIMT one (KS_TSQR_TC=0): parity tests + c4/c3/c2 timing.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tsqr or lowrank or solve or inplace or host" > gpurun_out/tc_tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/tc_tests.txt
for cfg in "512 262144 8" "256 65536 16" "128 16384 8"; do
  echo "== $cfg default(tc)" >> gpurun_out/tc_timing.txt
  timeout 120 python tools/tsqr_one.py $cfg 5 >> gpurun_out/tc_timing.txt 2>&1
  echo "== $cfg KS_TSQR_TC=0" >> gpurun_out/tc_timing.txt
  KS_TSQR_TC=0 timeout 120 python tools/tsqr_one.py $cfg 5 >> gpurun_out/tc_timing.txt 2>&1
done
