#!/bin/bash
# Run the GPU test groups one by one, each under its own timeout (a hung kernel only costs its group).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/env.txt; nproc >> gpurun_out/env.txt; nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv >> gpurun_out/env.txt
for grp in "$@"; do
  echo "=== group: $grp" >> gpurun_out/gpu_tests.log
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "$grp" -p no:cacheprovider -rf 2>&1 | tail -40 >> gpurun_out/gpu_tests.log
  echo "exit=$?" >> gpurun_out/gpu_tests.log
done
