#!/bin/bash
# One GPU session: build check, smoke, parity tests, diagnostics, bench lines, ncu launch list.
# Usage: tools/gpu_run.sh <tag> [steps...]   steps: smoke tests prec bench bench_all ncu ncufull
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
tag=${1:-run}; shift
out=gpurun_out/$tag
mkdir -p $out
nvidia-smi -L > $out/env.txt; nproc >> $out/env.txt
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv >> $out/env.txt
for step in "$@"; do
  echo "=== $step $(date +%T)" >> $out/summary.txt
  case $step in
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1 ;;
    tests) timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -rf --timeout 600 > $out/tests.log 2>&1 ;;
    testsall) timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > $out/tests.log 2>&1 ;;
    prec) timeout 600 python tools/gauss_precision.py > $out/prec.log 2>&1 ;;
    bench) timeout 900 python bench.py --steps 5 --warmup 3 > $out/bench.log 2>&1 ;;
    bench_all) for c in c1 c2 c3 c4 c5; do
                 timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_$c.log 2>&1
               done ;;
    ncu) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
           --log-file $out/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu.log 2>&1 ;;
    ncufull) timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sketch -c 1 \
           -o $out/sketch python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncufull.log 2>&1 ;;
    *) eval "$step" >> $out/custom.log 2>&1 ;;
  esac
  echo "exit=$? $(date +%T)" >> $out/summary.txt
done
