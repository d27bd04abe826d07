#!/bin/bash
# Gaussian-sketch A/B: parity tests of each variant .so (swapped in), bench lines c3 / c3h / p50k of the in-tree
# library and the variants, and the KS_GAUSS_DEBUG decomposition (1: no MMAs, 2: no producer arithmetic).
# usage (GPU box): tools/gauss_ab.sh <outdir> variant ...
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/$1; shift; mkdir -p $out
lib=paper_1312_1869_b200/libks_b200.so
cp $lib /tmp/ks_cur.so
for v in "$@"; do
  cp paper_1312_1869_b200/variants/$v.so $lib.tmp; mv $lib.tmp $lib
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gp.py tests/test_gpu_planted.py -q -x -k "sketch or trig or gauss or planted or nystrom or randomness or repeat" > $out/tests_$v.txt 2>&1
  echo "rc=$?" >> $out/tests_$v.txt
done
cp /tmp/ks_cur.so $lib.tmp; mv $lib.tmp $lib
rm -f gpurun_out/ab_bench.txt
bash tools/ab_bench.sh "c3 c3h p50k" "$@" > /dev/null 2>&1
mv gpurun_out/ab_bench.txt $out/ab_bench.txt
for dbg in 1 2 3; do
  KS_GAUSS_DEBUG=$dbg timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('KS_GAUSS_DEBUG=$dbg sketch', d['sketch_ms'])" >> $out/debug.txt
done
