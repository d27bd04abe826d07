#!/bin/bash
# Round-end evidence: smoke, GPU tests, bench lines c1-c5 + default, c4 launch list, ncu --set full of the top
# kernels (SRHT c4 / c5, TSQR apply + panel QR, Gaussian c3).  Usage: tools/round_profiles.sh <tag>
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
tag=${1:-rp}; out=gpurun_out/$tag; mkdir -p $out
nvidia-smi -L > $out/env.txt; nproc >> $out/env.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit=$?" >> $out/summary.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --timeout 600 > $out/tests.log 2>&1; echo "tests exit=$?" >> $out/summary.txt
timeout 900 python bench.py --steps 5 --warmup 3 > $out/bench_default.log 2>&1; echo "bench exit=$?" >> $out/summary.txt
for c in ${CONFIGS:-c1 c2 c3 c4 c5}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $out/bench_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file $out/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $out/ncu_launch.log 2>&1
python tools/launches.py $out/launches_c4.csv > $out/launches_c4.txt 2>&1
NCU="ncu --clock-control none --set full --import-source on"
timeout 900 $NCU -k regex:k_sketch_srht -c 1 -o $out/srht_c4 python tools/profile_step.py c4 --warm 0 > $out/ncu1.log 2>&1
timeout 900 $NCU -k regex:k_sketch_srht -c 1 -o $out/srht_c5 python tools/profile_step.py c5 --warm 0 > $out/ncu2.log 2>&1
timeout 900 $NCU -k regex:k_sketch_gauss -c 1 -o $out/gauss_c3 python tools/profile_step.py c3 --warm 0 > $out/ncu3.log 2>&1
KS_TSQR_GRAPH=0 timeout 900 $NCU -k regex:k_leaf_apply_tc -c 1 -o $out/apply_leaf python tools/tsqr_one.py > $out/ncu4.log 2>&1
KS_TSQR_GRAPH=0 timeout 900 $NCU -k regex:k_panel_qr -c 1 -o $out/panel_qr python tools/tsqr_one.py > $out/ncu5.log 2>&1
KS_TSQR_GRAPH=0 timeout 900 $NCU -k regex:k_qtx_fast -c 1 -o $out/qtx python tools/profile_step.py c4 --warm 0 > $out/ncu6.log 2>&1
echo "done" >> $out/summary.txt
