#!/bin/bash
# ncu of the tcgen05 leaf apply: the first factor launch (--set full) and the launch list of one c4 factor + Q
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-tcprof}; mkdir -p $out
NCU="ncu --clock-control none --set full --import-source on"
KS_TSQR_GRAPH=0 $NCU -k regex:k_leaf_apply_tc -c 1 -o $out/tc_first python tools/tsqr_one.py > $out/ncu1.log 2>&1
KS_TSQR_GRAPH=0 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches.csv python tools/tsqr_one.py > $out/ncu2.log 2>&1
KS_TSQR_GRAPH=0 KS_TSQR_TC=0 ncu --clock-control none --metrics gpu__time_duration.sum --csv --log-file $out/launches_simt.csv python tools/tsqr_one.py > $out/ncu3.log 2>&1
ls $out
