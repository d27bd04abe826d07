#!/bin/bash
# Launch list (ncu gpu__time_duration) of one c4-sized TSQR factor + Q.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-tsqrl}; mkdir -p $out
KS_TSQR_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python tools/tsqr_one.py 512 262144 8 1 > $out/ncu.log 2>&1
python tools/launches.py $out/launches.csv > $out/launches.txt 2>&1; head -30 $out/launches.txt
