#!/bin/bash
# TSQR change check: TSQR / solve parity tests, then timing of one c4-sized factor+Q and a c4 bench line.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-tsqrchk}; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "tsqr or lowrank or apply or qform or cond or gp" > $out/tests.log 2>&1
echo "tests exit=$?" >> $out/tests.log
timeout 300 python tools/tsqr_one.py 512 262144 8 5 > $out/tsqr_one.log 2>&1
timeout 300 python tools/tsqr_timing.py > $out/tsqr_timing.log 2>&1
[ "$2" = "bench" ] && timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/bench.log 2>&1
tail -3 $out/tests.log; cat $out/tsqr_one.log $out/tsqr_timing.log; tail -c 600 $out/bench.log 2>/dev/null
