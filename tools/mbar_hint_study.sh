#!/bin/bash
# mbarrier try_wait with / without the suspend-time hint (-DKS_MBAR_NO_HINT): Gaussian c3 sketch (full and the
# KS_GAUSS_DEBUG=3 skeleton), c3h, and the TC TSQR factor+Q.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/$1; shift; mkdir -p $out
lib=paper_1312_1869_b200/libks_b200.so
cp $lib /tmp/ks_cur.so
for v in cur "$@"; do
  if [ $v != cur ]; then cp paper_1312_1869_b200/variants/$v.so $lib.tmp; mv $lib.tmp $lib; fi
  for cfg in c3 c3h; do for dbg in 0 3; do
    KS_GAUSS_DEBUG=$dbg timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $cfg KS_GAUSS_DEBUG=$dbg sketch', round(d['sketch_ms'],4))" >> $out/timing.txt
  done; done
  timeout 60 python tools/tsqr_one.py 512 262144 8 6 2>&1 | tail -1 | sed "s/^/$v c4 tsqr /" >> $out/timing.txt
  cp /tmp/ks_cur.so $lib.tmp; mv $lib.tmp $lib
done
