#!/bin/bash
# TSQR parity tests + repeatability of the in-tree library, factor+Q timing (c4 / c3 / c2 shapes) of the
# in-tree library and of each variant .so given, and the phase timeline of the KS_TC_TIMING variant.
# usage (GPU box): tools/tc_apply_ab.sh <outdir> [variant ...]
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/$1; shift; mkdir -p $out
timeout 420 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "tsqr or lowrank or solve or inplace or host or full or repeat" > $out/tests.txt 2>&1
echo "tests rc=$?" >> $out/tests.txt
lib=paper_1312_1869_b200/libks_b200.so
cp $lib /tmp/ks_cur.so
for v in cur "$@"; do
  if [ $v = cur ]; then cp /tmp/ks_cur.so $lib.tmp; else cp paper_1312_1869_b200/variants/$v.so $lib.tmp; fi
  mv $lib.tmp $lib
  for cfg in "512 262144 8" "256 65536 16" "128 16384 8"; do
    echo "== $v $cfg" >> $out/timing.txt
    timeout 60 python tools/tsqr_one.py $cfg 6 2>&1 | tail -2 >> $out/timing.txt
  done
done
cp /tmp/ks_cur.so $lib.tmp; mv $lib.tmp $lib
[ -f paper_1312_1869_b200/variants/tctime.so ] && timeout 300 python tools/tc_stamps.py paper_1312_1869_b200/variants/tctime.so > $out/stamps.txt 2>&1
