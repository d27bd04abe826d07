#!/bin/bash
# factor+Q timing (c4 / c3 / c2 shapes) of each variant .so given (no tests), and the phase timeline of each
# variant whose name ends in "t" (a KS_TC_TIMING build).  usage (GPU box): tools/tc_variant_timing.sh <outdir> v1 [v2 ...]
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/$1; shift; mkdir -p $out
lib=paper_1312_1869_b200/libks_b200.so
cp $lib /tmp/ks_cur.so
for v in "$@"; do
  case $v in
    *t) timeout 300 python tools/tc_stamps.py paper_1312_1869_b200/variants/$v.so > $out/stamps_$v.txt 2>&1 ;;
    *) cp paper_1312_1869_b200/variants/$v.so $lib.tmp; mv $lib.tmp $lib
       for cfg in "512 262144 8" "256 65536 16" "128 16384 8"; do
         echo "== $v $cfg" >> $out/timing.txt
         timeout 60 python tools/tsqr_one.py $cfg 6 2>&1 | tail -1 >> $out/timing.txt
       done
       cp /tmp/ks_cur.so $lib.tmp; mv $lib.tmp $lib ;;
  esac
done
