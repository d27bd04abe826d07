cd $GRAFT_REPO_ROOT
lib=paper_1312_1869_b200/libks_b200.so
cp $lib /tmp/ks_cur.so
for v in cur relaxed; do
  if [ $v = relaxed ]; then cp paper_1312_1869_b200/variants/relaxed.so $lib.tmp; mv $lib.tmp $lib; fi
  for dbg in 0 3 7; do
    KS_GAUSS_DEBUG=$dbg timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v KS_GAUSS_DEBUG=$dbg sketch', d['sketch_ms'])" >> gpurun_out/relax.txt
  done
done
cp /tmp/ks_cur.so $lib.tmp; mv $lib.tmp $lib
