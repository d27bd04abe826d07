#!/bin/bash
# Bench lines of the NEXT rows (planted-spectrum stored-K sweep, Hartley / cosine c3) and the NEXT-4 timing.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-nextrows}; mkdir -p $out
for c in p1k p5k p10k p50k p50kh p50kc p50ks c3h c3c; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > $out/bench_$c.log 2>&1
done
timeout 600 python tools/next4_timing.py > $out/next4.log 2>&1; timeout 600 python tools/next4_timing.py c3 >> $out/next4.log 2>&1; timeout 600 python tools/next4_timing.py c2 >> $out/next4.log 2>&1
for c in p1k p5k p10k p50k p50kh p50kc p50ks c3h c3c; do
  python -c "import json; l=[x for x in open('$out/bench_$c.log').read().splitlines() if x.startswith('{')][-1]; d=json.loads(l); print('$c', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phase_ms'].items()}, d['roofline']['bound'], round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
tail -3 $out/next4.log
