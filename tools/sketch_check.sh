#!/bin/bash
# Sketch change check: sketch / randomness parity tests, then c4 and c5 bench lines (no e2e, no CPU baseline).
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-skchk}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_planted.py -m gpu -q -x -p no:cacheprovider -k "sketch or random or lowrank or planted" > $out/tests.log 2>&1
echo "tests exit=$?" >> $out/tests.log; tail -2 $out/tests.log
for c in ${CONFIGS:-c4 c5}; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $out/bench_$c.log 2>&1
  python -c "import json,sys; d=json.loads(open('$out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['phase_ms'], d['roofline']['frac'])"
done
