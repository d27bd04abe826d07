#!/bin/bash
# Summarize a gpu_run.sh output directory: tests, bench lines, launch list.
d=${1:-gpurun_out/r1f}
tail -1 $d/tests.log 2>/dev/null
for f in $d/bench_c*.log $d/bench.log; do [ -f $f ] || continue; grep "^{" $f | python3 -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['config']['workload'], 'step %.2f ms'%d['ms_per_step'], {k:round(v,2) for k,v in d['phase_ms'].items()}, 'e2e', d['e2e'] and round(d['e2e']['ms_per_step'],2), 'frac %.3f'%d['roofline']['frac'])
"; done
for f in $d/launches_*.csv; do [ -f $f ] && python3 tools/launches.py $f --last-frac 0.5 | head -12; done
