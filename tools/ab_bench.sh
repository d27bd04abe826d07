#!/bin/bash
# A/B: bench.py lines (sketch ms, step ms, roofline frac) for the in-tree library and each variant .so given.
# usage (GPU box): tools/ab_bench.sh "c4 c5" variant1 [variant2 ...]
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
cfgs=$1; shift
lib=paper_1312_1869_b200/libks_b200.so
cp $lib /tmp/ks_default.so
mkdir -p gpurun_out
for v in default "$@"; do
  if [ "$v" = default ]; then cp /tmp/ks_default.so $lib; else cp paper_1312_1869_b200/variants/$v.so $lib; fi
  for c in $cfgs; do
    st=3; [ "$c" = c5 ] && st=2
    timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.json 2>/tmp/ab.err
    python - "$v" "$c" <<'PY' >> gpurun_out/ab_bench.txt
import json, sys
try:
    d = json.loads(open('/tmp/ab.json').read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:>12s} {sys.argv[2]:>4s} step {d['ms_per_step']:9.3f} ms  sketch {d['sketch_ms']:9.3f} ms  "
          f"tsqr+q {d['phase_ms']['tsqr_qform']:7.3f}  solve {d['phase_ms']['solve']:6.3f}  frac {d['roofline']['frac']:.4f}  "
          f"sm {d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], sys.argv[2], "FAILED", e, open('/tmp/ab.err').read()[-500:])
PY
  done
done
cp /tmp/ks_default.so $lib
