cd $GRAFT_REPO_ROOT
for s in 16 24 32; do
  KS_GAUSS_SEG=$s timeout 300 python bench.py --config c3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/g.json 2>/dev/null
  python -c "
import json;d=json.loads(open('/tmp/g.json').read().strip().splitlines()[-1]);print('seg $s', round(d['sketch_ms'],3), round(d['roofline']['frac'],4))" >> gpurun_out/gseg.txt
  KS_GAUSS_SEG=$s timeout 300 python -m pytest tests/test_gpu_fullsize.py -k c3 -q -s 2>&1 | grep "c3:" >> gpurun_out/gseg.txt
done
