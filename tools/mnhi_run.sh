cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/mnhi
timeout 60 tools/tc_probe4.bin > gpurun_out/mnhi/probe4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tsqr or lowrank or solve or inplace or host" > gpurun_out/mnhi/tests.txt 2>&1
echo "tests rc=$?" >> gpurun_out/mnhi/tests.txt
cp paper_1312_1869_b200/libks_b200.so /tmp/ks_new.so
for v in new mnhi0; do
  if [ $v = new ]; then cp /tmp/ks_new.so paper_1312_1869_b200/libks_b200.so; else cp paper_1312_1869_b200/variants/mnhi0.so paper_1312_1869_b200/libks_b200.so; fi
  for cfg in "512 262144 8" "256 65536 16" "128 16384 8"; do
    echo "== $v $cfg" >> gpurun_out/mnhi/timing.txt
    timeout 120 python tools/tsqr_one.py $cfg 5 2>&1 | tail -2 >> gpurun_out/mnhi/timing.txt
  done
done
cp /tmp/ks_new.so paper_1312_1869_b200/libks_b200.so
timeout 300 python tools/tsqr_precision.py > gpurun_out/mnhi/precision.txt 2>&1
