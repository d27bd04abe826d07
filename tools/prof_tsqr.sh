cd $GRAFT_REPO_ROOT; out=gpurun_out/tsqrprof; mkdir -p $out
python tools/tsqr_one.py 512 262144 8 3 > $out/plain.log 2>&1
ncu --clock-control none --set full --import-source on -k regex:k_panel_apply_staged -c 1 -o $out/apply_leaf python tools/tsqr_one.py > $out/ncu1.log 2>&1
ncu --clock-control none --set full --import-source on -k regex:k_panel_qr -c 2 -o $out/qr python tools/tsqr_one.py > $out/ncu2.log 2>&1
ncu --clock-control none --set full --import-source on -k regex:k_panel_apply_staged --launch-skip 96 -c 1 -o $out/apply_q python tools/tsqr_one.py > $out/ncu3.log 2>&1
ls -la $out
