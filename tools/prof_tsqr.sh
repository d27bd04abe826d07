#!/bin/bash
# ncu --set full captures of the TSQR kernels (first leaf-level QR, first leaf-level staged apply of the
# factorisation and of the Q formation) of one c4-sized factor + Q.
cd "${GRAFT_REPO_ROOT:-$(dirname $0)/..}"
out=gpurun_out/${1:-tsqrprof}; mkdir -p $out
NCU="ncu --clock-control none --set full --import-source on"
KS_TSQR_GRAPH=0 $NCU -k regex:k_panel_apply_staged -c 1 -o $out/apply_leaf python tools/tsqr_one.py > $out/ncu1.log 2>&1
KS_TSQR_GRAPH=0 $NCU -k regex:k_panel_qr -c 1 -o $out/qr python tools/tsqr_one.py > $out/ncu2.log 2>&1
KS_TSQR_GRAPH=0 $NCU -k regex:k_panel_apply_staged --launch-skip 90 -c 1 -o $out/apply_q python tools/tsqr_one.py > $out/ncu3.log 2>&1
ls $out
