for s in 2 4 8 16 64; do echo "seg=$s"; KS_GAUSS_SEG=$s timeout 300 python tools/gauss_precision.py 8192 65536; done
