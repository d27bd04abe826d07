cd $GRAFT_REPO_ROOT
for t in 0 8 16 24 32; do echo "KS_TREE_SMS=$t" >> gpurun_out/treesms.txt; KS_TREE_SMS=$t python tools/tsqr_one.py 512 262144 8 4 2>&1 | tail -1 >> gpurun_out/treesms.txt; KS_TREE_SMS=$t python tools/tsqr_one.py 256 65536 16 4 2>&1 | tail -1 >> gpurun_out/treesms.txt; done
