"""One TSQR factorisation + explicit Q of a random rows x d matrix (for ncu captures of the TSQR kernels).
Usage (GPU box): python tools/tsqr_one.py [d] [rows] [blocks] [reps]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1312_1869_b200 as ks  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
b = int(sys.argv[3]) if len(sys.argv) > 3 else 8
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
Y = torch.randn(n, d, device=dev, generator=g)
plan = ks.TsqrPlan(n, d, b, dev)
Q = torch.empty(n, d, device=dev)
R = torch.empty(d, d, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(reps):
    e0.record()
    ks.ks_tsqr(plan.h, Y, Q, R)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {r}: factor+Q {e0.elapsed_time(e1):.3f} ms", flush=True)
