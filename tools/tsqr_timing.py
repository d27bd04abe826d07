"""TSQR timing on one GPU for the per-rank shares of a multi-GPU run (rows/P x d, blocks per rank) and the
cross-rank merge (P*d x d).  Usage (GPU box): python tools/tsqr_timing.py [d] [rows_total] [blocks_per_rank]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1312_1869_b200 as ks  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 512
n = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
bpr = int(sys.argv[3]) if len(sys.argv) > 3 else 8
dev = torch.device("cuda:0")


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for P in (1, 2, 4, 8):
    rows = n // P
    Y = torch.randn(rows, d, device=dev)
    plan = ks.TsqrPlan(rows, d, bpr, dev)
    Q = torch.empty(rows, d, device=dev)
    R = torch.empty(d, d, device=dev)
    t_f = timed(lambda: ks.ks_tsqr(plan.h, Y, None, R))
    t_fq = timed(lambda: ks.ks_tsqr(plan.h, Y, Q, R))
    line = f"P={P} rows/rank={rows} d={d} blocks/rank={bpr}: factor {t_f:.2f} ms, factor+Q {t_fq:.2f} ms"
    if P > 1:
        Rs = torch.randn(P * d, d, device=dev).triu_()
        mp = ks.TsqrPlan(P * d, d, 1, dev)   # as dist.py: one block of <= 512-row leaves, one flat merge
        Q2 = torch.empty(P * d, d, device=dev)
        t_m = timed(lambda: ks.ks_tsqr(mp.h, Rs, Q2, R))
        line += f", merge ({P * d}x{d}) {t_m:.2f} ms"
    print(line, flush=True)
