"""Second-level TSQR merge timing (the multi-GPU critical path): QR + Q2 of P stacked d x d R's
through a persistent plan (CUDA-graph replay, as dist.CudaOps), flat single block vs the pairwise tree with
triangular blocks.  Usage (GPU box): python tools/merge_timing.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1312_1869_b200 as ks  # noqa: E402

dev = torch.device("cuda:0")
for d in (512, 256):
    for P in (2, 4, 8):
        rng = np.random.default_rng(P + d)
        st = np.concatenate([np.linalg.qr(rng.standard_normal((2 * d, d)), mode="r") for _ in range(P)], 0)
        S = torch.as_tensor(st.astype(np.float32), device=dev)
        Q2 = torch.empty_like(S)
        R = torch.empty((d, d), device=dev)
        line = f"d={d} P={P}:"
        for name, blocks, topo in (("flat", 1, ks.TSQR_TREE), ("flat-tri", 1, ks.TSQR_TREE | ks.TSQR_TRIANGULAR),
                                   ("pairwise-tri", P, ks.TSQR_TREE | ks.TSQR_TRIANGULAR),
                                   ("pairwise", P, ks.TSQR_TREE)):
            plan = ks.TsqrPlan(P * d, d, blocks, dev, topology=topo)
            for _ in range(3):
                plan.factor(S, Q2, R)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(10):
                a.record(); plan.factor(S, Q2, R); b.record(); b.synchronize()
                ts.append(a.elapsed_time(b))
            line += f"  {name} {np.median(ts):.3f} ms"
        print(line, flush=True)
