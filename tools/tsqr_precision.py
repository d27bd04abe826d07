"""R / Q accuracy of the GPU TSQR vs the fp64 oracle on the sketches of config-shaped problems (and random Y).
Usage (GPU box): python tools/tsqr_precision.py   (set KS_TSQR_TC=0 for the SIMT trailing update)"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import paper_1312_1869_b200 as ks  # noqa: E402
from _problems import align_rows, desc_of, problem, relF  # noqa: E402

dev = torch.device("cuda:0")
for name, over in (("c3", dict(n=8192, blocks=4)), ("c4", dict(n=8192, blocks=4)), ("c1", {}), ("c2", {})):
    cfg, pts, A, prob = problem(name, **over)
    sk = ks.Sketch(desc_of(cfg), dev)
    Y = sk(torch.as_tensor(pts, device=dev))
    plan = ks.TsqrPlan(cfg["n"], cfg["d"], cfg["blocks"], dev)
    Q, R = plan.factor(Y)
    torch.cuda.synchronize()
    Y64 = Y.cpu().numpy().astype(np.float64)
    Qr, Rr = oracle.tsqr_tree(Y64, cfg["blocks"], want_q=True)
    Rg, Qg = R.cpu().numpy().astype(np.float64), Q.cpu().numpy().astype(np.float64)
    d = cfg["d"]
    print(f"{name} n={cfg['n']} d={d}: R relF {relF(align_rows(Rg, Rr), Rr):.3e}  QR=Y {relF(Qg @ Rg, Y64):.3e}  "
          f"|QtQ-I| {np.linalg.norm(Qg.T @ Qg - np.eye(d)):.3e}  cond(R) {np.linalg.cond(Rr):.2e}", flush=True)
