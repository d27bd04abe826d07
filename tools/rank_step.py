"""Per-rank step of a P-GPU run, measured on one B200: rank 0's exact kernel sequence (dist.CudaOps with world = P,
rows [0, n/P)): sketch, local TSQR (R), the merge of the (P d) x d stack (filled with copies of the local R as a
stand-in for the all-gathered R's: the merge's cost does not depend on the values), Q_p = Q1 Q2_p, Q^T A, the
truncated solve, X = Omega Z; the two collectives (one d x d all-gather, one d x m all-reduce, ~10-30 us over
NVLink) are not included.  Usage (GPU box): python tools/rank_step.py c4 [P ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ks_inputs  # noqa: E402
from paper_1312_1869_b200 import dist as ksd  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
cfg, pts, A = ks_inputs.make_problem(name)
dev = torch.device("cuda:0")
desc = dict(n=cfg["n"], dim=cfg["dim"], kernel=cfg["kernel"], sigma2=cfg["sigma2"], ell=cfg["ell"],
            nugget=cfg["nugget"], d=cfg["d"], seed=cfg["seed"], omega=cfg["omega"])
P_d = torch.as_tensor(pts, device=dev)
res = {"config": name, "n": cfg["n"], "d": cfg["d"]}
for P in Ps:
    bpr = cfg["blocks"] if cfg.get("blocks_per_gpu") else max(1, cfg["blocks"] // P)
    ops = ksd.CudaOps(desc, cfg["m"], bpr, 1e-5, 0, P, dev, inplace=True)
    A_loc = torch.as_tensor(np.ascontiguousarray(A[ops.rb:ops.re]), device=dev)
    d = cfg["d"]

    def step():
        Y = ops.sketch(P_d)
        Rp = ops.local_r(Y)
        if P > 1:
            ops.Rstack.copy_(Rp.repeat(P, 1))
            Q2, R = ops.merge(ops.Rstack)
            Q = ops.qform(Q2[0:d].contiguous())
        else:
            R = Rp
            Q = ops.qform(None)
        Cm = ops.qt(Q, A_loc)
        Z, k = ops.trsolve(R, Cm)
        ops.omega_apply(Z)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); step(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    res[f"P{P}_rank_step_ms"] = float(np.median(ts))
t1 = res.get("P1_rank_step_ms")
if t1:
    for P in Ps:
        if P > 1:
            res[f"P{P}_projected_strong_eff"] = t1 / (P * res[f"P{P}_rank_step_ms"])
print(json.dumps(res))
