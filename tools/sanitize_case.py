"""Small end-to-end cases for compute-sanitizer (one tool per gpurun call, B200_PROFILING.md):
c1 (SRHT sketch + TSQR + solve), a 4096-row c3 (tcgen05 CTA-pair Gaussian sketch), a 16384 x 128 TSQR whose
leaf level runs the tcgen05 trailing update (k_leaf_apply_tc), and a small Nystrom core + core likelihood.
Usage (GPU box): compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ks_inputs  # noqa: E402
import paper_1312_1869_b200 as ks  # noqa: E402

dev = torch.device("cuda:0")


def desc_of(cfg):
    return dict(n=cfg["n"], dim=cfg["dim"], kernel=cfg["kernel"], sigma2=cfg["sigma2"], ell=cfg["ell"],
                nugget=cfg["nugget"], d=cfg["d"], seed=cfg["seed"], omega=cfg["omega"])


for name, over in (("c1", {}), ("c3", dict(n=4096, d=128, blocks=2, m=8))):
    cfg, pts, A = ks_inputs.make_problem(name, **over)
    pipe = ks.Pipeline(desc_of(cfg), cfg["m"], cfg["blocks"], device=dev)
    pipe(torch.as_tensor(pts, device=dev), torch.as_tensor(A, device=dev))
    torch.cuda.synchronize()
    print(name, "k", int(pipe.k.item()), flush=True)
Y = torch.randn(16384, 128, device=dev, generator=torch.Generator(device=dev).manual_seed(3))
plan = ks.TsqrPlan(16384, 128, 4, dev)
Q, R = plan.factor(Y)
torch.cuda.synchronize()
print("tsqr QR=Y", float(torch.linalg.norm(Q @ R - Y) / torch.linalg.norm(Y)), flush=True)
cfg, pts, A = ks_inputs.make_problem("c2", n=2048, d=64, blocks=2, m=4)
pipe = ks.Pipeline(desc_of(cfg), cfg["m"], cfg["blocks"], device=dev)
pipe(torch.as_tensor(pts, device=dev), torch.as_tensor(A, device=dev))
W, B = ks.nystrom_core(desc_of(cfg), torch.as_tensor(pts, device=dev), pipe.Q)
ll = ks.gp_loglik_core(pipe.Q, B, 0.01, torch.as_tensor(A[:, 0], device=dev))
torch.cuda.synchronize()
print("nystrom loglik", ll.cpu().numpy(), flush=True)
print("SANITIZE_CASE_OK")
