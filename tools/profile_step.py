"""One warm pass of the hot path for a config (for ncu launch lists / captures).
Usage: python tools/profile_step.py c4 [--passes 1] [--warm 1]"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ks_inputs  # noqa: E402
from paper_1312_1869_b200 import dist as ksd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--passes", type=int, default=1)
ap.add_argument("--warm", type=int, default=1)
a = ap.parse_args()
cfg, pts, A = ks_inputs.make_problem(a.config)
dev = torch.device("cuda:0")
desc = dict(n=cfg["n"], dim=cfg["dim"], kernel=cfg["kernel"], sigma2=cfg["sigma2"], ell=cfg["ell"],
            nugget=cfg["nugget"], d=cfg["d"], seed=cfg["seed"], omega=cfg["omega"])
ops = ksd.CudaOps(desc, cfg["m"], cfg["blocks"], 1e-5, 0, 1, dev, inplace=True)
P = torch.as_tensor(pts, device=dev)
Ad = torch.as_tensor(A, device=dev)
for _ in range(a.warm + a.passes):
    ksd.lowrank_solve_sharded(ops, P, Ad)
torch.cuda.synchronize()
print("ok", a.config)
