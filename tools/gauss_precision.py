"""Diagnostic: relative Frobenius error of the tcgen05 Gaussian sketch vs the fp64 oracle as n grows
(c3 parameters, sampled rows).  Error growing ~linearly in n points at the accumulator, not the
operand split.  Usage (GPU box): python tools/gauss_precision.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1312_1869_b200 as ks  # noqa: E402
from _problems import desc_of, problem, relF  # noqa: E402

dev = torch.device("cuda:0")
for n in [int(a) for a in (sys.argv[1:] or ["2048", "8192", "16384", "32768", "65536"])]:
    cfg, pts, A, prob = problem("c3", n=n)
    Y = ks.Sketch(desc_of(cfg), dev)(torch.as_tensor(pts, device=dev)).cpu().numpy()
    rows = np.sort(np.random.default_rng(0).choice(n, size=48, replace=False))
    Yr = prob.sketch_rows(rows)
    print(f"n={n:6d}  relF(Y)={relF(Y[rows], Yr):.3e}", flush=True)
