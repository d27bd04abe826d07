"""Bitwise repeatability stress of the GPU kernels at config sizes (study tool, not product): every kernel of the
path is deterministic (fixed reduction orders, no atomics), so a run that differs from run 0 exposes a race.
  TSQR factor + Q (tcgen05 leaf apply, node levels) at the c4 / c3 / c2 shapes,
  the sketch at full c3 (Gaussian, CTA pairs), c2 / c4 (SRHT), and the whole Pipeline at c2.
usage (GPU box): python tools/stress_repeat.py [reps_scale]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import ks_inputs  # noqa: E402
import paper_1312_1869_b200 as ks  # noqa: E402
from _problems import desc_of  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
dev = torch.device("cuda:0")


def report(name, runs, bad):
    print(f"{name}: {bad} of {runs} runs differ from run 0", flush=True)


for (rows, d, blocks, reps) in [(262144, 512, 8, 40), (65536, 256, 16, 150), (16384, 128, 8, 300)]:
    reps = max(2, int(reps * scale))
    g = torch.Generator(device=dev).manual_seed(rows + d)
    Y = torch.randn(rows, d, device=dev, generator=g)
    plan = ks.TsqrPlan(rows, d, blocks, dev)
    Q0, R0 = (t.clone() for t in plan.factor(Y))
    bad = 0
    for _ in range(reps - 1):
        Q, R = plan.factor(Y)
        bad += int(not (bool((Q == Q0).all()) and bool((R == R0).all())))
    report(f"tsqr factor+Q {rows}x{d} blocks {blocks}", reps, bad)

for name, reps in [("c3", 20), ("c2", 100), ("c4", 4)]:
    reps = max(2, int(reps * scale))
    cfg, pts, A = ks_inputs.make_problem(name)
    sk = ks.Sketch(desc_of(cfg), dev)
    P = torch.as_tensor(np.ascontiguousarray(pts), device=dev)
    Y0 = sk(P).clone()
    Y = torch.empty_like(Y0)
    bad = 0
    for _ in range(reps - 1):
        sk(P, Y=Y)
        bad += int(not bool((Y == Y0).all()))
    report(f"sketch {name} (omega {cfg['omega']})", reps, bad)

cfg, pts, A = ks_inputs.make_problem("c2")
pipe = ks.Pipeline(desc_of(cfg), cfg["m"], cfg["blocks"], device=dev)
P = torch.as_tensor(np.ascontiguousarray(pts), device=dev)
Ad = torch.as_tensor(np.ascontiguousarray(A), device=dev)
X0 = pipe(P, Ad).clone()
reps, bad = max(2, int(100 * scale)), 0
for _ in range(reps - 1):
    bad += int(not bool((pipe(P, Ad) == X0).all()))
report("Pipeline c2 (X)", reps, bad)
