"""Can the TSQR of one row block run concurrently with the sketch of the next?  c4: the sketch of 1/8 of the rows
on one stream and the TSQR (+Q) of a 32768 x 512 block on a second (optionally high-priority) stream.
Usage (GPU box): python tools/overlap_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import ks_inputs  # noqa: E402
import paper_1312_1869_b200 as ks  # noqa: E402

dev = torch.device("cuda:0")
cfg, pts, A = ks_inputs.make_problem("c4")
desc = dict(n=cfg["n"], dim=cfg["dim"], kernel=cfg["kernel"], sigma2=cfg["sigma2"], ell=cfg["ell"],
            nugget=cfg["nugget"], d=cfg["d"], seed=cfg["seed"], omega=cfg["omega"])
sk = ks.Sketch(desc, dev)
P = torch.as_tensor(pts, device=dev)
rows = cfg["n"] // 8
Yb = torch.empty((rows, 512), device=dev)
Y0 = torch.randn(rows, 512, device=dev)
plan = ks.TsqrPlan(rows, 512, 1, dev)
Q = torch.empty_like(Y0)
R = torch.empty((512, 512), device=dev)
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
s1 = torch.cuda.Stream(device=dev)
for prio in (0, -1, -2, -5):
    s2 = torch.cuda.Stream(device=dev, priority=prio)
    def sk_blk(i, st):
        ks.ks_sketch(desc, P, i * rows, (i + 1) * rows, Yb, sk.ws, st)
    def ts(st):
        ks.ks_tsqr(plan.h, Y0, Q, R, st)
    for _ in range(2):   # warm (graph capture)
        sk_blk(1, s1); ts(s2)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    e[0].record(s1); sk_blk(1, s1); e[1].record(s1); torch.cuda.synchronize()
    e[2].record(s2); ts(s2); e[3].record(s2); torch.cuda.synchronize()
    e[4].record(s1); s2.wait_event(e[4]); sk_blk(1, s1); ts(s2); s1.wait_stream(s2); e[5].record(s1)
    torch.cuda.synchronize()
    a, b, c = e[0].elapsed_time(e[1]), e[2].elapsed_time(e[3]), e[4].elapsed_time(e[5])
    print(f"priority {prio}: sketch block {a:.2f} ms, TSQR+Q block {b:.2f} ms, both concurrently {c:.2f} ms "
          f"(sum {a + b:.2f}, saved {a + b - c:.2f})", flush=True)
