"""Repeatability study of the tensor-core sketch (study tool, not product): runs each Hartley / cosine /
Gaussian case R times on fresh workspaces and counts the runs whose Y differs from the fp64 oracle by more
than the parity bound (and from run 0 bitwise), printing the rows / columns of each bad run.
usage: python tools/repro_trig.py R [case ...]      (KS_LIB=path swaps the library for A/B runs)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1312_1869_b200 as ks  # noqa: E402
from _problems import desc_of, problem, relF  # noqa: E402

if os.environ.get("KS_LIB"):
    ks.library_path = os.path.abspath(os.environ["KS_LIB"])

CASES = [
    (2, dict(n=4096, d=128, dim=2)),
    (3, dict(n=3000, d=64, dim=1, kernel=1, ell=0.05)),
    (2, dict(n=1000, d=16, dim=3)),
    (3, dict(n=8192, d=256, dim=2)),
    (2, dict(n=5000, d=96, dim=2, kernel=1)),
    (1, dict(n=3000, d=64, dim=1, kernel=1, ell=0.05)),
    (1, dict(n=20000, d=128, dim=2)),
]


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    pick = [int(a) for a in sys.argv[2:]] or range(len(CASES))
    cuda = torch.device("cuda:0")
    print(f"library {ks.library_path}", flush=True)
    for ci in pick:
        omega, over = CASES[ci]
        cfg, pts, A, prob = problem("c2", omega=omega, seed=4321 + over["n"], **over)
        Yref = prob.sketch_rows()
        P = torch.from_numpy(np.ascontiguousarray(pts, np.float32)).to(cuda)
        first, errs, ndiff, nbad = None, [], 0, 0
        sk = ks.Sketch(desc_of(cfg), cuda)
        for r in range(R):
            if r % 10 == 0:
                sk = ks.Sketch(desc_of(cfg), cuda)
            Y = sk(P).cpu().numpy()
            errs.append(relF(Y, Yref))
            if first is None:
                first = Y
            elif not np.array_equal(Y, first):
                ndiff += 1
            if errs[-1] > 1e-5:
                nbad += 1
                big = np.abs(Y - Yref) > 1e-4 * np.abs(Yref).max()
                rows, cols = np.nonzero(big.any(axis=1))[0], np.nonzero(big.any(axis=0))[0]
                print(f"  run {r}: relF {errs[-1]:.3e}, rows {rows.min()}..{rows.max()} ({len(rows)}), "
                      f"cols {cols.min()}..{cols.max()} ({len(cols)})", flush=True)
        print(f"case {ci} omega {omega} {over}: {nbad}/{R} runs above 1e-5 (relF min {min(errs):.3e} max "
              f"{max(errs):.3e}); {ndiff}/{R - 1} differ from run 0", flush=True)


if __name__ == "__main__":
    main()
