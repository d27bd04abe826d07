"""NEXT-4 timing on the c4 shape: Theorem 5 diagnostic (ks_cond_diag) and the GP likelihood / Woodbury solve
with the c4 pipeline's own Y, Q, R (sketch + TSQR through the C-ABI), CUDA events, 1 B200."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ks_inputs  # noqa: E402
import paper_1312_1869_b200 as ks  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record(); fn(); b.record(); b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    cfg, pts, A = ks_inputs.make_problem(name)
    dev = torch.device("cuda", 0)
    desc = dict(n=cfg["n"], dim=cfg["dim"], kernel=cfg["kernel"], sigma2=cfg["sigma2"], ell=cfg["ell"],
                nugget=cfg["nugget"], d=cfg["d"], seed=cfg["seed"], omega=cfg["omega"])
    Y = ks.Sketch(desc, dev)(torch.as_tensor(pts, device=dev))
    n, d = Y.shape
    Q, R = ks.TsqrPlan(n, d, cfg["blocks"], dev).factor(Y)
    res = {"config": name, "n": n, "d": d}
    ws = torch.empty(ks.ks_cond_diag_workspace_size(n, d), dtype=torch.uint8, device=dev)
    out = torch.empty(4, dtype=torch.float32, device=dev)
    res["cond_diag_ms"] = timed(lambda: ks.ks_cond_diag(Y, R, out, ws))
    res["cond"], res["eps"], res["l_min"], res["l_max"] = [float(x) for x in out.cpu()]
    lam = torch.as_tensor(np.exp(-0.01 * np.arange(1, d + 1)), dtype=torch.float32, device=dev)
    y = torch.as_tensor(A[:, 0].copy(), device=dev)
    wsg = torch.empty(ks.ks_gp_workspace_size(n, d, 1), dtype=torch.uint8, device=dev)
    o3 = torch.empty(3, dtype=torch.float64, device=dev)
    res["gp_loglik_ms"] = timed(lambda: ks.ks_gp_loglik(Q, lam, 1e-2, y, o3, wsg))
    res["loglik"] = float(o3[0].cpu())
    B = torch.as_tensor(A, device=dev)
    wsb = torch.empty(ks.ks_gp_workspace_size(n, d, B.shape[1]), dtype=torch.uint8, device=dev)
    X = torch.empty_like(B)
    res["gp_woodbury_ms_m%d" % B.shape[1]] = timed(lambda: ks.ks_gp_woodbury_solve(Q, lam, 1e-2, B, X, wsb))
    if d <= 256 and d % 16 == 0:   # the Nystrom core (second K pass on the tensor cores) and the core likelihood
        pts_d = torch.as_tensor(pts, device=dev)
        wsn = torch.empty(ks.ks_nystrom_workspace_size(desc), dtype=torch.uint8, device=dev)
        W = torch.empty_like(Q)
        Bc = torch.empty((d, d), dtype=torch.float32, device=dev)
        res["nystrom_core_ms"] = timed(lambda: ks.ks_nystrom_core(desc, pts_d, Q, W, Bc, wsn))
        # tensor-pipe FLOPs of W = K Q: 2 n^2 d per product, 3 products (K_hi Q_hi, K_lo Q_hi, K_hi Q_lo)
        res["nystrom_tensor_tflops"] = 3 * 2.0 * n * n * d / (res["nystrom_core_ms"] * 1e-3) / 1e12
        wsc = torch.empty(ks.ks_gp_core_workspace_size(n, d, 1), dtype=torch.uint8, device=dev)
        res["gp_loglik_core_ms"] = timed(lambda: ks.ks_gp_loglik_core(Q, Bc, 1e-2, y, o3, wsc))
        res["loglik_core"] = float(o3[0].cpu())
        wsw = torch.empty(ks.ks_gp_core_workspace_size(n, d, B.shape[1]), dtype=torch.uint8, device=dev)
        res["gp_woodbury_core_ms_m%d" % B.shape[1]] = timed(lambda: ks.ks_gp_woodbury_core(Q, Bc, 1e-2, B, X, wsw))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
