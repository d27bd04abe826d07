"""Multi-rank orchestration (paper_1312_1869_b200.dist) on CPU: world size 2 over gloo.

The row-sharded path -- local sketch, local TSQR, all_gather of the d x d R's, redundant
merge QR (eq. (5)'s final merge), Q_p = Q_p^(1) Q2_p, all_reduce of Q^T A,
redundant truncated solve, local X -- runs here with the local steps supplied by the fp64
oracle (test infrastructure).  It must give the world-size-1 answer: the same R (unique,
r_jj >= 0), the same k and Z, and X rows that concatenate to the single-rank X.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ks_inputs
import oracle
from paper_1312_1869_b200 import dist as ksd


class OracleOps:
    """The seven local steps of dist.lowrank_solve_sharded, done by the oracle on CPU tensors."""

    def __init__(self, cfg, pts, blocks_per_rank, rank, world):
        self.prob = oracle.Problem.from_cfg(cfg, pts)
        self.rb, self.re = ksd.shard_rows(cfg["n"], world, rank)
        self.blocks = blocks_per_rank
        self.Q1 = None

    def sketch(self, pts):
        return torch.from_numpy(self.prob.sketch_rows(np.arange(self.rb, self.re)))

    def local_r(self, Y):
        self.Q1, R = oracle.tsqr_tree(Y.numpy(), self.blocks, want_q=True)
        return torch.from_numpy(R)

    def merge(self, Rstack):
        Q2, R = oracle.householder_qr(Rstack.numpy(), want_q=True)
        return torch.from_numpy(Q2), torch.from_numpy(R)

    def qform(self, Cblk):
        return torch.from_numpy(self.Q1 if Cblk is None else oracle.matmul(self.Q1, Cblk.numpy()))

    def qt(self, Q, A):
        return torch.from_numpy(oracle.matmul(np.ascontiguousarray(Q.numpy().T), A.numpy().astype(np.float64)))

    def trsolve(self, R, Cm):
        k = oracle.truncation_rank(R.numpy())
        return torch.from_numpy(oracle.back_substitute(R.numpy(), Cm.numpy(), k)), torch.tensor([k])

    def omega_apply(self, Z):
        return torch.from_numpy(self.prob.omega_apply(Z.numpy())[self.rb:self.re])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, over, blocks_per_rank, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, pts, A = ks_inputs.make_problem(name, **over)
    ops = OracleOps(cfg, pts, blocks_per_rank, rank, world)
    X, Z, k, R = ksd.lowrank_solve_sharded(ops, pts, torch.from_numpy(A[ops.rb:ops.re].astype(np.float64)))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), X=X.numpy(), Z=Z.numpy(), k=int(k[0]), R=R.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,over,bpr", [("c2", dict(n=2048, d=32, m=3), 2), ("c5", dict(n=1536, d=24, m=2), 1),
                                           ("c3", dict(n=1024, d=32, m=4), 2)])
def test_world2_equals_world1(tmp_path, name, over, bpr):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), name, over, bpr, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    cfg, pts, A = ks_inputs.make_problem(name, **over)
    prob = oracle.Problem.from_cfg(cfg, pts)
    ref = oracle.lowrank_solve(prob, A, bpr * world)
    for p in parts:                                   # redundant steps agree on every rank
        np.testing.assert_array_equal(p["R"], parts[0]["R"])
        np.testing.assert_array_equal(p["Z"], parts[0]["Z"])
        assert p["k"] == parts[0]["k"] == ref["k"]
    R = parts[0]["R"]
    assert np.linalg.norm(R - ref["R"]) <= 1e-10 * np.linalg.norm(ref["R"])
    X = np.concatenate([p["X"] for p in parts], 0)
    k = ref["k"]
    # Z is unique on the leading k rows (full-rank prefix); compare through K X = Y Z.
    assert abs(oracle.rho_of(ref["Y"], parts[0]["Z"], A) - ref["rho"][k]) <= 1e-10
    np.testing.assert_allclose(X, prob.omega_apply(parts[0]["Z"]), rtol=0, atol=1e-12 * np.abs(X).max())


def test_shard_rows_partition():
    for n in (1, 7, 2048, 1 << 20):
        for w in (1, 2, 3, 8):
            b = [ksd.shard_rows(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1
