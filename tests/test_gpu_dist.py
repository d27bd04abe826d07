"""The multi-rank path (paper_1312_1869_b200.dist with CudaOps) on the GPU: world size 2.

Two processes share cuda:0 (gpurun and the round-end driver give one GPU); their collectives go through
a gloo group with the CUDA tensors staged via host memory (dist.all_gather_into / all_reduce_sum), so
neither rank's kernels wait on the other's -- each rank runs exactly the kernels it would run on its own
GPU: its row block's sketch and local TSQR, the redundant merge QR of the stacked R's (ks_tsqr on the
(2d) x d stack), ks_qform with its Q2 block, its Q^T A, the redundant truncated solve and its
rows of X = Omega Z.  The answer must be the world-size-1 answer: R against the oracle (<= 1e-4), k within
1, rho(Z) within 1e-4 of rho_ref(k) (L15), bitwise agreement of the redundant R, Z, k across ranks, and the
rows of X against the oracle's Omega Z of the same Z.
"""
import os
import socket

import numpy as np
import pytest

import ks_inputs
import oracle
from _problems import align_rows, desc_of, relF

pytestmark = pytest.mark.gpu

CASES = [("c2", dict(n=8192, m=16), 4), ("c4", dict(n=8192, m=8), 4), ("c5", dict(n=6144, m=8), 2)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, over, bpr, out_dir):
    import torch
    import torch.distributed as dist
    from paper_1312_1869_b200 import dist as ksd
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg, pts, A = ks_inputs.make_problem(name, **over)
    ops = ksd.CudaOps(desc_of(cfg), cfg["m"], bpr, oracle.TAU, rank, world, dev, inplace=True)
    A_loc = torch.as_tensor(np.ascontiguousarray(A[ops.rb:ops.re]), device=dev)
    for _ in range(2):   # the second pass reuses every buffer and the cached graphs
        X, Z, k, R = ksd.lowrank_solve_sharded(ops, torch.as_tensor(pts, device=dev), A_loc)
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), X=X.cpu().numpy(), Z=Z.cpu().numpy(), k=int(k.item()),
             R=R.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,over,bpr", CASES)
def test_world2_cudaops_on_one_gpu(tmp_path, cuda, name, over, bpr):
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), name, over, bpr, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    parts = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    for p in parts:                                   # the redundant steps agree bit for bit on every rank
        np.testing.assert_array_equal(p["R"], parts[0]["R"])
        np.testing.assert_array_equal(p["Z"], parts[0]["Z"])
        assert p["k"] == parts[0]["k"]
    cfg, pts, A = ks_inputs.make_problem(name, **over)
    prob = oracle.Problem.from_cfg(cfg, pts)
    ref = oracle.lowrank_solve(prob, A, bpr * world)
    R = parts[0]["R"].astype(np.float64)
    assert np.all(np.tril(R, -1) == 0) and np.all(np.diag(R) >= 0)
    assert relF(align_rows(R, ref["R"]), ref["R"]) <= 1e-4
    kg = int(parts[0]["k"])
    assert abs(kg - ref["k"]) <= 1
    Zg = parts[0]["Z"].astype(np.float64)
    assert abs(oracle.rho_of(ref["Y"], Zg, A) - ref["rho"][kg]) <= 1e-4
    X = np.concatenate([p["X"] for p in parts], 0)
    assert relF(X, prob.omega_apply(Zg)) <= 1e-5
