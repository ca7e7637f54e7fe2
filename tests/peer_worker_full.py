"""Worker for the full-size distributed parity tests (tests/test_gpu_fullsize.py).

One rank of a P-process peer-memory group on cuda:0 (one process and one
CUDA context per rank, IPC windows swapped over gloo -- the one-process-
per-GPU deployment folded onto one device).  Builds cfg4 (CG, 7-pt Poisson
256^3, b = A*1) and cfg5 (BiCGSTAB, 7-pt upwind gamma 0.5 256^3, b = A x*)
on the device, keeps its contiguous row block, solves row-partitioned and
writes iterations / history / flops as JSON to <out>/r<rank>.json and its
slice of x to <out>/r<rank>_<case>.npy.  Env: RANK, WORLD_SIZE,
MASTER_ADDR/PORT; argv: out dir, cases ("cg", "bicgstab", "cg_rec")."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2011_08879_b200 import dist as D, gen, larch as lk  # noqa: E402


def local_problem(ex, gamma, rank, world):
    A = gen.stencil(ex, "7pt", 256, gamma)
    n = A.nrows
    xs = np.ones(n) if gamma == 0.0 else gen.seeded_values(n, 11)
    b = lk.make_vector(ex, n)
    lk.spmv(A, lk.vector_from(ex, xs), b)
    lo, hi = D.part_range(n, world, rank)
    rp = A.row_ptr[lo:hi + 1].cpu().numpy().astype(np.int64)
    j0, j1 = int(rp[0]), int(rp[-1])
    cols = A.col_idx[j0:j1].cpu().numpy()
    vals = A.vals[j0:j1].cpu().numpy()
    nnz = A.nnz()
    b_loc = b.values[lo:hi].clone()
    del A, b
    torch.cuda.empty_cache()
    return n, nnz, (rp - j0).astype(np.int32), cols, vals, b_loc


def main():
    out_dir, cases = sys.argv[1], sys.argv[2].split(",")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ex = lk.CudaExecutor(0)
    res = {}
    comm = None
    for case in cases:
        kind = "bicgstab" if case == "bicgstab" else "cg"
        n, nnz, rp, cols, vals, b_loc = local_problem(ex, 0.5 if kind == "bicgstab" else 0.0,
                                                      rank, world)
        m = D.DistMap(n, world, rank, rp, cols)
        D.exchange_requests(m)
        if comm is None:  # same sparsity for every case: one halo capacity
            comm = D.Communicator.peer(0, D.peer_halo_cap(m))
        M = D.DistCsrMatrix(ex, m, rp, vals, nnz)
        x = torch.zeros(M.n_local, dtype=torch.float64, device="cuda")
        mode = "recurrence" if case == "cg_rec" else "true"
        r = M.solve(comm, b_loc, x, lk.SolverConfig(kind=kind, rel_tol=1e-8, max_iters=20000,
                                                     residual_mode=mode))
        res[case] = {"iters": r.iterations, "hist": list(r.residual_history),
                     "flops": r.flop_count, "conv": r.converged}
        np.save(os.path.join(out_dir, f"r{rank}_{case}.npy"), x.cpu().numpy())
        del M, m, x
        torch.cuda.empty_cache()
    comm.close()
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
