"""Worker for the peer-memory communicator tests (tests/test_gpu_dist.py).

One rank of a P-process peer group; every process drives cuda:0, so P
ranks share one B200 exactly as P GPUs of one node would be driven (one
process and one CUDA context per rank; CUDA IPC windows swapped over
gloo). Env: RANK, WORLD_SIZE, MASTER_ADDR/PORT. Runs every case and writes
its results as JSON to argv[1]. Test infrastructure: the oracle is only the
checker."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2011_08879_b200 import dist as D, larch as lk  # noqa: E402


KEEP = []


def setup(A, comm=None):
    rank, world = dist.get_rank(), dist.get_world_size()
    rp, cols, vals = D.local_rows(A.row_ptr, A.cols, A.vals, world, rank)
    m = D.DistMap(A.nrows, world, rank, rp, cols)
    D.exchange_requests(m)
    if comm is None:
        comm = D.Communicator.peer(0, D.peer_halo_cap(m))
        KEEP.append(comm)  # windows stay mapped until every rank is done
    M = D.DistCsrMatrix(EX, m, rp, vals, A.nnz)
    lo, hi = D.part_range(A.nrows, world, rank)
    return M, comm, lo, hi


def solve(kind, A, b, **kw):
    M, comm, lo, hi = setup(A)
    x = torch.zeros(hi - lo, dtype=torch.float64, device="cuda")
    cfg = lk.SolverConfig(kind=kind, rel_tol=kw.get("tol", 1e-8), max_iters=20000,
                          gmres_restart=20, fixed_iters=kw.get("fixed", 0))
    r = M.solve(comm, torch.from_numpy(b[lo:hi].copy()).cuda(), x, cfg)
    return {"iters": r.iterations, "hist": r.residual_history, "conv": r.converged,
            "flops": r.flop_count, "x": x.cpu().numpy().tolist()}


def main():
    global EX
    dist.init_process_group("gloo")
    EX = lk.CudaExecutor(0)
    out = {}
    # SpMV bit-exact vs the oracle (three stencils)
    for kind, m in (("7pt", 16), ("27pt", 12), ("5pt", 60)):
        A = O.stencil(kind, m, 0.5 if kind == "7pt" else 0.0)
        M, comm, lo, hi = setup(A)
        x = O.seeded_values(A.ncols, 11)
        y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        M.spmv(comm, M.ext_vector(x[lo:hi]), y)
        out[f"spmv_{kind}"] = bool(np.array_equal(y.cpu().numpy(), O.spmv_csr(A, x)[lo:hi]))
    # five SpMVs back to back, no sync or reduction between (slot hand-back)
    A = O.stencil("7pt", 14, 0.5)
    M, comm, lo, hi = setup(A)
    xs = [O.seeded_values(A.ncols, 20 + k) for k in range(5)]
    ys = [torch.empty(hi - lo, dtype=torch.float64, device="cuda") for _ in xs]
    xe = [M.ext_vector(x[lo:hi]) for x in xs]
    for k in range(5):
        M.spmv(comm, xe[k], ys[k], sync=False)
    comm.sync(EX)
    out["spmv_back_to_back"] = all(
        np.array_equal(ys[k].cpu().numpy(), O.spmv_csr(A, xs[k])[lo:hi]) for k in range(5))
    # two matrices with different neighbour sets on ONE communicator, applied
    # A, B, B, A (B = diagonal: no halo at all) -- ADVICE r1: the per-
    # communicator halo epoch advanced on B while only A's peers handed back
    A = O.stencil("7pt", 12)
    rk, world = dist.get_rank(), dist.get_world_size()
    rp, cols, _ = D.local_rows(A.row_ptr, A.cols, A.vals, world, rk)
    mA = D.DistMap(A.nrows, world, rk, rp, cols)
    D.exchange_requests(mA)
    shared = D.Communicator.peer(0, D.peer_halo_cap(mA))
    KEEP.append(shared)
    Bm = O.Csr(A.nrows, A.ncols, np.arange(A.nrows + 1, dtype=np.int32),
               np.arange(A.nrows, dtype=np.int32), np.full(A.nrows, 2.0))
    MA, _, lo, hi = setup(A, shared)
    MB, _, _, _ = setup(Bm, shared)
    xg = O.seeded_values(A.ncols, 31)
    ok = True
    for M, ref in ((MA, O.spmv_csr(A, xg)), (MB, 2.0 * xg), (MB, 2.0 * xg), (MA, O.spmv_csr(A, xg))):
        y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        M.spmv(shared, M.ext_vector(xg[lo:hi]), y)
        ok = ok and bool(np.array_equal(y.cpu().numpy(), ref[lo:hi]))
    out["shared_comm_abba"] = ok
    # allreduce
    t = torch.tensor([float(dist.get_rank() + 1), 0.25], dtype=torch.float64, device="cuda")
    comm.allreduce_sum(EX, t)
    comm.sync(EX)
    out["allreduce"] = t.tolist()
    # solvers
    A = O.stencil("7pt", 32)
    out["cg"] = solve("cg", A, O.spmv_csr(A, np.ones(A.nrows)))
    os.environ["LBK_CG_MERGE"] = "0"  # three exchanges per iteration
    out["cg_3x"] = solve("cg", A, O.spmv_csr(A, np.ones(A.nrows)))
    os.environ.pop("LBK_CG_MERGE")
    out["cg_fixed"] = solve("cg", A, O.spmv_csr(A, np.ones(A.nrows)), fixed=50)
    A = O.stencil("7pt", 20, 0.5)
    b = O.spmv_csr(A, O.seeded_values(A.nrows, 11))
    out["bicgstab"] = solve("bicgstab", A, b)
    os.environ["LBK_SOLVER_GRAPH"] = "0"
    out["bicgstab_eager"] = solve("bicgstab", A, b)
    os.environ.pop("LBK_SOLVER_GRAPH")
    os.environ["LBK_CG_MERGE"] = "0"  # the residual exchanged on its own
    out["bicgstab_unmerged"] = solve("bicgstab", A, b)
    os.environ.pop("LBK_CG_MERGE")
    out["bicgstab_fixed"] = solve("bicgstab", A, b, fixed=23)
    # the exact exchange's wide-range encoding (sign-magnitude digits) on
    # ordinary data: the same bits as the raw-limb posts
    os.environ["LBK_XRED_DIGITS"] = "1"
    out["bicgstab_digits"] = solve("bicgstab", A, b)
    os.environ.pop("LBK_XRED_DIGITS")
    A = O.stencil("7pt", 14, 0.5)
    b = O.spmv_csr(A, O.seeded_values(A.nrows, 11))
    out["cgs"] = solve("cgs", A, b)
    out["gmres"] = solve("gmres", A, b)
    # a peer that never arrives: rank 0 alone runs an SpMV and must time out
    os.environ["LBK_PEER_TIMEOUT"] = "2"
    A = O.stencil("7pt", 10)
    M, comm, lo, hi = setup(A)
    if dist.get_rank() == 0:
        try:
            y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
            M.spmv(comm, M.ext_vector(np.ones(hi - lo)), y)
            out["timeout"] = "no error"
        except lk.DeviceError as e:
            out["timeout"] = str(e)
    dist.barrier()
    KEEP.clear()
    with open(sys.argv[1], "w") as f:
        json.dump(out, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
