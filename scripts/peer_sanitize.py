"""Dev tool: one rank of a 2-process peer group (cuda:0) doing a few
distributed SpMVs and a short CG, small enough to run under
compute-sanitizer (env: RANK, WORLD_SIZE, MASTER_ADDR/PORT)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2011_08879_b200 import dist as D, larch as lk  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
ex = lk.CudaExecutor(0)
A = O.stencil("7pt", 12, 0.5)
rp, cols, vals = D.local_rows(A.row_ptr, A.cols, A.vals, world, rank)
m = D.DistMap(A.nrows, world, rank, rp, cols)
D.exchange_requests(m)
comm = D.Communicator.peer(0, D.peer_halo_cap(m))
M = D.DistCsrMatrix(ex, m, rp, vals, A.nnz)
lo, hi = D.part_range(A.nrows, world, rank)
x = O.seeded_values(A.ncols, 11)
y = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
for _ in range(3):
    M.spmv(comm, M.ext_vector(x[lo:hi]), y)
ok = np.array_equal(y.cpu().numpy(), O.spmv_csr(A, x)[lo:hi])
b = O.spmv_csr(A, np.ones(A.nrows))[lo:hi]
for kind in ("cg", "bicgstab"):
    r = M.solve(comm, torch.from_numpy(b.copy()).cuda(), torch.zeros(hi - lo, dtype=torch.float64,
                device="cuda"), lk.SolverConfig(kind=kind, rel_tol=1e-8, fixed_iters=20))
    print(f"rank {rank} {kind}: {r.iterations} iterations", flush=True)
print(f"rank {rank} spmv bit-exact: {ok}", flush=True)
comm.close()
dist.destroy_process_group()
