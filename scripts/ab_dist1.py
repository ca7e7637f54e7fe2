"""Dev tool: cost of the distributed solver path at one rank (cfg4 CG):
fused single-GPU vs dist (no communicator) vs dist (NCCL, 1 rank)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import dist as D, gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = gen.stencil(ex, "7pt", m)
b = lk.make_vector(ex, A.nrows)
lk.spmv(A, lk.vector_from(ex, np.ones(A.ncols)), b)
cfg = lk.SolverConfig(kind="cg", rel_tol=1e-8, fixed_iters=200)
x = lk.zeros(ex, A.nrows)
r = lk.solve(A, b, x, cfg)
print(f"fused       {r.iterations / r.elapsed:8.1f} it/s")
rp = A.row_ptr.cpu().numpy()
m_ = D.DistMap(A.nrows, 1, 0, rp, A.col_idx.cpu().numpy())
D.exchange_requests_local([m_])
M = D.DistCsrMatrix(ex, m_, rp, A.vals.cpu().numpy(), A.nnz())
for name, comm in [("dist/none", None), ("dist/nccl1", D.Communicator.nccl_single(0))]:
    for g in ("0", "1"):
        os.environ["LBK_SOLVER_GRAPH"] = g
        xx = torch.zeros(A.nrows, dtype=torch.float64, device="cuda")
        r = M.solve(comm, b.values, xx, cfg)
        print(f"{name:11s} graph={g} {r.iterations / r.elapsed:8.1f} it/s")
