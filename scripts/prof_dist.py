"""Dev tool: 20 fixed cfg4 CG iterations, fused single-GPU then the
distributed path at one rank (no communicator), for an ncu launch list."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import dist as D, gen, larch as lk  # noqa: E402

os.environ["LBK_SOLVER_GRAPH"] = "0"
ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "7pt", 256)
b = lk.make_vector(ex, A.nrows)
lk.spmv(A, lk.vector_from(ex, np.ones(A.ncols)), b)
cfg = lk.SolverConfig(kind="cg", rel_tol=1e-8, fixed_iters=20)
x = lk.zeros(ex, A.nrows)
torch.cuda.nvtx.range_push("fused")
lk.solve(A, b, x, cfg)
torch.cuda.nvtx.range_pop()
rp = A.row_ptr.cpu().numpy()
m_ = D.DistMap(A.nrows, 1, 0, rp, A.col_idx.cpu().numpy())
D.exchange_requests_local([m_])
M = D.DistCsrMatrix(ex, m_, rp, A.vals.cpu().numpy(), A.nnz())
xx = torch.zeros(A.nrows, dtype=torch.float64, device="cuda")
M.solve(None, b.values, xx, cfg)
