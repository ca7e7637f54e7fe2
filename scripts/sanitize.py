"""Dev tool: small runs of every kernel family for compute-sanitizer."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "27pt", 12)
x = lk.vector_from(ex, gen.seeded_values(A.ncols, 11))
y = lk.make_vector(ex, A.nrows)
for M in (A, lk.csr_to_coo(A), lk.csr_to_ell(A), lk.csr_to_sellp(A, 32)):
    lk.spmv(M, x, y)
    lk.spmv(M, x, y, alpha=2.0, beta=0.5)
R = O.powerlaw(1 << 14, window=2048, max_len=3000)
P = lk.csr_from_host(ex, R.nrows, R.ncols, R.row_ptr, R.cols, R.vals)
xp = lk.vector_from(ex, O.seeded_values(R.ncols, 11))
yp = lk.make_vector(ex, R.nrows)
lk.spmv(P, xp, yp)
lk.spmv(lk.csr_to_coo(P), xp, yp)
A7 = gen.stencil(ex, "7pt", 10, 0.5)
b = lk.make_vector(ex, A7.nrows)
lk.spmv(A7, lk.vector_from(ex, np.ones(A7.ncols)), b)
for kind in ("cg", "bicgstab", "cgs", "gmres"):
    xs = lk.zeros(ex, A7.nrows)
    lk.solve(A7, b, xs, lk.SolverConfig(kind=kind, rel_tol=1e-8, max_iters=200, gmres_restart=10))
lk.dot(x, x)
# exact reductions: the direct-to-limbs path (600 decades of range),
# cancellation, subnormals, inf/nan (xred.cuh)
rng = np.random.default_rng(1)
w = rng.standard_normal(200000) * 10.0 ** rng.integers(-300, 300, 200000)
lk.dot(lk.vector_from(ex, w), lk.vector_from(ex, np.ones(w.size)))
w[5] = np.inf
w[7] = np.nan
lk.dot(lk.vector_from(ex, w), lk.vector_from(ex, np.ones(w.size)))
v = rng.standard_normal(4096) * 1e-160
lk.dot(lk.vector_from(ex, v), lk.vector_from(ex, v))
# calibration set, flops sweep, one GMRES cycle with its basis
sa, sb, sc = (lk.vector_from(ex, rng.standard_normal(1 << 16)) for _ in range(3))
for op in lk.STREAM_OPS:
    lk.stream_kernel(op, sa, sb, sc, 0.4)
lk.flops_sweep(sa, 9)
lk.gmres_restart_cycle(A7, b, lk.zeros(ex, A7.nrows), 8, [])
M = lk.coo_from_entries(ex, 5, 5, [(0, 1, 1.0), (4, 4, 2.0), (0, 1, 3.0)])
lk.coo_to_csr(M)
torch.cuda.synchronize()
print("sanitize run done")
