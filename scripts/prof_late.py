"""Dev tool: CG (cfg4) or BiCGSTAB (cfg5) with fixed_iters=N, for ncu
captures of late-iteration kernels (argv: cg|bicgstab N)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

kind, n_it = sys.argv[1], int(sys.argv[2])
gamma = 0.5 if kind == "bicgstab" else 0.0
ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "7pt", 256, gamma)
b = lk.make_vector(ex, A.nrows)
lk.spmv(A, lk.vector_from(ex, gen.seeded_values(A.ncols) if gamma else np.ones(A.ncols)), b)
r = lk.solve(A, b, lk.zeros(ex, A.nrows), lk.SolverConfig(kind=kind, rel_tol=1e-8,
                                                         fixed_iters=n_it))
print(r.iterations)
