"""Dev tool: a short cfg4 CG solve (for ncu captures of the solver kernels)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "7pt", 256)
b = lk.make_vector(ex, A.nrows)
lk.spmv(A, lk.vector_from(ex, np.ones(A.ncols)), b)
x = lk.zeros(ex, A.nrows)
r = lk.solve(A, b, x, lk.SolverConfig(kind="cg", rel_tol=1e-8, fixed_iters=int(sys.argv[1]) if len(sys.argv) > 1 else 20))
print(r.iterations, r.elapsed)
