"""Dev tool: one plain CSR SpMV and a 2-iteration CG on cfg4 (7-pt 256^3),
for an ncu comparison of csr_stream_kernel<EpiStore> with the CG kernels."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "7pt", 256)
x = lk.vector_from(ex, np.ones(A.ncols))
b = lk.make_vector(ex, A.nrows)
lk.spmv(A, x, b)
lk.spmv(A, x, b)
r = lk.solve(A, b, lk.zeros(ex, A.nrows), lk.SolverConfig(kind="cg", rel_tol=1e-8, fixed_iters=2))
print(r.iterations)
