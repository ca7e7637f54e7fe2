"""Dev tool: a 3-iteration BiCGSTAB on cfg5 (7-pt upwind 256^3) for ncu
launch lists of the B2-B6 kernels."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "7pt", 256, 0.5)
b = lk.make_vector(ex, A.nrows)
lk.spmv(A, lk.vector_from(ex, gen.seeded_values(A.ncols)), b)
r = lk.solve(A, b, lk.zeros(ex, A.nrows), lk.SolverConfig(kind="bicgstab", rel_tol=1e-8,
                                                         fixed_iters=3))
print(r.iterations)
