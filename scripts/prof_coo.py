"""Dev tool: cfg2 (27-pt 128^3) COO SpMV launches for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "27pt", 128)
C = lk.csr_to_coo(A)
x = lk.vector_from(ex, gen.seeded_values(A.ncols, 11))
y = lk.make_vector(ex, A.nrows)
for _ in range(4):
    lk.spmv(C, x, y)
