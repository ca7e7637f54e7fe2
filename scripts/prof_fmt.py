"""Dev tool: run one format's SpMV a few times on cfg2 (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "27pt", 128)
fmt = sys.argv[1] if len(sys.argv) > 1 else "sellp"
M = {"csr": lambda: A, "coo": lambda: lk.csr_to_coo(A), "ell": lambda: lk.csr_to_ell(A),
     "sellp": lambda: lk.csr_to_sellp(A, 32)}[fmt]()
x = lk.vector_from(ex, gen.seeded_values(A.ncols))
y = lk.make_vector(ex, A.nrows)
for _ in range(4):
    lk.spmv(M, x, y)
print("done", fmt)
