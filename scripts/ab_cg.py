"""Dev tool: solver A/B for the library selected by LBK_LIB -- cfg4 CG
(both residual modes) and cfg5 BiCGSTAB, best of 3 after a warm-up."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
tag = os.path.basename(os.environ.get("LBK_LIB", "default"))
out = []
for kind, gamma, modes in (("cg", 0.0, ("true", "recurrence")), ("bicgstab", 0.5, ("true",)),
                           ("cgs", 0.5, ("true",))):
    A = gen.stencil(ex, "7pt", 256, gamma)
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, lk.vector_from(ex, gen.seeded_values(A.ncols) if gamma else np.ones(A.ncols)), b)
    for mode in modes:
        lk.solve(A, b, lk.zeros(ex, A.nrows), lk.SolverConfig(kind=kind, rel_tol=1e-8, max_iters=40,
                                                             residual_mode=mode))
        best = 0.0
        for _ in range(3):
            r = lk.solve(A, b, lk.zeros(ex, A.nrows),
                         lk.SolverConfig(kind=kind, rel_tol=1e-8, residual_mode=mode))
            best = max(best, r.iterations / r.elapsed)
        out.append(f"{kind}/{mode} {r.iterations} {best:7.1f}")
    del A, b
print(f"{tag:45s}", " | ".join(out), flush=True)
