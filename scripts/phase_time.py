"""Dev tool: solver time per iteration window (fixed_iters = k, 2k, ...),
cfg4 CG and cfg5 BiCGSTAB, for the library selected by LBK_LIB."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
tag = os.path.basename(os.environ.get("LBK_LIB", "default"))
for kind, gamma in (("cg", 0.0), ("bicgstab", 0.5)):
    A = gen.stencil(ex, "7pt", 256, gamma)
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, lk.vector_from(ex, gen.seeded_values(A.ncols) if gamma else np.ones(A.ncols)), b)
    lk.solve(A, b, lk.zeros(ex, A.nrows), lk.SolverConfig(kind=kind, rel_tol=1e-8, fixed_iters=5))
    prev_t, prev_k, out = 0.0, 0, []
    for k in (50, 100, 200, 300, 400, 480):
        r = lk.solve(A, b, lk.zeros(ex, A.nrows), lk.SolverConfig(kind=kind, rel_tol=1e-8,
                                                                 fixed_iters=k))
        out.append(f"{prev_k}-{k}: {(r.elapsed - prev_t) / (k - prev_k) * 1e6:6.0f}us")
        prev_t, prev_k = r.elapsed, k
    print(f"{tag:28s} {kind:8s}", " ".join(out), flush=True)
