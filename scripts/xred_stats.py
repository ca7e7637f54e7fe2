"""Dev tool: exact-reduction lane statistics (flushes / slides / re-centres)
per solver iteration, with a library built -DLBK_XRED_STATS
(scripts/variants.sh LBK_XRED_STATS; run with LBK_LIB pointing at it)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import _lib as L, gen, larch as lk  # noqa: E402

lib = L.load()
f = lib.lbk_dbg_xred_stats
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
ex = lk.CudaExecutor(0)
st = (C.c_ulonglong * 4)()
for kind, gamma in (("cg", 0.0), ("bicgstab", 0.5)):
    A = gen.stencil(ex, "7pt", 256, gamma)
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, lk.vector_from(ex, gen.seeded_values(A.ncols) if gamma else np.ones(A.ncols)), b)
    f(st, 1)
    r = lk.solve(A, b, lk.zeros(ex, A.nrows), lk.SolverConfig(kind=kind, rel_tol=1e-8))
    f(st, 0)
    print(f"{kind}: {r.iterations} it, per iteration: direct {st[0]/r.iterations:.0f} "
          f"placements {st[2]/r.iterations:.0f}", flush=True)
