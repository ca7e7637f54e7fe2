"""Generates tests/golden/cfg45.npz from the REFERENCE LIBRARY (oracle/_ref,
ReferenceExecutor = sequential, FMA-free) at full size -- about 11 minutes
of CPU:

  cfg4  CG, 7-pt Poisson 256^3, b = A*1, x0 = 0, tol 1e-8: iterations,
        residual history, flop_count (581 iterations,
        final 9.589270e-09)
  cfg5  BiCGSTAB, 7-pt upwind gamma 0.5 256^3, b = A x*, x* =
        seeded_values(n, 11): iterations, history, flop_count (495)

    python tests/golden/make_golden_cfg45.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def main():
    O.build()
    out = {}
    t = time.time()
    A = O.stencil("7pt", 256)
    b, _ = O.ref_spmv(A, np.ones(A.nrows))
    r = O.ref_solve(A, b, "cg", rel_tol=1e-8, max_iters=20000)
    out.update(cg_iters=np.array(r.iterations), cg_hist=r.history, cg_flops=np.array(r.flop_count))
    print("cfg4", r.iterations, r.history[-1], time.time() - t, flush=True)
    del A, b
    A = O.stencil("7pt", 256, 0.5)
    b, _ = O.ref_spmv(A, O.seeded_values(A.nrows, 11))
    r = O.ref_solve(A, b, "bicgstab", rel_tol=1e-8, max_iters=20000)
    out.update(bicg_iters=np.array(r.iterations), bicg_hist=r.history,
               bicg_flops=np.array(r.flop_count))
    print("cfg5", r.iterations, r.history[-1], time.time() - t, flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg45.npz"),
                        **out)


if __name__ == "__main__":
    main()
