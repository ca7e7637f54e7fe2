"""Generates tests/golden/cfg45_exact.npz: the krylov.cpp CG / BiCGSTAB
recurrences with EXACTLY ROUNDED dot products (oracle/xkrylov.cpp, the
product's partition-independent reduction; port_xdot is pinned to
Python's math.fsum in tests/test_oracle.py) at full size -- about 5 minutes
on 8 host cores:

  cfg4  CG, 7-pt Poisson 256^3, b = A*1, x0 = 0, tol 1e-8
  cfg5  BiCGSTAB, 7-pt upwind gamma 0.5 256^3, b = A x*, x* =
        seeded_values(n, 11), x0 = 0, tol 1e-8

For each: iterations, the full residual history, flop_count and the
SHA-256 of the solution's bytes.  The GPU solver reproduces all of them
bit for bit on one GPU and row-partitioned over any number of ranks
(tests/test_gpu_fullsize.py).

    python tests/golden/make_golden_cfg45_exact.py
"""
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def main():
    O.build(ref=False)
    out = {}
    for tag, kind, gamma in (("cg", "cg", 0.0), ("bicg", "bicgstab", 0.5)):
        t = time.time()
        A = O.stencil("7pt", 256, gamma)
        xs = np.ones(A.nrows) if kind == "cg" else O.seeded_values(A.nrows, 11)
        b = O.spmv_csr(A, xs)
        r = O.xsolve(A, b, kind, tol=1e-8, max_iters=20000)
        out[f"{tag}_iters"] = np.int64(r["iterations"])
        out[f"{tag}_hist"] = r["history"]
        out[f"{tag}_flops"] = np.int64(r["flops"])
        out[f"{tag}_x_sha256"] = np.array(hashlib.sha256(r["x"].tobytes()).hexdigest())
        print(tag, r["iterations"], r["history"][-1], f"{time.time() - t:.0f}s", flush=True)
        del A, b
    np.savez(os.path.join(ROOT, "tests", "golden", "cfg45_exact.npz"), **out)


if __name__ == "__main__":
    main()
