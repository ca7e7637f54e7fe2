"""Generates tests/golden/golden.npz from the REFERENCE LIBRARY itself
(oracle/_ref/liblarch_ref.so = /root/reference/proj/src compiled FMA-free,
see oracle/Makefile).  Run in the container that holds /root/reference:

    python tests/golden/make_golden.py

Fixtures (all small; the GPU box reads only the .npz):
  kat_*        SPEC.md:416-420 SpMV examples and SPEC.md:311-324 conversions
  rnd{i}_*     random COO entry lists with duplicates -> coo_from_entries,
               coo_to_csr, spmv_csr / spmv_coo on seeded x
  st5_*        2D 5-pt 32x32 stencil, spmv with seeded_values(., 11)
  cg16_*       CG, 7-pt Poisson 16^3, b = A*1, tol 1e-8 (iterations, history,
               flop_count, x)
  bicg16_*     BiCGSTAB, 7-pt upwind gamma 0.5 16^3, b = A*x*, tol 1e-8
  cg2_*        CG 2x2 KAT [[4,1],[1,3]] x = [1,2]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402


def main():
    O.build()
    g = {}
    # ---- SPEC KATs
    # I3 * [1,2,3]
    g["kat_eye_y"], _ = O.ref_spmv(O.Csr(3, 3, np.array([0, 1, 2, 3], np.int32),
                                         np.array([0, 1, 2], np.int32), np.ones(3)),
                                   np.array([1.0, 2.0, 3.0]))
    g["kat_up_y"], _ = O.ref_spmv(O.Csr(2, 2, np.array([0, 2, 3], np.int32),
                                        np.array([0, 1, 1], np.int32),
                                        np.array([1.0, 2.0, 3.0])), np.array([1.0, 1.0]))
    g["kat_empty_y"], _ = O.ref_spmv(O.Csr(2, 2, np.array([0, 1, 1], np.int32),
                                           np.array([0], np.int32), np.array([5.0])),
                                     np.array([2.0, 7.0]))
    rp, _, _ = O.ref_coo_to_csr(2, 2, np.array([0, 0, 1]), np.array([0, 1, 1]),
                                np.array([1.0, 2.0, 3.0]))
    g["kat_c2c_rowptr"] = rp
    rp, _, _ = O.ref_coo_to_csr(3, 3, np.zeros(0), np.zeros(0), np.zeros(0))
    g["kat_c2c_empty_rowptr"] = rp
    # ---- random entry lists with duplicates
    rng = np.random.default_rng(20240611)
    for i in range(6):
        nr, nc = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        n = int(rng.integers(0, 4 * nr))
        rows = rng.integers(0, nr, n).astype(np.int32)
        cols = rng.integers(0, nc, n).astype(np.int32)
        vals = rng.uniform(-1, 1, n)
        vals[rng.random(n) < 0.05] = 0.0  # explicit zeros are kept
        ro, co, vo = O.ref_coo_from_entries(nr, nc, rows, cols, vals)
        rp, _, _ = O.ref_coo_to_csr(nr, nc, ro, co, vo)
        x = O.seeded_values(nc, 11 + i)
        y_csr, _ = O.ref_spmv(O.Csr(nr, nc, rp, co, vo), x, "csr")
        y_coo, _ = O.ref_spmv(O.Csr(nr, nc, rp, co, vo), x, "coo")
        for k, v in dict(shape=np.array([nr, nc]), in_rows=rows, in_cols=cols, in_vals=vals,
                         rows=ro, cols=co, vals=vo, rowptr=rp, x=x, y_csr=y_csr,
                         y_coo=y_coo).items():
            g[f"rnd{i}_{k}"] = v
    # ---- 5-pt stencil
    A = O.stencil("5pt", 32)
    x = O.seeded_values(A.ncols, 11)
    g["st5_x"] = x
    g["st5_y"], _ = O.ref_spmv(A, x)
    # ---- CG 16^3
    A = O.stencil("7pt", 16)
    b, _ = O.ref_spmv(A, np.ones(A.nrows))
    r = O.ref_solve(A, b, "cg", rel_tol=1e-8, max_iters=20000)
    g.update(cg16_b=b, cg16_iters=np.array(r.iterations), cg16_hist=r.history,
             cg16_flops=np.array(r.flop_count), cg16_x=r.x)
    # ---- BiCGSTAB 16^3, gamma 0.5, b = A x*
    A = O.stencil("7pt", 16, 0.5)
    b, _ = O.ref_spmv(A, O.seeded_values(A.nrows, 11))
    r = O.ref_solve(A, b, "bicgstab", rel_tol=1e-8, max_iters=20000)
    g.update(bicg16_b=b, bicg16_iters=np.array(r.iterations), bicg16_hist=r.history,
             bicg16_flops=np.array(r.flop_count), bicg16_x=r.x)
    # ---- CG 2x2 KAT
    A = O.Csr(2, 2, np.array([0, 2, 4], np.int32), np.array([0, 1, 0, 1], np.int32),
              np.array([4.0, 1.0, 1.0, 3.0]))
    r = O.ref_solve(A, np.array([1.0, 2.0]), "cg", rel_tol=1e-12, max_iters=10)
    g.update(cg2_x=r.x, cg2_iters=np.array(r.iterations), cg2_hist=r.history)
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, len(g), "arrays")


if __name__ == "__main__":
    main()
