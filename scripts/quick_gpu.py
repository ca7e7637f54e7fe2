"""First-light GPU check: parity vs the oracle + rough timings (dev tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
print(ex.describe())
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=20):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts)), float(np.min(ts))


def relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


for cfg in ["cfg1", "cfg2"]:
    c = gen.CONFIGS[cfg]
    A = gen.stencil(ex, c["kind"], c["m"], c["gamma"])
    ref = O.stencil(c["kind"], c["m"], c["gamma"])
    print(cfg, "gen bit-exact:",
          np.array_equal(A.row_ptr.cpu().numpy(), ref.row_ptr),
          np.array_equal(A.col_idx.cpu().numpy(), ref.cols),
          np.array_equal(A.vals.cpu().numpy(), ref.vals))
    xh = gen.seeded_values(A.ncols)
    x = lk.vector_from(ex, xh)
    y = lk.make_vector(ex, A.nrows)
    yref = O.spmv_csr(ref, xh)
    n, nnz = A.nrows, A.nnz()
    for name, M in [("csr", A), ("coo", lk.csr_to_coo(A)), ("ell", lk.csr_to_ell(A)),
                    ("sellp", lk.csr_to_sellp(A, 32))]:
        lk.spmv(M, x, y)
        yy = lk.vector_to_host(y)
        bytes_ = {"csr": 12 * nnz + 4 * (n + 1) + 16 * n, "coo": 16 * nnz + 16 * n,
                  "ell": 12 * getattr(M, "width", 0) * n + 16 * n,
                  "sellp": 12 * (M.col_idx.numel() if name == "sellp" else 0) + 16 * n + 8 * (n // 32)}[name]
        med, mn = timeit(lambda: lk.spmv(M, x, y, sync=False))
        print(f"  {name:6s} bitexact={np.array_equal(yy, yref)} rel={relerr(yy, yref):.2e} "
              f"t={med*1e6:.1f}us (min {mn*1e6:.1f}) {bytes_/med/1e9:.0f} GB/s "
              f"{2*nnz/med/1e9:.0f} GFLOP/s")

# small solves vs the reference library
for kind, m, gamma in [("cg", 32, 0.0), ("bicgstab", 32, 0.5)]:
    ref = O.stencil("7pt", m, gamma)
    if kind == "cg":
        bh, _ = O.ref_spmv(ref, np.ones(ref.nrows))
    else:
        bh, _ = O.ref_spmv(ref, O.seeded_values(ref.nrows, 11))
    r = O.ref_solve(ref, bh, kind, rel_tol=1e-8, max_iters=20000)
    A = lk.csr_from_host(ex, ref.nrows, ref.ncols, ref.row_ptr, ref.cols, ref.vals)
    b = lk.vector_from(ex, bh)
    x = lk.zeros(ex, ref.nrows)
    t0 = time.time()
    g = lk.solve(A, b, x, lk.SolverConfig(kind=kind, rel_tol=1e-8, max_iters=20000))
    h = np.array(g.residual_history)
    hr = r.history
    k = min(len(h), len(hr), 40)
    print(f"{kind} {m}^3: ref iters {r.iterations} flops {r.flop_count} | gpu iters {g.iterations} "
          f"flops {g.flop_count} final {g.final_rel_residual:.3e} hist40 maxrel "
          f"{np.max(np.abs(h[:k]-hr[:k])/hr[:k]):.2e} t={time.time()-t0:.3f}s")

# power-law (reduced) csr/coo parity
rp, ci, va = gen.powerlaw_host(1 << 20)
A = lk.csr_from_host(ex, 1 << 20, 1 << 20, rp, ci, va)
ref = O.Csr(1 << 20, 1 << 20, rp, ci, va)
xh = gen.seeded_values(A.ncols)
x = lk.vector_from(ex, xh)
y = lk.make_vector(ex, A.nrows)
yref = O.spmv_csr(ref, xh)
for name, M in [("csr", A), ("coo", lk.csr_to_coo(A))]:
    lk.spmv(M, x, y)
    yy = lk.vector_to_host(y)
    print(f"powerlaw 2^20 {name}: rel={relerr(yy, yref):.2e} bit-equal rows "
          f"{np.mean(yy == yref):.4f}")
print("DONE")
