"""Dev tool: cfg3 power-law SpMV (CSR f64, COO f64, CSR f32) for ncu captures
and quick timings.  `python scripts/prof_pl.py [csr|coo|f32 ...]`."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

which = sys.argv[1:] or ["csr", "coo", "f32"]
ex = lk.CudaExecutor(0)
n = 1 << 24
rp, ci, va = gen.powerlaw_host(n)
A = lk.csr_from_host(ex, n, n, rp, ci, va)
del rp, ci, va
nnz = A.nnz()
x = lk.vector_from(ex, gen.seeded_values(n, 11))
y = lk.make_vector(ex, n)


def timeit(M, xx, yy, reps=10):
    for _ in range(3):
        lk.spmv(M, xx, yy, sync=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        lk.spmv(M, xx, yy, sync=False)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


for w in which:
    if w == "csr":
        t = timeit(A, x, y)
        b = 12 * nnz + 4 * (n + 1) + 16 * n
    elif w == "coo":
        C = lk.csr_to_coo(A)
        t = timeit(C, x, y)
        b = 16 * nnz + 16 * n
        del C
    else:
        A32 = A.astype(torch.float32)
        x32 = lk.DenseVector(x.values.float(), ex)
        y32 = lk.make_vector(ex, n, torch.float32)
        t = timeit(A32, x32, y32)
        b = 8 * nnz + 4 * (n + 1) + 8 * n
        del A32
    print(f"cfg3 {w}: {t*1e6:.1f} us  {b/t/1e9:.0f} GB/s", flush=True)
