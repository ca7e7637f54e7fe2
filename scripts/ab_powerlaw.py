"""Dev tool: power-law CSR/COO SpMV timing vs the row-length cap (which
part of cfg3 costs)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3 / reps


n = 1 << 24
for max_len in [int(a) for a in (sys.argv[1:] or ["32", "128", "896", "10000"])]:
    rp, ci, va = gen.powerlaw_host(n, max_len=max_len)
    A = lk.csr_from_host(ex, n, n, rp, ci, va)
    x = lk.vector_from(ex, gen.seeded_values(n))
    y = lk.make_vector(ex, n)
    nnz = A.nnz()
    for f, M in [("csr", A), ("coo", lk.csr_to_coo(A))]:
        b = 12 * nnz + 4 * (n + 1) + 16 * n if f == "csr" else 16 * nnz + 16 * n
        t = timeit(lambda: lk.spmv(M, x, y, sync=False))
        print(f"max_len {max_len:6d} nnz {nnz:10d} {f} {t*1e6:9.1f}us {b/t/1e9:7.0f} GB/s", flush=True)
    del A, M
    torch.cuda.empty_cache()
