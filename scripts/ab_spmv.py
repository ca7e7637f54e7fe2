"""A/B timing of SpMV kernels (dev tool): prints one line per format/config
for the library selected by LBK_LIB (default in-tree liblbk.so)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
tag = os.path.basename(os.environ.get("LBK_LIB", "default"))


def timeit(fn, reps=20):
    ts = []
    for _ in range(3):
        fn()
    for _ in range(reps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def run(name, A, fmts):
    x = lk.vector_from(ex, gen.seeded_values(A.ncols))
    y = lk.make_vector(ex, A.nrows)
    n, nnz = A.nrows, A.nnz()
    for f in fmts:
        M = A if f == "csr" else lk.csr_to_coo(A)
        b = 12 * nnz + 4 * (n + 1) + 16 * n if f == "csr" else 16 * nnz + 16 * n
        t = timeit(lambda: lk.spmv(M, x, y, sync=False))
        print(f"{tag:28s} {name:6s} {f:4s} {t*1e6:8.1f}us {b/t/1e9:7.0f} GB/s", flush=True)


for cfg in ["cfg1", "cfg2"]:
    c = gen.CONFIGS[cfg]
    run(cfg, gen.stencil(ex, c["kind"], c["m"], c["gamma"]), ["csr", "coo"])
if "--cfg4" in sys.argv:  # the CG operator: 7-pt 256^3
    run("cfg4", gen.stencil(ex, "7pt", 256, 0.0), ["csr"])
if "--powerlaw" in sys.argv:
    rp, ci, va = gen.powerlaw_host(1 << 24)
    run("cfg3", lk.csr_from_host(ex, 1 << 24, 1 << 24, rp, ci, va), ["csr", "coo"])
