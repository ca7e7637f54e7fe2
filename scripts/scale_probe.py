"""Dev tool: per-rank work of cfg4 CG at P GPUs, on one GPU. Runs the
distributed solver (peer communicator, one rank) on one row block of the
7-pt 256^3 matrix -- n/P rows with a one-plane halo on each side -- so the
per-iteration device time at P ranks can be read off without P GPUs
(communication latency excluded)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import dist as D, gen, larch as lk  # noqa: E402

ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "7pt", 256)
rp = A.row_ptr.cpu().numpy()
cols = A.col_idx.cpu().numpy()
vals = A.vals.cpu().numpy()
n = A.nrows
b = lk.make_vector(ex, n)
lk.spmv(A, lk.vector_from(ex, np.ones(n)), b)
bh = b.values.cpu().numpy()
del A
PS = [int(a) for a in sys.argv[1:2]] or [1, 2, 4, 8]
ITERS = int(sys.argv[2]) if len(sys.argv) > 2 else 300
for P in PS:
    r = P // 2  # an interior rank: halo on both sides
    lo, hi = D.part_range(n, P, r)
    k0, k1 = int(rp[lo]), int(rp[hi])
    m = D.DistMap(n, P, r, (rp[lo:hi + 1] - k0).astype(np.int32), cols[k0:k1])
    # a one-rank solve of the block: treat ghosts as zero-valued columns by
    # restricting to owned columns (same kernels and sizes as rank r's)
    own = (cols[k0:k1] >= lo) & (cols[k0:k1] < hi)
    rows = np.repeat(np.arange(hi - lo), np.diff(rp[lo:hi + 1]))
    cnt = np.bincount(rows[own], minlength=hi - lo)
    lrp = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
    m1 = D.DistMap(hi - lo, 1, 0, lrp, (cols[k0:k1][own] - lo).astype(np.int32))
    D.exchange_requests_local([m1])
    M = D.DistCsrMatrix(ex, m1, lrp, vals[k0:k1][own], int(rp[-1]))
    comm = D.Communicator.peer_group([0], 1)[0]
    bb = torch.from_numpy(bh[lo:hi].copy()).cuda()
    cfg = lk.SolverConfig(kind="cg", rel_tol=1e-30, fixed_iters=ITERS)
    M.solve(comm, bb, torch.zeros(hi - lo, dtype=torch.float64, device="cuda"), cfg)
    res = M.solve(comm, bb, torch.zeros(hi - lo, dtype=torch.float64, device="cuda"), cfg)
    print(f"P={P}: rank block {hi - lo} rows, halo {m.n_ghost}: "
          f"{res.elapsed / res.iterations * 1e6:7.1f} us/iteration", flush=True)
