"""GPU: the distributed path on one B200.

P virtual ranks run as P host threads, each with its own executor and
stream, through the in-process communicator (the same partition, halo,
deferred-reduction and allreduce logic as NCCL, with device copies for
the exchange). The one-rank NCCL communicator checks the NCCL path itself.

Bars:
* distributed SpMV is bit-identical to the global oracle SpMV, because
  every row keeps its ascending-k order;
* distributed CG/BiCGSTAB iteration counts are within the reference's
  spread (±1 for CG);
* every rank reports the same result."""
import threading

import numpy as np
import pytest
import torch

from conftest import relerr

pytestmark = pytest.mark.gpu


def build(O, lk, A, P):
    from paper_2011_08879_b200 import dist as D
    maps, parts = [], []
    for rank in range(P):
        rp, cols, vals = D.local_rows(A.row_ptr, A.cols, A.vals, P, rank)
        maps.append(D.DistMap(A.nrows, P, rank, rp, cols))
        parts.append((rp, vals))
    D.exchange_requests_local(maps)
    exs = [lk.CudaExecutor(0, stream=torch.cuda.Stream()) for _ in range(P)]
    mats = [D.DistCsrMatrix(exs[r], maps[r], parts[r][0], parts[r][1], A.nnz) for r in range(P)]
    comms = D.Communicator.threads(P) if P > 1 else [None]
    return exs, mats, comms


def run_threads(P, fn):
    errs, out = [], [None] * P

    def w(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=w, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("kind,m,P", [("7pt", 16, 1), ("7pt", 16, 2), ("27pt", 14, 3),
                                      ("5pt", 70, 4), ("7pt", 12, 8)])
def test_dist_spmv_bitexact(O, lk, kind, m, P):
    A = O.stencil(kind, m, 0.5 if kind == "7pt" else 0.0)
    x = O.seeded_values(A.ncols, 11)
    yref = O.spmv_csr(A, x)
    exs, mats, comms = build(O, lk, A, P)
    from paper_2011_08879_b200 import dist as D
    xs = [mats[r].ext_vector(x[slice(*D.part_range(A.nrows, P, r))]) for r in range(P)]
    ys = [torch.full((mats[r].n_local,), float("nan"), dtype=torch.float64, device="cuda")
          for r in range(P)]
    torch.cuda.synchronize()
    run_threads(P, lambda r: mats[r].spmv(comms[r], xs[r], ys[r]))
    torch.cuda.synchronize()
    y = np.concatenate([t.cpu().numpy() for t in ys])
    assert np.array_equal(y, yref)


@pytest.mark.parametrize("P", [1, 2, 4])
def test_dist_cg(O, lk, P):
    A = O.stencil("7pt", 32)
    b = O.spmv_csr(A, np.ones(A.nrows))
    exs, mats, comms = build(O, lk, A, P)
    from paper_2011_08879_b200 import dist as D
    rng = [D.part_range(A.nrows, P, r) for r in range(P)]
    bs = [torch.from_numpy(b[lo:hi].copy()).cuda() for lo, hi in rng]
    xs = [torch.zeros(hi - lo, dtype=torch.float64, device="cuda") for lo, hi in rng]
    torch.cuda.synchronize()
    cfg = lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000)
    res = run_threads(P, lambda r: mats[r].solve(comms[r], bs[r], xs[r], cfg))
    torch.cuda.synchronize()
    assert all(r.iterations == res[0].iterations for r in res)
    assert all(r.residual_history == res[0].residual_history for r in res)
    assert abs(res[0].iterations - 81) <= 1  # golden
    assert res[0].converged
    # reference flop accounting over the GLOBAL sizes
    I = res[0].iterations
    assert res[0].flop_count == I * (4 * A.nnz + 16 * A.nrows) + 2 * A.nnz + 4 * A.nrows
    x = np.concatenate([t.cpu().numpy() for t in xs])
    assert np.max(np.abs(x - 1.0)) < 1e-5


@pytest.mark.parametrize("P", [2, 3])
def test_dist_bicgstab(O, lk, P):
    A = O.stencil("7pt", 24, 0.5)
    b = O.spmv_csr(A, O.seeded_values(A.nrows, 11))
    exs, mats, comms = build(O, lk, A, P)
    from paper_2011_08879_b200 import dist as D
    rng = [D.part_range(A.nrows, P, r) for r in range(P)]
    bs = [torch.from_numpy(b[lo:hi].copy()).cuda() for lo, hi in rng]
    xs = [torch.zeros(hi - lo, dtype=torch.float64, device="cuda") for lo, hi in rng]
    torch.cuda.synchronize()
    cfg = lk.SolverConfig(kind="bicgstab", rel_tol=1e-8, max_iters=20000)
    res = run_threads(P, lambda r: mats[r].solve(comms[r], bs[r], xs[r], cfg))
    torch.cuda.synchronize()
    assert all(r.iterations == res[0].iterations for r in res)
    if O.ref_available():
        rr = O.ref_solve(A, b, "bicgstab", rel_tol=1e-8, max_iters=20000)
        rp = O.ref_solve(A, b, "bicgstab", rel_tol=1e-8, max_iters=20000, exec_kind=1, workers=8)
        assert abs(res[0].iterations - rr.iterations) <= max(1, abs(rp.iterations - rr.iterations))
        x = np.concatenate([t.cpu().numpy() for t in xs])
        assert relerr(x, rr.x) <= 1e-6


def test_nccl_single_rank(O, lk):
    """The NCCL communicator path (1 rank: init, allreduce, solve)."""
    from paper_2011_08879_b200 import dist as D
    comm = D.Communicator.nccl_single(0)
    ex = lk.CudaExecutor(0)
    t = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
    comm.allreduce_sum(ex, t)
    ex.synchronize()
    assert t.tolist() == [1.5, -2.0]
    A = O.stencil("7pt", 16)
    b = O.spmv_csr(A, np.ones(A.nrows))
    m = D.DistMap(A.nrows, 1, 0, A.row_ptr, A.cols)
    D.exchange_requests_local([m])
    M = D.DistCsrMatrix(ex, m, A.row_ptr, A.vals, A.nnz)
    x = torch.zeros(A.nrows, dtype=torch.float64, device="cuda")
    r = M.solve(comm, torch.from_numpy(b).cuda(), x, lk.SolverConfig(kind="cg", rel_tol=1e-8))
    assert abs(r.iterations - 41) <= 1
    # chunks after the first run as a captured CUDA graph (NCCL allreduce
    # inside); the 32^3 solve (81 iterations) replays it several times
    A = O.stencil("7pt", 32)
    b = O.spmv_csr(A, np.ones(A.nrows))
    m = D.DistMap(A.nrows, 1, 0, A.row_ptr, A.cols)
    D.exchange_requests_local([m])
    M = D.DistCsrMatrix(ex, m, A.row_ptr, A.vals, A.nnz)
    x = torch.zeros(A.nrows, dtype=torch.float64, device="cuda")
    r = M.solve(comm, torch.from_numpy(b).cuda(), x, lk.SolverConfig(kind="cg", rel_tol=1e-8))
    assert abs(r.iterations - 81) <= 1 and r.converged


@pytest.mark.parametrize("kind,P", [("cgs", 2), ("gmres", 3)])
def test_dist_cgs_gmres(O, lk, kind, P):
    """The other solvers run unchanged on the distributed environment."""
    A = O.stencil("7pt", 14, 0.5)
    b = O.spmv_csr(A, O.seeded_values(A.nrows, 11))
    exs, mats, comms = build(O, lk, A, P)
    from paper_2011_08879_b200 import dist as D
    rng = [D.part_range(A.nrows, P, r) for r in range(P)]
    bs = [torch.from_numpy(b[lo:hi].copy()).cuda() for lo, hi in rng]
    xs = [torch.zeros(hi - lo, dtype=torch.float64, device="cuda") for lo, hi in rng]
    torch.cuda.synchronize()
    cfg = lk.SolverConfig(kind=kind, rel_tol=1e-8, max_iters=20000, gmres_restart=20)
    res = run_threads(P, lambda r: mats[r].solve(comms[r], bs[r], xs[r], cfg))
    torch.cuda.synchronize()
    assert all(r.iterations == res[0].iterations for r in res)
    if O.ref_available():
        rr = O.ref_solve(A, b, kind, rel_tol=1e-8, max_iters=20000, restart=20)
        rp = O.ref_solve(A, b, kind, rel_tol=1e-8, max_iters=20000, restart=20, exec_kind=1,
                         workers=8)
        assert abs(res[0].iterations - rr.iterations) <= max(1, abs(rp.iterations - rr.iterations))
    x = np.concatenate([t.cpu().numpy() for t in xs])
    assert res[0].converged
    assert np.max(np.abs(O.spmv_csr(A, x) - b)) <= 1e-7 * np.max(np.abs(b))



@pytest.fixture(scope="module", params=[2, 4])
def peer_run(request, tmp_path_factory):
    """P processes on cuda:0, one peer-memory rank each (tests/peer_worker.py):
    one CUDA context per rank, windows swapped as CUDA IPC handles over
    gloo -- the one-process-per-GPU deployment, with the GPUs folded onto
    one device. (Ranks must not share a context: a kernel spinning on a
    peer's flag would block device-synchronising calls of the other ranks'
    host threads.)"""
    import json
    import os
    import socket
    import subprocess
    import sys
    P = request.param
    tmp = tmp_path_factory.mktemp(f"peer{P}")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    here = os.path.dirname(os.path.abspath(__file__))
    procs = []
    for r in range(P):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(r),
                   WORLD_SIZE=str(P), LBK_PEER_TIMEOUT="120")
        procs.append(subprocess.Popen([sys.executable, os.path.join(here, "peer_worker.py"),
                                       str(tmp / f"r{r}.json")], env=env))
    try:
        codes = [p.wait(timeout=900) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert codes == [0] * P, codes
    return P, [json.loads((tmp / f"r{r}.json").read_text()) for r in range(P)]


def test_peer_spmv_bitexact(peer_run):
    P, out = peer_run
    for o in out:
        assert o["spmv_7pt"] and o["spmv_27pt"] and o["spmv_5pt"]
        assert o["spmv_back_to_back"]
        assert o["shared_comm_abba"]
        assert o["allreduce"] == [P * (P + 1) / 2, 0.25 * P]


def test_peer_solvers(peer_run, O):
    P, out = peer_run
    for kind in ("cg", "bicgstab", "bicgstab_eager", "cgs", "gmres"):
        r0 = out[0][kind]
        for o in out[1:]:  # every rank: the same iterations and history bits
            assert o[kind]["iters"] == r0["iters"] and o[kind]["hist"] == r0["hist"], kind
        assert r0["conv"], kind
    assert abs(out[0]["cg"]["iters"] - 81) <= 1  # golden
    # two exchanges per CG iteration (K3's residual rides with the next
    # <p,Ap>) give exactly the three-exchange path's history and x
    assert out[0]["cg"]["hist"] == out[0]["cg_3x"]["hist"]
    assert out[0]["cg"]["x"] == out[0]["cg_3x"]["x"]
    # fixed iteration count: the loop ends on a deferred residual (flush)
    assert out[0]["cg_fixed"]["iters"] == 50 and len(out[0]["cg_fixed"]["hist"]) == 51
    A = O.stencil("7pt", 32)
    I = out[0]["cg"]["iters"]
    assert out[0]["cg"]["flops"] == I * (4 * A.nnz + 16 * A.nrows) + 2 * A.nnz + 4 * A.nrows
    x = np.concatenate([o["cg"]["x"] for o in out])
    assert np.max(np.abs(x - 1.0)) < 1e-5
    # captured graph and eager launches give the same bits
    assert out[0]["bicgstab"]["hist"] == out[0]["bicgstab_eager"]["hist"]
    assert out[0]["bicgstab"]["hist"] == out[0]["bicgstab_unmerged"]["hist"]
    assert out[0]["bicgstab"]["hist"] == out[0]["bicgstab_digits"]["hist"]
    assert out[0]["bicgstab"]["x"] == out[0]["bicgstab_digits"]["x"]
    assert out[0]["bicgstab"]["x"] == out[0]["bicgstab_unmerged"]["x"]
    assert out[0]["bicgstab_fixed"]["iters"] == 23
    assert len(out[0]["bicgstab_fixed"]["hist"]) == 24
    A = O.stencil("7pt", 20, 0.5)
    b = O.spmv_csr(A, O.seeded_values(A.nrows, 11))
    x = np.concatenate([o["bicgstab"]["x"] for o in out])
    assert np.max(np.abs(O.spmv_csr(A, x) - b)) <= 1e-7 * np.max(np.abs(b))
    if O.ref_available():
        rr = O.ref_solve(A, b, "bicgstab", rel_tol=1e-8, max_iters=20000)
        rp = O.ref_solve(A, b, "bicgstab", rel_tol=1e-8, max_iters=20000, exec_kind=1, workers=8)
        assert abs(out[0]["bicgstab"]["iters"] - rr.iterations) <= max(
            1, abs(rp.iterations - rr.iterations))


def test_peer_timeout_reported(peer_run):
    P, out = peer_run
    assert "timed out waiting for halo values" in out[0]["timeout"], out[0]["timeout"]
