"""GPU: full-size parity of the Krylov configs (cfg4 CG, cfg5 BiCGSTAB, 256^3)
on one GPU and row-partitioned over P = 2, 4, 8 ranks.

Two goldens, both generated on the CPU and committed:
* tests/golden/cfg45.npz -- the REFERENCE LIBRARY (oracle/_ref,
  ReferenceExecutor, krylov.cpp:119-230); the north-star bands hold against
  it (CG 581 +-1 and every history entry within 1e-7;
  BiCGSTAB in the reference's own spread [495, 498], the 1e-6 crossing at
  275, the first 40 entries within 1e-6, final <= 1e-8);
* tests/golden/cfg45_exact.npz -- krylov.cpp with exactly rounded dots
  (oracle/xkrylov.cpp, the product's reduction): the GPU reproduces its
  history, flop count and x (SHA-256) BIT FOR BIT -- on one GPU and at
  every rank count, which is what makes the iteration count independent
  of the partition."""
import hashlib
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "cfg45.npz")), np.load(os.path.join(GOLD, "cfg45_exact.npz"))


def check_cg(hist, iters, flops, gold):
    ref, ex = gold
    assert abs(iters - int(ref["cg_iters"])) <= 1
    h = np.asarray(hist)
    rh = ref["cg_hist"]
    k = min(len(h), len(rh))
    assert np.max(np.abs(h[:k] - rh[:k]) / rh[:k]) <= 1e-7
    assert h[-1] <= 1e-8
    assert iters == int(ex["cg_iters"]) and flops == int(ex["cg_flops"])
    assert h.tolist() == ex["cg_hist"].tolist()  # bit for bit


def check_bicg(hist, iters, flops, gold):
    ref, ex = gold
    assert 495 <= iters <= 498  # the reference's own executor spread
    h = np.asarray(hist)
    assert int(np.argmax(h <= 1e-6)) == 275
    rh = ref["bicg_hist"]
    assert np.max(np.abs(h[:41] - rh[:41]) / rh[:41]) <= 1e-6
    assert h[-1] <= 1e-8
    assert iters == int(ex["bicg_iters"]) and flops == int(ex["bicg_flops"])
    assert h.tolist() == ex["bicg_hist"].tolist()  # bit for bit


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x, np.float64).tobytes()).hexdigest()


def test_cfg4_cg_single_gpu(lk, ex, gold):
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, "7pt", 256)
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, lk.vector_from(ex, np.ones(A.ncols)), b)
    x = lk.zeros(ex, A.nrows)
    r = lk.solve(A, b, x, lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000))
    check_cg(r.residual_history, r.iterations, r.flop_count, gold)
    assert sha(lk.vector_to_host(x)) == str(gold[1]["cg_x_sha256"])
    # residual_mode 'recurrence' stops at the same iteration
    r2 = lk.solve(A, b, lk.zeros(ex, A.nrows),
                  lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000,
                                  residual_mode="recurrence"))
    assert r2.iterations == r.iterations and r2.final_rel_residual == r.final_rel_residual


def test_cfg5_bicgstab_single_gpu(lk, ex, gold):
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, "7pt", 256, 0.5)
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, lk.vector_from(ex, gen.seeded_values(A.ncols, 11)), b)
    x = lk.zeros(ex, A.nrows)
    r = lk.solve(A, b, x, lk.SolverConfig(kind="bicgstab", rel_tol=1e-8, max_iters=20000))
    check_bicg(r.residual_history, r.iterations, r.flop_count, gold)
    assert sha(lk.vector_to_host(x)) == str(gold[1]["bicg_x_sha256"])


def _run_peer(P, cases, tmp):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(P):
        env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(r),
                   WORLD_SIZE=str(P), LBK_PEER_TIMEOUT="300")
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests",
                                                                     "peer_worker_full.py"),
                                       str(tmp), ",".join(cases)], env=env))
    try:
        codes = [p.wait(timeout=1500) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert codes == [0] * P, codes
    return [json.loads((tmp / f"r{r}.json").read_text()) for r in range(P)]


@pytest.mark.parametrize("P", [2, 4, 8])
def test_full_size_distributed(P, gold, tmp_path):
    """cfg4 CG (both residual modes) and cfg5 BiCGSTAB over P peer-memory
    ranks: every rank reports the single-GPU golden bits; the assembled x
    hashes to the golden."""
    cases = ["cg", "bicgstab", "cg_rec"]
    out = _run_peer(P, cases, tmp_path)
    for o in out:
        check_cg(o["cg"]["hist"], o["cg"]["iters"], o["cg"]["flops"], gold)
        check_bicg(o["bicgstab"]["hist"], o["bicgstab"]["iters"], o["bicgstab"]["flops"], gold)
        assert o["cg_rec"]["iters"] == o["cg"]["iters"]
        assert o["cg_rec"]["hist"] == out[0]["cg_rec"]["hist"]
    for case, key in (("cg", "cg_x_sha256"), ("bicgstab", "bicg_x_sha256")):
        x = np.concatenate([np.load(tmp_path / f"r{r}_{case}.npy") for r in range(P)])
        assert sha(x) == str(gold[1][key]), case


# ------------------------------------------------------------------ cfg3
@pytest.fixture(scope="module")
def cfg3(O):
    """cfg3 at full size: the product's power-law generator (lbk_gen_powerlaw,
    the one bench.py uses) next to the oracle's (port_powerlaw_new), both
    SURVEY.md App. B (2^24 rows, window 65,536, max row 10,000)."""
    from paper_2011_08879_b200 import gen
    n = 1 << 24
    rp, ci, va = gen.powerlaw_host(n)
    R = O.powerlaw(n)
    return n, rp, ci, va, R


def test_cfg3_generator_matches_oracle(cfg3):
    n, rp, ci, va, R = cfg3
    assert int(rp[-1]) == R.nnz == 268_195_029  # App. B nnz KAT
    assert int(np.diff(R.row_ptr).max()) == 10_000
    assert np.array_equal(rp, R.row_ptr)
    assert np.array_equal(ci, R.cols)
    assert np.array_equal(va, R.vals)


def test_cfg3_fp64_csr_coo_full(O, lk, ex, cfg3):
    """FP64 CSR and COO SpMV on the full cfg3 matrix (16.7M rows, 268M nnz,
    x of 128 MiB > L2, int32 offsets near 2^28): rows of <= 256 entries are
    bit-identical to the reference order, the whole vector within 1e-12."""
    from conftest import relerr
    n, rp, ci, va, R = cfg3
    xh = O.seeded_values(n, 11)
    yref = O.spmv_csr(R, xh)
    A = lk.csr_from_host(ex, n, n, rp, ci, va)
    x = lk.vector_from(ex, xh)
    short = np.diff(rp) <= 256
    for name, M in (("csr", A), ("coo", lk.csr_to_coo(A))):
        y = lk.make_vector(ex, n)
        y.values.fill_(float("nan"))
        lk.spmv(M, x, y)
        yh = lk.vector_to_host(y)
        assert relerr(yh, yref) <= 1e-12, name
        assert np.array_equal(yh[short], yref[short]), name
        del M, y


def test_cfg3_fp32_csr_full(O, lk, ex, cfg3):
    """FP32 CSR on the full cfg3 matrix: within 1e-5 of the FP64 product of
    the FP32-rounded inputs; rows <= 256 equal the FP32 restatement."""
    import torch
    from conftest import relerr
    n, rp, ci, va, R = cfg3
    x32 = O.seeded_values(n, 11).astype(np.float32)
    v32 = va.astype(np.float32)
    ref64 = O.spmv_csr(O.Csr(n, n, R.row_ptr, R.cols, v32.astype(np.float64)),
                       x32.astype(np.float64))
    ref32 = O.spmv_csr(O.Csr(n, n, R.row_ptr, R.cols, v32), x32)
    A = lk.csr_from_host(ex, n, n, rp, ci, v32, dtype=torch.float32)
    x = lk.vector_from(ex, x32)
    y = lk.make_vector(ex, n, torch.float32)
    lk.spmv(A, x, y)
    yh = lk.vector_to_host(y)
    assert yh.dtype == np.float32
    assert relerr(yh, ref64) <= 1e-5
    short = np.diff(rp) <= 256
    assert np.array_equal(yh[short], ref32[short])
