"""GPU parity: device-resident CG / BiCGSTAB (lbk_solve_csr/coo) against the
reference library and the survey goldens:

* iteration counts: |I_gpu - I_ref| <= max(1, reference spread);
* residual histories within 1e-7 relative (CG) of the oracle's; BiCGSTAB
  over the first 40 iterations within 1e-6 (its trajectory is chaotic);
* flop_count equal to the reference accounting (krylov.cpp:41-69);
* KATs: 2x2 CG -> [1/11, 7/11]; A = I in 1 iteration; b = 0 -> 0 iterations;
  fixed_iters runs exactly that many; breakdown raises with its iteration.
"""
import os

import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def up(lk, ex, A):
    return lk.csr_from_host(ex, A.nrows, A.ncols, A.row_ptr, A.cols, A.vals)


def solve(lk, ex, M, bh, **cfg):
    b = lk.vector_from(ex, bh)
    x = lk.zeros(ex, M.nrows)
    r = lk.solve(M, b, x, lk.SolverConfig(**cfg))
    return r, lk.vector_to_host(x)


@pytest.mark.parametrize("fmt", ["csr", "coo"])
def test_cg16_golden(O, ex, lk, fmt):
    A = up(lk, ex, O.stencil("7pt", 16))
    M = A if fmt == "csr" else lk.csr_to_coo(A)
    r, x = solve(lk, ex, M, G["cg16_b"], kind="cg", rel_tol=1e-8, max_iters=20000)
    assert abs(r.iterations - int(G["cg16_iters"])) <= 1
    h, hr = np.array(r.residual_history), G["cg16_hist"]
    k = min(len(h), len(hr))
    # the reference's own executor spread at 16^3 is 1.3e-7 (reference vs
    # parallel(4)); allow ~8x that
    assert np.max(np.abs(h[:k] - hr[:k]) / hr[:k]) <= 1e-6
    if r.iterations == int(G["cg16_iters"]):
        assert r.flop_count == int(G["cg16_flops"])
    assert relerr(x, G["cg16_x"]) <= 1e-9
    assert r.converged and r.final_rel_residual <= 1e-8


def test_bicgstab16_golden(O, ex, lk):
    A = up(lk, ex, O.stencil("7pt", 16, 0.5))
    r, x = solve(lk, ex, A, G["bicg16_b"], kind="bicgstab", rel_tol=1e-8, max_iters=20000)
    assert abs(r.iterations - int(G["bicg16_iters"])) <= 1
    h, hr = np.array(r.residual_history), G["bicg16_hist"]
    # BiCGSTAB is chaotic under rounding: the reference's own executors agree
    # to ~1e-8 over 20 iterations but differ by up to 7e-5 by iteration 36
    k = min(len(h), len(hr), 20)
    assert np.max(np.abs(h[:k] - hr[:k]) / hr[:k]) <= 1e-6
    if r.iterations == int(G["bicg16_iters"]):
        assert r.flop_count == int(G["bicg16_flops"])
    assert r.converged


def test_kats(ex, lk):
    A = lk.csr_from_host(ex, 2, 2, [0, 2, 4], [0, 1, 0, 1], [4.0, 1.0, 1.0, 3.0])
    r, x = solve(lk, ex, A, np.array([1.0, 2.0]), kind="cg", rel_tol=1e-12, max_iters=10)
    assert np.allclose(x, [1 / 11, 7 / 11], rtol=0, atol=1e-12)
    assert np.allclose(x, G["cg2_x"], rtol=0, atol=1e-15)
    n = 1000
    I = lk.csr_from_host(ex, n, n, np.arange(n + 1), np.arange(n), np.ones(n))
    for kind in ("cg", "bicgstab"):
        r, x = solve(lk, ex, I, np.linspace(1, 2, n), kind=kind, rel_tol=1e-10)
        assert r.iterations == 1 and r.converged
        r, x = solve(lk, ex, I, np.zeros(n), kind=kind, rel_tol=1e-10)
        assert r.iterations == 0 and r.converged and r.residual_history == [0.0]
        assert np.all(x == 0)


def test_fixed_iters_and_freeze(O, ex, lk):
    R = O.stencil("7pt", 12)
    A = up(lk, ex, R)
    b = O.spmv_csr(R, np.ones(R.nrows))
    for kind in ("cg", "bicgstab"):
        r, _ = solve(lk, ex, A, b, kind=kind, rel_tol=1e-8, fixed_iters=300)
        assert r.iterations == 300 and len(r.residual_history) == 301
        if O.ref_available():
            rr = O.ref_solve(R, b, kind, rel_tol=1e-8, fixed_iters=300)
            assert rr.iterations == 300
            # the freeze (krylov.cpp:150-153) makes the tail constant
            assert r.residual_history[-1] == r.residual_history[-2]


def test_breakdown(R, ex, lk):
    O = R
    # <p, Ap> = 0 on the first iteration: A = [[0,1],[1,0]], b = [1,0]
    A = O.Csr(2, 2, np.array([0, 1, 2], np.int32), np.array([1, 0], np.int32), np.ones(2))
    with pytest.raises(O.OracleError) as e_ref:
        O.ref_solve(A, np.array([1.0, 0.0]), "cg", rel_tol=1e-10)
    with pytest.raises(lk.BreakdownError) as e:
        solve(lk, ex, up(lk, ex, A), np.array([1.0, 0.0]), kind="cg", rel_tol=1e-10)
    assert e.value.iteration == e_ref.value.iteration == 1


def test_config_errors(ex, lk):
    A = lk.csr_from_host(ex, 2, 2, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(lk.ConfigurationError):
        solve(lk, ex, A, np.ones(2), kind="cg", max_iters=0)
    with pytest.raises(lk.ConfigurationError):
        solve(lk, ex, A, np.ones(2), kind="cg", rel_tol=0.0)
    with pytest.raises(lk.ConfigurationError):
        solve(lk, ex, A, np.ones(2), kind="gmres", gmres_restart=0)
    with pytest.raises(lk.ConfigurationError):
        solve(lk, ex, A, np.ones(2), kind="gmres", max_iters=10, gmres_restart=11)
    with pytest.raises(lk.ConfigurationError):
        solve(lk, ex, A, np.ones(2), kind="minres")
    B = lk.csr_from_host(ex, 2, 3, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(lk.ShapeError):
        solve(lk, ex, B, np.ones(2), kind="cg")


@pytest.mark.parametrize("m,iters", [(32, 81), (64, 158), (128, 296)])
def test_cg_iteration_goldens(ex, lk, m, iters):
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, "7pt", m)
    ones = lk.vector_from(ex, np.ones(A.ncols))
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, ones, b)
    for mode in ("true", "recurrence"):
        x = lk.zeros(ex, A.nrows)
        r = lk.solve(A, b, x, lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000,
                                               residual_mode=mode))
        assert abs(r.iterations - iters) <= 1, (mode, r.iterations)
        assert r.converged and r.final_rel_residual <= 1e-8


def test_cg_history_vs_reference(R, ex, lk):
    O = R
    Rm = O.stencil("7pt", 32)
    b = O.spmv_csr(Rm, np.ones(Rm.nrows))
    rr = O.ref_solve(Rm, b, "cg", rel_tol=1e-8, max_iters=20000)
    spread = max(np.max(np.abs(p.history - rr.history) / rr.history)
                 for p in (O.ref_solve(Rm, b, "cg", rel_tol=1e-8, max_iters=20000, exec_kind=1,
                                       workers=w) for w in (2, 3, 4, 8)))
    r, x = solve(lk, ex, up(lk, ex, Rm), b, kind="cg", rel_tol=1e-8, max_iters=20000)
    assert r.iterations == rr.iterations
    assert r.flop_count == rr.flop_count
    h = np.array(r.residual_history)
    # within 10x the reference's own reduction-order spread (3.8e-8 here)
    assert np.max(np.abs(h - rr.history) / rr.history) <= max(1e-7, 10 * spread)
    assert relerr(x, rr.x) <= 1e-9


def test_bicgstab_history_vs_reference(R, ex, lk):
    O = R
    Rm = O.stencil("7pt", 32, 0.5)
    b = O.spmv_csr(Rm, O.seeded_values(Rm.nrows, 11))
    rr = O.ref_solve(Rm, b, "bicgstab", rel_tol=1e-8, max_iters=20000)
    rp = O.ref_solve(Rm, b, "bicgstab", rel_tol=1e-8, max_iters=20000, exec_kind=1, workers=8)
    r, _ = solve(lk, ex, up(lk, ex, Rm), b, kind="bicgstab", rel_tol=1e-8, max_iters=20000)
    spread = max(1, abs(rp.iterations - rr.iterations))
    assert abs(r.iterations - rr.iterations) <= spread
    h = np.array(r.residual_history)
    k = min(20, len(h), len(rr.history))
    assert np.max(np.abs(h[:k] - rr.history[:k]) / rr.history[:k]) <= 1e-6
    # over 40 iterations: within 3x the reference's own executor spread
    k = min(40, len(h), len(rr.history), len(rp.history))
    ref_spread = np.max(np.abs(rp.history[:k] - rr.history[:k]) / rr.history[:k])
    assert np.max(np.abs(h[:k] - rr.history[:k]) / rr.history[:k]) <= max(1e-6, 3 * ref_spread)


def test_cfg4_cg_256(ex, lk):
    """cfg4 at full size: 581 +- 1 iterations (golden), final
    true residual <= 1e-8, hist[1] = 5.037289e-01."""
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, "7pt", 256)
    ones = lk.vector_from(ex, np.ones(A.ncols))
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, ones, b)
    x = lk.zeros(ex, A.nrows)
    r = lk.solve(A, b, x, lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000))
    assert abs(r.iterations - 581) <= 1 and r.final_rel_residual <= 1e-8
    assert abs(r.residual_history[1] - 5.037289e-01) <= 1e-6
    assert r.flop_count == r.iterations * (4 * A.nnz() + 16 * A.nrows) + 2 * A.nnz() + 4 * A.nrows
    xh = lk.vector_to_host(x)
    assert np.max(np.abs(xh - 1.0)) < 1e-5


def test_cfg5_bicgstab_256(ex, lk):
    """cfg5: 7-pt upwind gamma 0.5, b = A x*, x* = seeded_values(n, 11):
    oracle 495 (reference) / 498 (parallel) -> accept 495 +- 3."""
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, "7pt", 256, 0.5)
    xs = lk.vector_from(ex, gen.seeded_values(A.ncols, 11))
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, xs, b)  # bit-identical to the oracle's CSR SpMV (rows <= 32)
    x = lk.zeros(ex, A.nrows)
    r = lk.solve(A, b, x, lk.SolverConfig(kind="bicgstab", rel_tol=1e-8, max_iters=20000))
    assert abs(r.iterations - 495) <= 3, r.iterations
    assert r.final_rel_residual <= 1e-8
    assert abs(r.residual_history[1] - 1.136784e-01) <= 1e-6


@pytest.mark.parametrize("m,gamma", [(16, 0.0), (24, 0.5)])
def test_cgs_vs_reference(R, ex, lk, m, gamma):
    """CGS (krylov.cpp:233-297, §8f.2): iterations within the reference's
    own executor spread, flop accounting equal, early history agreement."""
    O = R
    Rm = O.stencil("7pt", m, gamma)
    b = O.spmv_csr(Rm, O.seeded_values(Rm.nrows, 11))
    rr = O.ref_solve(Rm, b, "cgs", rel_tol=1e-8, max_iters=20000)
    rp = O.ref_solve(Rm, b, "cgs", rel_tol=1e-8, max_iters=20000, exec_kind=1, workers=8)
    r, x = solve(lk, ex, up(lk, ex, Rm), b, kind="cgs", rel_tol=1e-8, max_iters=20000)
    spread = max(1, abs(rp.iterations - rr.iterations))
    assert abs(r.iterations - rr.iterations) <= spread, (r.iterations, rr.iterations)
    if r.iterations == rr.iterations:
        assert r.flop_count == rr.flop_count
    h = np.array(r.residual_history)
    k = min(10, len(h), len(rr.history))
    assert np.max(np.abs(h[:k] - rr.history[:k]) / rr.history[:k]) <= 1e-6
    assert r.converged and r.final_rel_residual <= 1e-8
    assert relerr(x, rr.x) <= 1e-6


def test_cgs_fixed_iters(R, ex, lk):
    O = R
    Rm = O.stencil("7pt", 10)
    b = O.spmv_csr(Rm, np.ones(Rm.nrows))
    rr = O.ref_solve(Rm, b, "cgs", rel_tol=1e-8, fixed_iters=120)
    r, _ = solve(lk, ex, up(lk, ex, Rm), b, kind="cgs", rel_tol=1e-8, fixed_iters=120)
    assert r.iterations == rr.iterations == 120
    assert len(r.residual_history) == 121


@pytest.mark.parametrize("m,gamma,restart", [(12, 0.0, 30), (16, 0.5, 30), (12, 0.5, 5)])
def test_gmres_vs_reference(R, ex, lk, m, gamma, restart):
    """Restarted GMRES (krylov.cpp:308-443, §8f.2): MGS on the device, the
    Givens / back-substitution scalars advanced by finisher threads."""
    O = R
    Rm = O.stencil("7pt", m, gamma)
    b = O.spmv_csr(Rm, O.seeded_values(Rm.nrows, 11))
    rr = O.ref_solve(Rm, b, "gmres", rel_tol=1e-8, max_iters=20000, restart=restart)
    rp = O.ref_solve(Rm, b, "gmres", rel_tol=1e-8, max_iters=20000, restart=restart,
                     exec_kind=1, workers=8)
    r, x = solve(lk, ex, up(lk, ex, Rm), b, kind="gmres", rel_tol=1e-8, max_iters=20000,
                 gmres_restart=restart)
    spread = max(1, abs(rp.iterations - rr.iterations))
    assert abs(r.iterations - rr.iterations) <= spread, (r.iterations, rr.iterations)
    if r.iterations == rr.iterations:
        assert r.flop_count == rr.flop_count
    h = np.array(r.residual_history)
    k = min(10, len(h), len(rr.history))
    assert np.max(np.abs(h[:k] - rr.history[:k]) / rr.history[:k]) <= 1e-6
    assert r.converged and r.final_rel_residual <= 1e-8
    assert relerr(x, rr.x) <= 1e-6


def test_gmres_fixed_iters(R, ex, lk):
    O = R
    Rm = O.stencil("7pt", 8, 0.5)
    b = O.spmv_csr(Rm, np.ones(Rm.nrows))
    rr = O.ref_solve(Rm, b, "gmres", rel_tol=1e-8, fixed_iters=50, restart=7)
    r, _ = solve(lk, ex, up(lk, ex, Rm), b, kind="gmres", rel_tol=1e-8, fixed_iters=50,
                 gmres_restart=7)
    assert r.iterations == rr.iterations == 50
    assert len(r.residual_history) == 51


@pytest.mark.parametrize("kind", ["cg", "bicgstab", "cgs"])
def test_graph_captured_chunks_identical(O, ex, lk, kind, monkeypatch):
    """Chunks after the first replayed as one CUDA graph give the same
    iterations, history and x, bit for bit."""
    A = O.stencil("7pt", 24, 0.5 if kind != "cg" else 0.0)
    b = O.spmv_csr(A, O.seeded_values(A.nrows, 11))
    M = up(lk, ex, A)
    monkeypatch.setenv("LBK_SOLVER_GRAPH", "0")
    r0, x0 = solve(lk, ex, M, b, kind=kind, rel_tol=1e-8, max_iters=20000)
    monkeypatch.setenv("LBK_SOLVER_GRAPH", "1")
    r1, x1 = solve(lk, ex, M, b, kind=kind, rel_tol=1e-8, max_iters=20000)
    assert r0.iterations == r1.iterations and r0.iterations > 32
    assert r0.residual_history == r1.residual_history
    assert np.array_equal(x0, x1) and r0.flop_count == r1.flop_count


@pytest.mark.parametrize("kind", ["cg", "bicgstab", "cgs", "gmres"])
def test_paper_fixed_10000_protocol(R, ex, lk, kind):
    """Paper §6.2 / SPEC.md:645 #10: benchmark mode runs exactly 10,000
    iterations (COO SpMV, the harness's default), freezing the history once
    the residual reaches the machine floor (krylov.cpp:150-153) -- or stops
    with the same BreakdownError the reference raises (CGS's rho vanishes
    after convergence on this problem, in the reference too)."""
    O = R
    A = O.stencil("7pt", 10, 0.5 if kind != "cg" else 0.0)
    b = O.spmv_csr(A, np.ones(A.nrows))
    M = lk.csr_to_coo(up(lk, ex, A))
    try:
        rr = O.ref_solve(A, b, kind, rel_tol=1e-8, fixed_iters=10000, max_iters=10000,
                         restart=30, fmt="coo")
        ref_breakdown = None
    except O.OracleError as e:
        ref_breakdown = e
    if ref_breakdown is not None:
        with pytest.raises(lk.BreakdownError):
            solve(lk, ex, M, b, kind=kind, rel_tol=1e-8, fixed_iters=10000, max_iters=10000,
                  gmres_restart=30)
        return
    r, x = solve(lk, ex, M, b, kind=kind, rel_tol=1e-8, fixed_iters=10000, max_iters=10000,
                 gmres_restart=30)
    assert r.iterations == rr.iterations == 10000 and len(r.residual_history) == 10001
    # the converged prefix agrees; past convergence the runs are rounding noise
    k = next(i for i, h in enumerate(rr.history) if h <= 1e-8)
    assert abs(next(i for i, h in enumerate(r.residual_history) if h <= 1e-8) - k) <= 1


def _g45():
    p = os.path.join(os.path.dirname(__file__), "golden", "cfg45.npz")
    if not os.path.exists(p):
        pytest.skip("tests/golden/cfg45.npz not generated")
    return np.load(p)


def test_cfg4_full_history_vs_reference():
    """SURVEY.md §8c recommended cfg4 report: iterations 581 +- 1, every
    residual_history entry within 1e-7 relative of the reference's (~17x the
    reference's own executor spread), final true residual <= 1e-8, flops."""
    import torch
    from paper_2011_08879_b200 import gen, larch as lk
    g = _g45()
    ex = lk.CudaExecutor(0)
    A = gen.stencil(ex, "7pt", 256)
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, lk.vector_from(ex, np.ones(A.ncols)), b)
    x = lk.zeros(ex, A.nrows)
    r = lk.solve(A, b, x, lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000))
    assert int(g["cg_iters"]) == 581 and abs(r.iterations - 581) <= 1
    h, hr = np.array(r.residual_history), g["cg_hist"]
    k = min(len(h), len(hr))
    assert np.max(np.abs(h[:k] - hr[:k]) / hr[:k]) <= 1e-7
    assert r.final_rel_residual <= 1e-8
    if r.iterations == int(g["cg_iters"]):
        assert r.flop_count == int(g["cg_flops"])


def test_cfg5_report_vs_reference():
    """SURVEY.md §8c recommended cfg5 report: (1) iterations inside the
    oracle band (reference 495 / parallel 498, +-3), (2) exact match of the
    first crossing of tol 1e-6 (275 on both oracle executors), (3) history
    within 1e-6 relative over the first 40 iterations, (4) final true
    residual <= tol."""
    from paper_2011_08879_b200 import gen, larch as lk
    g = _g45()
    ex = lk.CudaExecutor(0)
    A = gen.stencil(ex, "7pt", 256, 0.5)
    xs = lk.vector_from(ex, gen.seeded_values(A.ncols, 11))
    b = lk.make_vector(ex, A.nrows)
    lk.spmv(A, xs, b)
    x = lk.zeros(ex, A.nrows)
    r = lk.solve(A, b, x, lk.SolverConfig(kind="bicgstab", rel_tol=1e-8, max_iters=20000))
    ref_iters = int(g["bicg_iters"])
    assert ref_iters == 495
    assert abs(r.iterations - ref_iters) <= 3
    h, hr = np.array(r.residual_history), g["bicg_hist"]
    first = lambda hh, tol: int(np.argmax(hh <= tol))  # noqa: E731
    assert first(h, 1e-6) == first(hr, 1e-6) == 275
    assert np.max(np.abs(h[:40] - hr[:40]) / hr[:40]) <= 1e-6
    assert r.final_rel_residual <= 1e-8


# ------------------------------------------------------ gmres_restart_cycle
@pytest.mark.parametrize("m,restart", [(12, 10), (10, 40)])
def test_gmres_restart_cycle_vs_reference(R, lk, ex, m, restart):
    """gmres_restart_cycle (krylov.hpp:78-89) against the reference
    library's: the same step count and happy flag, the residual and x to
    rounding, an orthonormal basis matching the reference's to rounding."""
    O = R
    A = O.stencil("7pt", m, 0.5)
    b = O.spmv_csr(A, O.seeded_values(A.nrows, 11))
    ref = O.ref_gmres_cycle(A, b, restart=restart)
    Ad = lk.csr_from_host(ex, A.nrows, A.ncols, A.row_ptr, A.cols, A.vals)
    x = lk.zeros(ex, A.nrows)
    basis = []
    r = lk.gmres_restart_cycle(Ad, lk.vector_from(ex, b), x, restart, basis)
    assert r.steps == ref["steps"] and r.happy_breakdown == ref["happy"]
    assert abs(r.rel_residual - ref["rel_residual"]) <= 1e-6 * ref["rel_residual"] + 1e-15
    assert np.max(np.abs(lk.vector_to_host(x) - ref["x"])) <= 1e-9 * np.max(np.abs(ref["x"]))
    assert len(basis) == len(ref["basis"])
    V = np.stack([lk.vector_to_host(v) for v in basis])
    # the leading Krylov vectors to rounding; later ones amplify the dot
    # rounding differences as the residual falls (ill-conditioned
    # directions), so they are held to the orthonormality both bases share
    k = min(6, len(basis))
    assert np.max(np.abs(V[:k] - ref["basis"][:k])) <= 1e-8
    G = V[:k] @ V[:k].T
    assert np.max(np.abs(G - np.eye(k))) <= 1e-10
    assert np.allclose(np.linalg.norm(V, axis=1), 1.0, atol=1e-12)


def test_gmres_restart_cycle_edge_cases(lk, ex, O):
    A = O.stencil("7pt", 6)
    Ad = lk.csr_from_host(ex, A.nrows, A.ncols, A.row_ptr, A.cols, A.vals)
    # x already exact: zero residual -> happy, no steps, empty basis
    b = O.spmv_csr(A, np.ones(A.nrows))
    basis = []
    r = lk.gmres_restart_cycle(Ad, lk.vector_from(ex, b), lk.vector_from(ex, np.ones(A.nrows)), 5,
                               basis)
    assert r.steps == 0 and r.happy_breakdown and r.rel_residual == 0.0 and basis == []
    with pytest.raises(lk.ConfigurationError):
        lk.gmres_restart_cycle(Ad, lk.vector_from(ex, b), lk.zeros(ex, A.nrows), 0)
