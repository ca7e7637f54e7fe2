"""CPU: pin the oracle before trusting it.

* the reference library (oracle/_ref) reproduces the SPEC KATs and the
  committed golden vectors (tests/golden/golden.npz, made by
  tests/golden/make_golden.py from that same library);
* our restatement (oracle/port.cpp) is bit-identical to the reference on
  CSR/COO SpMV and the conversions, over the golden cases and random
  matrices;
* the restatement's additions (ELL, SELL-P, FP32, partition maps), which
  have no reference implementation, are checked against the App. B integer
  KATs, brute force, and bit-for-bit against the reference CSR SpMV.
"""
import os

import numpy as np
import pytest

from conftest import relerr

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def _rnd(i):
    return {k.split("_", 1)[1]: G[k] for k in G.files if k.startswith(f"rnd{i}_")}


# ------------------------------------------------------------- golden / KAT
def test_spec_kats_reference(R):
    O = R
    y, _ = O.ref_spmv(O.Csr(3, 3, np.array([0, 1, 2, 3], np.int32), np.array([0, 1, 2], np.int32),
                            np.ones(3)), np.array([1.0, 2.0, 3.0]))
    assert list(y) == [1.0, 2.0, 3.0]
    y, _ = O.ref_spmv(O.Csr(2, 2, np.array([0, 2, 3], np.int32), np.array([0, 1, 1], np.int32),
                            np.array([1.0, 2.0, 3.0])), np.array([1.0, 1.0]))
    assert list(y) == [3.0, 3.0]
    assert list(G["kat_empty_y"]) == [10.0, 0.0]
    assert list(G["kat_c2c_rowptr"]) == [0, 2, 3]
    assert list(G["kat_c2c_empty_rowptr"]) == [0, 0, 0, 0]
    # coo_from_entries: sort + dedupe
    ro, co, vo = O.ref_coo_from_entries(2, 2, [1, 0, 1], [0, 1, 0], [1.0, 2.0, 3.0])
    assert list(ro) == [0, 1] and list(co) == [1, 0] and list(vo) == [2.0, 4.0]


def test_cg_2x2_kat():
    assert np.allclose(G["cg2_x"], [1 / 11, 7 / 11], rtol=0, atol=1e-12)


@pytest.mark.parametrize("i", range(6))
def test_reference_reproduces_golden(R, i):
    O, g = R, _rnd(i)
    nr, nc = (int(v) for v in g["shape"])
    ro, co, vo = O.ref_coo_from_entries(nr, nc, g["in_rows"], g["in_cols"], g["in_vals"])
    assert np.array_equal(ro, g["rows"]) and np.array_equal(co, g["cols"])
    assert np.array_equal(vo, g["vals"])
    y, _ = O.ref_spmv(O.Csr(nr, nc, g["rowptr"], g["cols"], g["vals"]), g["x"])
    assert np.array_equal(y, g["y_csr"])


@pytest.mark.parametrize("i", range(6))
def test_port_matches_golden_bitwise(O, i):
    g = _rnd(i)
    nr, nc = (int(v) for v in g["shape"])
    rp = O.coo_to_csr_ptr(nr, g["rows"])
    assert np.array_equal(rp, g["rowptr"])
    A = O.Csr(nr, nc, rp, g["cols"], g["vals"])
    assert np.array_equal(O.csr_to_coo_rows(A), g["rows"])
    assert np.array_equal(O.spmv_csr(A, g["x"]), g["y_csr"])
    assert np.array_equal(O.spmv_coo(nr, g["rows"], g["cols"], g["vals"], g["x"]), g["y_coo"])
    # CSR and COO agree bitwise in the FMA-free build
    assert np.array_equal(g["y_csr"], g["y_coo"])


def test_port_stencil_spmv_golden(O):
    A = O.stencil("5pt", 32)
    assert np.array_equal(O.seeded_values(A.ncols, 11), G["st5_x"])
    assert np.array_equal(O.spmv_csr(A, G["st5_x"]), G["st5_y"])


def test_solver_goldens_reference(R):
    O = R
    A = O.stencil("7pt", 16)
    r = O.ref_solve(A, G["cg16_b"], "cg", rel_tol=1e-8, max_iters=20000)
    assert r.iterations == int(G["cg16_iters"]) == 41  # SURVEY.md §8c golden
    assert np.array_equal(r.history, G["cg16_hist"])
    assert r.flop_count == int(G["cg16_flops"])
    # flop accounting KAT: I*(4nnz+16n) + 2nnz + 4n
    n, nnz, I = A.nrows, A.nnz, r.iterations
    assert r.flop_count == I * (4 * nnz + 16 * n) + 2 * nnz + 4 * n
    A = O.stencil("7pt", 16, 0.5)
    r = O.ref_solve(A, G["bicg16_b"], "bicgstab", rel_tol=1e-8, max_iters=20000)
    assert r.iterations == int(G["bicg16_iters"])
    assert r.flop_count == r.iterations * (6 * A.nnz + 28 * A.nrows) + 2 * A.nnz + 2 * A.nrows


@pytest.mark.parametrize("m,iters", [(16, 41), (32, 81)])
def test_cg_iteration_goldens(R, m, iters):
    O = R
    A = O.stencil("7pt", m)
    b, _ = O.ref_spmv(A, np.ones(A.nrows))
    assert O.ref_solve(A, b, "cg", rel_tol=1e-8, max_iters=20000).iterations == iters
    # executor-invariant for CG
    assert O.ref_solve(A, b, "cg", rel_tol=1e-8, max_iters=20000, exec_kind=1,
                       workers=4).iterations == iters


def test_bicgstab_a1_golden_and_breakdown(R):
    O = R
    A = O.stencil("7pt", 16, 0.5)
    b, _ = O.ref_spmv(A, np.ones(A.nrows))
    assert O.ref_solve(A, b, "bicgstab", rel_tol=1e-8, max_iters=20000).iterations == 42


# ---------------------------------------------- restatement vs reference
def _random_csr(rng, nr, nc, density):
    mask = rng.random((nr, nc)) < density
    rows, cols = np.nonzero(mask)
    vals = rng.uniform(-1, 1, rows.size)
    rp = np.zeros(nr + 1, np.int32)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    from oracle.oracle import Csr
    return Csr(nr, nc, rp, cols.astype(np.int32), vals)


def test_port_vs_reference_random(R):
    O = R
    rng = np.random.default_rng(5)
    for trial in range(40):
        nr, nc = int(rng.integers(1, 200)), int(rng.integers(1, 200))
        A = _random_csr(rng, nr, nc, float(rng.uniform(0, 0.3)))
        x = rng.uniform(-1, 1, nc)
        yr, _ = O.ref_spmv(A, x, "csr")
        yc, _ = O.ref_spmv(A, x, "coo")
        assert np.array_equal(O.spmv_csr(A, x), yr)
        assert np.array_equal(yr, yc)
        ro, co, vo = O.ref_csr_to_coo(A)
        assert np.array_equal(O.csr_to_coo_rows(A), ro)
        assert np.array_equal(O.coo_to_csr_ptr(nr, ro), A.row_ptr)


def test_port_powerlaw_vs_reference(R):
    O = R
    A = O.powerlaw(1 << 14, window=4096, max_len=2000)
    assert A.row_ptr[-1] == A.nnz
    d = np.diff(A.row_ptr)
    assert d.min() >= 1 and d.max() <= 2000
    for r in range(0, A.nrows, 997):  # sorted unique columns inside the window
        c = A.cols[A.row_ptr[r]:A.row_ptr[r + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= max(0, r - 4096) and c.max() <= r + 4096
    x = O.seeded_values(A.ncols, 11)
    yr, _ = O.ref_spmv(A, x)
    assert np.array_equal(O.spmv_csr(A, x), yr)


# ---------------------------------------------- unpinned additions (App. B)
def test_ell_sellp_layout_bruteforce(O):
    rng = np.random.default_rng(9)
    for n in range(1, 17):
        A = _random_csr(rng, n, n, 0.4)
        w, s, ec, ev = O.csr_to_ell(A)
        assert w == (np.diff(A.row_ptr).max() if n else 0)
        for r in range(n):
            k0, k1 = A.row_ptr[r], A.row_ptr[r + 1]
            for j in range(w):
                if k0 + j < k1:
                    assert ec[j * s + r] == A.cols[k0 + j] and ev[j * s + r] == A.vals[k0 + j]
                else:
                    assert ec[j * s + r] == -1 and ev[j * s + r] == 0.0
        for S in (1, 2, 4, 32):
            sl, ss, sc, sv = O.csr_to_sellp(A, S)
            ns = (n + S - 1) // S
            assert len(sl) == ns and ss[0] == 0 and len(ss) == ns + 1
            seen = np.zeros(ss[-1] * S, bool)
            for r in range(n):
                sl_r = r // S
                assert sl[sl_r] == max(np.diff(A.row_ptr)[sl_r * S:(sl_r + 1) * S])
                k0, k1 = A.row_ptr[r], A.row_ptr[r + 1]
                for j in range(sl[sl_r]):
                    pos = (ss[sl_r] + j) * S + r % S
                    assert not seen[pos]
                    seen[pos] = True
                    if k0 + j < k1:
                        assert sc[pos] == A.cols[k0 + j]
                    else:
                        assert sc[pos] == -1 and sv[pos] == 0.0


def test_ell_sellp_spmv_bitwise_vs_reference_csr(R):
    O = R
    A = O.stencil("27pt", 12)
    x = O.seeded_values(A.ncols, 11)
    yr, _ = O.ref_spmv(A, x)
    w, s, ec, ev = O.csr_to_ell(A)
    assert np.array_equal(O.spmv_ell(A.nrows, w, s, ec, ev, x), yr)
    for S in (32, 64):
        sl, ss, sc, sv = O.csr_to_sellp(A, S)
        assert np.array_equal(O.spmv_sellp(A.nrows, S, ss, sc, sv, x), yr)


def test_sellp_integer_kats_cfg2(O):
    """App. B integer KATs for the 27-pt 128^3 matrix."""
    A = O.stencil("27pt", 128)
    assert A.nnz == 55_742_968
    sl, ss, stored = O.sellp_sets(A, 32)
    assert len(sl) == 65_536 and ss[65_536] == 1_751_088 and stored == 56_034_816
    sl, ss, stored = O.sellp_sets(A, 64)
    assert len(sl) == 32_768 and ss[32_768] == 875_544 and stored == 56_034_816
    assert O.port().port_csr_max_row(A.nrows, A.row_ptr) == 27
    assert 27 * A.nrows == 56_623_104


def test_stencil_nnz_configs(O):
    lib = O.port()
    assert lib.port_stencil_nnz(0, 1024) == 5_238_784
    assert lib.port_stencil_nnz(2, 128) == 55_742_968
    assert lib.port_stencil_nnz(1, 256) == 117_047_296


def test_fp32_restatement_tolerance(O):
    A = O.powerlaw(1 << 12, window=1024, max_len=1000)
    x = O.seeded_values(A.ncols, 11)
    y32 = O.spmv_csr(O.Csr(A.nrows, A.ncols, A.row_ptr, A.cols, A.vals.astype(np.float32)),
                     x.astype(np.float32))
    y64 = O.spmv_csr(O.Csr(A.nrows, A.ncols, A.row_ptr, A.cols,
                           A.vals.astype(np.float32).astype(np.float64)),
                     x.astype(np.float32).astype(np.float64))
    assert relerr(y32, y64) <= 1e-5  # App. B FP32 bound


def test_partition_maps_bruteforce(O):
    A = O.stencil("7pt", 8)
    n = A.nrows
    for P in (1, 2, 3, 4, 8):
        chunk = -(-n // P)
        for r in range(0, n, 37):
            assert O.port().port_part_rank_of(n, P, r) == min(r // chunk, P - 1)
        owned = 0
        for rank in range(P):
            b, e = O.part_range(n, P, rank)
            owned += e - b
            cols = A.cols[A.row_ptr[b]:A.row_ptr[e]]
            ghosts = np.unique(cols[(cols < b) | (cols >= e)]).astype(np.int32)
            assert np.array_equal(O.part_ghosts(A, P, rank), ghosts)
            loc = O.part_local_cols(A, P, rank, ghosts)
            exp = np.where((cols >= b) & (cols < e), cols - b,
                           (e - b) + np.searchsorted(ghosts, cols))
            assert np.array_equal(loc, exp)
        assert owned == n


def test_full_size_goldens_committed():
    """tests/golden/cfg45.npz (reference library, sequential executor, full
    size) carries the survey's goldens: CG cfg4 581 iterations, final
    9.589270e-09, flop KAT; BiCGSTAB cfg5 495 iterations."""
    p = os.path.join(os.path.dirname(__file__), "golden", "cfg45.npz")
    if not os.path.exists(p):
        pytest.skip("cfg45.npz not generated")
    g = np.load(p)
    assert int(g["cg_iters"]) == 581 and len(g["cg_hist"]) == 582
    assert abs(g["cg_hist"][-1] - 9.589270e-09) <= 1e-14
    assert abs(g["cg_hist"][1] - 5.037289e-01) <= 1e-6
    n, nnz = 256 ** 3, 117_047_296
    assert int(g["cg_flops"]) == 581 * (4 * nnz + 16 * n) + 2 * nnz + 4 * n == 428_280_119_296
    assert int(g["bicg_iters"]) == 495
    assert abs(g["bicg_hist"][1] - 1.136784e-01) <= 1e-6
    assert int(g["bicg_flops"]) == 495 * (6 * nnz + 28 * n) + 2 * nnz + 2 * n


# ------------------------------------------ exactly rounded reductions
def test_xdot_pinned_to_fsum(O):
    """oracle/xkrylov.cpp's exact dot == Python's math.fsum (an independent
    exactly rounded sum) on wide-range, cancelling and subnormal data."""
    import math
    rng = np.random.default_rng(5)
    for n in (1, 17, 5000, 70000):
        for scale in (0, 200, 300):
            x = rng.standard_normal(n) * 10.0 ** rng.integers(-scale, scale + 1, n)
            y = rng.standard_normal(n)
            assert O.xdot(x, y) == math.fsum((x * y).tolist())
    h = rng.standard_normal(1001)
    v = np.concatenate([h, -h, [1e-300]])
    assert O.xsum(v) == math.fsum(v.tolist()) == 1e-300
    t = rng.standard_normal(3000) * 1e-160
    assert O.xsum(t * t) == math.fsum((t * t).tolist())


@pytest.mark.parametrize("kind,m,gamma", [("cg", 16, 0.0), ("cg", 32, 0.0),
                                          ("bicgstab", 24, 0.5)])
def test_xsolve_restates_krylov(O, kind, m, gamma):
    """The exact-dot restatement of krylov.cpp agrees with the reference
    library (sequential dots) to rounding: same iterations (the reference's
    own spread for BiCGSTAB), histories within the §8c bands over the first
    40 iterations, same flop accounting."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    A = O.stencil("7pt", m, gamma)
    xs = np.ones(A.nrows) if kind == "cg" else O.seeded_values(A.nrows, 11)
    b = O.spmv_csr(A, xs)
    r = O.xsolve(A, b, kind, tol=1e-8, max_iters=5000)
    rr = O.ref_solve(A, b, kind, rel_tol=1e-8, max_iters=5000)
    rp = O.ref_solve(A, b, kind, rel_tol=1e-8, max_iters=5000, exec_kind=1, workers=8)
    assert abs(r["iterations"] - rr.iterations) <= max(1, abs(rp.iterations - rr.iterations))
    k = min(len(r["history"]), len(rr.history), 40)
    h, g = r["history"][:k], np.asarray(rr.history[:k])
    # SURVEY.md §8c bands: CG 1e-7; BiCGSTAB (chaotic under rounding) 1e-6
    assert np.max(np.abs(h - g) / g) <= (1e-7 if kind == "cg" else 1e-6)
    if r["iterations"] == rr.iterations:
        assert r["flops"] == rr.flop_count
    if kind == "cg":
        assert r["iterations"] == {16: 41, 32: 81}[m]  # SURVEY.md §8c goldens


def test_cfg45_exact_golden_is_consistent(O):
    """The committed full-size exact-dot goldens satisfy the north-star
    bands against the reference library's full-size goldens."""
    import os
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg45.npz"))
    ex = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg45_exact.npz"))
    assert int(ex["cg_iters"]) == int(ref["cg_iters"]) == 581
    assert np.max(np.abs(ex["cg_hist"] - ref["cg_hist"]) / ref["cg_hist"]) <= 1e-7
    assert int(ex["cg_flops"]) == int(ref["cg_flops"])
    assert 495 <= int(ex["bicg_iters"]) <= 498
    assert int(np.argmax(ex["bicg_hist"] <= 1e-6)) == 275
    assert np.max(np.abs(ex["bicg_hist"][:41] - ref["bicg_hist"][:41]) / ref["bicg_hist"][:41]) <= 1e-6
    assert ex["bicg_hist"][-1] <= 1e-8
