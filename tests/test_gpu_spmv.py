"""GPU parity: SpMV in every format, conversions, assembly, validation and
BLAS-1 through the C ABI (liblbk.so) against the oracle (reference library
/ restatement) and the committed golden vectors.

Bars: integer/index work bit-exact; FP64 SpMV normwise
relative error <= 1e-12 (rows <= 32 entries are in fact bit-identical to
the FMA-free reference, asserted where it holds); FP32 <= 1e-5 vs the FP64
oracle applied to FP32-rounded inputs (App. B).
"""
import os

import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
TOL64 = 1e-12
TOL32 = 1e-5


def _rnd(i):
    return {k.split("_", 1)[1]: G[k] for k in G.files if k.startswith(f"rnd{i}_")}


def up(lk, ex, A, dtype=None):
    import torch
    return lk.csr_from_host(ex, A.nrows, A.ncols, A.row_ptr, A.cols, A.vals,
                            dtype=dtype or torch.float64)


def all_formats(lk, A):
    return {"csr": A, "coo": lk.csr_to_coo(A), "ell": lk.csr_to_ell(A),
            "sellp32": lk.csr_to_sellp(A, 32), "sellp64": lk.csr_to_sellp(A, 64),
            "sellp7": lk.csr_to_sellp(A, 7)}


def spmv_host(lk, ex, M, xh):
    x = lk.vector_from(ex, xh)
    y = lk.make_vector(ex, M.nrows, x.values.dtype)
    y.values.fill_(float("nan"))
    lk.spmv(M, x, y)
    return lk.vector_to_host(y)


# ------------------------------------------------------------ generators
@pytest.mark.parametrize("kind,m,gamma", [("5pt", 64, 0.0), ("27pt", 24, 0.0), ("7pt", 20, 0.5),
                                          ("5pt", 1024, 0.0)])
def test_device_stencil_bitexact(O, ex, lk, kind, m, gamma):
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, kind, m, gamma)
    R = O.stencil(kind, m, gamma)
    assert np.array_equal(A.row_ptr.cpu().numpy(), R.row_ptr)
    assert np.array_equal(A.col_idx.cpu().numpy(), R.cols)
    assert np.array_equal(A.vals.cpu().numpy(), R.vals)


# ------------------------------------------------------------ golden
@pytest.mark.parametrize("i", range(6))
def test_golden_assembly_conversion_spmv(ex, lk, i):
    g = _rnd(i)
    nr, nc = (int(v) for v in g["shape"])
    M = lk.coo_from_entries(ex, nr, nc, (g["in_rows"], g["in_cols"], g["in_vals"]))
    assert np.array_equal(M.row_idx.cpu().numpy(), g["rows"])
    assert np.array_equal(M.col_idx.cpu().numpy(), g["cols"])
    assert np.array_equal(M.vals.cpu().numpy(), g["vals"])  # duplicates summed in input order
    A = lk.coo_to_csr(M)
    assert np.array_equal(A.row_ptr.cpu().numpy(), g["rowptr"])
    assert np.array_equal(lk.csr_to_coo(A).row_idx.cpu().numpy(), g["rows"])
    for name, F in all_formats(lk, A).items():
        y = spmv_host(lk, ex, F, g["x"])
        assert np.array_equal(y, g["y_csr"]), name


def test_spec_kats(ex, lk):
    A = lk.csr_from_host(ex, 2, 2, [0, 1, 1], [0], [5.0])
    assert list(spmv_host(lk, ex, A, np.array([2.0, 7.0]))) == [10.0, 0.0]
    A = lk.csr_from_host(ex, 2, 2, [0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0])
    for F in all_formats(lk, A).values():
        assert list(spmv_host(lk, ex, F, np.array([1.0, 1.0]))) == [3.0, 3.0]
    M = lk.coo_from_entries(ex, 3, 3, [])
    assert list(lk.coo_to_csr(M).row_ptr.cpu().numpy()) == [0, 0, 0, 0]


# ------------------------------------------------------------ cfg parity
def test_cfg1_all_formats_bitexact(O, ex, lk):
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, "5pt", 1024)
    R = O.stencil("5pt", 1024)
    xh = O.seeded_values(A.ncols, 11)
    yref = O.spmv_csr(R, xh)
    if O.ref_available():
        yr, _ = O.ref_spmv(R, xh)
        assert np.array_equal(yr, yref)
    for name, F in all_formats(lk, A).items():
        assert np.array_equal(spmv_host(lk, ex, F, xh), yref), name


def test_cfg2_csr_coo_bitexact_and_layout_kats(O, ex, lk):
    from paper_2011_08879_b200 import gen
    A = gen.stencil(ex, "27pt", 128)
    R = O.stencil("27pt", 128)
    xh = O.seeded_values(A.ncols, 11)
    yref = O.spmv_csr(R, xh)
    assert np.array_equal(spmv_host(lk, ex, A, xh), yref)
    assert np.array_equal(spmv_host(lk, ex, lk.csr_to_coo(A), xh), yref)
    E = lk.csr_to_ell(A)
    assert E.width == 27 and E.col_idx.numel() == 56_623_104
    assert np.array_equal(spmv_host(lk, ex, E, xh), yref)
    del E
    S = lk.csr_to_sellp(A, 32)
    ss = S.slice_sets.cpu().numpy()
    assert S.nslices == 65_536 and ss[65_536] == 1_751_088 and S.col_idx.numel() == 56_034_816
    sl, ss_ref, stored = O.sellp_sets(R, 32)
    assert np.array_equal(ss, ss_ref) and np.array_equal(S.slice_lengths.cpu().numpy(), sl)
    assert np.array_equal(spmv_host(lk, ex, S, xh), yref)


def test_ell_sellp_conversion_bitexact(O, ex, lk):
    R = O.powerlaw(1 << 12, window=512, max_len=200)
    A = up(lk, ex, R)
    w, s, ec, ev = O.csr_to_ell(R)
    E = lk.csr_to_ell(A)
    assert E.width == w
    assert np.array_equal(E.col_idx.cpu().numpy()[: w * s], ec)
    assert np.array_equal(E.vals.cpu().numpy()[: w * s], ev)
    for S in (32, 64, 5):
        sl, ss, sc, sv = O.csr_to_sellp(R, S)
        D = lk.csr_to_sellp(A, S)
        assert np.array_equal(D.slice_lengths.cpu().numpy(), sl)
        assert np.array_equal(D.slice_sets.cpu().numpy(), ss)
        assert np.array_equal(D.col_idx.cpu().numpy()[: len(sc)], sc)
        assert np.array_equal(D.vals.cpu().numpy()[: len(sv)], sv)


@pytest.mark.parametrize("n,window,max_len", [(1 << 18, 65536, 10000), (1 << 16, 1 << 16, 3000)])
def test_powerlaw_csr_coo(O, ex, lk, n, window, max_len):
    """Load-balance stress (cfg3 shape, reduced): giant rows take the wide-
    tile path; rows <= 256 (kSeqRow, including a short row that overflowed
    its tile's slot) stay bit-exact, the whole vector within 1e-12."""
    R = O.powerlaw(n, window=window, max_len=max_len)
    A = up(lk, ex, R)
    xh = O.seeded_values(n, 11)
    yref = O.spmv_csr(R, xh)
    short = np.diff(R.row_ptr) <= 256
    for name, F in [("csr", A), ("coo", lk.csr_to_coo(A)), ("sellp", lk.csr_to_sellp(A, 32))]:
        y = spmv_host(lk, ex, F, xh)
        assert relerr(y, yref) <= TOL64, name
        assert np.array_equal(y[short], yref[short]), name


def test_random_shapes_and_edge_cases(O, ex, lk):
    rng = np.random.default_rng(3)
    cases = []
    for _ in range(20):
        nr, nc = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
        dens = float(rng.choice([0.0, 0.001, 0.01, 0.05]))
        cases.append((nr, nc, dens))
    cases += [(1, 1, 1.0), (5000, 7, 0.3), (7, 5000, 0.5), (1, 20000, 0.9)]
    for nr, nc, dens in cases:
        mask = rng.random((nr, nc)) < dens
        rows, cols = np.nonzero(mask)
        vals = rng.uniform(-1, 1, rows.size)
        rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=nr))]).astype(np.int32)
        R = O.Csr(nr, nc, rp, cols.astype(np.int32), vals)
        xh = rng.uniform(-1, 1, nc)
        yref = O.spmv_csr(R, xh)
        A = up(lk, ex, R)
        short = np.diff(rp) <= 32
        for name, F in all_formats(lk, A).items():
            y = spmv_host(lk, ex, F, xh)
            assert relerr(y, yref) <= TOL64, (nr, nc, dens, name)
            assert np.array_equal(y[short], yref[short]), (nr, nc, dens, name)


def test_empty_matrix_zero_rows(ex, lk):
    import torch
    A = lk.csr_from_host(ex, 4, 3, [0, 0, 0, 0, 0], np.zeros(0, np.int32), np.zeros(0))
    for F in [A, lk.csr_to_coo(A), lk.csr_to_ell(A), lk.csr_to_sellp(A, 32)]:
        assert list(spmv_host(lk, ex, F, np.ones(3))) == [0.0] * 4
    Z = lk.csr_from_host(ex, 0, 0, [0], np.zeros(0, np.int32), np.zeros(0))
    x = lk.make_vector(ex, 0)
    y = lk.make_vector(ex, 0)
    lk.spmv(Z, x, y)


# ------------------------------------------------------------ FP32 / advanced apply
def test_fp32_formats(O, ex, lk):
    import torch
    R = O.powerlaw(1 << 16, window=4096, max_len=1000)
    xh = O.seeded_values(R.ncols, 11).astype(np.float32)
    v32 = R.vals.astype(np.float32)
    ref64 = O.spmv_csr(O.Csr(R.nrows, R.ncols, R.row_ptr, R.cols, v32.astype(np.float64)),
                       xh.astype(np.float64))
    ref32 = O.spmv_csr(O.Csr(R.nrows, R.ncols, R.row_ptr, R.cols, v32), xh)
    A = up(lk, ex, R, torch.float32)
    short = np.diff(R.row_ptr) <= 32
    for name, F in [("csr", A), ("coo", lk.csr_to_coo(A)), ("ell", lk.csr_to_ell(A)),
                    ("sellp", lk.csr_to_sellp(A, 32))]:
        y = spmv_host(lk, ex, F, xh)
        assert y.dtype == np.float32
        assert relerr(y, ref64) <= TOL32, name
        assert np.array_equal(y[short], ref32[short]), name


def test_advanced_apply(O, ex, lk):
    R = O.stencil("27pt", 20)
    A = up(lk, ex, R)
    xh = O.seeded_values(R.ncols, 11)
    y0 = O.seeded_values(R.nrows, 12)
    ax = O.spmv_csr(R, xh)
    for alpha, beta in [(1.0, 0.0), (2.5, -0.5), (-1.0, 1.0), (0.0, 3.0)]:
        exp = alpha * ax + beta * y0
        for name, F in [("csr", A), ("coo", lk.csr_to_coo(A)), ("ell", lk.csr_to_ell(A)),
                        ("sellp", lk.csr_to_sellp(A, 32))]:
            x = lk.vector_from(ex, xh)
            y = lk.vector_from(ex, y0)
            lk.spmv(F, x, y, alpha=alpha, beta=beta)
            assert relerr(lk.vector_to_host(y), exp) <= 1e-14, (name, alpha, beta)
    # FP32 advanced apply in every format
    import torch
    A32 = A.astype(torch.float32)
    x32, y32 = xh.astype(np.float32), y0.astype(np.float32)
    ax32 = O.spmv_csr(O.Csr(R.nrows, R.ncols, R.row_ptr, R.cols, R.vals.astype(np.float32)), x32)
    exp32 = np.float32(2.5) * ax32 + np.float32(-0.5) * y32
    for name, F in [("csr", A32), ("coo", lk.csr_to_coo(A32)), ("ell", lk.csr_to_ell(A32)),
                    ("sellp", lk.csr_to_sellp(A32, 32))]:
        xv, yv = lk.vector_from(ex, x32), lk.vector_from(ex, y32)
        lk.spmv(F, xv, yv, alpha=2.5, beta=-0.5)
        assert relerr(lk.vector_to_host(yv), exp32) <= 1e-6, name
    # beta == 0 must not read y (NaN in y stays out)
    x = lk.vector_from(ex, xh)
    y = lk.make_vector(ex, R.nrows)
    y.values.fill_(float("nan"))
    lk.spmv(A, x, y, alpha=1.0, beta=0.0)
    assert np.array_equal(lk.vector_to_host(y), ax)


# ------------------------------------------------------------ errors
def test_shape_type_errors(ex, lk):
    import torch
    A = lk.csr_from_host(ex, 2, 3, [0, 1, 2], [0, 2], [1.0, 2.0])
    with pytest.raises(lk.ShapeError):
        lk.spmv(A, lk.make_vector(ex, 2), lk.make_vector(ex, 2))
    with pytest.raises(lk.ShapeError):
        lk.spmv(A, lk.make_vector(ex, 3), lk.make_vector(ex, 3))
    with pytest.raises(lk.TypeError_):
        lk.spmv(A, lk.make_vector(ex, 3, torch.float32), lk.make_vector(ex, 2, torch.float32))
    with pytest.raises(lk.ShapeError):
        lk.axpy(1.0, lk.make_vector(ex, 3), lk.make_vector(ex, 4))


def test_validate_matches_reference(R, ex, lk):
    O = R
    bad = [
        (2, 2, [0, 2, 1], [0, 1], [1.0, 1.0]),        # row_ptr decreasing
        (2, 2, [0, 2, 2], [1, 0], [1.0, 1.0]),        # columns not increasing
        (2, 2, [0, 1, 2], [0, 2], [1.0, 1.0]),        # column out of range
        (2, 2, [1, 1, 2], [0, 1], [1.0, 1.0]),        # row_ptr[0] != 0
        (2, 2, [0, 1, 2], [0, 0], [1.0, 1.0]),        # fine
    ]
    for nr, nc, rp, cols, vals in bad:
        want = O.ref_validate("csr", nr, nc, rp, cols, vals)
        A = lk.csr_from_host(ex, nr, nc, rp, cols, vals)
        if want == 0:
            lk.validate(A)
        else:
            with pytest.raises(lk.FormatError):
                lk.validate(A)
    # COO: unsorted / duplicate
    for rows, cols in [([1, 0], [0, 0]), ([0, 0], [1, 1]), ([0, 1], [0, 1])]:
        want = O.ref_validate("coo", 2, 2, rows, cols, [1.0, 1.0])
        M = lk.coo_from_host(ex, 2, 2, rows, cols, [1.0, 1.0])
        if want == 0:
            lk.validate(M)
        else:
            with pytest.raises(lk.FormatError):
                lk.validate(M)
    with pytest.raises(lk.FormatError):  # coo_from_entries bounds check
        lk.coo_from_entries(ex, 2, 2, [(0, 0, 1.0), (2, 0, 1.0)])


# ------------------------------------------------------------ BLAS-1
def test_blas1(O, ex, lk):
    n = 1_000_003
    a = O.seeded_values(n, 1)
    b = O.seeded_values(n, 2)
    x, y = lk.vector_from(ex, a), lk.vector_from(ex, b)
    d = lk.dot(x, y)
    assert abs(d - O.port().port_dot(n, a, b)) <= 1e-12 * np.dot(np.abs(a), np.abs(b))
    assert lk.dot(x, y) == d  # deterministic two-stage reduction
    assert abs(lk.nrm2(x) - np.linalg.norm(a)) <= 1e-12 * np.linalg.norm(a)
    lk.axpy(0.5, x, y)
    assert np.array_equal(lk.vector_to_host(y), b + 0.5 * a)
    lk.scal(-2.0, y)
    assert np.array_equal(lk.vector_to_host(y), -2.0 * (b + 0.5 * a))
    lk.fill(y, 3.25)
    assert np.all(lk.vector_to_host(y) == 3.25)


def test_sellp_stream_kernel_opt_in():
    """The warp-pipelined SELL-P kernel (LBK_SELLP_ALGO=stream, read once per
    process) is exercised in a subprocess: bit-exact with the reference."""
    import subprocess
    import sys
    import textwrap
    code = textwrap.dedent("""
        import sys, numpy as np
        sys.path.insert(0, %r)
        from oracle import oracle as O
        from paper_2011_08879_b200 import larch as lk
        ex = lk.CudaExecutor(0)
        for R in (O.stencil("27pt", 20), O.powerlaw(1 << 14, window=2048, max_len=3000)):
            A = lk.csr_from_host(ex, R.nrows, R.ncols, R.row_ptr, R.cols, R.vals)
            xh = O.seeded_values(R.ncols, 11)
            x = lk.vector_from(ex, xh)
            y = lk.make_vector(ex, R.nrows)
            lk.spmv(lk.csr_to_sellp(A, 32), x, y)
            yref = O.spmv_csr(R, xh)
            short = np.diff(R.row_ptr) <= 32
            yy = lk.vector_to_host(y)
            assert np.array_equal(yy[short], yref[short])
            assert np.max(np.abs(yy - yref)) <= 1e-12 * np.max(np.abs(yref))
        print("ok")
    """) % (os.path.dirname(os.path.dirname(os.path.abspath(__file__))),)
    env = dict(os.environ, LBK_SELLP_ALGO="stream")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


# ------------------------------------------------ stream set / flops sweep
def test_stream_ops_and_flops_sweep(O, ex, lk):
    """The rest of the reference's StreamOp set and flops_sweep
    (kernels.hpp:58-113, reference.cpp:92-130): closed-form values as the
    harness verifies them (harness.cpp:166-195, 236-249), bit-exact."""
    import math
    n = 1 << 20
    rng = np.random.default_rng(4)
    ah, bh, ch = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    mk = lambda h: lk.vector_from(ex, h)  # noqa: E731
    a, b, c = mk(ah), mk(bh), mk(ch)
    assert lk.stream_kernel("copy", a, b, c, 0.4) == 0.0
    assert np.array_equal(lk.vector_to_host(c), ah)
    a, b, c = mk(ah), mk(bh), mk(ch)
    lk.stream_kernel("mul", a, b, c, 0.4)
    assert np.array_equal(lk.vector_to_host(b), 0.4 * ch)
    a, b, c = mk(ah), mk(bh), mk(ch)
    lk.stream_kernel("add", a, b, c, 0.4)
    assert np.array_equal(lk.vector_to_host(c), ah + bh)
    a, b, c = mk(ah), mk(bh), mk(ch)
    lk.stream_kernel("triad", a, b, c, 0.4)
    assert np.array_equal(lk.vector_to_host(a), bh + 0.4 * ch)
    a, b, c = mk(ah), mk(bh), mk(ch)
    assert lk.stream_kernel("dot", a, b, c, 0.4) == math.fsum((ah * bh).tolist())
    assert lk.stream_bytes("add", n) == 24 * n and lk.stream_bytes("dot", n) == 16 * n
    # flops sweep: the fma chain bit for bit (seeded_values(n, 7) as the harness)
    x0 = O.seeded_values(4099, 7)
    for fma in (0, 1, 2, 7, 64):
        want = x0.copy()
        for k in range(fma):
            want = (2.0 if k % 2 == 0 else 0.5) * want + 3.0
        x = lk.vector_from(ex, x0)
        lk.flops_sweep(x, fma)
        assert np.array_equal(lk.vector_to_host(x), want), fma
    with pytest.raises(lk.UsageError):
        lk.flops_sweep(lk.vector_from(ex, x0), -1)
