"""GPU: the MatrixMarket corpus sweep (scripts/mm_sweep.py)
on a small generated corpus -- the reference's run_spmv_bench protocol
(harness.cpp:284-364): every loadable file gives a verified spmv.csr and
spmv.coo record, a malformed file a failed spmv.load record."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_mm_sweep_small_corpus(tmp_path):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "scripts"))
    import mm_sweep as M
    from paper_2011_08879_b200 import report as R
    n, r, c, v = M._stencil("7pt", 12)
    M._write_mtx(str(tmp_path / "p7.mtx"), n, n, r, c, v)
    lo = r >= c
    M._write_mtx(str(tmp_path / "p7_sym.mtx"), n, n, r[lo], c[lo], v[lo], symmetry="symmetric")
    rng = np.random.default_rng(1)
    rr, cc = rng.integers(0, 300, 2000), rng.integers(0, 500, 2000)
    M._write_mtx(str(tmp_path / "rand.mtx"), 300, 500, rr, cc, rng.uniform(-1, 1, 2000))
    (tmp_path / "bad.mtx").write_text("%%MatrixMarket matrix array real general\n1 1\n1\n")
    recs = M.sweep(str(tmp_path), reps=3)
    ids = sorted((x.problem_id, x.benchmark_id, x.failed) for x in recs)
    assert ids == [("bad", "spmv.load", True), ("p7", "spmv.coo", False), ("p7", "spmv.csr", False),
                   ("p7_sym", "spmv.coo", False), ("p7_sym", "spmv.csr", False),
                   ("rand", "spmv.coo", False), ("rand", "spmv.csr", False)]
    for x in recs:
        if not x.failed:
            assert x.elapsed > 0 and x.flops > 0 and x.bound > 0
    # the report round-trips in the reference schema
    assert len(R.parse_records_json(R.emit_report(recs, "json"))) == len(recs)
