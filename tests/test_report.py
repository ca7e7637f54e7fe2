"""BenchRecord reports in the reference's schema (record.hpp:22-51,
report.cpp, roofline.cpp:14-26): field order, CSV header, bounds, JSON
round trip, SVG frame."""
import json
import os

import pytest

from paper_2011_08879_b200 import report as R


def test_bounds_anchor():
    # SPEC.md:576-578 anchors: 920 GB/s -> CSR 153.3, COO/solver 115 GFLOP/s
    m = R.compute_bounds(920.0)
    assert abs(m["csr_bound"] - 153.333) < 1e-3 and m["coo_bound"] == 115.0
    assert m["solver_bound"] == 115.0
    with pytest.raises(ValueError):
        R.compute_bounds(0.0)


def test_spmv_record_model():
    r = R.spmv_record("csr", "p", "cuda", 10, 10, 40, 1e-6, 920.0)
    assert r.bytes_moved == 12 * 40 + 4 * 11 + 8 * 20 and r.flops == 80
    assert abs(r.achieved - 80 / 1e-6 / 1e9) < 1e-9
    c = R.spmv_record("coo", "p", "cuda", 10, 10, 40, 1e-6, 920.0)
    assert c.bytes_moved == 16 * 40 + 8 * 20 and c.bound == 115.0


def test_emit_and_parse():
    recs = [R.spmv_record("csr", "a,b", "cuda", 5, 5, 9, 2e-6, 6000.0),
            R.solver_record("cg.true", "cfg4", "cuda", 1000, 0.5, 6000.0)]
    csv = R.emit_report(recs, "csv").splitlines()
    assert csv[0] == ("benchmark_id,executor_kind,problem_id,bytes_moved,flops,elapsed,"
                      "achieved,bound,fraction_of_peak,failed")
    assert csv[1].startswith('spmv.csr,cuda,"a,b",') and csv[1].endswith(",false")
    assert R.parse_records_json(R.emit_report(recs, "json")) == recs
    assert list(json.loads(R.emit_report(recs, "json"))[0]) == [
        "benchmark_id", "executor_kind", "problem_id", "bytes_moved", "flops", "elapsed",
        "achieved", "bound", "fraction_of_peak", "failed"]
    svg = R.emit_report(recs, "svg")
    assert svg.startswith("<svg") and "stroke-dasharray" in svg
    with pytest.raises(ValueError):
        R.emit_report([], "svg")
    with pytest.raises(ValueError):
        R.emit_report(recs, "xml")


def test_records_from_committed_bench_line():
    p = os.path.join(os.path.dirname(os.path.dirname(__file__)), "profiles", "r1_bench_N1.json")
    line = json.load(open(p))
    recs = R.records_from_bench(line)
    ids = {r.benchmark_id for r in recs}
    assert {"spmv.csr.f64", "spmv.coo.f64", "spmv.ell.f64", "spmv.sellp.f64"} <= ids
    assert any(r.benchmark_id.startswith("solve.cg") for r in recs)
