"""BenchRecord reports in the reference's schema.

Mirrors include/larch/bench/record.hpp:22-51 and src/bench/report.cpp:
the same fields in the same order, JSON / CSV / SVG roofline scatter, and
the same byte/flop/bound model (harness.cpp:284-446, roofline.cpp:14-26):
spmv.csr bound = BW/6, spmv.coo (and the solver model) = BW/8 GFLOP/s;
achieved = flops / elapsed in GFLOP/s.  GPU rows and the reference's CPU
rows therefore land in one report.  Additions keep the schema: ELL/SELL-P
records use the CSR bound over their stored-slot byte count.
"""
from __future__ import annotations

import io
import json
import math
from dataclasses import asdict, dataclass, fields
from typing import Iterable, List, Sequence


@dataclass
class BenchRecord:
    benchmark_id: str
    executor_kind: str
    problem_id: str
    bytes_moved: int = 0
    flops: int = 0
    elapsed: float = 0.0  # seconds
    achieved: float = 0.0  # GFLOP/s
    bound: float = 0.0
    fraction_of_peak: float = 0.0
    failed: bool = False


def compute_bounds(peak_bandwidth_gbs: float) -> dict:
    """roofline.cpp:14-26"""
    if not peak_bandwidth_gbs > 0.0:
        raise ValueError(f"peak bandwidth must be positive, got {peak_bandwidth_gbs}")
    return {"peak_bandwidth": peak_bandwidth_gbs, "coo_bound": peak_bandwidth_gbs / 8.0,
            "csr_bound": peak_bandwidth_gbs / 6.0, "solver_bound": peak_bandwidth_gbs / 8.0}


def spmv_record(fmt: str, problem: str, executor: str, nrows: int, ncols: int, nnz: int,
                elapsed: float, peak_gbs: float, stored: int | None = None,
                nslices: int = 0) -> BenchRecord:
    """harness.cpp:338-361 (+ ELL / SELL-P over stored slots)."""
    m = compute_bounds(peak_gbs)
    vec = 8 * (nrows + ncols)
    if fmt == "coo":
        nbytes, bound = 16 * nnz + vec, m["coo_bound"]
    elif fmt == "csr":
        nbytes, bound = 12 * nnz + 4 * (nrows + 1) + vec, m["csr_bound"]
    else:
        nbytes, bound = 12 * int(stored) + 8 * nslices + vec, m["csr_bound"]
    flops = 2 * nnz
    ach = flops / elapsed / 1e9 if elapsed > 0 else 0.0
    return BenchRecord(f"spmv.{fmt}", executor, problem, int(nbytes), int(flops), elapsed, ach,
                       bound, ach / bound if bound > 0 else 0.0)


def solver_record(kind: str, problem: str, executor: str, flop_count: int, elapsed: float,
                  peak_gbs: float) -> BenchRecord:
    """harness.cpp:432-434: bytes_moved = flops (intensity 1), bound BW/8."""
    m = compute_bounds(peak_gbs)
    ach = flop_count / elapsed / 1e9 if elapsed > 0 else 0.0
    return BenchRecord(f"solve.{kind}", executor, problem, int(flop_count), int(flop_count),
                       elapsed, ach, m["solver_bound"], ach / m["solver_bound"])


def _csv_field(v: str) -> str:
    if not any(c in v for c in ',"\n'):
        return v
    return '"' + v.replace('"', '""') + '"'


def _num(v) -> str:
    # the reference streams doubles with operator<< (6 significant digits)
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return f"{v:.6g}"
    return str(v)


def emit_report(records: Sequence[BenchRecord], fmt: str) -> str:
    """report.cpp:173-190: 'json' | 'csv' | 'svg'."""
    if fmt == "json":
        return json.dumps([asdict(r) for r in records], indent=2) + "\n"
    if fmt == "csv":
        out = io.StringIO()
        out.write(",".join(f.name for f in fields(BenchRecord)) + "\n")
        for r in records:
            out.write(",".join([_csv_field(r.benchmark_id), _csv_field(r.executor_kind),
                                _csv_field(r.problem_id)] +
                               [_num(getattr(r, f.name)) for f in fields(BenchRecord)[3:]]) + "\n")
        return out.getvalue()
    if fmt == "svg":
        return _svg(records)
    raise ValueError(f"unknown report format '{fmt}', expected json, csv, or svg")


def parse_records_json(text: str) -> List[BenchRecord]:
    return [BenchRecord(**d) for d in json.loads(text)]


def _svg(records: Sequence[BenchRecord]) -> str:
    """report.cpp:72-150: log-x bytes moved vs achieved, dashed bound lines."""
    if not records:
        raise ValueError("svg scatter needs at least one record")
    W, H, ml, mr, mt, mb = 840, 520, 70, 30, 30, 50
    pw, ph = W - ml - mr, H - mt - mb
    ok = [r for r in records if not r.failed]
    xs = [max(r.bytes_moved, 1) for r in ok] or [1, 10]
    x0, x1 = min(xs), max(xs)
    if x1 <= x0:
        x1 = x0 + 1
    bounds = sorted({r.bound for r in ok if r.bound > 0})
    ymax = max([r.achieved for r in ok] + bounds + [1e-300]) * 1.08
    lx0, lx1 = math.log10(x0), math.log10(x1)

    def mx(x):
        return ml + (math.log10(x) - lx0) / (lx1 - lx0) * pw

    def my(y):
        return mt + (1.0 - y / ymax) * ph
    o = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{W}" height="{H}">',
         f'<rect x="{ml}" y="{mt}" width="{pw}" height="{ph}" fill="none" stroke="black"/>',
         f'<text x="{ml + pw / 2}" y="{H - 12}" text-anchor="middle">bytes moved</text>',
         f'<text x="18" y="{mt + ph / 2}" text-anchor="middle" '
         f'transform="rotate(-90 18 {mt + ph / 2})">achieved rate</text>']
    for b in bounds:
        o.append(f'<line x1="{ml}" y1="{my(b)}" x2="{ml + pw}" y2="{my(b)}" stroke="red" '
                 f'stroke-dasharray="6 3"/>')
        o.append(f'<text x="{ml + pw - 4}" y="{my(b) - 5}" text-anchor="end" fill="red">'
                 f'bound {b:.6g}</text>')
    for r in ok:
        o.append(f'<circle cx="{mx(max(r.bytes_moved, 1))}" cy="{my(r.achieved)}" r="4" '
                 f'fill="steelblue" fill-opacity="0.7"><title>{r.benchmark_id} {r.problem_id}'
                 f'</title></circle>')
    o.append("</svg>")
    return "\n".join(o) + "\n"


def records_from_bench(line: dict) -> List[BenchRecord]:
    """BenchRecords from one bench.py JSON line (GPU rows; the CPU baseline
    row is the reference's own spmv.csr record on the same problem)."""
    peak = line.get("roofline", {}).get("peak") or 6650.0
    recs: List[BenchRecord] = []
    fm = line.get("formats") or {}
    meta = {"cfg1": ("2d5pt-1024", 1048576, 5238784), "cfg2": ("3d27pt-128", 2097152, 55742968),
            "cfg3": ("powerlaw-2^24", 16777216, None)}
    for key, v in fm.items():
        if not isinstance(v, dict) or "us" not in v:
            continue
        cfg, fmt, prec = key.split("_")
        pid, n, nnz = meta[cfg]
        nnz = v.get("nnz") or nnz or int(round(v["gflops"] * 1e9 * v["us"] * 1e-6 / 2))
        t = v["us"] * 1e-6
        base = fmt.rstrip("0123456789")
        r = BenchRecord(f"spmv.{base}.{prec}", "cuda", pid, int(v["bytes"]), 2 * nnz, t,
                        2 * nnz / t / 1e9, peak / (8.0 if base == "coo" else 6.0))
        r.fraction_of_peak = r.achieved / r.bound
        recs.append(r)
    cg = line.get("cg") or {}
    for mode in ("true", "recurrence"):
        if mode in cg:
            d = cg[mode]
            fl = d.get("flop_count") or d["gflops_ref_model"] * 1e9 * d["seconds"]
            recs.append(solver_record(f"cg.{mode}", "cfg4-7pt-256", "cuda", int(fl), d["seconds"],
                                      peak))
    if "bicgstab_cfg5" in cg:
        d = cg["bicgstab_cfg5"]
        recs.append(solver_record("bicgstab", "cfg5-7pt-256-g0.5", "cuda",
                                  int(d.get("flop_count") or d["gflops_ref_model"] * 1e9 *
                                      d["seconds"]), d["seconds"], peak))
    cb = line.get("cpu_baseline") or {}
    if cb.get("value"):
        t = cb["ms_per_step"] * 1e-3
        recs.append(BenchRecord("spmv.csr", f"reference-parallel({cb['cores']})", "3d27pt-128",
                                710858660, 2 * 55742968, t, 2 * 55742968 / t / 1e9, 0.0, 0.0))
    return recs
