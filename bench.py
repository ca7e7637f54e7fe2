#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 sparse backend.

Metric (BASELINE.json): "FP64 CSR SpMV GB/s (% of HBM roofline) and CG
iters/s at 1/2/4/8 B200".  A *step* is one CSR SpMV y = A x (reference
spmv_csr, src/kernels/reference.cpp:74-89) over the config's matrix:

  workload  cfg2 -- FP64 CSR SpMV, 3D 27-pt Poisson 128^3 (n = 2,097,152,
            nnz = 55,742,968), x = seeded_values(n, 11) (harness.cpp:90-99);
            the matrix is generated on the device (bit-exact vs the oracle,
            tests/test_gpu_spmv.py).
  value     algorithmic GB/s = (12 nnz + 4 (n+1) + 8 (n + n)) bytes per step
            (reference byte model, harness.cpp:342-354) x N / device time,
            inputs resident in HBM; matrix streams (670 MB) exceed L2, so no
            flush is needed between steps (x, 16.8 MB, stays L2-resident as
            it would inside a solver).
  e2e       same metric through the C ABI (lbk_memcpy_h2d of x from pinned
            host memory -> lbk_spmv_csr_f64 -> lbk_memcpy_d2h of y), copies
            inside the timed region; the operator (matrix + plan) is set up
            once, as the reference's clone_to does.
  cg        CG iterations/s on cfg4 (7-pt Poisson 256^3, b = A*1, x0 = 0, tol
            1e-8) with reference semantics (true residual every iteration)
            and with the recurrence stop (verified true residual).
N > 1 (torchrun): every rank runs the same SpMV replica on its own GPU (cfg1-3
are single-GPU configs: "replicas only"); time = max over
ranks; value = N x bytes / time ("scaling": "weak").

--impl reference times the reference's own CPU implementation (oracle/_ref:
the reference library compiled from /root/reference/proj/src, FMA-free) with
ParallelExecutor(all host threads) on the same config; rank 0 only.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# keep stdout to the one JSON line: NCCL's version banner goes to stdout
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"
# a failed peer must cost minutes, not the driver's whole budget
os.environ.setdefault("LBK_NCCL_TIMEOUT", "180")
os.environ.setdefault("LBK_PEER_TIMEOUT", "120")

METRIC = "FP64 CSR SpMV GB/s (% of HBM roofline) and CG iters/s at 1/2/4/8 B200"
WORKLOAD = {"workload": "cfg2: FP64 CSR SpMV, 3D 27-pt Poisson 128^3 (2,097,152 rows, "
                        "55,742,968 nnz), single RHS",
            "format": "csr", "matrix": "27pt-128^3", "rows": 2097152, "nnz": 55742968,
            "l2": "inputs larger than L2 (matrix streams 670 MB > 126 MB); no flush"}
PEAK_FALLBACK = 6650.0


def csr_bytes(n: int, ncols: int, nnz: int) -> int:
    """Reference byte model for CSR (harness.cpp:342-354)."""
    return 12 * nnz + 4 * (n + 1) + 8 * (n + ncols)


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return PEAK_FALLBACK, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str):
    """DRAM bytes per launch from the committed `ncu --set full` summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed phases."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = f"/tmp/lbk_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons, util = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for row in csv.reader(f):
                if len(row) < 8:
                    continue
                try:
                    s, m, u = float(row[0]), float(row[1]), float(row[7])
                except ValueError:
                    continue
                util.append(u)
                if u < 50:  # only samples under load
                    continue
                sm.append(s)
                smax.append(m)
                for nm, v in zip(names, row[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples_under_load": len(sm)}


# ------------------------------------------------------------ our arm
def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist
    import ctypes as C

    from paper_2011_08879_b200 import _lib as L, gen, larch as lk

    torch.cuda.set_device(local_rank)
    ex = lk.CudaExecutor(local_rank)
    lib = L.load()
    dev = ex.device

    A = gen.stencil(ex, "27pt", 128)
    n, nnz, ncols = A.nrows, A.nnz(), A.ncols
    bytes_step = csr_bytes(n, A.ncols, nnz)
    xh = gen.seeded_values(A.ncols, 11)
    x = lk.vector_from(ex, xh)
    y = lk.make_vector(ex, n)
    desc = A.desc()  # builds + caches the load-balance plan once
    xp, yp = C.c_void_p(x.values.data_ptr()), C.c_void_p(y.values.data_ptr())
    ctx = ex.ctx
    stream = ex.stream

    def step():
        st = lib.lbk_spmv_csr_f64(ctx, C.byref(desc), xp, yp)
        if st:
            lk._check(st, ctx)

    def barrier():
        if world > 1:
            dist.barrier()

    sampler = ClockSampler(local_rank)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region: K steps, one kernel each
    K = args.steps
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K)]
    barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for i in range(K):
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    elapsed = t0.elapsed_time(t1) * 1e-3
    launch_s = [a.elapsed_time(b) * 1e-3 for a, b in evs]
    t_max = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    elapsed_max = float(t_max.item())

    # ---- end-to-end through the C ABI with host buffers
    # (a) sequential: each step = H2D x -> SpMV -> D2H y on one stream;
    # (b) pipelined: the same calls on three contexts/streams (copy-in,
    #     compute, copy-out) with double-buffered device x/y, so step i's
    #     SpMV overlaps step i+1's upload and step i-1's download (PCIe is
    #     full duplex).  Every step still moves its own input and result.
    xh_pin = torch.from_numpy(xh).pin_memory()
    yh_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    xhp, yhp = C.c_void_p(xh_pin.data_ptr()), C.c_void_p(yh_pin.data_ptr())
    nb = 8 * n

    def e2e_step():
        lk._check(lib.lbk_memcpy_h2d(ctx, xp, xhp, 8 * ncols), ctx)
        step()
        lk._check(lib.lbk_memcpy_d2h(ctx, yhp, yp, nb), ctx)

    def timed(body):
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        last = body(e0)
        e1.record(last)
        torch.cuda.synchronize()
        barrier()
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def run_seq(_e0):
        for _ in range(K):
            e2e_step()
        return stream

    for _ in range(args.warmup):
        e2e_step()
    e2e_seq_s = timed(run_seq)

    # three non-default streams: work on the legacy default stream would
    # serialise against the copy streams
    s_in, s_out, s_mv = (torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    ex_in = lk.CudaExecutor(local_rank, stream=s_in)
    ex_out = lk.CudaExecutor(local_rank, stream=s_out)
    ex_mv = lk.CudaExecutor(local_rank, stream=s_mv)
    NB = int(os.environ.get("LBK_E2E_BUFFERS", "2"))  # device buffers in flight (3, 4: no gain)
    xb = [x.values] + [torch.empty_like(x.values) for _ in range(NB - 1)]
    yb = [y.values] + [torch.empty_like(y.values) for _ in range(NB - 1)]
    descs = desc

    def run_pipe(e0):
        s_in.wait_event(e0)
        s_mv.wait_event(e0)
        up_done = [torch.cuda.Event() for _ in range(K)]
        mv_done = [torch.cuda.Event() for _ in range(K)]
        dn_done = [torch.cuda.Event() for _ in range(K)]
        for i in range(K):
            j = i % NB
            if i >= NB:
                s_in.wait_event(mv_done[i - NB])  # x buffer j free again
            lk._check(lib.lbk_memcpy_h2d(ex_in.ctx, C.c_void_p(xb[j].data_ptr()), xhp, 8 * ncols),
                      ex_in.ctx)
            up_done[i].record(s_in)
            s_mv.wait_event(up_done[i])
            if i >= NB:
                s_mv.wait_event(dn_done[i - NB])  # y buffer j drained
            st = lib.lbk_spmv_csr_f64(ex_mv.ctx, C.byref(descs), C.c_void_p(xb[j].data_ptr()),
                                      C.c_void_p(yb[j].data_ptr()))
            if st:
                lk._check(st, ex_mv.ctx)
            mv_done[i].record(s_mv)
            s_out.wait_event(mv_done[i])
            lk._check(lib.lbk_memcpy_d2h(ex_out.ctx, yhp, C.c_void_p(yb[j].data_ptr()), nb),
                      ex_out.ctx)
            dn_done[i].record(s_out)
        return s_out

    run_pipe_warm = timed(run_pipe)  # warm-up pass (events, streams)
    e2e_s = timed(run_pipe)
    e2e_step_ok = bool(torch.equal(yb[0], yb[1]))
    del run_pipe_warm

    # ---- every format / config of §8d on this GPU (rank 0 of a replica run)
    formats = None
    if not args.no_formats and rank == 0:
        try:
            formats = run_formats(ex, lib, A, x, y, args.steps, args.warmup, args.no_cfg3)
        except Exception as e:
            formats = {"error": f"{type(e).__name__}: {e}"}

    # ---- CG iterations/s (cfg4): fused single-GPU solver at N = 1, the
    # row-partitioned solver over NCCL (halo exchange + allreduce) at N > 1
    cg = None
    del A, desc
    torch.cuda.empty_cache()
    if not args.no_cg:
        try:
            cg = run_cg(ex, world, rank, local_rank, args.cg_dist)
        except Exception as e:  # reported in the line, never fatal for the SpMV metric
            cg = {"error": f"{type(e).__name__}: {e}"}
    clocks = sampler.stop()

    if rank != 0:
        return
    value = world * bytes_step * K / elapsed_max
    peak, peak_src = measured_peak()
    avg_launch = sum(launch_s) / len(launch_s)
    achieved = bytes_step / avg_launch / 1e9
    traffic = ncu_traffic("csr_stream_kernel")
    line = {
        "metric": METRIC, "value": round(value / 1e9, 2), "unit": "GB/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": elapsed_max / K * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (App. B 27-pt stencil generated on device; x = seeded_values(n, 11))",
        "config": WORKLOAD,
        "parallelism": f"replicas x{world}",
        "gflops": round(world * 2 * nnz * K / elapsed_max / 1e9, 1),
        "roofline": {"bound": "hbm", "kernel": "csr_stream_kernel", "achieved": round(achieved, 1),
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "frac_of_8000": round(achieved / 8000, 4),
                     "traffic": traffic, "algorithmic_bytes_per_launch": bytes_step,
                     "avg_launch_us": avg_launch * 1e6},
        "e2e": {"value": round(world * bytes_step * K / e2e_s / 1e9, 2), "unit": "GB/s",
                "h2d_bytes_per_step": 8 * ncols, "d2h_bytes_per_step": nb,
                "ms_per_step": e2e_s / K * 1e3,
                "path": "lbk_memcpy_h2d(x) + lbk_spmv_csr_f64 + lbk_memcpy_d2h(y), pinned host, "
                        "three contexts/streams, double-buffered (step i's SpMV overlaps step "
                        "i+1's upload and step i-1's download)",
                "results_equal": e2e_step_ok,
                "sequential": {"value": round(world * bytes_step * K / e2e_seq_s / 1e9, 2),
                               "ms_per_step": e2e_seq_s / K * 1e3,
                               "path": "the same three calls back to back on one stream"}},
        "gpu_launches": K,
        "clocks": clocks,
    }
    if formats is not None:
        line["formats"] = formats
    if cg is not None:
        line["cg"] = cg
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample()
    print(json.dumps(line), flush=True)
    if args.report_dir:
        from paper_2011_08879_b200 import report as R
        os.makedirs(args.report_dir, exist_ok=True)
        recs = R.records_from_bench(line)
        for fmt in ("json", "csv", "svg"):
            with open(os.path.join(args.report_dir, f"bench_records.{fmt}"), "w") as f:
                f.write(R.emit_report(recs, fmt))


def cfg3_check(rp, ci, va, xh, y_csr, y_coo) -> dict:
    """cfg3 output check (measured but never verified): CSR and
    COO y agree bit for bit on every row of <= 256 entries and normwise
    everywhere, and a 65,536-row sample matches a host recomputation in the
    reference's order (sum from 0.0 in ascending k, reference.cpp:82-88)
    within 1e-12 normwise (bit-exact for rows <= 256)."""
    import numpy as np
    yc, yo = y_csr.cpu().numpy(), y_coo.cpu().numpy()
    lens = np.diff(rp.astype(np.int64))
    short = lens <= 256
    rng = np.random.default_rng(3)
    rows = np.sort(rng.choice(len(lens), 65536, replace=False))
    ref = np.empty(rows.size)
    for i, r in enumerate(rows):  # sequential sums: the reference's bits
        s = 0.0
        for k in range(int(rp[r]), int(rp[r + 1])):
            s += va[k] * xh[ci[k]]
        ref[i] = s
    d = np.abs(yc[rows] - ref).max() / max(np.abs(ref).max(), 1e-300)
    sh = short[rows]
    out = {"rows": int(len(lens)), "nnz": int(rp[-1]), "max_row": int(lens.max()),
           "csr_eq_coo_rows_le_256": bool(np.array_equal(yc[short], yo[short])),
           "csr_vs_coo_normwise": float(np.abs(yc - yo).max() / np.abs(yc).max()),
           "sample_rows": int(rows.size), "sample_normwise_vs_host": float(d),
           "sample_bitexact_rows_le_256": bool(np.array_equal(yc[rows][sh], ref[sh]))}
    out["ok"] = (out["csr_eq_coo_rows_le_256"] and out["sample_bitexact_rows_le_256"]
                 and out["sample_normwise_vs_host"] <= 1e-12 and out["csr_vs_coo_normwise"] <= 1e-12)
    if not out["ok"]:
        print(f"bench: cfg3 check FAILED {out}", file=sys.stderr)
    return out


def time_launches(ex, call, steps: int, warmup: int, flush=None) -> float:
    """Mean device time of one launch (CUDA event pair per launch, launches
    back to back on the executor's stream; with `flush`, that buffer is
    rewritten before every launch, outside the event pair)."""
    import torch
    for _ in range(warmup):
        call()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    for a, b in evs:
        if flush is not None:
            with torch.cuda.stream(ex.stream):
                flush.fill_(1)
        a.record(ex.stream)
        call()
        b.record(ex.stream)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / steps * 1e-3


def run_formats(ex, lib, A, x, y, steps: int, warmup: int, no_cfg3: bool) -> dict:
    """SpMV of every format and precision on the §8d configs: GB/s under the
    reference byte model (harness.cpp:342-354), GFLOP/s = 2 nnz / t."""
    import ctypes as C
    import numpy as np
    import torch

    from paper_2011_08879_b200 import gen, larch as lk

    peak, _ = measured_peak()
    out = {"peak_gbs": peak, "note": "GB/s = algorithmic bytes / mean launch time"}

    def meas(key, M, xv, yv, nbytes, nnz, flush=None):
        fn = {lk.CsrMatrix: "csr", lk.CooMatrix: "coo", lk.EllMatrix: "ell",
              lk.SellpMatrix: "sellp"}[type(M)]
        fn = getattr(lib, f"lbk_spmv_{fn}_{'f32' if xv.values.dtype == torch.float32 else 'f64'}")
        d = M.desc()
        xp, yp = C.c_void_p(xv.values.data_ptr()), C.c_void_p(yv.values.data_ptr())

        def call():
            st = fn(ex.ctx, C.byref(d), xp, yp)
            if st:
                lk._check(st, ex.ctx)
        t = time_launches(ex, call, max(steps, 10), max(warmup, 3), flush)
        out[key] = {"us": round(t * 1e6, 2), "gbs": round(nbytes / t / 1e9, 1),
                    "gflops": round(2 * nnz / t / 1e9, 1), "frac": round(nbytes / t / 1e9 / peak, 3),
                    "bytes": int(nbytes), "nnz": int(nnz)}

    # in-run bandwidth calibration (BabelStream copy / triad, 2 x 1 GiB + 1 GiB)
    ns = 1 << 27
    sa = torch.empty(ns, dtype=torch.float64, device=ex.device).fill_(1.0)
    sb = torch.empty_like(sa).fill_(2.0)
    sc = torch.empty_like(sa)
    pa, pb, pc = (C.c_void_p(t.data_ptr()) for t in (sa, sb, sc))
    t = time_launches(ex, lambda: lk._check(lib.lbk_stream_copy_f64(ex.ctx, ns, pa, pc), ex.ctx),
                      20, 3)
    out["stream_copy_gbs"] = round(16 * ns / t / 1e9, 1)
    t = time_launches(ex, lambda: lk._check(lib.lbk_stream_triad_f64(ex.ctx, ns, 0.4, pb, pc, pa),
                                            ex.ctx), 20, 3)
    out["stream_triad_gbs"] = round(24 * ns / t / 1e9, 1)
    del sa, sb, sc
    torch.cuda.empty_cache()

    n, nnz = A.nrows, A.nnz()
    meas("cfg2_csr_f64", A, x, y, 12 * nnz + 4 * (n + 1) + 16 * n, nnz)

    # device-side assembly and conversions (§8f.1; the reference does these
    # on the host: 12.2 s for cfg2)
    def wall(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ex.stream)
        for _ in range(reps):
            fn()
        e1.record(ex.stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    Co = lk.csr_to_coo(A)
    perm = torch.randperm(nnz, device=ex.device)
    rows_s, cols_s, vals_s = Co.row_idx[perm].contiguous(), Co.col_idx[perm].contiguous(), \
        Co.vals[perm].contiguous()
    del perm
    ro = torch.empty_like(rows_s)
    co = torch.empty_like(cols_s)
    vo = torch.empty_like(vals_s)
    nz = C.c_int64()

    def assemble():
        lk._check(lib.lbk_coo_assemble_f64(ex.ctx, n, n, nnz, C.c_void_p(rows_s.data_ptr()),
                                           C.c_void_p(cols_s.data_ptr()), C.c_void_p(vals_s.data_ptr()),
                                           C.c_void_p(ro.data_ptr()), C.c_void_p(co.data_ptr()),
                                           C.c_void_p(vo.data_ptr()), C.byref(nz)), ex.ctx)
    conv = {"coo_from_entries_shuffled_ms": round(wall(assemble), 2)}
    assert nz.value == nnz and torch.equal(ro, Co.row_idx) and torch.equal(co, Co.col_idx)
    del rows_s, cols_s, vals_s, ro, co, vo
    conv["coo_to_csr_ms"] = round(wall(lambda: lk.coo_to_csr(Co)), 3)
    conv["csr_to_coo_ms"] = round(wall(lambda: lk.csr_to_coo(A)), 3)
    conv["csr_to_ell_ms"] = round(wall(lambda: lk.csr_to_ell(A)), 3)
    conv["csr_to_sellp32_ms"] = round(wall(lambda: lk.csr_to_sellp(A, 32)), 3)
    conv["note"] = ("cfg2 (55.7M entries), device; coo_from_entries = bounds check + stable "
                    "(row, col) sort + duplicate sum (formats.cpp:78-116); output checked equal")
    out["conversions_cfg2"] = conv
    torch.cuda.empty_cache()
    Co = lk.csr_to_coo(A)
    meas("cfg2_coo_f64", Co, x, y, 16 * nnz + 16 * n, nnz)
    del Co
    E = lk.csr_to_ell(A)
    meas("cfg2_ell_f64", E, x, y, 12 * E.width * E.stride + 16 * n, nnz)
    del E
    S = lk.csr_to_sellp(A, 32)
    meas("cfg2_sellp32_f64", S, x, y, 12 * S.col_idx.numel() + 8 * S.nslices + 16 * n, nnz)
    del S
    A32 = A.astype(torch.float32)
    x32 = lk.DenseVector(x.values.float(), ex)
    y32 = lk.make_vector(ex, n, torch.float32)
    meas("cfg2_csr_f32", A32, x32, y32, 8 * nnz + 4 * (n + 1) + 8 * n, nnz)
    del A32
    torch.cuda.empty_cache()
    A1 = gen.stencil(ex, "5pt", 1024)
    x1 = lk.vector_from(ex, gen.seeded_values(A1.ncols, 11))
    y1 = lk.make_vector(ex, A1.nrows)
    n1, z1 = A1.nrows, A1.nnz()
    # cfg1's 84 MB fit in the 126 MB L2: flush it between launches (a 512 MB
    # write outside the timed event pair), SURVEY.md §8d
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=ex.device)
    meas("cfg1_csr_f64", A1, x1, y1, 12 * z1 + 4 * (n1 + 1) + 16 * n1, z1, flush=flush)
    out["cfg1_csr_f64"]["l2"] = "flushed (512 MB write) before every timed launch"
    del flush
    del A1
    if not no_cfg3:
        nn = 1 << 24
        rp, ci, va = gen.powerlaw_host(nn)
        A3 = lk.csr_from_host(ex, nn, nn, rp, ci, va)
        z3 = A3.nnz()
        x3h = gen.seeded_values(nn, 11)
        x3 = lk.vector_from(ex, x3h)
        y3 = lk.make_vector(ex, nn)
        meas("cfg3_csr_f64", A3, x3, y3, 12 * z3 + 4 * (nn + 1) + 16 * nn, z3)
        y_csr = y3.values.clone()
        C3 = lk.csr_to_coo(A3)
        meas("cfg3_coo_f64", C3, x3, y3, 16 * z3 + 16 * nn, z3)
        del C3
        out["cfg3_check"] = cfg3_check(rp, ci, va, x3h, y_csr, y3.values)
        del rp, ci, va, y_csr
        A3f = A3.astype(torch.float32)
        del A3
        x3f = lk.DenseVector(x3.values.float(), ex)
        y3f = lk.make_vector(ex, nn, torch.float32)
        meas("cfg3_csr_f32", A3f, x3f, y3f, 8 * z3 + 4 * (nn + 1) + 8 * nn, z3)
        del A3f
    torch.cuda.empty_cache()
    return out


def band_check(iters: int) -> bool:
    """cfg5 BiCGSTAB: the reference's own executor spread [495, 498]
    (SURVEY.md §8c-note); a miss is reported on stderr and in the line."""
    ok = 495 <= iters <= 498
    if not ok:
        print(f"bench: cfg5 BiCGSTAB {iters} iterations outside [495, 498]", file=sys.stderr)
    return ok


def run_cg(ex, world: int, rank: int, local_rank: int, force_dist: bool = False) -> dict:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2011_08879_b200 import dist as D, gen, larch as lk

    dev = ex.device
    A4 = gen.stencil(ex, "7pt", 256)
    n, nnz = A4.nrows, A4.nnz()
    ones = lk.vector_from(ex, np.ones(A4.ncols))
    b = lk.make_vector(ex, n)
    lk.spmv(A4, ones, b)  # b = A*1 (harness.cpp:376-378); rows <= 32 -> bit-exact
    cg = {"config": "cfg4: 7-pt Poisson 256^3, b = A*1, x0 = 0, tol 1e-8",
          "golden_iterations": 581}

    def tmax(v: float) -> float:
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if world == 1 and not force_dist:
        cg["mode"] = "single GPU, fused device-resident solver"
        for mode in ("true", "recurrence"):
            xs = lk.zeros(ex, n)
            # warm-up (the reference harness's 1 warm-up run, harness.cpp:55-61):
            # first-launch module loading stays out of the timed solve
            lk.solve(A4, b, lk.zeros(ex, n), lk.SolverConfig(kind="cg", rel_tol=1e-8, fixed_iters=3,
                                                             residual_mode="true"))
            if mode == "recurrence":
                lk.solve(A4, b, lk.zeros(ex, n), lk.SolverConfig(kind="cg", rel_tol=0.5,
                                                                 max_iters=20000,
                                                                 residual_mode=mode))
            r = lk.solve(A4, b, xs, lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000,
                                                     residual_mode=mode))
            cg[mode] = {"iterations": r.iterations, "final_rel_residual": r.final_rel_residual,
                        "seconds": r.elapsed, "iters_per_s": r.iterations / r.elapsed,
                        "flop_count": r.flop_count,
                        "gflops_ref_model": r.flop_count / r.elapsed / 1e9}
        del A4, ones, b, xs
        torch.cuda.empty_cache()
        # cfg5: BiCGSTAB, 7-pt upwind gamma 0.5, b = A x*, x* = seeded_values(n, 11)
        A5 = gen.stencil(ex, "7pt", 256, 0.5)
        xstar = lk.vector_from(ex, gen.seeded_values(A5.ncols, 11))
        b5 = lk.make_vector(ex, n)
        lk.spmv(A5, xstar, b5)
        xs = lk.zeros(ex, n)
        lk.solve(A5, b5, lk.zeros(ex, n), lk.SolverConfig(kind="bicgstab", rel_tol=1e-8,
                                                          fixed_iters=3))
        r = lk.solve(A5, b5, xs, lk.SolverConfig(kind="bicgstab", rel_tol=1e-8, max_iters=20000))
        cg["bicgstab_cfg5"] = {"config": "cfg5: 7-pt upwind gamma 0.5 256^3, b = A x*, tol 1e-8",
                               "golden_iterations": "495 (reference) / 498 (parallel)",
                               "in_band": band_check(r.iterations),
                               "iterations": r.iterations,
                               "final_rel_residual": r.final_rel_residual, "seconds": r.elapsed,
                               "iters_per_s": r.iterations / r.elapsed,
                               "flop_count": r.flop_count,
                               "gflops_ref_model": r.flop_count / r.elapsed / 1e9}
        xs = lk.zeros(ex, n)
        lk.solve(A5, b5, lk.zeros(ex, n), lk.SolverConfig(kind="cgs", rel_tol=1e-8, fixed_iters=3))
        r = lk.solve(A5, b5, xs, lk.SolverConfig(kind="cgs", rel_tol=1e-8, max_iters=20000))
        cg["cgs_cfg5"] = {"config": "cfg5 matrix and rhs, CGS (krylov.cpp:233-297), tol 1e-8",
                          "iterations": r.iterations, "final_rel_residual": r.final_rel_residual,
                          "seconds": r.elapsed, "iters_per_s": r.iterations / r.elapsed,
                          "flop_count": r.flop_count,
                          "gflops_ref_model": r.flop_count / r.elapsed / 1e9}
        return cg
    # distributed: this rank's rows of the same matrix
    lo, hi = D.part_range(n, world, rank)
    rp = A4.row_ptr[lo:hi + 1].cpu().numpy().astype(np.int64)
    k0, k1 = int(rp[0]), int(rp[-1])
    cols = A4.col_idx[k0:k1].cpu().numpy()
    vals = A4.vals[k0:k1].cpu().numpy()
    b_loc = b.values[lo:hi].clone()
    del A4, ones, b
    torch.cuda.empty_cache()
    rp = (rp - k0).astype(np.int32)
    def all_ok(ok: bool, what: str) -> None:
        # a rank that failed must not leave its peers blocked in a collective
        if world > 1:
            f = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            ok = bool(f.item())
        if not ok:
            raise RuntimeError(f"distributed CG: {what} failed on some rank")

    m = None
    try:
        m = D.DistMap(n, world, rank, rp, cols)
    except Exception:
        pass
    all_ok(m is not None, "partition maps")
    # communicator: "peer" (default; halo and reductions in lbk's own kernels
    # over IPC-mapped peer windows) or "nccl" (LBK_BENCH_COMM=nccl)
    comm_kind = os.environ.get("LBK_BENCH_COMM", "peer")
    if world > 1:
        D.exchange_requests(m)
        if comm_kind == "nccl":
            comm = D.Communicator.nccl(local_rank)
        else:
            comm = D.Communicator.peer(local_rank, D.peer_halo_cap(m))
    else:  # --cg-dist at N = 1: the same path on a one-rank communicator
        D.exchange_requests_local([m])
        if comm_kind == "nccl":
            comm = D.Communicator.nccl_single(local_rank)
        else:
            comm = D.Communicator.peer_group([local_rank], m.halo_count())[0]
    M = None
    try:
        M = D.DistCsrMatrix(ex, m, rp, vals, nnz)
    except Exception:
        pass
    all_ok(M is not None, "device matrix")
    if comm_kind == "nccl":
        cg["mode"] = (f"row-partitioned over {world} GPUs: NCCL halo exchange overlapped with "
                      f"the interior rows, ncclAllReduce per reduction (strong scaling)")
    else:
        cg["mode"] = (f"row-partitioned over {world} GPUs: halo stored into the neighbours' "
                      f"peer windows before the interior rows, each reduction summed over the "
                      f"peers in one kernel (strong scaling)")
    cg["comm"] = comm_kind
    cg["n_ghost_rank0"] = M.n_ghost
    for mode in ("true", "recurrence"):
        x = torch.zeros(M.n_local, dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        # warm-up: module loading and the CUDA-graph capture of a chunk
        M.solve(comm, b_loc, torch.zeros(M.n_local, dtype=torch.float64, device=dev),
                lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=40, residual_mode=mode))
        torch.cuda.synchronize()
        r = M.solve(comm, b_loc, x, lk.SolverConfig(kind="cg", rel_tol=1e-8, max_iters=20000,
                                                     residual_mode=mode))
        el = tmax(r.elapsed)
        cg[mode] = {"iterations": r.iterations, "final_rel_residual": r.final_rel_residual,
                    "seconds": el, "iters_per_s": r.iterations / el, "flop_count": r.flop_count,
                    "gflops_ref_model": r.flop_count / el / 1e9}
    # cfg5: BiCGSTAB on the nonsymmetric 7-pt upwind stencil, same partition
    # and communicator (same sparsity pattern, so the same halo)
    A5 = gen.stencil(ex, "7pt", 256, 0.5)
    xstar = lk.vector_from(ex, gen.seeded_values(A5.ncols, 11))
    b5 = lk.make_vector(ex, n)
    lk.spmv(A5, xstar, b5)
    rp5 = A5.row_ptr[lo:hi + 1].cpu().numpy().astype(np.int64)
    j0, j1 = int(rp5[0]), int(rp5[-1])
    cols5 = A5.col_idx[j0:j1].cpu().numpy()
    vals5 = A5.vals[j0:j1].cpu().numpy()
    nnz5 = A5.nnz()
    b5_loc = b5.values[lo:hi].clone()
    del A5, xstar, b5
    torch.cuda.empty_cache()
    rp5 = (rp5 - j0).astype(np.int32)
    M5 = None
    try:
        m5 = D.DistMap(n, world, rank, rp5, cols5)
    except Exception:
        m5 = None
    all_ok(m5 is not None, "cfg5 partition maps")
    if world > 1:
        D.exchange_requests(m5)
    else:
        D.exchange_requests_local([m5])
    try:
        M5 = D.DistCsrMatrix(ex, m5, rp5, vals5, nnz5)
    except Exception:
        M5 = None
    all_ok(M5 is not None, "cfg5 device matrix")
    M5.solve(comm, b5_loc, torch.zeros(M5.n_local, dtype=torch.float64, device=dev),
             lk.SolverConfig(kind="bicgstab", rel_tol=1e-8, max_iters=3))
    torch.cuda.synchronize()
    x5 = torch.zeros(M5.n_local, dtype=torch.float64, device=dev)
    r = M5.solve(comm, b5_loc, x5, lk.SolverConfig(kind="bicgstab", rel_tol=1e-8,
                                                  max_iters=20000))
    el = tmax(r.elapsed)
    cg["bicgstab_cfg5"] = {"config": "cfg5: 7-pt upwind gamma 0.5 256^3, b = A x*, tol 1e-8, "
                                     f"row-partitioned over {world} GPUs",
                           "golden_iterations": "495 (reference) / 498 (parallel)",
                           "in_band": band_check(r.iterations),
                           "iterations": r.iterations, "final_rel_residual": r.final_rel_residual,
                           "seconds": el, "iters_per_s": r.iterations / el,
                           "flop_count": r.flop_count,
                           "gflops_ref_model": r.flop_count / el / 1e9}
    comm.close()  # collective: peers may still be storing into this rank's window
    return cg


# ------------------------------------------------------------ CPU legs
def _cfg2_host():
    from oracle import oracle as O
    return O, O.stencil("27pt", 128)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_sample(reps: int = 5) -> dict:
    """The reference library (oracle/_ref) on this host (CPU
    timing beside it): cfg2 CSR SpMV with ParallelExecutor(nproc) (the
    `value`, median of `reps`) and ReferenceExecutor (1 core, median of 3);
    the reference's own host stream-copy peak (measure_peak_bandwidth,
    harness.cpp:125-141) on both executors; and cfg4 CG seconds per
    iteration at fixed_iters = 50 (krylov.hpp:30) on ParallelExecutor(nproc).
    About 15 s of host work."""
    try:
        O, A = _cfg2_host()
        if not O.ref_available():
            raise RuntimeError("oracle/_ref not built")
        cores = os.cpu_count() or 1
        x = O.seeded_values(A.ncols, 11)
        b2 = csr_bytes(A.nrows, A.ncols, A.nnz)
        _, med = O.ref_spmv(A, x, "csr", exec_kind=O.EXEC_PARALLEL, workers=cores, reps=reps)
        _, med1 = O.ref_spmv(A, x, "csr", exec_kind=0, workers=1, reps=3)
        out = {"value": round(b2 / med / 1e9, 3), "unit": "GB/s", "cores": cores,
               "kind": "reference", "cpu_model": cpu_model(),
               "sample": f"cfg2 CSR SpMV, reference ParallelExecutor({cores}), median of {reps}",
               "ms_per_step": med * 1e3,
               "reference_executor_1core": {"gbs": round(b2 / med1 / 1e9, 3),
                                            "ms_per_step": med1 * 1e3,
                                            "sample": "cfg2 CSR SpMV, ReferenceExecutor, median of 3"}}
        del A
        out["host_stream_copy_gbs"] = {
            f"parallel({cores})": round(O.ref_peak_bandwidth(O.EXEC_PARALLEL, cores, 1 << 27, 3), 2),
            "reference(1)": round(O.ref_peak_bandwidth(0, 1, 1 << 27, 3), 2),
            "note": "the reference's measure_peak_bandwidth (harness.cpp:125-141), 128 MiB arrays"}
        import numpy as np
        A4 = O.stencil("7pt", 256)
        b4 = O.spmv_csr(A4, np.ones(A4.nrows))
        r = O.ref_solve(A4, b4, "cg", rel_tol=1e-8, fixed_iters=50, exec_kind=O.EXEC_PARALLEL,
                        workers=cores)
        out["cg_cfg4_fixed50"] = {"s_per_iter": r.elapsed / 50, "iters_per_s": 50 / r.elapsed,
                                  "executor": f"ParallelExecutor({cores})",
                                  "note": "reference solve(), fixed_iters = 50 (krylov.hpp:30)"}
        return out
    except Exception as e:  # reported, never fatal for the GPU arm
        return {"value": None, "unit": "GB/s", "cores": 0, "kind": "reference",
                "sample": f"unavailable: {e}"}


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    O, A = _cfg2_host()
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    cores = os.cpu_count() or 1
    x = O.seeded_values(A.ncols, 11)
    for _ in range(args.warmup):
        O.ref_spmv(A, x, "csr", exec_kind=O.EXEC_PARALLEL, workers=cores, reps=1)
    times = []
    for _ in range(args.steps):
        _, s = O.ref_spmv(A, x, "csr", exec_kind=O.EXEC_PARALLEL, workers=cores, reps=1)
        times.append(s)
    total = sum(times)
    b = csr_bytes(A.nrows, A.ncols, A.nnz)
    v = round(b * len(times) / total / 1e9, 3)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / len(times) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (App. B 27-pt stencil, oracle generator)",
            "config": WORKLOAD,
            "parallelism": f"host ParallelExecutor({cores})", "cpu_model": cpu_model(),
            "gflops": round(2 * A.nnz * len(times) / total / 1e9, 3),
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "reference",
                             "sample": f"cfg2 CSR SpMV through the reference's spmv_csr, "
                                       f"{len(times)} steps"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-formats", action="store_true")
    ap.add_argument("--report-dir", default=None,
                    help="also write BenchRecord json/csv/svg (reference schema) here")
    ap.add_argument("--no-cfg3", action="store_true")
    ap.add_argument("--cg-dist", action="store_true",
                    help="use the row-partitioned solver for the CG leg even at N = 1")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # dev-only: LBK_BENCH_FOLD=1 folds every rank onto cuda:0 (gloo
    # bootstrap) to exercise the N > 1 code paths on a one-GPU box; its
    # numbers are meaningless (the ranks' contexts time-slice)
    fold = os.environ.get("LBK_BENCH_FOLD") == "1"
    if fold:
        local_rank = 0
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        import datetime
        if fold:
            dist.init_process_group("gloo", timeout=datetime.timedelta(minutes=10))
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank),
                                    timeout=datetime.timedelta(minutes=5))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
