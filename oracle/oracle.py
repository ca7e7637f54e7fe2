"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes front-end over the two CPU checkers built by ``oracle/Makefile``:

* ``ref``  -- ``oracle/_ref/liblarch_ref.so``: the reference library itself
  (``/root/reference/proj/src`` compiled out of tree, FMA-free, plus
  ``ref_driver.cpp``).  Present wherever ``build()`` ran in the container
  that holds ``/root/reference``; the built ``.so`` travels to the GPU box.
* ``port`` -- ``oracle/_build/liboracle_port.so``: our restatement
  (``port.cpp``), incl. ELL / SELL-P / FP32 / partition maps / generators.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "liblarch_ref.so")
PORT_SO = os.path.join(HERE, "_build", "liboracle_port.so")

i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
i64 = C.c_int64

_port = None
_ref = None


def build(ref: bool | None = None) -> None:
    """Compile the checkers (make -C oracle).  ``ref`` defaults to building
    the reference library only when /root/reference is present."""
    import subprocess

    if ref is None:
        ref = os.path.isdir(os.environ.get("LARCH_REF_DIR", "/root/reference/proj"))
    targets = ["port"] + (["ref"] if ref else [])
    env = dict(os.environ)
    if "LARCH_REF_DIR" in env:
        env["REF_DIR"] = env["LARCH_REF_DIR"]
    subprocess.run(["make", "-s", "-j8", "-C", HERE] + targets, check=True, env=env)


def port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        lib = C.CDLL(PORT_SO)
        sig = {
            "port_stencil_nnz": (i64, [C.c_int, C.c_int]),
            "port_stencil_csr": (None, [C.c_int, C.c_int, C.c_double, i32p, i32p, f64p]),
            "port_seeded_values": (None, [i64, C.c_uint64, f64p]),
            "port_powerlaw_new": (C.c_void_p, [C.c_int32, C.c_uint64, C.c_int32, C.c_int32, C.POINTER(i64)]),
            "port_powerlaw_fill": (None, [C.c_void_p, i32p, i32p, f64p]),
            "port_free": (None, [C.c_void_p]),
            "port_spmv_csr_f64": (None, [C.c_int32, i32p, i32p, f64p, f64p, f64p]),
            "port_spmv_csr_f32": (None, [C.c_int32, i32p, i32p, f32p, f32p, f32p]),
            "port_spmv_coo_f64": (None, [C.c_int32, i64, i32p, i32p, f64p, f64p, f64p]),
            "port_spmv_ell_f64": (None, [C.c_int32, C.c_int32, i64, i32p, f64p, f64p, f64p]),
            "port_spmv_sellp_f64": (None, [C.c_int32, C.c_int32, i32p, i32p, f64p, f64p, f64p]),
            "port_csr_max_row": (C.c_int32, [C.c_int32, i32p]),
            "port_csr_to_ell": (None, [C.c_int32, i32p, i32p, f64p, C.c_int32, i64, i32p, f64p]),
            "port_sellp_sets": (i64, [C.c_int32, i32p, C.c_int32, i32p, i32p]),
            "port_csr_to_sellp": (None, [C.c_int32, i32p, i32p, f64p, C.c_int32, i32p, i32p, f64p]),
            "port_coo_to_csr": (None, [C.c_int32, i64, i32p, i32p]),
            "port_csr_to_coo": (None, [C.c_int32, i32p, i32p]),
            "port_part_rank_of": (C.c_int32, [C.c_int32, C.c_int32, C.c_int32]),
            "port_part_range": (None, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
            "port_part_ghosts": (i64, [C.c_int32, C.c_int32, C.c_int32, i32p, i32p, C.c_void_p, i64]),
            "port_part_local_cols": (None, [C.c_int32, C.c_int32, C.c_int32, i32p, i32p, i32p, i64, i32p]),
            "port_dot": (C.c_double, [i64, f64p, f64p]),
            "port_xdot": (C.c_double, [i64, f64p, f64p]),
            "port_xsum": (C.c_double, [i64, f64p]),
            "port_xsolve": (C.c_int, [C.c_int, C.c_int32, i32p, i32p, f64p, f64p, f64p, C.c_double,
                                      C.c_int, C.c_int, f64p, i64, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), C.POINTER(i64), C.POINTER(C.c_int)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_buildable() -> bool:
    return os.path.isdir(os.environ.get("LARCH_REF_DIR", "/root/reference/proj"))


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"reference oracle not built: {REF_SO}")
        lib = C.CDLL(REF_SO)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_last_breakdown_iter": (C.c_int, []),
            "ref_spmv": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i64, i32p, i32p, f64p, f64p, f64p, C.c_int, C.POINTER(C.c_double)]),
            "ref_dot": (C.c_int, [C.c_int, C.c_int, i64, f64p, f64p, C.POINTER(C.c_double)]),
            "ref_axpy": (C.c_int, [i64, C.c_double, f64p, f64p]),
            "ref_coo_from_entries": (C.c_int, [C.c_int, C.c_int, i64, i32p, i32p, f64p, C.POINTER(i64), i32p, i32p, f64p]),
            "ref_coo_to_csr": (C.c_int, [C.c_int, C.c_int, i64, i32p, i32p, f64p, i32p, i32p, f64p]),
            "ref_csr_to_coo": (C.c_int, [C.c_int, C.c_int, i64, i32p, i32p, f64p, i32p, i32p, f64p]),
            "ref_validate": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, i32p, i32p, f64p]),
            "ref_read_mm": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(i64), C.c_void_p, C.c_void_p, C.c_void_p]),
            "ref_gmres_cycle": (C.c_int, [C.c_int, C.c_int, C.c_int, i64, i32p, i32p, f64p, f64p,
                                          f64p, C.c_int, C.POINTER(C.c_double), i32p, C.c_void_p,
                                          C.c_int]),
            "ref_measure_peak_bandwidth": (C.c_int, [C.c_int, C.c_int, i64, C.c_int,
                                                     C.POINTER(C.c_double)]),
            "ref_solve": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, i64, i32p, i32p, f64p, f64p, f64p, C.c_int, C.c_double, C.c_int, C.c_int, f64p, C.c_int, i32p, f64p, C.POINTER(i64)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _ref = lib
    return _ref


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str, iteration: int = -1):
        super().__init__(f"status {status}: {msg}")
        self.msg = msg
        self.status = status
        self.iteration = iteration


def _chk(st: int) -> None:
    if st != 0:
        lib = ref()
        raise OracleError(st, lib.ref_last_error().decode(), lib.ref_last_breakdown_iter())


# ----------------------------------------------------------------- matrices
@dataclass
class Csr:
    nrows: int
    ncols: int
    row_ptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.vals.size)


def stencil(kind: str, m: int, gamma: float = 0.0) -> Csr:
    """kind in {'5pt', '7pt', '27pt'} -- SURVEY.md App. B stencils."""
    k = {"5pt": 0, "7pt": 1, "27pt": 2}[kind]
    lib = port()
    nnz = lib.port_stencil_nnz(k, m)
    n = m * m if k == 0 else m * m * m
    rp = np.empty(n + 1, np.int32)
    ci = np.empty(nnz, np.int32)
    va = np.empty(nnz, np.float64)
    lib.port_stencil_csr(k, m, gamma, rp, ci, va)
    return Csr(n, n, rp, ci, va)


def powerlaw(n: int, seed: int = 42, max_len: int = 10000, window: int = 65536) -> Csr:
    lib = port()
    nnz = i64(0)
    h = lib.port_powerlaw_new(n, seed, max_len, window, C.byref(nnz))
    rp = np.empty(n + 1, np.int32)
    ci = np.empty(nnz.value, np.int32)
    va = np.empty(nnz.value, np.float64)
    lib.port_powerlaw_fill(h, rp, ci, va)
    lib.port_free(h)
    return Csr(n, n, rp, ci, va)


def seeded_values(n: int, seed: int = 11) -> np.ndarray:
    out = np.empty(n, np.float64)
    port().port_seeded_values(n, seed, out)
    return out


# ------------------------------------------------------------ SpMV (port)
def spmv_csr(a: Csr, x: np.ndarray) -> np.ndarray:
    y = np.empty(a.nrows, x.dtype)
    if x.dtype == np.float32:
        port().port_spmv_csr_f32(a.nrows, a.row_ptr, a.cols, a.vals.astype(np.float32), x, y)
    else:
        port().port_spmv_csr_f64(a.nrows, a.row_ptr, a.cols, a.vals, x, y)
    return y


def csr_to_coo_rows(a: Csr) -> np.ndarray:
    rows = np.empty(a.nnz, np.int32)
    port().port_csr_to_coo(a.nrows, a.row_ptr, rows)
    return rows


def coo_to_csr_ptr(nrows: int, rows: np.ndarray) -> np.ndarray:
    rp = np.empty(nrows + 1, np.int32)
    port().port_coo_to_csr(nrows, rows.size, np.ascontiguousarray(rows, np.int32), rp)
    return rp


def spmv_coo(nrows: int, rows, cols, vals, x) -> np.ndarray:
    y = np.empty(nrows, np.float64)
    port().port_spmv_coo_f64(nrows, vals.size, rows, cols, vals, x, y)
    return y


def csr_to_ell(a: Csr, width: int | None = None, stride: int | None = None):
    lib = port()
    w = lib.port_csr_max_row(a.nrows, a.row_ptr) if width is None else width
    s = a.nrows if stride is None else stride
    ec = np.empty(max(w * s, 0), np.int32)
    ev = np.empty(max(w * s, 0), np.float64)
    lib.port_csr_to_ell(a.nrows, a.row_ptr, a.cols, a.vals, w, s, ec, ev)
    return w, s, ec, ev


def spmv_ell(nrows, width, stride, ec, ev, x) -> np.ndarray:
    y = np.empty(nrows, np.float64)
    port().port_spmv_ell_f64(nrows, width, stride, ec, ev, x, y)
    return y


def sellp_sets(a: Csr, S: int = 32):
    lib = port()
    ns = (a.nrows + S - 1) // S
    sl = np.empty(ns, np.int32)
    ss = np.empty(ns + 1, np.int32)
    stored = lib.port_sellp_sets(a.nrows, a.row_ptr, S, sl, ss)
    return sl, ss, int(stored)


def csr_to_sellp(a: Csr, S: int = 32):
    sl, ss, stored = sellp_sets(a, S)
    sc = np.empty(stored, np.int32)
    sv = np.empty(stored, np.float64)
    port().port_csr_to_sellp(a.nrows, a.row_ptr, a.cols, a.vals, S, ss, sc, sv)
    return sl, ss, sc, sv


def spmv_sellp(nrows, S, ss, sc, sv, x) -> np.ndarray:
    y = np.empty(nrows, np.float64)
    port().port_spmv_sellp_f64(nrows, S, ss, sc, sv, x, y)
    return y


# -------------------------------------------------------- partition maps
def part_range(n: int, P: int, rank: int):
    b, e = C.c_int32(), C.c_int32()
    port().port_part_range(n, P, rank, C.byref(b), C.byref(e))
    return b.value, e.value


def part_ghosts(a: Csr, P: int, rank: int) -> np.ndarray:
    lib = port()
    cnt = lib.port_part_ghosts(a.nrows, P, rank, a.row_ptr, a.cols, None, 0)
    g = np.empty(cnt, np.int32)
    lib.port_part_ghosts(a.nrows, P, rank, a.row_ptr, a.cols, g.ctypes.data_as(C.c_void_p), cnt)
    return g


def part_local_cols(a: Csr, P: int, rank: int, ghosts: np.ndarray) -> np.ndarray:
    b, e = part_range(a.nrows, P, rank)
    out = np.empty(int(a.row_ptr[e] - a.row_ptr[b]), np.int32)
    port().port_part_local_cols(a.nrows, P, rank, a.row_ptr, a.cols, ghosts, ghosts.size, out)
    return out


# ---------------------------------------------------- reference library
EXEC_REFERENCE = 0
EXEC_PARALLEL = 1


def ref_spmv(a: Csr, x: np.ndarray, fmt: str = "csr", exec_kind: int = 0,
             workers: int = 1, reps: int = 0):
    """Returns (y, median_seconds) through the reference's spmv_csr/spmv_coo."""
    y = np.empty(a.nrows, np.float64)
    sec = C.c_double(0.0)
    if fmt == "csr":
        ptr = a.row_ptr
    else:
        ptr = csr_to_coo_rows(a)
    _chk(ref().ref_spmv(exec_kind, workers, 1 if fmt == "csr" else 0, a.nrows, a.ncols,
                        a.nnz, ptr, a.cols, a.vals, np.ascontiguousarray(x, np.float64), y,
                        reps, C.byref(sec)))
    return y, sec.value


def ref_dot(x, y, exec_kind=0, workers=1) -> float:
    out = C.c_double()
    _chk(ref().ref_dot(exec_kind, workers, x.size, x, y, C.byref(out)))
    return out.value


def ref_coo_from_entries(nrows, ncols, rows, cols, vals):
    n = len(vals)
    ro = np.empty(max(n, 1), np.int32)
    co = np.empty(max(n, 1), np.int32)
    vo = np.empty(max(n, 1), np.float64)
    nnz = i64()
    _chk(ref().ref_coo_from_entries(nrows, ncols, n, np.ascontiguousarray(rows, np.int32),
                                    np.ascontiguousarray(cols, np.int32),
                                    np.ascontiguousarray(vals, np.float64), C.byref(nnz), ro, co, vo))
    k = nnz.value
    return ro[:k].copy(), co[:k].copy(), vo[:k].copy()


def ref_coo_to_csr(nrows, ncols, rows, cols, vals):
    rp = np.empty(nrows + 1, np.int32)
    co = np.empty(max(len(vals), 1), np.int32)
    vo = np.empty(max(len(vals), 1), np.float64)
    _chk(ref().ref_coo_to_csr(nrows, ncols, len(vals), np.ascontiguousarray(rows, np.int32),
                              np.ascontiguousarray(cols, np.int32),
                              np.ascontiguousarray(vals, np.float64), rp, co, vo))
    return rp, co[: len(vals)], vo[: len(vals)]


def ref_csr_to_coo(a: Csr):
    ro = np.empty(max(a.nnz, 1), np.int32)
    co = np.empty(max(a.nnz, 1), np.int32)
    vo = np.empty(max(a.nnz, 1), np.float64)
    _chk(ref().ref_csr_to_coo(a.nrows, a.ncols, a.nnz, a.row_ptr, a.cols, a.vals, ro, co, vo))
    return ro[: a.nnz], co[: a.nnz], vo[: a.nnz]


def ref_validate(fmt: str, nrows, ncols, ptr, cols, vals) -> int:
    """Returns the reference status code (0 = valid, 8 = FormatError)."""
    return ref().ref_validate(1 if fmt == "csr" else 0, nrows, ncols, len(vals),
                              np.ascontiguousarray(ptr, np.int32),
                              np.ascontiguousarray(cols, np.int32),
                              np.ascontiguousarray(vals, np.float64))


def ref_read_mm(path: str):
    """The reference's read_matrix_market -> (nrows, ncols, rows, cols, vals),
    or raises OracleError (status 8 FormatError, 11 UnsupportedFormatError)."""
    nr, nc, nz = C.c_int(), C.c_int(), i64()
    _chk(ref().ref_read_mm(path.encode(), C.byref(nr), C.byref(nc), C.byref(nz), None, None, None))
    rows = np.empty(max(nz.value, 1), np.int32)
    cols = np.empty(max(nz.value, 1), np.int32)
    vals = np.empty(max(nz.value, 1), np.float64)
    _chk(ref().ref_read_mm(path.encode(), C.byref(nr), C.byref(nc), C.byref(nz),
                           rows.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p),
                           vals.ctypes.data_as(C.c_void_p)))
    k = nz.value
    return nr.value, nc.value, rows[:k], cols[:k], vals[:k]


@dataclass
class RefSolve:
    converged: bool
    iterations: int
    final_rel_residual: float
    history: np.ndarray
    flop_count: int
    elapsed: float
    x: np.ndarray


SOLVERS = {"cg": 0, "bicgstab": 1, "cgs": 2, "gmres": 3}


def ref_solve(a: Csr, b: np.ndarray, kind: str = "cg", x0=None, max_iters=1000,
              rel_tol=1e-10, fixed_iters=0, restart=30, fmt="csr", exec_kind=0,
              workers=1) -> RefSolve:
    n = a.nrows
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64)
    cap = (fixed_iters or max_iters) + 2
    hist = np.empty(cap, np.float64)
    oi = np.zeros(3, np.int32)
    od = np.zeros(2, np.float64)
    fl = i64()
    ptr = a.row_ptr if fmt == "csr" else csr_to_coo_rows(a)
    _chk(ref().ref_solve(exec_kind, workers, 1 if fmt == "csr" else 0, SOLVERS[kind], n,
                         a.nnz, ptr, a.cols, a.vals, np.ascontiguousarray(b, np.float64), x,
                         max_iters, rel_tol, fixed_iters, restart, hist, cap, oi, od, C.byref(fl)))
    return RefSolve(bool(oi[0]), int(oi[1]), float(od[0]), hist[: oi[2]].copy(), fl.value,
                    float(od[1]), x)


# ------------------------------------------------- exactly rounded reductions
def xdot(x: np.ndarray, y: np.ndarray) -> float:
    """RNE(sum RN(x_i y_i)) -- the product's partition-independent dot."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return port().port_xdot(x.size, x, y)


def xsum(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, np.float64)
    return port().port_xsum(v.size, v)


def xsolve(a: Csr, b: np.ndarray, kind: str = "cg", x0=None, tol: float = 1e-8,
           max_iters: int = 1000, fixed_iters: int = 0) -> dict:
    """krylov.cpp CG / BiCGSTAB with exactly rounded dots (oracle/xkrylov.cpp)."""
    k = {"cg": 0, "bicgstab": 1}[kind]
    x = np.zeros(a.nrows) if x0 is None else np.array(x0, np.float64)
    cap = (fixed_iters or max_iters) + 2
    hist = np.zeros(cap)
    it, conv, bd = C.c_int(), C.c_int(), C.c_int()
    fl = i64(0)
    st = port().port_xsolve(k, a.nrows, a.row_ptr, a.cols, a.vals,
                            np.ascontiguousarray(b, np.float64), x, tol, max_iters,
                            fixed_iters, hist, cap, C.byref(it), C.byref(conv), C.byref(fl),
                            C.byref(bd))
    return {"status": st, "iterations": it.value, "converged": bool(conv.value),
            "history": hist[: it.value + 1].copy(), "flops": fl.value,
            "breakdown_iter": bd.value, "x": x}


def ref_peak_bandwidth(exec_kind: int = 1, workers: int = 1, bytes_: int = 1 << 27,
                       reps: int = 3) -> float:
    """The reference's measure_peak_bandwidth (harness.cpp:125-141), GB/s."""
    out = C.c_double()
    _chk(ref().ref_measure_peak_bandwidth(exec_kind, workers, bytes_, reps, C.byref(out)))
    return out.value


def ref_gmres_cycle(a: Csr, b: np.ndarray, x0=None, restart: int = 10) -> dict:
    """The reference's gmres_restart_cycle (krylov.hpp:78-89) on CSR."""
    n = a.nrows
    x = np.zeros(n) if x0 is None else np.array(x0, np.float64)
    rel = C.c_double()
    oi = np.zeros(3, np.int32)
    basis = np.zeros((restart + 1, n))
    _chk(ref().ref_gmres_cycle(0, 1, n, a.nnz, a.row_ptr, a.cols, a.vals,
                               np.ascontiguousarray(b, np.float64), x, restart, C.byref(rel), oi,
                               basis.ctypes.data_as(C.c_void_p), restart + 1))
    return {"rel_residual": rel.value, "steps": int(oi[0]), "happy": bool(oi[1]),
            "basis": basis[: int(oi[2])].copy(), "x": x}
