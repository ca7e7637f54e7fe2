"""Python mirror of the reference's operator surface, on the B200 backend.

The names, argument meanings and error behaviour follow the reference's
public headers (paths relative to /root/reference/proj):

  executors   include/larch/core/executor.hpp:130-262
  vectors     include/larch/matrix/formats.hpp:20-34
  matrices    include/larch/matrix/formats.hpp:37-94
  kernels     include/larch/kernels/kernels.hpp:79-97
  solvers     include/larch/solver/krylov.hpp:17-60
  errors      include/larch/core/error.hpp:16-131

Everything below calls the C ABI in ``liblbk.so`` (``include/lbk.h``)
through ctypes; device memory and the stream come from PyTorch (plumbing
only).  There is no CPU path: without a CUDA device the executor cannot be
created, and without the library the import fails.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """error.hpp:16 -- base of every library error."""


class ConfigurationError(Error):
    pass


class OutOfMemoryError(Error):
    pass


class ShapeError(Error):
    pass


class TypeError_(Error):
    pass


class PlacementError(Error):
    pass


class UsageError(Error):
    pass


class DispatchError(Error):
    pass


class FormatError(Error):
    pass


class UnsupportedFormatError(FormatError):
    """error.hpp:108"""


class BreakdownError(Error):
    def __init__(self, what: str, iteration: int):
        super().__init__(what)
        self.iteration = iteration


class BenchmarkIntegrityError(Error):
    pass


class DeviceError(Error):
    """CUDA / NCCL failure (no reference counterpart)."""


_STATUS = {
    L.SHAPE_ERROR: ShapeError,
    L.PLACEMENT_ERROR: PlacementError,
    L.TYPE_ERROR: TypeError_,
    L.DISPATCH_ERROR: DispatchError,
    L.USAGE_ERROR: UsageError,
    L.CONFIGURATION_ERROR: ConfigurationError,
    L.OUT_OF_MEMORY: OutOfMemoryError,
    L.FORMAT_ERROR: FormatError,
    L.UNSUPPORTED_FORMAT: UnsupportedFormatError,
    L.BENCHMARK_INTEGRITY: BenchmarkIntegrityError,
    L.CUDA_ERROR: DeviceError,
    L.NCCL_ERROR: DeviceError,
    L.INTERNAL: Error,
}


def _check(status: int, ctx=None, iteration: int = -1) -> None:
    if status == L.OK:
        return
    msg = L.load().lbk_last_error(ctx).decode(errors="replace")
    if status == L.BREAKDOWN:
        raise BreakdownError(msg, iteration)
    raise _STATUS.get(status, Error)(msg)


# --------------------------------------------------------------- executor
class CudaExecutor:
    """B200 executor: one device, one stream (torch's current stream).

    Plays the role of the reference's Executor (executor.hpp:130-170):
    synchronize(), describe(), and an arena capacity whose excess raises
    OutOfMemoryError (executor.cpp:254-265)."""

    def __init__(self, device: int = 0, arena_capacity: Optional[int] = None,
                 stream: Optional["torch.cuda.Stream"] = None):
        if not torch.cuda.is_available():
            raise DispatchError("CudaExecutor needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", device)
        self.lib = L.load()
        stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        ctx = C.c_void_p()
        _check(self.lib.lbk_ctx_create_on_stream(device, C.c_void_p(stream.cuda_stream), C.byref(ctx)))
        self.ctx = ctx
        self.stream = stream
        self.arena_capacity = arena_capacity
        self.arena_used = 0

    def kind(self) -> str:
        return "cuda"

    def synchronize(self) -> None:
        _check(self.lib.lbk_sync(self.ctx), self.ctx)

    def describe(self) -> dict:
        dev, sms = C.c_int(), C.c_int()
        cap, used = C.c_size_t(), C.c_size_t()
        self.lib.lbk_ctx_info(self.ctx, C.byref(dev), C.byref(sms), C.byref(cap), C.byref(used))
        return {"kind": "cuda", "device": dev.value, "num_sms": sms.value,
                "arena_capacity": self.arena_capacity, "arena_used": self.arena_used,
                "name": torch.cuda.get_device_name(self.device)}

    # torch-backed arena accounting
    def empty(self, n: int, dtype) -> torch.Tensor:
        nbytes = int(n) * torch.tensor([], dtype=dtype).element_size()
        if self.arena_capacity is not None and nbytes > self.arena_capacity - self.arena_used:
            raise OutOfMemoryError(
                f"out of memory on {self.device}: requested {nbytes} bytes, available "
                f"{self.arena_capacity - self.arena_used}")
        self.arena_used += nbytes
        return torch.empty(int(n), dtype=dtype, device=self.device)

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.lib.lbk_ctx_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass


_default_exec: Optional[CudaExecutor] = None


def create_executor(kind: str = "cuda", device: int = 0, **params) -> CudaExecutor:
    """executor.hpp:261-262 create_executor; only the B200 kind exists here."""
    if kind != "cuda":
        raise ConfigurationError(f"unknown executor kind {kind!r} (this backend provides 'cuda')")
    return CudaExecutor(device, **params)


def default_executor() -> CudaExecutor:
    global _default_exec
    if _default_exec is None:
        _default_exec = CudaExecutor(0)
    return _default_exec


def _ptr(t: Optional[torch.Tensor]):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else C.c_void_p(0)


# ----------------------------------------------------------------- vectors
@dataclass
class DenseVector:
    """formats.hpp:20-34.  `values` is a contiguous CUDA tensor."""
    values: torch.Tensor
    exec: CudaExecutor

    def size(self) -> int:
        return int(self.values.numel())

    def executor(self) -> CudaExecutor:
        return self.exec

    def clone_to(self, exec: CudaExecutor) -> "DenseVector":
        v = exec.empty(self.size(), self.values.dtype)
        v.copy_(self.values)
        return DenseVector(v, exec)


def make_vector(exec: CudaExecutor, size: int, dtype=torch.float64) -> DenseVector:
    return DenseVector(exec.empty(size, dtype), exec)


def vector_from(exec: CudaExecutor, values, dtype=None) -> DenseVector:
    arr = np.asarray(values)
    if dtype is None:
        dtype = torch.float32 if arr.dtype == np.float32 else torch.float64
    v = exec.empty(arr.size, dtype)
    v.copy_(torch.from_numpy(np.ascontiguousarray(arr)).to(dtype))
    return DenseVector(v, exec)


def zeros(exec: CudaExecutor, size: int, dtype=torch.float64) -> DenseVector:
    v = make_vector(exec, size, dtype)
    v.values.zero_()
    return v


def vector_to_host(vec: DenseVector) -> np.ndarray:
    return vec.values.cpu().numpy()


# ---------------------------------------------------------------- matrices
def _dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float64:
        return L.F64
    if t.dtype == torch.float32:
        return L.F32
    raise TypeError_(f"unsupported value dtype {t.dtype}")


@dataclass
class CsrMatrix:
    """formats.hpp:65-76 (+ a lazily built load-balance plan)."""
    nrows: int
    ncols: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    vals: torch.Tensor
    exec: CudaExecutor
    _plan: Optional[torch.Tensor] = field(default=None, repr=False)

    def nnz(self) -> int:
        return int(self.vals.numel())

    def executor(self) -> CudaExecutor:
        return self.exec

    def desc(self, with_plan: bool = True) -> L.lbk_csr:
        d = L.lbk_csr(self.nrows, self.ncols, self.nnz(), _dt(self.vals), _ptr(self.row_ptr),
                      _ptr(self.col_idx), _ptr(self.vals), None, 0)
        if with_plan and self.nrows > 0:
            if self._plan is None:
                nt = C.c_int32()
                L.load().lbk_csr_plan_size(C.byref(d), C.byref(nt))
                plan = torch.empty(nt.value + 1, dtype=torch.int32, device=self.exec.device)
                _check(L.load().lbk_csr_plan(self.exec.ctx, C.byref(d), _ptr(plan)), self.exec.ctx)
                self._plan = plan
            d.tile_rows = _ptr(self._plan)
            d.ntiles = self._plan.numel() - 1
        return d

    def clone_to(self, exec: CudaExecutor) -> "CsrMatrix":
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr.to(exec.device).clone(),
                         self.col_idx.to(exec.device).clone(), self.vals.to(exec.device).clone(), exec)

    def astype(self, dtype) -> "CsrMatrix":
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr, self.col_idx, self.vals.to(dtype),
                         self.exec)


@dataclass
class CooMatrix:
    """formats.hpp:49-60 (+ lazily built row-aligned tile plan)."""
    nrows: int
    ncols: int
    row_idx: torch.Tensor
    col_idx: torch.Tensor
    vals: torch.Tensor
    exec: CudaExecutor
    _plan: Optional[torch.Tensor] = field(default=None, repr=False)

    def nnz(self) -> int:
        return int(self.vals.numel())

    def executor(self) -> CudaExecutor:
        return self.exec

    def desc(self, with_plan: bool = True) -> L.lbk_coo:
        d = L.lbk_coo(self.nrows, self.ncols, self.nnz(), _dt(self.vals), _ptr(self.row_idx),
                      _ptr(self.col_idx), _ptr(self.vals), None, 0)
        if with_plan and self.nnz() > 0:
            if self._plan is None:
                nt = C.c_int32()
                L.load().lbk_coo_plan_size(C.byref(d), C.byref(nt))
                plan = torch.empty(nt.value + 1, dtype=torch.int32, device=self.exec.device)
                _check(L.load().lbk_coo_plan(self.exec.ctx, C.byref(d), _ptr(plan)), self.exec.ctx)
                self._plan = plan
            d.tile_starts = _ptr(self._plan)
            d.ntiles = self._plan.numel() - 1
        return d

    def clone_to(self, exec: CudaExecutor) -> "CooMatrix":
        return CooMatrix(self.nrows, self.ncols, self.row_idx.to(exec.device).clone(),
                         self.col_idx.to(exec.device).clone(), self.vals.to(exec.device).clone(), exec)


@dataclass
class EllMatrix:
    """Ginkgo column-major ELL."""
    nrows: int
    ncols: int
    width: int
    stride: int
    col_idx: torch.Tensor
    vals: torch.Tensor
    nnz_logical: int
    exec: CudaExecutor

    def nnz(self) -> int:
        return self.nnz_logical

    def desc(self) -> L.lbk_ell:
        return L.lbk_ell(self.nrows, self.ncols, self.nnz_logical, _dt(self.vals), self.width,
                         self.stride, _ptr(self.col_idx), _ptr(self.vals))


@dataclass
class SellpMatrix:
    """Ginkgo SELL-P."""
    nrows: int
    ncols: int
    slice_size: int
    slice_lengths: torch.Tensor
    slice_sets: torch.Tensor
    col_idx: torch.Tensor
    vals: torch.Tensor
    nnz_logical: int
    exec: CudaExecutor
    stored: int = -1

    def nnz(self) -> int:
        return self.nnz_logical

    @property
    def nslices(self) -> int:
        return int(self.slice_lengths.numel())

    _plan: Optional[torch.Tensor] = field(default=None, repr=False)

    def desc(self) -> L.lbk_sellp:
        stored = self.stored if self.stored >= 0 else int(self.col_idx.numel())
        d = L.lbk_sellp(self.nrows, self.ncols, self.nnz_logical, _dt(self.vals),
                        self.slice_size, self.nslices, _ptr(self.slice_lengths),
                        _ptr(self.slice_sets), _ptr(self.col_idx), _ptr(self.vals), stored,
                        None, 0)
        if self.slice_size == 32 and stored > 0 and self.nrows > 0:
            if self._plan is None:
                nt = C.c_int32()
                _check(L.load().lbk_sellp_plan_size(C.byref(d), C.byref(nt)))
                plan = torch.empty(nt.value + 1, dtype=torch.int32, device=self.exec.device)
                _check(L.load().lbk_sellp_plan(self.exec.ctx, C.byref(d), _ptr(plan)), self.exec.ctx)
                self._plan = plan
            d.tile_slices = _ptr(self._plan)
            d.ntiles = self._plan.numel() - 1
        return d


def csr_from_host(exec: CudaExecutor, nrows: int, ncols: int, row_ptr, col_idx, vals,
                  dtype=torch.float64) -> CsrMatrix:
    """Upload host CSR arrays (the array_from_host staging path)."""
    dev = exec.device
    rp = torch.from_numpy(np.ascontiguousarray(row_ptr, np.int32)).to(dev)
    ci = torch.from_numpy(np.ascontiguousarray(col_idx, np.int32)).to(dev)
    va = torch.from_numpy(np.ascontiguousarray(vals)).to(dev).to(dtype)
    return CsrMatrix(nrows, ncols, rp, ci, va, exec)


def coo_from_host(exec: CudaExecutor, nrows: int, ncols: int, rows, cols, vals,
                  dtype=torch.float64) -> CooMatrix:
    dev = exec.device
    return CooMatrix(nrows, ncols,
                     torch.from_numpy(np.ascontiguousarray(rows, np.int32)).to(dev),
                     torch.from_numpy(np.ascontiguousarray(cols, np.int32)).to(dev),
                     torch.from_numpy(np.ascontiguousarray(vals)).to(dev).to(dtype), exec)


def coo_from_entries(exec: CudaExecutor, nrows: int, ncols: int, entries) -> CooMatrix:
    """formats.cpp:78-116 on the device: bounds check (FormatError), stable
    (row, col) sort, duplicates summed in input order, zeros kept.
    `entries` is a sequence of (row, col, value) or a (rows, cols, vals)
    triple of arrays."""
    if isinstance(entries, tuple) and len(entries) == 3 and hasattr(entries[0], "__len__") \
            and not isinstance(entries[0], (int, np.integer)):
        rows, cols, vals = (np.asarray(a) for a in entries)
    else:
        ent = list(entries)
        rows = np.array([e[0] for e in ent], np.int32)
        cols = np.array([e[1] for e in ent], np.int32)
        vals = np.array([e[2] for e in ent], np.float64)
    n = len(vals)
    dev = exec.device
    r_in = torch.from_numpy(np.ascontiguousarray(rows, np.int32)).to(dev)
    c_in = torch.from_numpy(np.ascontiguousarray(cols, np.int32)).to(dev)
    v_in = torch.from_numpy(np.ascontiguousarray(vals, np.float64)).to(dev)
    r_out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    c_out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    v_out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    nnz = C.c_int64()
    _check(L.load().lbk_coo_assemble_f64(exec.ctx, nrows, ncols, n, _ptr(r_in), _ptr(c_in),
                                         _ptr(v_in), _ptr(r_out), _ptr(c_out), _ptr(v_out),
                                         C.byref(nnz)), exec.ctx)
    k = nnz.value
    return CooMatrix(nrows, ncols, r_out[:k].clone(), c_out[:k].clone(), v_out[:k].clone(), exec)


def read_matrix_market_entries(path: str):
    """Host parse of a MatrixMarket coordinate file (reference io.cpp:71-191
    acceptance rules): (nrows, ncols, rows, cols, vals) before assembly."""
    lib = L.load()
    h = C.c_void_p()
    st = lib.lbk_mm_read(str(path).encode(), C.byref(h))
    if st != L.OK:
        msg = lib.lbk_mm_last_error().decode(errors="replace")
        raise _STATUS.get(st, Error)(msg)
    try:
        nr, nc, ne = C.c_int32(), C.c_int32(), C.c_int64()
        lib.lbk_mm_info(h, C.byref(nr), C.byref(nc), C.byref(ne))
        pr, pc, pv = C.c_void_p(), C.c_void_p(), C.c_void_p()
        lib.lbk_mm_entries(h, C.byref(pr), C.byref(pc), C.byref(pv))
        n = ne.value
        rows = np.ctypeslib.as_array((C.c_int32 * n).from_address(pr.value)).copy() if n else \
            np.zeros(0, np.int32)
        cols = np.ctypeslib.as_array((C.c_int32 * n).from_address(pc.value)).copy() if n else \
            np.zeros(0, np.int32)
        vals = np.ctypeslib.as_array((C.c_double * n).from_address(pv.value)).copy() if n else \
            np.zeros(0, np.float64)
        return nr.value, nc.value, rows, cols, vals
    finally:
        lib.lbk_mm_free(h)


def read_matrix_market(exec: CudaExecutor, path: str) -> CooMatrix:
    """io.hpp:25-28 read_matrix_market: host parse + device assembly
    (sort, duplicate sum) into canonical COO."""
    nr, nc, rows, cols, vals = read_matrix_market_entries(path)
    return coo_from_entries(exec, nr, nc, (rows, cols, vals))


def coo_to_entries(m: CooMatrix):
    return list(zip(m.row_idx.cpu().tolist(), m.col_idx.cpu().tolist(), m.vals.cpu().tolist()))


def coo_to_csr(m: CooMatrix) -> CsrMatrix:
    """formats.cpp:132-155: histogram + scan; col/vals carried verbatim."""
    rp = torch.empty(m.nrows + 1, dtype=torch.int32, device=m.exec.device)
    _check(L.load().lbk_coo_to_csr(m.exec.ctx, C.byref(m.desc(False)), _ptr(rp)), m.exec.ctx)
    return CsrMatrix(m.nrows, m.ncols, rp, m.col_idx.clone(), m.vals.clone(), m.exec)


def csr_to_coo(m: CsrMatrix) -> CooMatrix:
    """formats.cpp:158-179."""
    ri = torch.empty(m.nnz(), dtype=torch.int32, device=m.exec.device)
    _check(L.load().lbk_csr_to_coo(m.exec.ctx, C.byref(m.desc(False)), _ptr(ri)), m.exec.ctx)
    return CooMatrix(m.nrows, m.ncols, ri, m.col_idx.clone(), m.vals.clone(), m.exec)


def csr_to_ell(m: CsrMatrix, width: Optional[int] = None, stride: Optional[int] = None) -> EllMatrix:
    lib = L.load()
    d = m.desc(False)
    if width is None:
        w = C.c_int32()
        _check(lib.lbk_csr_ell_width(m.exec.ctx, C.byref(d), C.byref(w)), m.exec.ctx)
        width = w.value
    stride = m.nrows if stride is None else stride
    cols = torch.empty(max(width * stride, 1), dtype=torch.int32, device=m.exec.device)
    vals = torch.empty(max(width * stride, 1), dtype=m.vals.dtype, device=m.exec.device)
    _check(lib.lbk_csr_to_ell(m.exec.ctx, C.byref(d), width, stride, _ptr(cols), _ptr(vals)), m.exec.ctx)
    return EllMatrix(m.nrows, m.ncols, width, stride, cols, vals, m.nnz(), m.exec)


def csr_to_sellp(m: CsrMatrix, slice_size: int = 32) -> SellpMatrix:
    lib = L.load()
    d = m.desc(False)
    ns = (m.nrows + slice_size - 1) // slice_size
    sl = torch.empty(max(ns, 1), dtype=torch.int32, device=m.exec.device)
    ss = torch.empty(ns + 1, dtype=torch.int32, device=m.exec.device)
    stored = C.c_int64()
    _check(lib.lbk_csr_sellp_plan(m.exec.ctx, C.byref(d), slice_size, _ptr(sl), _ptr(ss),
                                  C.byref(stored)), m.exec.ctx)
    cols = torch.empty(max(stored.value, 1), dtype=torch.int32, device=m.exec.device)
    vals = torch.empty(max(stored.value, 1), dtype=m.vals.dtype, device=m.exec.device)
    _check(lib.lbk_csr_to_sellp(m.exec.ctx, C.byref(d), slice_size, _ptr(ss), _ptr(cols),
                                _ptr(vals)), m.exec.ctx)
    return SellpMatrix(m.nrows, m.ncols, slice_size, sl[:ns], ss, cols, vals, m.nnz(), m.exec,
                       stored.value)


def validate(m) -> None:
    """formats.cpp:182-242 -> FormatError."""
    lib = L.load()
    if isinstance(m, CsrMatrix):
        if m.row_ptr.numel() != m.nrows + 1 or m.col_idx.numel() != m.nnz():
            raise FormatError("csr arrays have inconsistent lengths")
        _check(lib.lbk_validate_csr(m.exec.ctx, C.byref(m.desc(False))), m.exec.ctx)
    elif isinstance(m, CooMatrix):
        if m.row_idx.numel() != m.nnz() or m.col_idx.numel() != m.nnz():
            raise FormatError("coo arrays have inconsistent lengths")
        _check(lib.lbk_validate_coo(m.exec.ctx, C.byref(m.desc(False))), m.exec.ctx)
    else:
        raise UsageError("validate: CsrMatrix or CooMatrix expected")


# ------------------------------------------------------------------ BLAS-1
def _same_size(a: int, b: int, what: str) -> None:
    if a != b:
        raise ShapeError(f"{what}: size mismatch, {a} vs {b}")


def _same_space(a: DenseVector, b, what: str) -> None:
    if a.exec is not b.exec:
        raise PlacementError(f"{what}: operands live on different executors")


def _f64(v: DenseVector, what: str) -> None:
    if v.values.dtype != torch.float64:
        raise TypeError_(f"{what}: float64 vectors expected")


def axpy(alpha: float, x: DenseVector, y: DenseVector) -> None:
    """y <- alpha x + y (kernels.hpp:80, api.cpp:69-76)."""
    _same_size(x.size(), y.size(), "axpy")
    _same_space(x, y, "axpy")
    _f64(x, "axpy")
    _f64(y, "axpy")
    _check(L.load().lbk_axpy_f64(y.exec.ctx, y.size(), float(alpha), _ptr(x.values), _ptr(y.values)), y.exec.ctx)
    y.exec.synchronize()


def scal(alpha: float, x: DenseVector) -> None:
    _f64(x, "scal")
    _check(L.load().lbk_scal_f64(x.exec.ctx, x.size(), float(alpha), _ptr(x.values)), x.exec.ctx)
    x.exec.synchronize()


def fill(x: DenseVector, value: float) -> None:
    _f64(x, "fill")
    _check(L.load().lbk_fill_f64(x.exec.ctx, x.size(), float(value), _ptr(x.values)), x.exec.ctx)
    x.exec.synchronize()


def dot(x: DenseVector, y: DenseVector) -> float:
    _same_size(x.size(), y.size(), "dot")
    _same_space(x, y, "dot")
    _f64(x, "dot")
    _f64(y, "dot")
    out = C.c_double()
    _check(L.load().lbk_dot_f64(x.exec.ctx, x.size(), _ptr(x.values), _ptr(y.values), C.byref(out)), x.exec.ctx)
    return out.value


def nrm2(x: DenseVector) -> float:
    _f64(x, "nrm2")
    out = C.c_double()
    _check(L.load().lbk_nrm2_f64(x.exec.ctx, x.size(), _ptr(x.values), C.byref(out)), x.exec.ctx)
    return out.value


# ---------------------------------------------- stream set / flops sweep
STREAM_OPS = ("copy", "mul", "add", "triad", "dot")


def stream_bytes(op: str, n: int) -> int:
    """Bytes touched by one stream op over n doubles (api.cpp:170-182)."""
    return (3 if op in ("add", "triad") else 2) * n * 8


def stream_kernel(op: str, a: DenseVector, b: DenseVector, c: DenseVector,
                  scalar: float) -> float:
    """kernels.hpp:99-103: copy c<-a, mul b<-scalar*c, add c<-a+b, triad
    a<-b+scalar*c; returns the dot product for 'dot' and 0 otherwise."""
    if op not in STREAM_OPS:
        raise UsageError(f"unknown stream op '{op}'")
    _same_size(a.size(), b.size(), "stream_kernel")
    _same_size(a.size(), c.size(), "stream_kernel")
    lib, ctx, n = L.load(), a.exec.ctx, a.size()
    pa, pb, pc = _ptr(a.values), _ptr(b.values), _ptr(c.values)
    out = C.c_double(0.0)
    if op == "copy":
        st = lib.lbk_stream_copy_f64(ctx, n, pa, pc)
    elif op == "mul":
        st = lib.lbk_stream_mul_f64(ctx, n, float(scalar), pc, pb)
    elif op == "add":
        st = lib.lbk_stream_add_f64(ctx, n, pa, pb, pc)
    elif op == "triad":
        st = lib.lbk_stream_triad_f64(ctx, n, float(scalar), pb, pc, pa)
    else:
        st = lib.lbk_stream_dot_f64(ctx, n, pa, pb, C.byref(out))
    _check(st, ctx)
    a.exec.synchronize()
    return out.value


def flops_sweep(x: DenseVector, fma_per_element: int) -> None:
    """kernels.hpp:105-109: x_i <- fma_chain(x_i, fma_per_element)."""
    if fma_per_element < 0:
        raise UsageError("fma count must be nonnegative")
    _check(L.load().lbk_flops_sweep_f64(x.exec.ctx, x.size(), int(fma_per_element), _ptr(x.values)),
           x.exec.ctx)
    x.exec.synchronize()


# -------------------------------------------------------------------- SpMV
_SPMV = {
    (CsrMatrix, torch.float64): ("lbk_spmv_csr_f64", "lbk_spmv_csr_adv_f64"),
    (CsrMatrix, torch.float32): ("lbk_spmv_csr_f32", "lbk_spmv_csr_adv_f32"),
    (CooMatrix, torch.float64): ("lbk_spmv_coo_f64", "lbk_spmv_coo_adv_f64"),
    (CooMatrix, torch.float32): ("lbk_spmv_coo_f32", "lbk_spmv_coo_adv_f32"),
    (EllMatrix, torch.float64): ("lbk_spmv_ell_f64", "lbk_spmv_ell_adv_f64"),
    (EllMatrix, torch.float32): ("lbk_spmv_ell_f32", "lbk_spmv_ell_adv_f32"),
    (SellpMatrix, torch.float64): ("lbk_spmv_sellp_f64", "lbk_spmv_sellp_adv_f64"),
    (SellpMatrix, torch.float32): ("lbk_spmv_sellp_f32", "lbk_spmv_sellp_adv_f32"),
}


def spmv(matrix, x: DenseVector, y: DenseVector, alpha: Optional[float] = None,
         beta: Optional[float] = None, sync: bool = True) -> None:
    """y <- A x (api.cpp:113-140 checks), or y <- alpha A x + beta y."""
    name = type(matrix).__name__
    _same_size(matrix.ncols, x.size(), f"spmv_{name} columns vs x")
    _same_size(matrix.nrows, y.size(), f"spmv_{name} rows vs y")
    _same_space(x, matrix, f"spmv_{name}")
    _same_space(y, matrix, f"spmv_{name}")
    key = (type(matrix), x.values.dtype)
    if key not in _SPMV or x.values.dtype != y.values.dtype:
        raise TypeError_(f"spmv: unsupported combination {name} / {x.values.dtype}")
    plain, adv = _SPMV[key]
    lib = L.load()
    d = matrix.desc()
    ctx = matrix.exec.ctx
    if alpha is None and beta is None:
        st = getattr(lib, plain)(ctx, C.byref(d), _ptr(x.values), _ptr(y.values))
    else:
        if adv is None:
            raise TypeError_(f"advanced apply not available for {name} / {x.values.dtype}")
        a = 1.0 if alpha is None else alpha
        b = 0.0 if beta is None else beta
        st = getattr(lib, adv)(ctx, a, C.byref(d), _ptr(x.values), b, _ptr(y.values))
    _check(st, ctx)
    if sync:
        matrix.exec.synchronize()


def spmv_csr(matrix: CsrMatrix, x: DenseVector, y: DenseVector) -> None:
    if not isinstance(matrix, CsrMatrix):
        raise UsageError("spmv_csr: CsrMatrix expected")
    spmv(matrix, x, y)


def spmv_coo(matrix: CooMatrix, x: DenseVector, y: DenseVector) -> None:
    if not isinstance(matrix, CooMatrix):
        raise UsageError("spmv_coo: CooMatrix expected")
    spmv(matrix, x, y)


def spmv_ell(matrix: EllMatrix, x: DenseVector, y: DenseVector) -> None:
    spmv(matrix, x, y)


def spmv_sellp(matrix: SellpMatrix, x: DenseVector, y: DenseVector) -> None:
    spmv(matrix, x, y)


def apply_operator(matrix, v: DenseVector) -> DenseVector:
    """krylov.cpp:601-616: y = A v into a fresh vector."""
    out = make_vector(matrix.exec, matrix.nrows, v.values.dtype)
    spmv(matrix, v, out)
    return out


# ----------------------------------------------------------------- solvers
SOLVER_KINDS = {"cg": 0, "bicgstab": 1, "cgs": 2, "gmres": 3}


@dataclass
class SolverConfig:
    """krylov.hpp:22-31 (+ residual_mode, the B200 addition)."""
    kind: str = "cg"
    max_iters: int = 1000
    rel_tol: float = 1e-10
    gmres_restart: int = 30
    fixed_iters: Optional[int] = None
    residual_mode: str = "true"  # "true" (reference) | "recurrence"


@dataclass
class SolveResult:
    """krylov.hpp:34-44."""
    converged: bool = False
    iterations: int = 0
    final_rel_residual: float = 0.0
    residual_history: list = field(default_factory=list)
    elapsed: float = 0.0
    flop_count: int = 0


@dataclass
class GmresCycleResult:
    """krylov.hpp:62-66."""
    rel_residual: float
    steps: int
    happy_breakdown: bool


def gmres_restart_cycle(matrix: "CsrMatrix", b: DenseVector, x: DenseVector, restart: int,
                        basis_out: Optional[list] = None) -> GmresCycleResult:
    """krylov.hpp:68-89: one restarted-GMRES cycle (modified Gram-Schmidt
    basis of dimension <= restart, Givens least squares, x updated); a
    subdiagonal below 1e-14 ends it early with the happy flag.  basis_out,
    when given, receives the cycle's orthonormal basis vectors."""
    if not isinstance(matrix, CsrMatrix):
        raise DispatchError("gmres_restart_cycle: CSR matrices only")
    if restart < 1:
        raise ConfigurationError("restart must be positive")
    _same_size(matrix.nrows, b.size(), "gmres_restart_cycle")
    _same_size(matrix.nrows, x.size(), "gmres_restart_cycle")
    ex = matrix.exec
    basis = ex.empty((restart + 1) * matrix.nrows, torch.float64) if basis_out is not None else None
    d = matrix.desc()
    r = L.lbk_gmres_cycle_result()
    _check(L.load().lbk_gmres_restart_cycle_csr(ex.ctx, C.byref(d), _ptr(b.values), _ptr(x.values),
                                                int(restart), _ptr(basis),
                                                restart + 1 if basis is not None else 0,
                                                C.byref(r)), ex.ctx)
    if basis_out is not None:
        basis_out.clear()
        for i in range(r.basis_count):
            basis_out.append(DenseVector(basis[i * matrix.nrows:(i + 1) * matrix.nrows].clone(), ex))
    return GmresCycleResult(r.rel_residual, r.steps, bool(r.happy_breakdown))


def solve(matrix, b: DenseVector, x: DenseVector, config: SolverConfig) -> SolveResult:
    """krylov.hpp:53-56 solve(A, b, x, cfg): x in/out, device-resident."""
    if isinstance(matrix, (CsrMatrix, CooMatrix)) and matrix.nrows != matrix.ncols:
        raise ShapeError(f"solve requires a square matrix, got {matrix.nrows}x{matrix.ncols}")
    if b.size() != matrix.nrows or x.size() != matrix.nrows:
        raise ShapeError("solve: operand sizes do not match the matrix")
    if b.exec is not matrix.exec or x.exec is not matrix.exec:
        raise PlacementError("solve: operands on a different executor than the matrix")
    if config.kind not in SOLVER_KINDS:
        raise ConfigurationError(f"solver kind {config.kind!r} not provided by the B200 backend")
    if config.fixed_iters is not None and config.fixed_iters < 1:
        raise ConfigurationError("fixed_iters must be positive")
    _f64(b, "solve")
    _f64(x, "solve")
    cfg = L.lbk_solver_cfg(SOLVER_KINDS[config.kind], int(config.max_iters), float(config.rel_tol),
                           int(config.fixed_iters or 0),
                           1 if config.residual_mode == "recurrence" else 0,
                           int(config.gmres_restart))
    res = L.lbk_solve_result()
    cap = int(config.fixed_iters or config.max_iters) + 2
    hist = np.empty(cap, np.float64)
    lib = L.load()
    ctx = matrix.exec.ctx
    if isinstance(matrix, CsrMatrix):
        st = lib.lbk_solve_csr(ctx, C.byref(matrix.desc()), _ptr(b.values), _ptr(x.values),
                               C.byref(cfg), C.byref(res), hist.ctypes.data_as(C.c_void_p), cap)
    elif isinstance(matrix, CooMatrix):
        st = lib.lbk_solve_coo(ctx, C.byref(matrix.desc()), _ptr(b.values), _ptr(x.values),
                               C.byref(cfg), C.byref(res), hist.ctypes.data_as(C.c_void_p), cap)
    else:
        raise UsageError("solve: CsrMatrix or CooMatrix expected")
    _check(st, ctx, res.breakdown_iter)
    return SolveResult(bool(res.converged), int(res.iterations), float(res.final_rel_residual),
                       hist[: res.history_len].tolist(), float(res.elapsed), int(res.flop_count))
