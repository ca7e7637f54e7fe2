"""Synthetic inputs of the benchmark configurations.

cfg1  2D 5-pt Poisson 1024^2              stencil("5pt", 1024)
cfg2  3D 27-pt 128^3                       stencil("27pt", 128)
cfg3  power-law 2^24 rows, mean ~16        powerlaw(1 << 24)
cfg4  3D 7-pt Poisson 256^3, b = A*1       stencil("7pt", 256)
cfg5  3D 7-pt upwind, gamma 0.5, b = A*x*  stencil("7pt", 256, 0.5)
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from .larch import CsrMatrix, CudaExecutor, _check, _ptr

KINDS = {"5pt": 0, "7pt": 1, "27pt": 2}

CONFIGS = {
    "cfg1": dict(kind="5pt", m=1024, gamma=0.0),
    "cfg2": dict(kind="27pt", m=128, gamma=0.0),
    "cfg4": dict(kind="7pt", m=256, gamma=0.0),
    "cfg5": dict(kind="7pt", m=256, gamma=0.5),
}


def stencil(exec: CudaExecutor, kind: str, m: int, gamma: float = 0.0) -> CsrMatrix:
    """Generates the stencil matrix directly in device memory."""
    lib = L.load()
    k = KINDS[kind]
    nnz = lib.lbk_gen_stencil_nnz(k, m)
    n = m * m if k == 0 else m * m * m
    dev = exec.device
    rp = torch.empty(n + 1, dtype=torch.int32, device=dev)
    ci = torch.empty(nnz, dtype=torch.int32, device=dev)
    va = torch.empty(nnz, dtype=torch.float64, device=dev)
    _check(lib.lbk_gen_stencil_csr(exec.ctx, k, m, float(gamma), _ptr(rp), _ptr(ci), _ptr(va)),
           exec.ctx)
    return CsrMatrix(n, n, rp, ci, va, exec)


def seeded_values(n: int, seed: int = 11) -> np.ndarray:
    """harness.cpp:90-99 seeded_values (mt19937_64, U(-1,1)), on the host."""
    out = np.empty(n, np.float64)
    L.load().lbk_gen_seeded_values(n, seed, out.ctypes.data_as(C.c_void_p))
    return out


def powerlaw_host(n: int = 1 << 24, seed: int = 42, max_len: int = 10000, window: int = 65536):
    """App. B power-law matrix as host CSR arrays (row_ptr, cols, vals)."""
    lib = L.load()
    nnz = C.c_int64()
    h = lib.lbk_gen_powerlaw(n, seed, max_len, window, C.byref(nnz))
    rp = np.empty(n + 1, np.int32)
    ci = np.empty(nnz.value, np.int32)
    va = np.empty(nnz.value, np.float64)
    lib.lbk_gen_powerlaw_fill(h, rp.ctypes.data_as(C.c_void_p), ci.ctypes.data_as(C.c_void_p),
                              va.ctypes.data_as(C.c_void_p))
    lib.lbk_gen_powerlaw_free(h)
    return rp, ci, va
