"""ctypes binding of ``liblbk.so`` (the C ABI declared in ``include/lbk.h``).

This is the reference-side binding a Python maintainer would add (see
INTEGRATION.md); the C++ façade ``include/lbk/larch.hpp`` is the C++ one.
There is no fallback: if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# LBK_LIB overrides the path (A/B timing of build variants); default in-tree.
LIB_PATH = os.environ.get("LBK_LIB") or os.path.join(HERE, "liblbk.so")

# ----------------------------------------------------------------- status
OK = 0
SHAPE_ERROR = 1
PLACEMENT_ERROR = 2
TYPE_ERROR = 3
DISPATCH_ERROR = 4
USAGE_ERROR = 5
CONFIGURATION_ERROR = 6
OUT_OF_MEMORY = 7
FORMAT_ERROR = 8
BREAKDOWN = 9
BENCHMARK_INTEGRITY = 10
UNSUPPORTED_FORMAT = 11
CUDA_ERROR = 20
NCCL_ERROR = 21
INTERNAL = 99

F64 = 0
F32 = 1


class lbk_csr(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("dtype", C.c_int), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("vals", C.c_void_p), ("tile_rows", C.c_void_p), ("ntiles", C.c_int32)]


class lbk_coo(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("dtype", C.c_int), ("row_idx", C.c_void_p), ("col_idx", C.c_void_p),
                ("vals", C.c_void_p), ("tile_starts", C.c_void_p), ("ntiles", C.c_int32)]


class lbk_ell(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("dtype", C.c_int), ("width", C.c_int32), ("stride", C.c_int64),
                ("col_idx", C.c_void_p), ("vals", C.c_void_p)]


class lbk_sellp(C.Structure):
    _fields_ = [("nrows", C.c_int32), ("ncols", C.c_int32), ("nnz", C.c_int64),
                ("dtype", C.c_int), ("slice_size", C.c_int32), ("nslices", C.c_int32),
                ("slice_lengths", C.c_void_p), ("slice_sets", C.c_void_p),
                ("col_idx", C.c_void_p), ("vals", C.c_void_p), ("stored", C.c_int64),
                ("tile_slices", C.c_void_p), ("ntiles", C.c_int32)]


class lbk_dist_map_info_t(C.Structure):
    _fields_ = [("begin", C.c_int32), ("end", C.c_int32), ("n_local", C.c_int32),
                ("n_ghost", C.c_int32), ("n_interior", C.c_int32), ("n_boundary", C.c_int32),
                ("nnz_local", C.c_int64), ("n_send", C.c_int32)]


class lbk_solver_cfg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("max_iters", C.c_int32), ("rel_tol", C.c_double),
                ("fixed_iters", C.c_int32), ("residual_mode", C.c_int32),
                ("gmres_restart", C.c_int32)]


class lbk_gmres_cycle_result(C.Structure):
    _fields_ = [("rel_residual", C.c_double), ("steps", C.c_int32),
                ("happy_breakdown", C.c_int32), ("basis_count", C.c_int32)]


class lbk_solve_result(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32),
                ("final_rel_residual", C.c_double), ("elapsed", C.c_double),
                ("flop_count", C.c_int64), ("breakdown_iter", C.c_int32),
                ("history_len", C.c_int32)]


vp = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
f64 = C.c_double
f32 = C.c_float
st = C.c_int
P = C.POINTER

SIGNATURES = {
    "lbk_ctx_create": (st, [C.c_int, P(vp)]),
    "lbk_ctx_create_on_stream": (st, [C.c_int, vp, P(vp)]),
    "lbk_ctx_set_stream": (st, [vp, vp]),
    "lbk_ctx_destroy": (st, [vp]),
    "lbk_last_error": (C.c_char_p, [vp]),
    "lbk_sync": (st, [vp]),
    "lbk_ctx_info": (st, [vp, P(C.c_int), P(C.c_int), P(C.c_size_t), P(C.c_size_t)]),
    "lbk_ctx_set_arena_capacity": (st, [vp, C.c_size_t]),
    "lbk_ctx_set_l2_persist": (st, [vp, C.c_int]),
    "lbk_alloc": (st, [vp, C.c_size_t, P(vp)]),
    "lbk_free": (st, [vp, vp, C.c_size_t]),
    "lbk_memcpy_h2d": (st, [vp, vp, vp, C.c_size_t]),
    "lbk_memcpy_d2h": (st, [vp, vp, vp, C.c_size_t]),
    "lbk_memcpy_d2d": (st, [vp, vp, vp, C.c_size_t]),
    "lbk_memcpy_peer": (st, [vp, vp, C.c_int, vp, C.c_int, C.c_size_t]),
    "lbk_spmv_csr_f64": (st, [vp, P(lbk_csr), vp, vp]),
    "lbk_spmv_csr_f32": (st, [vp, P(lbk_csr), vp, vp]),
    "lbk_spmv_csr_adv_f64": (st, [vp, f64, P(lbk_csr), vp, f64, vp]),
    "lbk_spmv_csr_adv_f32": (st, [vp, f32, P(lbk_csr), vp, f32, vp]),
    "lbk_spmv_coo_f64": (st, [vp, P(lbk_coo), vp, vp]),
    "lbk_spmv_coo_f32": (st, [vp, P(lbk_coo), vp, vp]),
    "lbk_spmv_coo_adv_f64": (st, [vp, f64, P(lbk_coo), vp, f64, vp]),
    "lbk_spmv_coo_adv_f32": (st, [vp, f32, P(lbk_coo), vp, f32, vp]),
    "lbk_spmv_ell_f64": (st, [vp, P(lbk_ell), vp, vp]),
    "lbk_spmv_ell_f32": (st, [vp, P(lbk_ell), vp, vp]),
    "lbk_spmv_ell_adv_f64": (st, [vp, f64, P(lbk_ell), vp, f64, vp]),
    "lbk_spmv_ell_adv_f32": (st, [vp, f32, P(lbk_ell), vp, f32, vp]),
    "lbk_spmv_sellp_f64": (st, [vp, P(lbk_sellp), vp, vp]),
    "lbk_spmv_sellp_f32": (st, [vp, P(lbk_sellp), vp, vp]),
    "lbk_spmv_sellp_adv_f64": (st, [vp, f64, P(lbk_sellp), vp, f64, vp]),
    "lbk_spmv_sellp_adv_f32": (st, [vp, f32, P(lbk_sellp), vp, f32, vp]),
    "lbk_csr_plan_size": (st, [P(lbk_csr), P(i32)]),
    "lbk_csr_plan": (st, [vp, P(lbk_csr), vp]),
    "lbk_coo_plan_size": (st, [P(lbk_coo), P(i32)]),
    "lbk_sellp_plan_size": (st, [P(lbk_sellp), P(i32)]),
    "lbk_sellp_plan": (st, [vp, P(lbk_sellp), vp]),
    "lbk_coo_plan": (st, [vp, P(lbk_coo), vp]),
    "lbk_axpy_f64": (st, [vp, i64, f64, vp, vp]),
    "lbk_scal_f64": (st, [vp, i64, f64, vp]),
    "lbk_fill_f64": (st, [vp, i64, f64, vp]),
    "lbk_copy_f64": (st, [vp, i64, vp, vp]),
    "lbk_dot_f64": (st, [vp, i64, vp, vp, P(f64)]),
    "lbk_nrm2_f64": (st, [vp, i64, vp, P(f64)]),
    "lbk_dot_f64_dev": (st, [vp, i64, vp, vp, vp]),
    "lbk_stream_copy_f64": (st, [vp, i64, vp, vp]),
    "lbk_stream_triad_f64": (st, [vp, i64, f64, vp, vp, vp]),
    "lbk_stream_mul_f64": (st, [vp, i64, f64, vp, vp]),
    "lbk_stream_add_f64": (st, [vp, i64, vp, vp, vp]),
    "lbk_stream_dot_f64": (st, [vp, i64, vp, vp, P(f64)]),
    "lbk_flops_sweep_f64": (st, [vp, i64, i32, vp]),
    "lbk_coo_to_csr": (st, [vp, P(lbk_coo), vp]),
    "lbk_csr_to_coo": (st, [vp, P(lbk_csr), vp]),
    "lbk_coo_assemble_f64": (st, [vp, i32, i32, i64, vp, vp, vp, vp, vp, vp, P(i64)]),
    "lbk_csr_ell_width": (st, [vp, P(lbk_csr), P(i32)]),
    "lbk_csr_to_ell": (st, [vp, P(lbk_csr), i32, i64, vp, vp]),
    "lbk_csr_sellp_plan": (st, [vp, P(lbk_csr), i32, vp, vp, P(i64)]),
    "lbk_csr_to_sellp": (st, [vp, P(lbk_csr), i32, vp, vp, vp]),
    "lbk_validate_csr": (st, [vp, P(lbk_csr)]),
    "lbk_validate_coo": (st, [vp, P(lbk_coo)]),
    "lbk_solve_csr": (st, [vp, P(lbk_csr), vp, vp, P(lbk_solver_cfg), P(lbk_solve_result), vp, i32]),
    "lbk_solve_coo": (st, [vp, P(lbk_coo), vp, vp, P(lbk_solver_cfg), P(lbk_solve_result), vp, i32]),
    "lbk_gmres_restart_cycle_csr": (st, [vp, P(lbk_csr), vp, vp, i32, vp, i32,
                                         P(lbk_gmres_cycle_result)]),
    "lbk_part_range": (st, [i32, i32, i32, P(i32), P(i32)]),
    "lbk_dist_map_create": (st, [i32, i32, i32, i32, i32, vp, vp, P(vp)]),
    "lbk_dist_map_info": (st, [vp, P(lbk_dist_map_info_t)]),
    "lbk_dist_map_ghosts": (st, [vp, vp, vp]),
    "lbk_dist_map_local_cols": (st, [vp, vp]),
    "lbk_dist_map_rows": (st, [vp, vp, vp]),
    "lbk_dist_map_set_sends": (st, [vp, vp, vp]),
    "lbk_dist_map_sends": (st, [vp, vp, vp]),
    "lbk_dist_map_destroy": (st, [vp]),
    "lbk_comm_nccl_unique_id": (st, [vp]),
    "lbk_comm_init_nccl": (st, [vp, i32, i32, i32, P(vp)]),
    "lbk_comm_init_threads": (st, [i32, vp]),
    "lbk_comm_init_peer": (st, [i32, i32, i32, i64, P(vp)]),
    "lbk_comm_peer_handle": (st, [vp, vp]),
    "lbk_comm_peer_open": (st, [vp, vp]),
    "lbk_comm_init_peer_group": (st, [i32, vp, i64, vp]),
    "lbk_comm_sync": (st, [vp, vp]),
    "lbk_comm_destroy": (st, [vp]),
    "lbk_comm_allreduce_sum_f64": (st, [vp, vp, vp, i32]),
    "lbk_dist_csr_create": (st, [vp, vp, vp, vp, i64, P(vp)]),
    "lbk_dist_csr_info": (st, [vp, P(i32), P(i32)]),
    "lbk_dist_csr_destroy": (st, [vp]),
    "lbk_dist_spmv_f64": (st, [vp, vp, vp, vp, vp]),
    "lbk_dist_solve": (st, [vp, vp, vp, vp, vp, P(lbk_solver_cfg), P(lbk_solve_result), vp, i32]),
    "lbk_mm_read": (st, [C.c_char_p, P(vp)]),
    "lbk_mm_last_error": (C.c_char_p, []),
    "lbk_mm_info": (st, [vp, P(i32), P(i32), P(i64)]),
    "lbk_mm_entries": (st, [vp, P(vp), P(vp), P(vp)]),
    "lbk_mm_free": (st, [vp]),
    "lbk_gen_stencil_nnz": (i64, [C.c_int, C.c_int]),
    "lbk_gen_stencil_csr": (st, [vp, C.c_int, C.c_int, f64, vp, vp, vp]),
    "lbk_gen_seeded_values": (None, [i64, C.c_uint64, vp]),
    "lbk_gen_powerlaw": (vp, [i32, C.c_uint64, i32, i32, P(i64)]),
    "lbk_gen_powerlaw_fill": (None, [vp, vp, vp, vp]),
    "lbk_gen_powerlaw_free": (None, [vp]),
}

_lib = None


def load() -> C.CDLL:
    """Load liblbk.so and bind every signature.  Raises if it is absent:
    there is deliberately no CPU path behind this API."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
