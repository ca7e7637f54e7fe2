"""CPU: the C-ABI library loads and exports every entry point include/lbk.h
declares (no compute calls without a GPU), and the Python mirror fails
loudly (no CPU fallback) when there is no device."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lbk.h")
LIB = os.path.join(ROOT, "paper_2011_08879_b200", "liblbk.so")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(lbk_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_header_declares_the_path():
    names = declared()
    for must in ["lbk_spmv_csr_f64", "lbk_spmv_coo_f64", "lbk_spmv_ell_f64", "lbk_spmv_sellp_f64",
                 "lbk_spmv_csr_f32", "lbk_coo_to_csr", "lbk_csr_to_coo", "lbk_coo_assemble_f64",
                 "lbk_csr_to_ell", "lbk_csr_to_sellp", "lbk_solve_csr", "lbk_solve_coo",
                 "lbk_dot_f64", "lbk_axpy_f64"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    assert os.path.exists(LIB), "liblbk.so not built (run __graft_entry__.build())"
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2011_08879_b200 import _lib
    bound = set(_lib.exported_symbols())
    assert set(declared()) <= bound | {"lbk_last_error"}, sorted(set(declared()) - bound)


def test_status_codes_match_header():
    from paper_2011_08879_b200 import _lib as L
    src = open(HEADER).read()
    codes = dict((k, int(v)) for k, v in re.findall(r"LBK_([A-Z_]+)\s*=\s*(\d+)", src))
    assert codes["OK"] == L.OK and codes["SHAPE_ERROR"] == L.SHAPE_ERROR
    assert codes["BREAKDOWN"] == L.BREAKDOWN and codes["FORMAT_ERROR"] == L.FORMAT_ERROR
    assert codes["OUT_OF_MEMORY"] == L.OUT_OF_MEMORY


def test_cpu_calls_fail_loudly_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2011_08879_b200 import larch as lk
    with pytest.raises(lk.DispatchError):
        lk.CudaExecutor(0)
    with pytest.raises(lk.ConfigurationError):
        lk.create_executor("reference")


def test_context_create_reports_cuda_error_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2011_08879_b200 import _lib as L
    lib = L.load()
    ctx = ctypes.c_void_p()
    st = lib.lbk_ctx_create(0, ctypes.byref(ctx))
    assert st == L.CUDA_ERROR
    assert b"" != lib.lbk_last_error(None)


def test_peer_communicator_fails_loudly_without_device():
    """The peer-memory communicator allocates its window on the device:
    without one it reports a CUDA error (no host fallback); bad arguments
    are usage errors before any device call."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2011_08879_b200 import _lib as L
    lib = L.load()
    h = ctypes.c_void_p()
    assert lib.lbk_comm_init_peer(2, 0, 0, 1024, ctypes.byref(h)) == L.CUDA_ERROR
    assert lib.lbk_comm_init_peer(17, 0, 0, 1024, ctypes.byref(h)) == L.USAGE_ERROR
    assert lib.lbk_comm_init_peer(2, 2, 0, 1024, ctypes.byref(h)) == L.USAGE_ERROR
    assert lib.lbk_comm_peer_handle(None, None) == L.USAGE_ERROR
    devs = (ctypes.c_int32 * 2)(0, 0)
    arr = (ctypes.c_void_p * 2)()
    assert lib.lbk_comm_init_peer_group(2, devs, 1024, arr) == L.USAGE_ERROR  # shared device


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2011_08879_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "larch_ref" not in txt, f
