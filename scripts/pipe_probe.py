"""Dev tool: does the three-stream e2e pipeline overlap H2D / SpMV / D2H?"""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_08879_b200 import _lib as L, gen, larch as lk  # noqa: E402

lib = L.load()
ex = lk.CudaExecutor(0)
A = gen.stencil(ex, "27pt", 128)
n = A.nrows
desc = A.desc()
xh = torch.from_numpy(gen.seeded_values(n)).pin_memory()
yh = torch.empty(n, dtype=torch.float64).pin_memory()
s_in, s_out, s_mv = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
e_in, e_out, e_mv = (lk.CudaExecutor(0, stream=s) for s in (s_in, s_out, s_mv))
xb = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
yb = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
K = 30


def pipe(use_lbk_copies, use_spmv=True, lbk_in=None, lbk_out=None):
    lbk_in = use_lbk_copies if lbk_in is None else lbk_in
    lbk_out = use_lbk_copies if lbk_out is None else lbk_out
    up = [torch.cuda.Event() for _ in range(K)]
    mv = [torch.cuda.Event() for _ in range(K)]
    dn = [torch.cuda.Event() for _ in range(K)]
    for i in range(K):
        j = i & 1
        if i >= 2:
            s_in.wait_event(mv[i - 2])
        if lbk_in:
            lib.lbk_memcpy_h2d(e_in.ctx, C.c_void_p(xb[j].data_ptr()), C.c_void_p(xh.data_ptr()), 8 * n)
        else:
            with torch.cuda.stream(s_in):
                xb[j].copy_(xh, non_blocking=True)
        up[i].record(s_in)
        s_mv.wait_event(up[i])
        if i >= 2:
            s_mv.wait_event(dn[i - 2])
        if use_spmv:
            lib.lbk_spmv_csr_f64(e_mv.ctx, C.byref(desc), C.c_void_p(xb[j].data_ptr()),
                                 C.c_void_p(yb[j].data_ptr()))
        mv[i].record(s_mv)
        s_out.wait_event(mv[i])
        if lbk_out == "raw":
            cudart.cudaMemcpyAsync(C.c_void_p(yh.data_ptr()), C.c_void_p(yb[j].data_ptr()),
                                   C.c_size_t(8 * n), 2, C.c_void_p(s_out.cuda_stream))
        elif lbk_out:
            lib.lbk_memcpy_d2h(e_out.ctx, C.c_void_p(yh.data_ptr()), C.c_void_p(yb[j].data_ptr()), 8 * n)
        else:
            with torch.cuda.stream(s_out):
                yh.copy_(yb[j], non_blocking=True)
        dn[i].record(s_out)


for lbkc in (False, True):
    for sp in (False, True):
        pipe(lbkc, sp)
        torch.cuda.synchronize()
        t0 = time.time()
        pipe(lbkc, sp)
        torch.cuda.synchronize()
        print(f"lbk copies={lbkc} spmv={sp}: {(time.time() - t0) / K * 1e3:.3f} ms/step")

import glob
cudart = C.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so.12"))[0])
cudart.cudaMemcpyAsync.restype = C.c_int
for li, lo in ((True, False), (False, True), (False, "raw")):
    pipe(False, False, li, lo)
    torch.cuda.synchronize()
    t0 = time.time()
    pipe(False, False, li, lo)
    torch.cuda.synchronize()
    print(f"lbk_in={li} lbk_out={lo}: {(time.time() - t0) / K * 1e3:.3f} ms/step")

# host-side duration of one async copy call
torch.cuda.synchronize()
t0 = time.time()
lib.lbk_memcpy_h2d(e_in.ctx, C.c_void_p(xb[0].data_ptr()), C.c_void_p(xh.data_ptr()), 8 * n)
t1 = time.time()
torch.cuda.synchronize()
t2 = time.time()
print(f"lbk_memcpy_h2d host call {1e3 * (t1 - t0):.3f} ms, to completion {1e3 * (t2 - t0):.3f} ms")
with torch.cuda.stream(s_in):
    t0 = time.time()
    xb[0].copy_(xh, non_blocking=True)
    t1 = time.time()
torch.cuda.synchronize()
print(f"torch copy_ host call {1e3 * (t1 - t0):.3f} ms")

def both_lbk():
    r1 = lib.lbk_memcpy_h2d(e_in.ctx, C.c_void_p(xb[0].data_ptr()), C.c_void_p(xh.data_ptr()), 8 * n)
    r2 = lib.lbk_memcpy_d2h(e_out.ctx, C.c_void_p(yh.data_ptr()), C.c_void_p(yb[1].data_ptr()), 8 * n)
    return r1, r2


def both_torch():
    with torch.cuda.stream(s_in):
        xb[0].copy_(xh, non_blocking=True)
    with torch.cuda.stream(s_out):
        yh.copy_(yb[1], non_blocking=True)


for name, fn in (("lbk", both_lbk), ("torch", both_torch)):
    fn()
    torch.cuda.synchronize()
    t0 = time.time()
    for _ in range(10):
        rr = fn()
    torch.cuda.synchronize()
    print(f"{name} H2D||D2H: {(time.time() - t0) / 10 * 1e3:.3f} ms  ret={rr}")
print("streams", hex(s_in.cuda_stream), hex(s_out.cuda_stream))
