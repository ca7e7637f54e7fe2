// integration/lbk_backend.cpp -- the reference-side binding of lbk.
//
// A file a maintainer adds to the reference tree (src/kernels/) to run its
// SpMV / BLAS-1 / Krylov hot path on the B200 through lbk's C ABI
// (include/lbk.h).  It is written against the reference's own headers and
// compiled against them by tests/test_integration.py (CPU, every round),
// with one seam patched in a scratch copy of executor.hpp:
//     enum class ExecutorKind { reference, parallel, sim_device, cuda };
// (executor.hpp:26; is_host_kind() already returns true for it, so the
// registry runs these entry points eagerly, dispatch.cpp:124-139).
//
// Seams:
//   KernelFn / KernelRegistry::register_host(name, kind, fn)  dispatch.hpp:23,33
//   argument blocks SpmvCsrArgs::matrix, DotArgs::result ...   kernels.hpp:24-56
//   DeviceArray::data()                                        device_array.hpp:80-81
//   solve(CsrMatrix, b, x, SolverConfig) -> SolveResult        krylov.hpp:53-56
//   the exception taxonomy                                     error.hpp:16-131
// The DeviceArrays of a `cuda` executor hold device (or managed) memory
// from lbk_alloc; the reference's wrappers are synchronous
// (dispatch.cpp:112-117), so every entry point ends in lbk_sync.
#include <lbk.h>

#include <any>
#include <cstdint>
#include <string>
#include <vector>

#include "larch/core/dispatch.hpp"
#include "larch/core/error.hpp"
#include "larch/kernels/kernels.hpp"
#include "larch/solver/krylov.hpp"

namespace larch {
namespace lbk_backend {
namespace {

lbk_ctx g_ctx = nullptr;  // one context: device 0, its own stream

// lbk_status -> the reference's exception classes (error.hpp:16-131; the
// status codes are defined 1:1 on them, lbk.h:36-52)
[[noreturn]] void raise(lbk_status s, int iteration = -1)
{
    const std::string msg = lbk_last_error(g_ctx);
    switch (s) {
    case LBK_SHAPE_ERROR: throw ShapeError(msg);
    case LBK_PLACEMENT_ERROR: throw PlacementError(msg);
    case LBK_TYPE_ERROR: throw TypeError(msg);
    case LBK_DISPATCH_ERROR: throw DispatchError(msg);
    case LBK_USAGE_ERROR: throw UsageError(msg);
    case LBK_CONFIGURATION_ERROR: throw ConfigurationError(msg);
    case LBK_OUT_OF_MEMORY: throw OutOfMemoryError(0, 0, 0);
    case LBK_FORMAT_ERROR: throw FormatError(msg);
    case LBK_UNSUPPORTED_FORMAT: throw UnsupportedFormatError(msg);
    case LBK_BREAKDOWN: throw BreakdownError(msg, iteration);
    case LBK_BENCHMARK_INTEGRITY: throw BenchmarkIntegrityError(msg);
    default: throw Error(msg);
    }
}

void check(lbk_status s)
{
    if (s != LBK_OK) raise(s);
}

const double* dptr(const DeviceArray* a) { return static_cast<const double*>(a->data()); }
double* dptr(DeviceArray* a) { return static_cast<double*>(a->data()); }

lbk_csr csr_desc(const CsrMatrix& A)
{
    return lbk_csr{A.nrows,
                   A.ncols,
                   static_cast<int64_t>(A.nnz()),
                   LBK_F64,
                   static_cast<const int32_t*>(A.row_ptr.data()),
                   static_cast<const int32_t*>(A.col_idx.data()),
                   A.vals.data(),
                   nullptr,
                   0};
}

lbk_coo coo_desc(const CooMatrix& A)
{
    return lbk_coo{A.nrows,
                   A.ncols,
                   static_cast<int64_t>(A.nnz()),
                   LBK_F64,
                   static_cast<const int32_t*>(A.row_idx.data()),
                   static_cast<const int32_t*>(A.col_idx.data()),
                   A.vals.data(),
                   nullptr,
                   0};
}

// KernelFn = std::function<void(Executor&, std::any&)> (dispatch.hpp:23)
void spmv_csr_kernel(Executor&, std::any& a)
{
    auto& args = std::any_cast<SpmvCsrArgs&>(a);  // kernels.hpp:52-56
    const lbk_csr d = csr_desc(*args.matrix);
    check(lbk_spmv_csr_f64(g_ctx, &d, dptr(args.x), dptr(args.y)));
    check(lbk_sync(g_ctx));
}

void spmv_coo_kernel(Executor&, std::any& a)
{
    auto& args = std::any_cast<SpmvCooArgs&>(a);  // kernels.hpp:46-50
    const lbk_coo d = coo_desc(*args.matrix);
    check(lbk_spmv_coo_f64(g_ctx, &d, dptr(args.x), dptr(args.y)));
    check(lbk_sync(g_ctx));
}

void dot_kernel(Executor&, std::any& a)
{
    auto& args = std::any_cast<DotArgs&>(a);  // kernels.hpp:40-44: result is a host double*
    check(lbk_dot_f64(g_ctx, static_cast<int64_t>(args.x->size()), dptr(args.x), dptr(args.y),
                      args.result));
}

void axpy_kernel(Executor&, std::any& a)
{
    auto& args = std::any_cast<AxpyArgs&>(a);
    check(lbk_axpy_f64(g_ctx, static_cast<int64_t>(args.x->size()), args.alpha, dptr(args.x),
                       dptr(args.y)));
    check(lbk_sync(g_ctx));
}

void scal_kernel(Executor&, std::any& a)
{
    auto& args = std::any_cast<ScalArgs&>(a);
    check(lbk_scal_f64(g_ctx, static_cast<int64_t>(args.x->size()), args.alpha, dptr(args.x)));
    check(lbk_sync(g_ctx));
}

void fill_kernel(Executor&, std::any& a)
{
    auto& args = std::any_cast<FillArgs&>(a);
    check(lbk_fill_f64(g_ctx, static_cast<int64_t>(args.x->size()), args.value, dptr(args.x)));
    check(lbk_sync(g_ctx));
}

// StreamOp {copy, mul, add, triad, dot} (kernels.hpp:58-68): the reference's
// bandwidth-calibration kernels, reference.cpp:92-130
void stream_kernel(StreamOp op, std::any& a)
{
    auto& args = std::any_cast<StreamArgs&>(a);
    const int64_t n = static_cast<int64_t>(args.a->size());
    switch (op) {
    case StreamOp::copy: check(lbk_stream_copy_f64(g_ctx, n, dptr(args.a), dptr(args.c))); break;
    case StreamOp::mul:
        check(lbk_stream_mul_f64(g_ctx, n, args.scalar, dptr(args.c), dptr(args.b)));
        break;
    case StreamOp::add:
        check(lbk_stream_add_f64(g_ctx, n, dptr(args.a), dptr(args.b), dptr(args.c)));
        break;
    case StreamOp::triad:
        check(lbk_stream_triad_f64(g_ctx, n, args.scalar, dptr(args.b), dptr(args.c),
                                   dptr(args.a)));
        break;
    case StreamOp::dot:
        check(lbk_stream_dot_f64(g_ctx, n, dptr(args.a), dptr(args.b), args.dot_result));
        break;
    }
    check(lbk_sync(g_ctx));
}

void flops_sweep_kernel(Executor&, std::any& a)
{
    auto& args = std::any_cast<FlopsSweepArgs&>(a);  // kernels.hpp:70-73
    check(lbk_flops_sweep_f64(g_ctx, static_cast<int64_t>(args.x->size()),
                              args.fma_per_element, dptr(args.x)));
    check(lbk_sync(g_ctx));
}

}  // namespace

// Called from register_builtin_kernels() (api.cpp:39-48) next to the
// reference's own backends: one host-style registration per kernel name
// for ExecutorKind::cuda.
void register_kernels()
{
    if (!g_ctx) check(lbk_ctx_create(0, &g_ctx));
    auto& r = KernelRegistry::instance();
    r.register_host("spmv_csr", ExecutorKind::cuda, spmv_csr_kernel);
    r.register_host("spmv_coo", ExecutorKind::cuda, spmv_coo_kernel);
    r.register_host("dot", ExecutorKind::cuda, dot_kernel);
    r.register_host("axpy", ExecutorKind::cuda, axpy_kernel);
    r.register_host("scal", ExecutorKind::cuda, scal_kernel);
    r.register_host("fill", ExecutorKind::cuda, fill_kernel);
    for (StreamOp op : {StreamOp::copy, StreamOp::mul, StreamOp::add, StreamOp::triad,
                        StreamOp::dot})
        r.register_host(std::string("stream_") + to_string(op), ExecutorKind::cuda,
                        [op](Executor&, std::any& a) { stream_kernel(op, a); });
    r.register_host("flops_sweep", ExecutorKind::cuda, flops_sweep_kernel);
}

// solve() routes here for the cuda kind (krylov.cpp:587-598): the whole
// Krylov loop stays on the device, one call, SolveResult filled 1:1.
SolveResult solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                  const SolverConfig& cfg)
{
    const lbk_csr d = csr_desc(A);
    lbk_solver_cfg c{};
    c.kind = static_cast<int32_t>(cfg.kind);  // SolverKind {cg, bicgstab, cgs, gmres}
    c.max_iters = cfg.max_iters;
    c.rel_tol = cfg.rel_tol;
    c.fixed_iters = cfg.fixed_iters ? *cfg.fixed_iters : 0;
    c.residual_mode = 0;  // reference semantics: true residual every iteration
    c.gmres_restart = cfg.gmres_restart;
    const int32_t cap = (cfg.fixed_iters ? *cfg.fixed_iters : cfg.max_iters) + 1;
    std::vector<double> hist(static_cast<size_t>(cap));
    lbk_solve_result r{};
    const lbk_status s = lbk_solve_csr(g_ctx, &d, dptr(&b.values), dptr(&x.values), &c, &r,
                                       hist.data(), cap);
    if (s != LBK_OK) raise(s, r.breakdown_iter);
    SolveResult out;
    out.converged = r.converged != 0;
    out.iterations = r.iterations;
    out.final_rel_residual = r.final_rel_residual;
    out.residual_history.assign(hist.begin(), hist.begin() + r.history_len);
    out.elapsed = r.elapsed;
    out.flop_count = r.flop_count;
    return out;
}

}  // namespace lbk_backend
}  // namespace larch
