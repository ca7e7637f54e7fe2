// oracle/ref_driver.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// A C-ABI over the *unmodified* reference library (larch, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  This is
// the reference run here, not a restatement: every entry point below calls
// the reference's own public API with host arrays, so parity tests and the
// bench's CPU baseline can drive it through ctypes.
//
// Reference API used (paths relative to /root/reference/proj):
//   ReferenceExecutor / ParallelExecutor ....... include/larch/core/executor.hpp:174-211
//   array_from_host / array_to_host ............ include/larch/core/device_array.hpp:166-171
//   coo_from_entries / coo_to_csr / csr_to_coo . include/larch/matrix/formats.hpp:82-90
//   validate ................................... include/larch/matrix/formats.hpp:93-94
//   spmv_coo / spmv_csr / dot / axpy ........... include/larch/kernels/kernels.hpp:79-97
//   solve / SolverConfig / SolveResult ......... include/larch/solver/krylov.hpp:22-56
//   Error taxonomy ............................. include/larch/core/error.hpp:16-131
//
// Status codes mirror include/lbk.h (LBK_*), so a test can compare the error
// behaviour of both sides directly.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "larch/bench/harness.hpp"
#include "larch/core/error.hpp"
#include "larch/core/executor.hpp"
#include "larch/kernels/kernels.hpp"
#include "larch/matrix/formats.hpp"
#include "larch/matrix/io.hpp"
#include "larch/solver/krylov.hpp"

namespace {

thread_local std::string g_last_error;

enum {
    ST_OK = 0,
    ST_SHAPE = 1,
    ST_PLACEMENT = 2,
    ST_TYPE = 3,
    ST_DISPATCH = 4,
    ST_USAGE = 5,
    ST_CONFIG = 6,
    ST_OOM = 7,
    ST_FORMAT = 8,
    ST_BREAKDOWN = 9,
    ST_INTEGRITY = 10,
    ST_UNSUPPORTED = 11,
    ST_INTERNAL = 99,
};

int breakdown_iter_slot = -1;

template <typename F>
int guarded(F&& body)
{
    g_last_error.clear();
    breakdown_iter_slot = -1;
    try {
        body();
        return ST_OK;
    } catch (const larch::BreakdownError& e) {
        g_last_error = e.what();
        breakdown_iter_slot = e.iteration;
        return ST_BREAKDOWN;
    } catch (const larch::ShapeError& e) {
        g_last_error = e.what();
        return ST_SHAPE;
    } catch (const larch::PlacementError& e) {
        g_last_error = e.what();
        return ST_PLACEMENT;
    } catch (const larch::TypeError& e) {
        g_last_error = e.what();
        return ST_TYPE;
    } catch (const larch::DispatchError& e) {
        g_last_error = e.what();
        return ST_DISPATCH;
    } catch (const larch::UsageError& e) {
        g_last_error = e.what();
        return ST_USAGE;
    } catch (const larch::ConfigurationError& e) {
        g_last_error = e.what();
        return ST_CONFIG;
    } catch (const larch::OutOfMemoryError& e) {
        g_last_error = e.what();
        return ST_OOM;
    } catch (const larch::UnsupportedFormatError& e) {
        g_last_error = e.what();
        return ST_UNSUPPORTED;
    } catch (const larch::FormatError& e) {
        g_last_error = e.what();
        return ST_FORMAT;
    } catch (const larch::BenchmarkIntegrityError& e) {
        g_last_error = e.what();
        return ST_INTEGRITY;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ST_INTERNAL;
    }
}

std::shared_ptr<larch::Executor> make_exec(int kind, int workers)
{
    if (kind == 0) {
        return larch::ReferenceExecutor::create();
    }
    return larch::ParallelExecutor::create(workers);
}

template <typename T>
std::span<const T> sp(const T* p, std::int64_t n)
{
    return {p, static_cast<std::size_t>(n)};
}

larch::CsrMatrix make_csr(std::shared_ptr<larch::Executor> exec, int nrows,
                          int ncols, std::int64_t nnz, const int* row_ptr,
                          const int* cols, const double* vals)
{
    larch::CsrMatrix a;
    a.nrows = nrows;
    a.ncols = ncols;
    a.row_ptr = larch::array_from_host<std::int32_t>(exec, sp(row_ptr, nrows + 1));
    a.col_idx = larch::array_from_host<std::int32_t>(exec, sp(cols, nnz));
    a.vals = larch::array_from_host<double>(exec, sp(vals, nnz));
    return a;
}

larch::CooMatrix make_coo(std::shared_ptr<larch::Executor> exec, int nrows,
                          int ncols, std::int64_t nnz, const int* rows,
                          const int* cols, const double* vals)
{
    larch::CooMatrix a;
    a.nrows = nrows;
    a.ncols = ncols;
    a.row_idx = larch::array_from_host<std::int32_t>(exec, sp(rows, nnz));
    a.col_idx = larch::array_from_host<std::int32_t>(exec, sp(cols, nnz));
    a.vals = larch::array_from_host<double>(exec, sp(vals, nnz));
    return a;
}

double median(std::vector<double> s)
{
    std::sort(s.begin(), s.end());
    if (s.empty()) return 0.0;
    auto n = s.size();
    return n % 2 ? s[n / 2] : 0.5 * (s[n / 2 - 1] + s[n / 2]);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }
int ref_last_breakdown_iter() { return breakdown_iter_slot; }

/// y = A x through the reference spmv_csr (fmt=1) or spmv_coo (fmt=0) on the
/// reference (exec_kind=0) or parallel(workers) (exec_kind=1) executor.
/// `ptr` is row_ptr for CSR and row_idx for COO.  With reps>0 the call is
/// repeated and the median wall time per call is written to *seconds
/// (the reference harness protocol, src/bench/harness.cpp:284-364).
int ref_spmv(int exec_kind, int workers, int fmt, int nrows, int ncols,
             std::int64_t nnz, const int* ptr, const int* cols,
             const double* vals, const double* x, double* y, int reps,
             double* seconds)
{
    return guarded([&] {
        auto exec = make_exec(exec_kind, workers);
        auto xv = larch::vector_from(exec, sp(x, ncols));
        auto yv = larch::make_vector(exec, static_cast<std::size_t>(nrows));
        std::vector<double> samples;
        if (fmt == 1) {
            auto a = make_csr(exec, nrows, ncols, nnz, ptr, cols, vals);
            larch::spmv_csr(a, xv, yv);
            for (int r = 0; r < reps; ++r) {
                auto t0 = std::chrono::steady_clock::now();
                larch::spmv_csr(a, xv, yv);
                samples.push_back(std::chrono::duration<double>(
                                      std::chrono::steady_clock::now() - t0)
                                      .count());
            }
        } else {
            auto a = make_coo(exec, nrows, ncols, nnz, ptr, cols, vals);
            larch::spmv_coo(a, xv, yv);
            for (int r = 0; r < reps; ++r) {
                auto t0 = std::chrono::steady_clock::now();
                larch::spmv_coo(a, xv, yv);
                samples.push_back(std::chrono::duration<double>(
                                      std::chrono::steady_clock::now() - t0)
                                      .count());
            }
        }
        auto out = larch::vector_to_host(yv);
        std::memcpy(y, out.data(), out.size() * sizeof(double));
        if (seconds) *seconds = median(samples);
    });
}

/// Reference dot (exec-dependent summation order, reference.cpp:46-56 vs
/// parallel.cpp:76-97).
int ref_dot(int exec_kind, int workers, std::int64_t n, const double* x,
            const double* y, double* out)
{
    return guarded([&] {
        auto exec = make_exec(exec_kind, workers);
        auto xv = larch::vector_from(exec, sp(x, n));
        auto yv = larch::vector_from(exec, sp(y, n));
        *out = larch::dot(xv, yv);
    });
}

/// Reference axpy: y <- alpha x + y (kernels.hpp:80).
int ref_axpy(std::int64_t n, double alpha, const double* x, double* y)
{
    return guarded([&] {
        auto exec = larch::ReferenceExecutor::create();
        auto xv = larch::vector_from(exec, sp(x, n));
        auto yv = larch::vector_from(exec, sp(static_cast<const double*>(y), n));
        larch::axpy(alpha, xv, yv);
        auto out = larch::vector_to_host(yv);
        std::memcpy(y, out.data(), out.size() * sizeof(double));
    });
}

/// coo_from_entries (formats.cpp:78-116).  Output arrays must hold n
/// entries; *nnz_out receives the canonical count.
int ref_coo_from_entries(int nrows, int ncols, std::int64_t n, const int* rows,
                         const int* cols, const double* vals,
                         std::int64_t* nnz_out, int* rows_out, int* cols_out,
                         double* vals_out)
{
    return guarded([&] {
        std::vector<larch::MatrixEntry> entries(static_cast<std::size_t>(n));
        for (std::int64_t k = 0; k < n; ++k) {
            entries[k] = larch::MatrixEntry{rows[k], cols[k], vals[k]};
        }
        auto exec = larch::ReferenceExecutor::create();
        auto coo = larch::coo_from_entries(exec, nrows, ncols, entries);
        auto r = larch::array_to_host<std::int32_t>(coo.row_idx);
        auto c = larch::array_to_host<std::int32_t>(coo.col_idx);
        auto v = larch::array_to_host<double>(coo.vals);
        *nnz_out = static_cast<std::int64_t>(v.size());
        std::memcpy(rows_out, r.data(), r.size() * sizeof(int));
        std::memcpy(cols_out, c.data(), c.size() * sizeof(int));
        std::memcpy(vals_out, v.data(), v.size() * sizeof(double));
    });
}

/// coo_to_csr (formats.cpp:132-155).
int ref_coo_to_csr(int nrows, int ncols, std::int64_t nnz, const int* rows,
                   const int* cols, const double* vals, int* row_ptr_out,
                   int* cols_out, double* vals_out)
{
    return guarded([&] {
        auto exec = larch::ReferenceExecutor::create();
        auto coo = make_coo(exec, nrows, ncols, nnz, rows, cols, vals);
        auto csr = larch::coo_to_csr(coo);
        auto p = larch::array_to_host<std::int32_t>(csr.row_ptr);
        auto c = larch::array_to_host<std::int32_t>(csr.col_idx);
        auto v = larch::array_to_host<double>(csr.vals);
        std::memcpy(row_ptr_out, p.data(), p.size() * sizeof(int));
        std::memcpy(cols_out, c.data(), c.size() * sizeof(int));
        std::memcpy(vals_out, v.data(), v.size() * sizeof(double));
    });
}

/// csr_to_coo (formats.cpp:158-179).
int ref_csr_to_coo(int nrows, int ncols, std::int64_t nnz, const int* row_ptr,
                   const int* cols, const double* vals, int* rows_out,
                   int* cols_out, double* vals_out)
{
    return guarded([&] {
        auto exec = larch::ReferenceExecutor::create();
        auto csr = make_csr(exec, nrows, ncols, nnz, row_ptr, cols, vals);
        auto coo = larch::csr_to_coo(csr);
        auto r = larch::array_to_host<std::int32_t>(coo.row_idx);
        auto c = larch::array_to_host<std::int32_t>(coo.col_idx);
        auto v = larch::array_to_host<double>(coo.vals);
        std::memcpy(rows_out, r.data(), r.size() * sizeof(int));
        std::memcpy(cols_out, c.data(), c.size() * sizeof(int));
        std::memcpy(vals_out, v.data(), v.size() * sizeof(double));
    });
}

/// read_matrix_market(path, exec) (io.cpp:71-191) -> canonical COO.  Call
/// with rows == nullptr first to learn the shape and nnz.
int ref_read_mm(const char* path, int* nrows, int* ncols, std::int64_t* nnz, int* rows,
                int* cols, double* vals)
{
    return guarded([&] {
        auto exec = larch::ReferenceExecutor::create();
        auto coo = larch::read_matrix_market(std::filesystem::path(path), exec);
        *nrows = coo.nrows;
        *ncols = coo.ncols;
        *nnz = static_cast<std::int64_t>(coo.nnz());
        if (rows) {
            auto r = larch::array_to_host<std::int32_t>(coo.row_idx);
            auto c = larch::array_to_host<std::int32_t>(coo.col_idx);
            auto v = larch::array_to_host<double>(coo.vals);
            std::memcpy(rows, r.data(), r.size() * sizeof(int));
            std::memcpy(cols, c.data(), c.size() * sizeof(int));
            std::memcpy(vals, v.data(), v.size() * sizeof(double));
        }
    });
}

/// validate(Csr) / validate(Coo) (formats.cpp:182-242); fmt as in ref_spmv.
int ref_validate(int fmt, int nrows, int ncols, std::int64_t nnz,
                 const int* ptr, const int* cols, const double* vals)
{
    return guarded([&] {
        auto exec = larch::ReferenceExecutor::create();
        if (fmt == 1) {
            larch::validate(make_csr(exec, nrows, ncols, nnz, ptr, cols, vals));
        } else {
            larch::validate(make_coo(exec, nrows, ncols, nnz, ptr, cols, vals));
        }
    });
}

/// solve() (krylov.cpp:587-598).  kind: 0 cg, 1 bicgstab, 2 cgs, 3 gmres.
/// fixed_iters <= 0 means "not set".  hist receives up to hist_cap entries.
/// out_i = {converged, iterations, hist_len}; out_d = {final_rel_residual,
/// elapsed}; *flops = flop_count.
int ref_solve(int exec_kind, int workers, int fmt, int kind, int n,
              std::int64_t nnz, const int* ptr, const int* cols,
              const double* vals, const double* b, double* x, int max_iters,
              double rel_tol, int fixed_iters, int restart, double* hist,
              int hist_cap, int* out_i, double* out_d, std::int64_t* flops)
{
    return guarded([&] {
        auto exec = make_exec(exec_kind, workers);
        auto bv = larch::vector_from(exec, sp(b, n));
        auto xv = larch::vector_from(exec, sp(static_cast<const double*>(x), n));
        larch::SolverConfig cfg;
        cfg.kind = static_cast<larch::SolverKind>(kind);
        cfg.max_iters = max_iters;
        cfg.rel_tol = rel_tol;
        cfg.gmres_restart = restart;
        if (fixed_iters > 0) cfg.fixed_iters = fixed_iters;
        larch::SolveResult res;
        if (fmt == 1) {
            auto a = make_csr(exec, n, n, nnz, ptr, cols, vals);
            res = larch::solve(a, bv, xv, cfg);
        } else {
            auto a = make_coo(exec, n, n, nnz, ptr, cols, vals);
            res = larch::solve(a, bv, xv, cfg);
        }
        auto xo = larch::vector_to_host(xv);
        std::memcpy(x, xo.data(), xo.size() * sizeof(double));
        out_i[0] = res.converged ? 1 : 0;
        out_i[1] = res.iterations;
        out_i[2] = static_cast<int>(res.residual_history.size());
        out_d[0] = res.final_rel_residual;
        out_d[1] = res.elapsed;
        *flops = res.flop_count;
        auto m = std::min<std::size_t>(res.residual_history.size(),
                                       static_cast<std::size_t>(hist_cap));
        std::memcpy(hist, res.residual_history.data(), m * sizeof(double));
    });
}

/// gmres_restart_cycle (krylov.hpp:78-89) on CSR: one cycle from x (updated
/// in place); out_i = {steps, happy, basis size}; *rel = rel_residual;
/// basis (n * cap, may be null) receives the basis vectors.
int ref_gmres_cycle(int exec_kind, int workers, int n, std::int64_t nnz, const int* ptr,
                    const int* cols, const double* vals, const double* b, double* x,
                    int restart, double* rel, int* out_i, double* basis, int cap)
{
    return guarded([&] {
        auto exec = make_exec(exec_kind, workers);
        auto bv = larch::vector_from(exec, sp(b, n));
        auto xv = larch::vector_from(exec, sp(static_cast<const double*>(x), n));
        auto a = make_csr(exec, n, n, nnz, ptr, cols, vals);
        std::vector<larch::DenseVector> V;
        auto r = larch::gmres_restart_cycle(a, bv, xv, restart, &V);
        auto xo = larch::vector_to_host(xv);
        std::memcpy(x, xo.data(), xo.size() * sizeof(double));
        *rel = r.rel_residual;
        out_i[0] = r.steps;
        out_i[1] = r.happy_breakdown ? 1 : 0;
        out_i[2] = static_cast<int>(V.size());
        for (int i = 0; basis && i < static_cast<int>(V.size()) && i < cap; ++i) {
            auto h = larch::vector_to_host(V[static_cast<std::size_t>(i)]);
            std::memcpy(basis + static_cast<std::size_t>(i) * n, h.data(), h.size() * sizeof(double));
        }
    });
}

/// The reference's own host bandwidth calibration: measure_peak_bandwidth
/// (harness.cpp:125-141) -- stream copy of `bytes` per array on the given
/// executor, median of `reps`; GB/s to *out.
int ref_measure_peak_bandwidth(int exec_kind, int workers, std::int64_t bytes, int reps,
                               double* out)
{
    return guarded([&] {
        auto exec = make_exec(exec_kind, workers);
        *out = larch::measure_peak_bandwidth(exec, static_cast<std::size_t>(bytes), reps);  // GB/s (safe_rate)
    });
}

}  // extern "C"
