// include/lbk/larch.hpp -- C++ host façade of the B200 backend.
//
// Mirrors the reference's public operator surface (paths relative to
// /root/reference/proj) in namespace lbk::larch, on top of the C ABI
// (include/lbk.h, liblbk.so):
//
//   errors      include/larch/core/error.hpp:16-131        (same classes)
//   executor    include/larch/core/executor.hpp:130-262     (cuda kind)
//   arrays      include/larch/core/device_array.hpp:57-171  (DeviceArray)
//   formats     include/larch/matrix/formats.hpp:20-94      (+ Ell, Sellp)
//   io          include/larch/matrix/io.hpp:25-28           (read_matrix_market)
//   kernels     include/larch/kernels/kernels.hpp:79-97     (+ alpha/beta)
//   solvers     include/larch/solver/krylov.hpp:17-60       (cg, bicgstab, cgs, gmres)
//
// Same names, argument meaning and error behaviour, so code written
// against the reference recompiles against this header with
// `namespace larch = lbk::larch;`.  Wrappers are synchronous like the
// reference's (dispatch.cpp:112-117).  Header-only; link -llbk -lcudart.
#ifndef LBK_LARCH_HPP
#define LBK_LARCH_HPP

#include <cstdint>
#include <filesystem>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lbk.h"

namespace lbk::larch {

// ------------------------------------------------------------------ errors
class Error : public std::runtime_error {
public:
    explicit Error(const std::string& what) : std::runtime_error(what) {}
};
class ConfigurationError : public Error { using Error::Error; };
class OutOfMemoryError : public Error { using Error::Error; };
class ShapeError : public Error { using Error::Error; };
class TypeError : public Error { using Error::Error; };
class PlacementError : public Error { using Error::Error; };
class UsageError : public Error { using Error::Error; };
class DispatchError : public Error { using Error::Error; };
class FormatError : public Error { using Error::Error; };
class UnsupportedFormatError : public FormatError { using FormatError::FormatError; };
class BenchmarkIntegrityError : public Error { using Error::Error; };
class DeviceError : public Error { using Error::Error; };  // CUDA/NCCL (new)
class BreakdownError : public Error {
public:
    BreakdownError(const std::string& what, int iter) : Error(what), iteration(iter) {}
    int iteration;
};

namespace detail {
inline void check(lbk_status s, lbk_ctx ctx = nullptr, int iter = -1)
{
    if (s == LBK_OK) return;
    const std::string m = lbk_last_error(ctx);
    switch (s) {
    case LBK_SHAPE_ERROR: throw ShapeError(m);
    case LBK_PLACEMENT_ERROR: throw PlacementError(m);
    case LBK_TYPE_ERROR: throw TypeError(m);
    case LBK_DISPATCH_ERROR: throw DispatchError(m);
    case LBK_USAGE_ERROR: throw UsageError(m);
    case LBK_CONFIGURATION_ERROR: throw ConfigurationError(m);
    case LBK_OUT_OF_MEMORY: throw OutOfMemoryError(m);
    case LBK_FORMAT_ERROR: throw FormatError(m);
    case LBK_UNSUPPORTED_FORMAT: throw UnsupportedFormatError(m);
    case LBK_BREAKDOWN: throw BreakdownError(m, iter);
    case LBK_BENCHMARK_INTEGRITY: throw BenchmarkIntegrityError(m);
    case LBK_CUDA_ERROR:
    case LBK_NCCL_ERROR: throw DeviceError(m);
    default: throw Error(m);
    }
}
}  // namespace detail

// ---------------------------------------------------------------- executor
// executor.hpp:26 ExecutorKind gains `cuda`; the host kinds stay in the
// reference (this backend replaces the kernels, not the host executors).
enum class ExecutorKind { cuda };
enum class ElementKind { float32, float64, int32 };

struct ExecutorParams {
    int device = 0;
    std::size_t arena_capacity = 0;  // 0: no cap (executor.hpp:57)
};

class Executor {
public:
    explicit Executor(const ExecutorParams& p) : device_(p.device)
    {
        detail::check(lbk_ctx_create(p.device, &ctx_));
        if (p.arena_capacity) detail::check(lbk_ctx_set_arena_capacity(ctx_, p.arena_capacity), ctx_);
    }
    Executor(const Executor&) = delete;
    Executor& operator=(const Executor&) = delete;
    ~Executor() { lbk_ctx_destroy(ctx_); }

    ExecutorKind kind() const { return ExecutorKind::cuda; }
    void synchronize() const { detail::check(lbk_sync(ctx_), ctx_); }
    std::string describe() const
    {
        int dev = 0, sms = 0;
        std::size_t cap = 0, used = 0;
        lbk_ctx_info(ctx_, &dev, &sms, &cap, &used);
        return "cuda(device=" + std::to_string(dev) + ", sms=" + std::to_string(sms) + ")";
    }
    // executor.cpp:254-279: arena accounting -> OutOfMemoryError
    void* raw_alloc(std::size_t bytes)
    {
        void* p = nullptr;
        detail::check(lbk_alloc(ctx_, bytes, &p), ctx_);
        return p;
    }
    void raw_free(void* p, std::size_t bytes) { lbk_free(ctx_, p, bytes); }
    lbk_ctx handle() const { return ctx_; }

private:
    int device_;
    lbk_ctx ctx_ = nullptr;
};

inline std::shared_ptr<Executor> create_executor(ExecutorKind, const ExecutorParams& p = {})
{
    return std::make_shared<Executor>(p);
}

// ------------------------------------------------------------- DeviceArray
// device_array.hpp:57-110: typed RAII buffer owned by its executor.
class DeviceArray {
public:
    DeviceArray() = default;
    DeviceArray(std::shared_ptr<Executor> exec, ElementKind kind, std::size_t n)
        : exec_(std::move(exec)), kind_(kind), n_(n)
    {
        if (n_) ptr_ = exec_->raw_alloc(bytes());
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    DeviceArray(DeviceArray&& o) noexcept { swap(o); }
    DeviceArray& operator=(DeviceArray&& o) noexcept
    {
        DeviceArray t(std::move(o));
        swap(t);
        return *this;
    }
    ~DeviceArray()
    {
        if (ptr_) exec_->raw_free(ptr_, bytes());
    }
    std::size_t size() const { return n_; }
    ElementKind kind() const { return kind_; }
    std::size_t element_size() const { return kind_ == ElementKind::float64 ? 8 : 4; }
    std::size_t bytes() const { return n_ * element_size(); }
    std::shared_ptr<Executor> owner() const { return exec_; }
    void* data() { return ptr_; }
    const void* data() const { return ptr_; }
    template <typename T>
    T* as() { return static_cast<T*>(ptr_); }
    template <typename T>
    const T* as() const { return static_cast<const T*>(ptr_); }

private:
    void swap(DeviceArray& o) noexcept
    {
        std::swap(exec_, o.exec_);
        std::swap(kind_, o.kind_);
        std::swap(n_, o.n_);
        std::swap(ptr_, o.ptr_);
    }
    std::shared_ptr<Executor> exec_;
    ElementKind kind_ = ElementKind::float64;
    std::size_t n_ = 0;
    void* ptr_ = nullptr;
};

template <typename T>
DeviceArray array_from_host(std::shared_ptr<Executor> exec, std::span<const T> host)
{
    constexpr ElementKind k = std::is_same_v<T, double>  ? ElementKind::float64
                              : std::is_same_v<T, float> ? ElementKind::float32
                                                         : ElementKind::int32;
    DeviceArray a(exec, k, host.size());
    if (!host.empty()) {
        detail::check(lbk_memcpy_h2d(exec->handle(), a.data(), host.data(), a.bytes()), exec->handle());
        exec->synchronize();
    }
    return a;
}

template <typename T>
std::vector<T> array_to_host(const DeviceArray& a)
{
    std::vector<T> out(a.size());
    if (!out.empty()) {
        auto e = a.owner();
        detail::check(lbk_memcpy_d2h(e->handle(), out.data(), a.data(), a.bytes()), e->handle());
        e->synchronize();
    }
    return out;
}

inline DeviceArray clone_array(const DeviceArray& a, std::shared_ptr<Executor> exec)
{
    DeviceArray b(exec, a.kind(), a.size());
    if (a.size()) {
        detail::check(lbk_memcpy_d2d(exec->handle(), b.data(), a.data(), a.bytes()), exec->handle());
        exec->synchronize();
    }
    return b;
}

// ------------------------------------------------------------------ formats
struct DenseVector {
    DeviceArray values;
    std::size_t size() const { return values.size(); }
    std::shared_ptr<Executor> executor() const { return values.owner(); }
    DenseVector clone_to(std::shared_ptr<Executor> exec) const { return {clone_array(values, exec)}; }
};

inline DenseVector make_vector(std::shared_ptr<Executor> exec, std::size_t size)
{
    return {DeviceArray(exec, ElementKind::float64, size)};
}
inline DenseVector vector_from(std::shared_ptr<Executor> exec, std::span<const double> values)
{
    return {array_from_host<double>(exec, values)};
}
inline DenseVector zeros(std::shared_ptr<Executor> exec, std::size_t size)
{
    DenseVector v = make_vector(exec, size);
    detail::check(lbk_fill_f64(exec->handle(), static_cast<int64_t>(size), 0.0, v.values.as<double>()),
                  exec->handle());
    exec->synchronize();
    return v;
}
inline std::vector<double> vector_to_host(const DenseVector& v) { return array_to_host<double>(v.values); }

struct MatrixEntry {
    std::int32_t row = 0;
    std::int32_t col = 0;
    double value = 0.0;
    friend bool operator==(const MatrixEntry&, const MatrixEntry&) = default;
};

struct CooMatrix {
    std::int32_t nrows = 0, ncols = 0;
    DeviceArray row_idx, col_idx, vals;
    std::size_t nnz() const { return vals.size(); }
    std::shared_ptr<Executor> executor() const { return vals.owner(); }
    CooMatrix clone_to(std::shared_ptr<Executor> e) const
    {
        return {nrows, ncols, clone_array(row_idx, e), clone_array(col_idx, e), clone_array(vals, e)};
    }
    lbk_coo desc() const
    {
        return lbk_coo{nrows, ncols, static_cast<int64_t>(nnz()), LBK_F64, row_idx.as<int32_t>(),
                       col_idx.as<int32_t>(), vals.data(), nullptr, 0};
    }
};

struct CsrMatrix {
    std::int32_t nrows = 0, ncols = 0;
    DeviceArray row_ptr, col_idx, vals;
    std::size_t nnz() const { return vals.size(); }
    std::shared_ptr<Executor> executor() const { return vals.owner(); }
    CsrMatrix clone_to(std::shared_ptr<Executor> e) const
    {
        return {nrows, ncols, clone_array(row_ptr, e), clone_array(col_idx, e), clone_array(vals, e)};
    }
    lbk_csr desc() const
    {
        return lbk_csr{nrows, ncols, static_cast<int64_t>(nnz()), LBK_F64, row_ptr.as<int32_t>(),
                       col_idx.as<int32_t>(), vals.data(), nullptr, 0};
    }
};

// Additions (absent from the reference).
struct EllMatrix {
    std::int32_t nrows = 0, ncols = 0, width = 0;
    std::int64_t stride = 0, logical_nnz = 0;
    DeviceArray col_idx, vals;
    std::shared_ptr<Executor> executor() const { return vals.owner(); }
    lbk_ell desc() const
    {
        return lbk_ell{nrows, ncols, logical_nnz, LBK_F64, width, stride, col_idx.as<int32_t>(),
                       vals.data()};
    }
};

struct SellpMatrix {
    std::int32_t nrows = 0, ncols = 0, slice_size = 32, nslices = 0;
    std::int64_t logical_nnz = 0;
    DeviceArray slice_lengths, slice_sets, col_idx, vals;
    std::shared_ptr<Executor> executor() const { return vals.owner(); }
    lbk_sellp desc() const
    {
        return lbk_sellp{nrows, ncols, logical_nnz, LBK_F64, slice_size, nslices,
                         slice_lengths.as<int32_t>(), slice_sets.as<int32_t>(), col_idx.as<int32_t>(),
                         vals.data(), static_cast<int64_t>(col_idx.size()), nullptr, 0};
    }
};

// formats.cpp:78-116 on the device.
inline CooMatrix coo_from_entries(std::shared_ptr<Executor> exec, std::int32_t nrows,
                                  std::int32_t ncols, std::span<const MatrixEntry> entries)
{
    const std::size_t n = entries.size();
    std::vector<int32_t> r(n), c(n);
    std::vector<double> v(n);
    for (std::size_t i = 0; i < n; ++i) {
        r[i] = entries[i].row;
        c[i] = entries[i].col;
        v[i] = entries[i].value;
    }
    auto rin = array_from_host<int32_t>(exec, r), cin = array_from_host<int32_t>(exec, c);
    auto vin = array_from_host<double>(exec, v);
    DeviceArray ro(exec, ElementKind::int32, n), co(exec, ElementKind::int32, n),
        vo(exec, ElementKind::float64, n);
    int64_t nnz = 0;
    detail::check(lbk_coo_assemble_f64(exec->handle(), nrows, ncols, static_cast<int64_t>(n),
                                       rin.as<int32_t>(), cin.as<int32_t>(), vin.as<double>(),
                                       ro.as<int32_t>(), co.as<int32_t>(), vo.as<double>(), &nnz),
                  exec->handle());
    CooMatrix m{nrows, ncols, DeviceArray(exec, ElementKind::int32, nnz),
                DeviceArray(exec, ElementKind::int32, nnz), DeviceArray(exec, ElementKind::float64, nnz)};
    if (nnz) {
        auto h = exec->handle();
        detail::check(lbk_memcpy_d2d(h, m.row_idx.data(), ro.data(), nnz * 4), h);
        detail::check(lbk_memcpy_d2d(h, m.col_idx.data(), co.data(), nnz * 4), h);
        detail::check(lbk_memcpy_d2d(h, m.vals.data(), vo.data(), nnz * 8), h);
        exec->synchronize();
    }
    return m;
}

// io.hpp:25-28: MatrixMarket coordinate file -> canonical COO (host parse
// with the reference's rules and messages, device assembly).
inline CooMatrix read_matrix_market(const std::filesystem::path& path, std::shared_ptr<Executor> exec)
{
    lbk_mm h = nullptr;
    const lbk_status s = lbk_mm_read(path.c_str(), &h);
    if (s != LBK_OK) {
        const std::string m = lbk_mm_last_error();
        if (s == LBK_UNSUPPORTED_FORMAT) throw UnsupportedFormatError(m);
        if (s == LBK_FORMAT_ERROR) throw FormatError(m);
        detail::check(s);
    }
    int32_t nr = 0, nc = 0;
    int64_t ne = 0;
    const int32_t *r = nullptr, *c = nullptr;
    const double* v = nullptr;
    lbk_mm_info(h, &nr, &nc, &ne);
    lbk_mm_entries(h, &r, &c, &v);
    std::vector<MatrixEntry> entries(static_cast<std::size_t>(ne));
    for (int64_t i = 0; i < ne; ++i) entries[i] = {r[i], c[i], v[i]};
    lbk_mm_free(h);
    return coo_from_entries(std::move(exec), nr, nc, entries);
}

inline std::vector<MatrixEntry> coo_to_entries(const CooMatrix& m)
{
    auto r = array_to_host<int32_t>(m.row_idx), c = array_to_host<int32_t>(m.col_idx);
    auto v = array_to_host<double>(m.vals);
    std::vector<MatrixEntry> out(v.size());
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = {r[i], c[i], v[i]};
    return out;
}

inline CsrMatrix coo_to_csr(const CooMatrix& m)
{
    auto e = m.executor();
    CsrMatrix out{m.nrows, m.ncols, DeviceArray(e, ElementKind::int32, std::size_t(m.nrows) + 1),
                  clone_array(m.col_idx, e), clone_array(m.vals, e)};
    auto d = m.desc();
    detail::check(lbk_coo_to_csr(e->handle(), &d, out.row_ptr.as<int32_t>()), e->handle());
    e->synchronize();
    return out;
}

inline CooMatrix csr_to_coo(const CsrMatrix& m)
{
    auto e = m.executor();
    CooMatrix out{m.nrows, m.ncols, DeviceArray(e, ElementKind::int32, m.nnz()),
                  clone_array(m.col_idx, e), clone_array(m.vals, e)};
    auto d = m.desc();
    detail::check(lbk_csr_to_coo(e->handle(), &d, out.row_idx.as<int32_t>()), e->handle());
    e->synchronize();
    return out;
}

inline EllMatrix csr_to_ell(const CsrMatrix& m)
{
    auto e = m.executor();
    auto d = m.desc();
    int32_t w = 0;
    detail::check(lbk_csr_ell_width(e->handle(), &d, &w), e->handle());
    const std::size_t slots = std::size_t(w) * m.nrows;
    EllMatrix out{m.nrows, m.ncols, w, m.nrows, static_cast<int64_t>(m.nnz()),
                  DeviceArray(e, ElementKind::int32, slots), DeviceArray(e, ElementKind::float64, slots)};
    detail::check(lbk_csr_to_ell(e->handle(), &d, w, m.nrows, out.col_idx.as<int32_t>(),
                                 out.vals.data()),
                  e->handle());
    e->synchronize();
    return out;
}

inline SellpMatrix csr_to_sellp(const CsrMatrix& m, int32_t slice_size = 32)
{
    auto e = m.executor();
    auto d = m.desc();
    const int32_t ns = (m.nrows + slice_size - 1) / slice_size;
    SellpMatrix out;
    out.nrows = m.nrows;
    out.ncols = m.ncols;
    out.slice_size = slice_size;
    out.nslices = ns;
    out.logical_nnz = static_cast<int64_t>(m.nnz());
    out.slice_lengths = DeviceArray(e, ElementKind::int32, ns);
    out.slice_sets = DeviceArray(e, ElementKind::int32, std::size_t(ns) + 1);
    int64_t stored = 0;
    detail::check(lbk_csr_sellp_plan(e->handle(), &d, slice_size, out.slice_lengths.as<int32_t>(),
                                     out.slice_sets.as<int32_t>(), &stored),
                  e->handle());
    out.col_idx = DeviceArray(e, ElementKind::int32, stored);
    out.vals = DeviceArray(e, ElementKind::float64, stored);
    detail::check(lbk_csr_to_sellp(e->handle(), &d, slice_size, out.slice_sets.as<int32_t>(),
                                   out.col_idx.as<int32_t>(), out.vals.data()),
                  e->handle());
    e->synchronize();
    return out;
}

inline void validate(const CooMatrix& m)
{
    auto e = m.executor();
    auto d = m.desc();
    detail::check(lbk_validate_coo(e->handle(), &d), e->handle());
}
inline void validate(const CsrMatrix& m)
{
    auto e = m.executor();
    auto d = m.desc();
    detail::check(lbk_validate_csr(e->handle(), &d), e->handle());
}

// ------------------------------------------------------------------ kernels
namespace detail {
inline void same_size(std::size_t a, std::size_t b, const char* what)
{
    if (a != b)
        throw ShapeError(std::string(what) + ": size mismatch, " + std::to_string(a) + " vs " +
                         std::to_string(b));
}
inline void same_space(const std::shared_ptr<Executor>& a, const std::shared_ptr<Executor>& b,
                       const char* what)
{
    if (a != b) throw PlacementError(std::string(what) + ": operands live on different executors");
}
}  // namespace detail

inline void axpy(double alpha, const DenseVector& x, DenseVector& y)
{
    detail::same_size(x.size(), y.size(), "axpy");
    detail::same_space(x.executor(), y.executor(), "axpy");
    auto e = y.executor();
    detail::check(lbk_axpy_f64(e->handle(), static_cast<int64_t>(x.size()), alpha,
                               x.values.as<double>(), y.values.as<double>()),
                  e->handle());
    e->synchronize();
}
inline void scal(double alpha, DenseVector& x)
{
    auto e = x.executor();
    detail::check(lbk_scal_f64(e->handle(), static_cast<int64_t>(x.size()), alpha, x.values.as<double>()),
                  e->handle());
    e->synchronize();
}
inline void fill(DenseVector& x, double value)
{
    auto e = x.executor();
    detail::check(lbk_fill_f64(e->handle(), static_cast<int64_t>(x.size()), value, x.values.as<double>()),
                  e->handle());
    e->synchronize();
}
inline double dot(const DenseVector& x, const DenseVector& y)
{
    detail::same_size(x.size(), y.size(), "dot");
    detail::same_space(x.executor(), y.executor(), "dot");
    auto e = x.executor();
    double r = 0.0;
    detail::check(lbk_dot_f64(e->handle(), static_cast<int64_t>(x.size()), x.values.as<double>(),
                              y.values.as<double>(), &r),
                  e->handle());
    return r;
}
inline double nrm2(const DenseVector& x)
{
    auto e = x.executor();
    double r = 0.0;
    detail::check(lbk_nrm2_f64(e->handle(), static_cast<int64_t>(x.size()), x.values.as<double>(), &r),
                  e->handle());
    return r;
}

// kernels.hpp:58-60, 99-113: the BabelStream-style calibration set and the
// flops sweep (reference.cpp:92-130, fma_chain.hpp)
enum class StreamOp { copy, mul, add, triad, dot };
inline const char* to_string(StreamOp op)
{
    switch (op) {
    case StreamOp::copy: return "copy";
    case StreamOp::mul: return "mul";
    case StreamOp::add: return "add";
    case StreamOp::triad: return "triad";
    case StreamOp::dot: return "dot";
    }
    return "?";
}
/// copy c<-a, mul b<-scalar*c, add c<-a+b, triad a<-b+scalar*c; returns the
/// dot product for StreamOp::dot and 0 otherwise (kernels.hpp:99-103).
inline double stream_kernel(StreamOp op, DenseVector& a, DenseVector& b, DenseVector& c,
                            double scalar)
{
    detail::same_size(a.size(), b.size(), "stream_kernel");
    detail::same_size(a.size(), c.size(), "stream_kernel");
    auto e = a.executor();
    const auto n = static_cast<int64_t>(a.size());
    double r = 0.0;
    lbk_status st = LBK_OK;
    switch (op) {
    case StreamOp::copy: st = lbk_stream_copy_f64(e->handle(), n, a.values.as<double>(), c.values.as<double>()); break;
    case StreamOp::mul: st = lbk_stream_mul_f64(e->handle(), n, scalar, c.values.as<double>(), b.values.as<double>()); break;
    case StreamOp::add:
        st = lbk_stream_add_f64(e->handle(), n, a.values.as<double>(), b.values.as<double>(), c.values.as<double>());
        break;
    case StreamOp::triad:
        st = lbk_stream_triad_f64(e->handle(), n, scalar, b.values.as<double>(), c.values.as<double>(),
                                  a.values.as<double>());
        break;
    case StreamOp::dot: st = lbk_stream_dot_f64(e->handle(), n, a.values.as<double>(), b.values.as<double>(), &r); break;
    }
    detail::check(st, e->handle());
    e->synchronize();
    return r;
}
/// x_i <- fma_chain(x_i, fma_per_element) (kernels.hpp:105-109).
inline void flops_sweep(DenseVector& x, int fma_per_element)
{
    if (fma_per_element < 0) throw UsageError("fma count must be nonnegative");
    auto e = x.executor();
    detail::check(lbk_flops_sweep_f64(e->handle(), static_cast<int64_t>(x.size()), fma_per_element,
                                      x.values.as<double>()),
                  e->handle());
    e->synchronize();
}
/// Bytes touched by one stream op over n doubles (api.cpp:170-182).
inline std::size_t stream_bytes(StreamOp op, std::size_t n)
{
    return (op == StreamOp::add || op == StreamOp::triad ? 3 : 2) * n * sizeof(double);
}

namespace detail {
template <class M>
void spmv_checks(const M& A, const DenseVector& x, const DenseVector& y, const char* what)
{
    same_size(static_cast<std::size_t>(A.ncols), x.size(), what);
    same_size(static_cast<std::size_t>(A.nrows), y.size(), what);
    same_space(A.executor(), x.executor(), what);
    same_space(A.executor(), y.executor(), what);
}
}  // namespace detail

// y <- A x (api.cpp:113-140), and the advanced apply y <- alpha A x + beta y.
inline void spmv_csr(const CsrMatrix& A, const DenseVector& x, DenseVector& y)
{
    detail::spmv_checks(A, x, y, "spmv_csr");
    auto e = A.executor();
    auto d = A.desc();
    detail::check(lbk_spmv_csr_f64(e->handle(), &d, x.values.as<double>(), y.values.as<double>()),
                  e->handle());
    e->synchronize();
}
inline void spmv_csr(double alpha, const CsrMatrix& A, const DenseVector& x, double beta, DenseVector& y)
{
    detail::spmv_checks(A, x, y, "spmv_csr");
    auto e = A.executor();
    auto d = A.desc();
    detail::check(lbk_spmv_csr_adv_f64(e->handle(), alpha, &d, x.values.as<double>(), beta,
                                       y.values.as<double>()),
                  e->handle());
    e->synchronize();
}
inline void spmv_coo(const CooMatrix& A, const DenseVector& x, DenseVector& y)
{
    detail::spmv_checks(A, x, y, "spmv_coo");
    auto e = A.executor();
    auto d = A.desc();
    detail::check(lbk_spmv_coo_f64(e->handle(), &d, x.values.as<double>(), y.values.as<double>()),
                  e->handle());
    e->synchronize();
}
inline void spmv_ell(const EllMatrix& A, const DenseVector& x, DenseVector& y)
{
    detail::spmv_checks(A, x, y, "spmv_ell");
    auto e = A.executor();
    auto d = A.desc();
    detail::check(lbk_spmv_ell_f64(e->handle(), &d, x.values.as<double>(), y.values.as<double>()),
                  e->handle());
    e->synchronize();
}
inline void spmv_sellp(const SellpMatrix& A, const DenseVector& x, DenseVector& y)
{
    detail::spmv_checks(A, x, y, "spmv_sellp");
    auto e = A.executor();
    auto d = A.desc();
    detail::check(lbk_spmv_sellp_f64(e->handle(), &d, x.values.as<double>(), y.values.as<double>()),
                  e->handle());
    e->synchronize();
}

// ------------------------------------------------------------------ solvers
enum class SolverKind { cg, bicgstab, cgs, gmres };
inline const char* to_string(SolverKind k)
{
    switch (k) {
    case SolverKind::cg: return "cg";
    case SolverKind::bicgstab: return "bicgstab";
    case SolverKind::cgs: return "cgs";
    default: return "gmres";
    }
}
enum class ResidualMode { true_residual, recurrence };

struct SolverConfig {
    SolverKind kind = SolverKind::cg;
    int max_iters = 1000;
    double rel_tol = 1e-10;
    int gmres_restart = 30;
    std::optional<int> fixed_iters{};
    ResidualMode residual_mode = ResidualMode::true_residual;  // B200 addition
};

struct SolveResult {
    bool converged = false;
    int iterations = 0;
    double final_rel_residual = 0.0;
    std::vector<double> residual_history;
    double elapsed = 0.0;
    std::int64_t flop_count = 0;
};

namespace detail {
template <class M, class F>
SolveResult solve_with(const M& A, const DenseVector& b, DenseVector& x, const SolverConfig& c, F&& call)
{
    if (c.fixed_iters && *c.fixed_iters < 1) throw ConfigurationError("fixed_iters must be positive");
    if (A.nrows != A.ncols)
        throw ShapeError("solve requires a square matrix, got " + std::to_string(A.nrows) + "x" +
                         std::to_string(A.ncols));
    same_size(b.size(), static_cast<std::size_t>(A.nrows), "solve");
    same_size(x.size(), static_cast<std::size_t>(A.nrows), "solve");
    same_space(A.executor(), b.executor(), "solve");
    same_space(A.executor(), x.executor(), "solve");
    lbk_solver_cfg cfg{static_cast<int32_t>(c.kind), c.max_iters, c.rel_tol,
                       c.fixed_iters ? *c.fixed_iters : 0,
                       c.residual_mode == ResidualMode::recurrence ? 1 : 0, c.gmres_restart};
    lbk_solve_result r{};
    std::vector<double> hist(static_cast<std::size_t>(c.fixed_iters ? *c.fixed_iters : c.max_iters) + 2);
    auto e = A.executor();
    const lbk_status s = call(e->handle(), &cfg, &r, hist.data(), static_cast<int32_t>(hist.size()));
    check(s, e->handle(), r.breakdown_iter);
    hist.resize(static_cast<std::size_t>(r.history_len));
    return SolveResult{r.converged != 0, r.iterations, r.final_rel_residual, std::move(hist), r.elapsed,
                       r.flop_count};
}
}  // namespace detail

inline SolveResult solve(const CsrMatrix& A, const DenseVector& b, DenseVector& x, const SolverConfig& c)
{
    const auto d = A.desc();
    return detail::solve_with(A, b, x, c, [&](lbk_ctx h, auto* cfg, auto* r, double* hist, int32_t cap) {
        return lbk_solve_csr(h, &d, b.values.as<double>(), x.values.as<double>(), cfg, r, hist, cap);
    });
}
inline SolveResult solve(const CooMatrix& A, const DenseVector& b, DenseVector& x, const SolverConfig& c)
{
    const auto d = A.desc();
    return detail::solve_with(A, b, x, c, [&](lbk_ctx h, auto* cfg, auto* r, double* hist, int32_t cap) {
        return lbk_solve_coo(h, &d, b.values.as<double>(), x.values.as<double>(), cfg, r, hist, cap);
    });
}

// krylov.cpp:601-616
inline DenseVector apply_operator(const CsrMatrix& A, const DenseVector& v)
{
    DenseVector y = make_vector(A.executor(), static_cast<std::size_t>(A.nrows));
    spmv_csr(A, v, y);
    return y;
}
inline DenseVector apply_operator(const CooMatrix& A, const DenseVector& v)
{
    DenseVector y = make_vector(A.executor(), static_cast<std::size_t>(A.nrows));
    spmv_coo(A, v, y);
    return y;
}

// krylov.hpp:62-89: one restarted-GMRES cycle
struct GmresCycleResult {
    double rel_residual = 0.0;
    int steps = 0;
    bool happy_breakdown = false;
};
inline GmresCycleResult gmres_restart_cycle(const CsrMatrix& A, const DenseVector& b, DenseVector& x,
                                            int restart,
                                            std::vector<DenseVector>* basis_out = nullptr)
{
    if (restart < 1) throw ConfigurationError("restart must be positive");
    detail::same_size(static_cast<std::size_t>(A.nrows), b.size(), "gmres_restart_cycle");
    detail::same_size(static_cast<std::size_t>(A.nrows), x.size(), "gmres_restart_cycle");
    auto e = A.executor();
    const auto n = static_cast<std::size_t>(A.nrows);
    DenseVector basis;
    if (basis_out) basis = make_vector(e, n * static_cast<std::size_t>(restart + 1));
    const auto d = A.desc();
    lbk_gmres_cycle_result r{};
    detail::check(lbk_gmres_restart_cycle_csr(e->handle(), &d, b.values.as<double>(),
                                              x.values.as<double>(), restart,
                                              basis_out ? basis.values.as<double>() : nullptr,
                                              basis_out ? restart + 1 : 0, &r),
                  e->handle());
    if (basis_out) {
        basis_out->clear();
        for (int i = 0; i < r.basis_count; ++i) {
            DenseVector v = make_vector(e, n);
            detail::check(lbk_memcpy_d2d(e->handle(), v.values.as<double>(),
                                         basis.values.as<double>() + static_cast<std::size_t>(i) * n,
                                         n * sizeof(double)),
                          e->handle());
            basis_out->push_back(std::move(v));
        }
        e->synchronize();
    }
    return GmresCycleResult{r.rel_residual, r.steps, r.happy_breakdown != 0};
}

}  // namespace lbk::larch

#endif  // LBK_LARCH_HPP
