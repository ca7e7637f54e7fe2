// tests/cpp/test_parity.cpp -- C++ parity tests of the host façade
// (include/lbk/larch.hpp) against the reference library itself.
//
// Written the way the reference's own (missing) tests/test_kernels.cpp and
// tests/test_krylov.cpp would be (tests/CMakeLists.txt:1-8):
// the code under test uses the reference's names through
// `namespace larch = lbk::larch`, and the oracle is the reference library
// (oracle/_ref/liblarch_ref.so, FMA-free) through its C driver
// (oracle/ref_driver.cpp) plus the restatement's generators
// (oracle/_build/liboracle_port.so).  Needs a GPU; exit status 0 = pass.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "lbk/larch.hpp"

namespace larch = lbk::larch;

extern "C" {
// oracle/ref_driver.cpp (the reference's public API, C-wrapped)
int ref_spmv(int exec_kind, int workers, int fmt, int nrows, int ncols, int64_t nnz, const int* ptr,
             const int* cols, const double* vals, const double* x, double* y, int reps, double* sec);
int ref_solve(int exec_kind, int workers, int fmt, int kind, int n, int64_t nnz, const int* ptr,
              const int* cols, const double* vals, const double* b, double* x, int max_iters,
              double rel_tol, int fixed_iters, int restart, double* hist, int hist_cap, int* oi,
              double* od, int64_t* flops);
int ref_csr_to_coo(int nrows, int ncols, int64_t nnz, const int* row_ptr, const int* cols,
                   const double* vals, int* rows_out, int* cols_out, double* vals_out);
// oracle/port.cpp generators
int64_t port_stencil_nnz(int kind, int m);
void port_stencil_csr(int kind, int m, double gamma, int32_t* row_ptr, int32_t* cols, double* vals);
}

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_fail;                                                                \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_AS(expr, Ex)      \
    do {                               \
        bool thrown_ = false;          \
        try {                          \
            expr;                      \
        } catch (const Ex&) {          \
            thrown_ = true;            \
        }                              \
        CHECK(thrown_ && #Ex);         \
    } while (0)

struct HostCsr {
    int n = 0, m = 0;
    std::vector<int> ptr, cols;
    std::vector<double> vals;
};

static larch::CsrMatrix upload(std::shared_ptr<larch::Executor> e, const HostCsr& h)
{
    return larch::CsrMatrix{h.n, h.m, larch::array_from_host<int32_t>(e, h.ptr),
                            larch::array_from_host<int32_t>(e, h.cols),
                            larch::array_from_host<double>(e, h.vals)};
}

static HostCsr stencil(int kind, int m, double gamma = 0.0)
{
    HostCsr h;
    h.n = h.m = kind == 0 ? m * m : m * m * m;
    const int64_t nnz = port_stencil_nnz(kind, m);
    h.ptr.resize(h.n + 1);
    h.cols.resize(nnz);
    h.vals.resize(nnz);
    port_stencil_csr(kind, m, gamma, h.ptr.data(), h.cols.data(), h.vals.data());
    return h;
}

static HostCsr random_csr(std::mt19937_64& rng, int n, int m, double density)
{
    HostCsr h;
    h.n = n;
    h.m = m;
    h.ptr.push_back(0);
    std::uniform_real_distribution<double> U(0, 1), V(-1, 1);
    for (int r = 0; r < n; ++r) {
        for (int c = 0; c < m; ++c)
            if (U(rng) < density) {
                h.cols.push_back(c);
                h.vals.push_back(V(rng));
            }
        h.ptr.push_back(static_cast<int>(h.cols.size()));
    }
    return h;
}

static void test_spec_kats(std::shared_ptr<larch::Executor> e)
{
    // SPEC.md:416-420
    HostCsr I{3, 3, {0, 1, 2, 3}, {0, 1, 2}, {1, 1, 1}};
    auto A = upload(e, I);
    std::vector<double> x123{1, 2, 3};
    auto y = larch::apply_operator(A, larch::vector_from(e, x123));
    CHECK((larch::vector_to_host(y) == std::vector<double>{1, 2, 3}));
    HostCsr U{2, 2, {0, 2, 3}, {0, 1, 1}, {1, 2, 3}};
    std::vector<double> ones{1, 1};
    auto yu = larch::apply_operator(larch::csr_to_coo(upload(e, U)), larch::vector_from(e, ones));
    CHECK((larch::vector_to_host(yu) == std::vector<double>{3, 3}));
    std::vector<larch::MatrixEntry> ent{{0, 0, 5.0}};
    auto C = larch::coo_from_entries(e, 2, 2, ent);
    std::vector<double> x27{2, 7};
    CHECK((larch::vector_to_host(larch::apply_operator(C, larch::vector_from(e, x27))) ==
           std::vector<double>{10, 0}));
    // canonical assembly and row pointers
    std::vector<larch::MatrixEntry> dup{{1, 0, 1.0}, {0, 1, 2.0}, {1, 0, 3.0}};
    auto D = larch::coo_from_entries(e, 2, 2, dup);
    CHECK((larch::coo_to_entries(D) == std::vector<larch::MatrixEntry>{{0, 1, 2.0}, {1, 0, 4.0}}));
    std::vector<larch::MatrixEntry> r001{{0, 0, 1.0}, {0, 1, 1.0}, {1, 1, 1.0}};
    auto P = larch::coo_to_csr(larch::coo_from_entries(e, 2, 2, r001));
    CHECK((larch::array_to_host<int32_t>(P.row_ptr) == std::vector<int32_t>{0, 2, 3}));
    auto Z = larch::coo_to_csr(larch::coo_from_entries(e, 3, 3, {}));
    CHECK((larch::array_to_host<int32_t>(Z.row_ptr) == std::vector<int32_t>{0, 0, 0, 0}));
    std::vector<larch::MatrixEntry> bad{{2, 0, 1.0}};
    CHECK_THROWS_AS(larch::coo_from_entries(e, 2, 2, bad), larch::FormatError);
}

// Normwise max-abs ratio (tests/support/test_utils.hpp max_rel_diff idea):
// <= 1e-12 everywhere, and bit-identical on rows of <= 32 entries, where the
// kernels keep the reference's sequential order.
static bool matches(const std::vector<double>& y, const std::vector<double>& yr, const HostCsr& h)
{
    double d = 0, m = 0;
    bool exact = true;
    for (size_t i = 0; i < y.size(); ++i) {
        d = std::max(d, std::fabs(y[i] - yr[i]));
        m = std::max(m, std::fabs(yr[i]));
        if (h.ptr[i + 1] - h.ptr[i] <= 32) exact = exact && y[i] == yr[i];
    }
    return exact && d <= 1e-12 * (m > 0 ? m : 1);
}

static void test_random_vs_reference(std::shared_ptr<larch::Executor> e)
{
    // SPEC.md:633-645 #4/#5: 100 random matrices, n <= 200, backends agree
    // (normwise 1e-12; ELL / SELL-P sum every row sequentially -> bit-for-bit)
    std::mt19937_64 rng(7);
    for (int t = 0; t < 100; ++t) {
        const int n = 1 + static_cast<int>(rng() % 200), m = 1 + static_cast<int>(rng() % 200);
        const double dens = (rng() % 100) / 300.0;
        HostCsr h = random_csr(rng, n, m, dens);
        std::vector<double> x(m);
        std::uniform_real_distribution<double> V(-1, 1);
        for (auto& v : x) v = V(rng);
        std::vector<double> yr(n);
        double sec = 0;
        CHECK(ref_spmv(0, 1, 1, n, m, h.vals.size(), h.ptr.data(), h.cols.data(), h.vals.data(), x.data(),
                       yr.data(), 0, &sec) == 0);
        auto A = upload(e, h);
        auto xv = larch::vector_from(e, x);
        auto y = larch::make_vector(e, n);
        larch::spmv_csr(A, xv, y);
        CHECK(matches(larch::vector_to_host(y), yr, h));
        auto C = larch::csr_to_coo(A);
        std::vector<int> rr(h.vals.size() + 1), rc(h.vals.size() + 1);
        std::vector<double> rv(h.vals.size() + 1);
        CHECK(ref_csr_to_coo(n, m, h.vals.size(), h.ptr.data(), h.cols.data(), h.vals.data(), rr.data(),
                             rc.data(), rv.data()) == 0);
        rr.resize(h.vals.size());
        CHECK(larch::array_to_host<int32_t>(C.row_idx) == rr);
        larch::spmv_coo(C, xv, y);
        CHECK(matches(larch::vector_to_host(y), yr, h));
        auto B = larch::coo_to_csr(C);
        CHECK(larch::array_to_host<int32_t>(B.row_ptr) == h.ptr);
        larch::validate(B);
        larch::validate(C);
        auto E = larch::csr_to_ell(A);
        larch::spmv_ell(E, xv, y);
        CHECK(larch::vector_to_host(y) == yr);
        auto S = larch::csr_to_sellp(A, 32);
        larch::spmv_sellp(S, xv, y);
        CHECK(larch::vector_to_host(y) == yr);
    }
}

static void test_blas1_and_errors(std::shared_ptr<larch::Executor> e)
{
    std::vector<double> a(1000), b(1000);
    for (int i = 0; i < 1000; ++i) {
        a[i] = std::sin(i);
        b[i] = std::cos(i);
    }
    auto x = larch::vector_from(e, a), y = larch::vector_from(e, b);
    double ref = 0;
    for (int i = 0; i < 1000; ++i) ref += a[i] * b[i];
    CHECK(std::fabs(larch::dot(x, y) - ref) <= 1e-12 * 1000);
    CHECK(larch::dot(x, y) == larch::dot(x, y));  // deterministic
    larch::axpy(2.0, x, y);
    auto yh = larch::vector_to_host(y);
    bool ok = true;
    for (int i = 0; i < 1000; ++i) ok = ok && yh[i] == b[i] + 2.0 * a[i];
    CHECK(ok);
    auto z = larch::make_vector(e, 999);
    CHECK_THROWS_AS(larch::axpy(1.0, x, z), larch::ShapeError);
    HostCsr h{2, 3, {0, 1, 2}, {0, 2}, {1, 2}};
    auto A = upload(e, h);
    auto y2 = larch::make_vector(e, 2), x2 = larch::make_vector(e, 2);
    CHECK_THROWS_AS(larch::spmv_csr(A, x2, y2), larch::ShapeError);
    auto e2 = larch::create_executor(larch::ExecutorKind::cuda);
    auto x3 = larch::make_vector(e2, 3);
    CHECK_THROWS_AS(larch::spmv_csr(A, x3, y2), larch::PlacementError);
    auto s = larch::zeros(e, 2);
    larch::SolverConfig cfg;
    cfg.kind = larch::SolverKind::gmres;
    cfg.gmres_restart = 0;  // krylov.cpp:466-471: must lie in [1, max_iters]
    HostCsr sq{2, 2, {0, 1, 2}, {0, 1}, {1, 1}};
    auto Sq = upload(e, sq);
    CHECK_THROWS_AS(larch::solve(Sq, s, s, cfg), larch::ConfigurationError);
    // arena capacity -> OutOfMemoryError (executor.cpp:254-265)
    auto small = larch::create_executor(larch::ExecutorKind::cuda, {0, 1024});
    CHECK_THROWS_AS(larch::make_vector(small, 1000), larch::OutOfMemoryError);
}

static void test_solvers(std::shared_ptr<larch::Executor> e)
{
    // [[4,1],[1,3]] x = [1,2] -> [1/11, 7/11]
    HostCsr h{2, 2, {0, 2, 4}, {0, 1, 0, 1}, {4, 1, 1, 3}};
    auto A = upload(e, h);
    std::vector<double> b{1, 2};
    auto bv = larch::vector_from(e, b);
    auto x = larch::zeros(e, 2);
    larch::SolverConfig cfg;
    cfg.rel_tol = 1e-12;
    auto r = larch::solve(A, bv, x, cfg);
    auto xh = larch::vector_to_host(x);
    CHECK(std::fabs(xh[0] - 1.0 / 11) <= 1e-12 && std::fabs(xh[1] - 7.0 / 11) <= 1e-12);
    CHECK(r.converged);
    // b = 0 -> 0 iterations, history [0] (krylov.cpp:479-482)
    auto z = larch::zeros(e, 2);
    auto r0 = larch::solve(A, z, x, cfg);
    CHECK(r0.iterations == 0 && r0.residual_history.size() == 1 && r0.residual_history[0] == 0.0);
    // breakdown: <p, Ap> = 0 at iteration 1
    HostCsr sw{2, 2, {0, 1, 2}, {1, 0}, {1, 1}};
    std::vector<double> b10{1, 0};
    auto xb = larch::zeros(e, 2);
    bool bd = false;
    try {
        larch::solve(upload(e, sw), larch::vector_from(e, b10), xb, cfg);
    } catch (const larch::BreakdownError& err) {
        bd = err.iteration == 1;
    }
    CHECK(bd);
    // CG / BiCGSTAB on 7-pt 24^3 against the reference solve
    for (int kind = 0; kind < 2; ++kind) {
        HostCsr s = stencil(1, 24, kind ? 0.5 : 0.0);
        std::vector<double> ones(s.n, 1.0), bb(s.n);
        double sec = 0;
        ref_spmv(0, 1, 1, s.n, s.n, s.vals.size(), s.ptr.data(), s.cols.data(), s.vals.data(), ones.data(),
                 bb.data(), 0, &sec);
        std::vector<double> xr(s.n, 0.0), hist(20002), od(2);
        int oi[3];
        int64_t fl = 0;
        CHECK(ref_solve(0, 1, 1, kind, s.n, s.vals.size(), s.ptr.data(), s.cols.data(), s.vals.data(),
                        bb.data(), xr.data(), 20000, 1e-8, 0, 30, hist.data(), 20002, oi, od.data(),
                        &fl) == 0);
        auto As = upload(e, s);
        auto xs = larch::zeros(e, s.n);
        larch::SolverConfig c2;
        c2.kind = kind ? larch::SolverKind::bicgstab : larch::SolverKind::cg;
        c2.rel_tol = 1e-8;
        c2.max_iters = 20000;
        auto rs = larch::solve(As, larch::vector_from(e, bb), xs, c2);
        CHECK(std::abs(rs.iterations - oi[1]) <= 1);
        if (rs.iterations == oi[1]) CHECK(rs.flop_count == fl);
        CHECK(rs.converged && rs.final_rel_residual <= 1e-8);
        std::printf("  %s 24^3: reference %d iterations, B200 %d\n", kind ? "bicgstab" : "cg", oi[1],
                    rs.iterations);
    }
}

static void test_matrix_market(std::shared_ptr<larch::Executor> e)
{
    // io.cpp:71-191: symmetric expansion, duplicates summed, 1-based indices
    const char* path = "/tmp/lbk_parity_test.mtx";
    {
        std::FILE* f = std::fopen(path, "w");
        std::fputs("%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 4\n1 1 2\n2 1 -1\n"
                   "3 3 5\n2 1 0.5\n", f);
        std::fclose(f);
    }
    auto M = larch::read_matrix_market(path, e);
    CHECK((larch::coo_to_entries(M) ==
           std::vector<larch::MatrixEntry>{{0, 0, 2.0}, {0, 1, -0.5}, {1, 0, -0.5}, {2, 2, 5.0}}));
    {
        std::FILE* f = std::fopen(path, "w");
        std::fputs("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", f);
        std::fclose(f);
    }
    CHECK_THROWS_AS(larch::read_matrix_market(path, e), larch::UnsupportedFormatError);
    std::remove(path);
}

int main()
{
    auto e = larch::create_executor(larch::ExecutorKind::cuda);
    std::printf("executor: %s\n", e->describe().c_str());
    test_spec_kats(e);
    test_random_vs_reference(e);
    test_blas1_and_errors(e);
    test_solvers(e);
    test_matrix_market(e);
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
