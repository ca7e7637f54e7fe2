// oracle/xkrylov.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/port.h).
//
// CPU restatement of the reference's CG and BiCGSTAB (src/solver/krylov.cpp
// :119-161 run_cg, :164-230 run_bicgstab; Workspace :36-88; paths relative
// to /root/reference/proj) with ONE deliberate change: every dot product
// and norm is the exactly rounded sum of the rounded products,
//     dot(x, y) = RNE( sum_i RN(x_i * y_i) ),
// instead of ref_dot's sequential sum (reference.cpp:46-56).  That is the
// reduction order of the product's partition-independent ("exact")
// reduction mode: with it the solver's scalars do not depend on how the
// rows are split over blocks, tiles or GPUs, so its histories are the same
// bits at every GPU count.  Element-wise ops restate reference.cpp:17-43
// FMA-free (y + (a x), two roundings), SpMV restates reference.cpp:74-89.
//
// The exact sum is pinned independently: tests/test_oracle.py checks
// port_xdot against Python's math.fsum (also an exactly rounded sum).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "port.h"

namespace {

// Exact accumulator: the sum as an integer in units of 2^-1074 (the
// smallest subnormal), held in 32-bit digits with signed 64-bit carry room.
struct XAcc {
    static constexpr int kLimbs = 67;
    int64_t l[kLimbs] = {};
    bool nonfinite = false;
    double nf = 0.0;  // inf/nan propagated like a plain sum

    void add(double v)
    {
        if (v == 0.0) return;
        if (!std::isfinite(v)) {
            nonfinite = true;
            nf += v;
            return;
        }
        uint64_t bits;
        std::memcpy(&bits, &v, 8);
        const int e = static_cast<int>((bits >> 52) & 0x7ff);
        uint64_t m = bits & ((uint64_t(1) << 52) - 1);
        if (e) m |= uint64_t(1) << 52;
        const int pos = e ? e - 1 : 0;  // bit position of m's lsb
        const int li = pos >> 5, off = pos & 31;
        // m << off spans at most 85 bits: three 32-bit digits
        const unsigned __int128 w = static_cast<unsigned __int128>(m) << off;
        const int64_t d0 = static_cast<int64_t>(static_cast<uint64_t>(w) & 0xffffffffu);
        const int64_t d1 = static_cast<int64_t>(static_cast<uint64_t>(w >> 32) & 0xffffffffu);
        const int64_t d2 = static_cast<int64_t>(static_cast<uint64_t>(w >> 64));
        if (bits >> 63) {
            l[li] -= d0;
            l[li + 1] -= d1;
            l[li + 2] -= d2;
        } else {
            l[li] += d0;
            l[li + 1] += d1;
            l[li + 2] += d2;
        }
    }

    void merge(const XAcc& o)
    {
        for (int i = 0; i < kLimbs; ++i) l[i] += o.l[i];
        if (o.nonfinite) {
            nonfinite = true;
            nf += o.nf;
        }
    }

    // Round to nearest, ties to even.
    double round() const
    {
        if (nonfinite) return nf;
        int64_t d[kLimbs];
        std::memcpy(d, l, sizeof d);
        for (int i = 0; i + 1 < kLimbs; ++i) {  // carry-normalise to [0, 2^32)
            const int64_t c = d[i] >> 32;  // arithmetic shift: floor division
            d[i] -= c * (int64_t(1) << 32);
            d[i + 1] += c;
        }
        bool neg = d[kLimbs - 1] < 0;
        if (neg) {  // magnitude = -value: complement digits and add 1
            int64_t carry = 1;
            for (int i = 0; i < kLimbs; ++i) {
                int64_t v = (0xffffffffLL - (d[i] & 0xffffffffLL)) + carry;
                carry = v >> 32;
                d[i] = v & 0xffffffffLL;
            }
        }
        int top = kLimbs - 1;
        while (top >= 0 && d[top] == 0) --top;
        if (top < 0) return 0.0;
        int hb = 31;
        while (!((d[top] >> hb) & 1)) --hb;
        const int msb = top * 32 + hb;  // bit position of the leading 1
        double r;
        if (msb < 53) {  // exact (subnormal or small): value < 2^53 units
            uint64_t v = 0;
            for (int i = top; i >= 0; --i) v = (v << 32) | static_cast<uint64_t>(d[i]);
            r = std::ldexp(static_cast<double>(v), -1074);
        } else {
            const int sh = msb - 52;  // drop sh low bits
            auto bit = [&](int p) -> uint64_t { return (d[p >> 5] >> (p & 31)) & 1; };
            uint64_t mant = 0;
            for (int p = msb; p >= sh; --p) mant = (mant << 1) | bit(p);
            const uint64_t rb = bit(sh - 1);
            bool sticky = false;
            for (int p = sh - 2; p >= 0 && !sticky; --p) sticky = bit(p) != 0;
            if (rb && (sticky || (mant & 1))) mant += 1;  // may carry to 2^53: still exact
            r = std::ldexp(static_cast<double>(mant), sh - 1074);
        }
        return neg ? -r : r;
    }
};

template <typename F>
void par_chunks(int64_t n, F&& f)
{
    unsigned t = std::max(1u, std::thread::hardware_concurrency());
    if (n < 65536) t = 1;
    std::vector<std::thread> th;
    for (unsigned w = 0; w < t; ++w)
        th.emplace_back([&, w] { f(n * w / t, n * (w + 1) / t, w); });
    for (auto& x : th) x.join();
}

double xdot(int64_t n, const double* x, const double* y)
{
    unsigned t = std::max(1u, std::thread::hardware_concurrency());
    std::vector<XAcc> part(t);
    par_chunks(n, [&](int64_t b, int64_t e, unsigned w) {
        for (int64_t i = b; i < e; ++i) part[w].add(x[i] * y[i]);
    });
    XAcc tot;
    for (auto& p : part) tot.merge(p);  // integer adds: order-free
    return tot.round();
}

struct Csr {
    int32_t n;
    const int32_t* rp;
    const int32_t* ci;
    const double* v;
    int64_t nnz;
};

// reference.cpp:74-89: y = A x, sum from 0.0 in ascending k, no FMA.
void spmv(const Csr& A, const double* x, double* y)
{
    par_chunks(A.n, [&](int64_t b, int64_t e, unsigned) {
        for (int64_t r = b; r < e; ++r) {
            double s = 0.0;
            for (int32_t k = A.rp[r]; k < A.rp[r + 1]; ++k) s += A.v[k] * x[A.ci[k]];
            y[r] = s;
        }
    });
}

// Workspace (krylov.cpp:36-88) with the exact dot and the reference flops.
struct Ws {
    Csr A;
    int64_t n;
    int64_t flops = 0;
    void apply(const double* in, double* out)
    {
        spmv(A, in, out);
        flops += 2 * A.nnz;
    }
    double dot(const double* x, const double* y)
    {
        flops += 2 * n;
        return xdot(n, x, y);
    }
    double norm(const double* x)
    {
        flops += 2 * n;
        return std::sqrt(xdot(n, x, x));
    }
    void axpy(double a, const double* x, double* y)
    {
        flops += 2 * n;
        par_chunks(n, [&](int64_t b, int64_t e, unsigned) {
            for (int64_t i = b; i < e; ++i) y[i] += a * x[i];
        });
    }
    void scal(double a, double* x)
    {
        flops += n;
        par_chunks(n, [&](int64_t b, int64_t e, unsigned) {
            for (int64_t i = b; i < e; ++i) x[i] *= a;
        });
    }
    double true_residual(const double* b, const double* x, double* scratch, double nb)
    {
        apply(x, scratch);
        scal(-1.0, scratch);
        axpy(1.0, b, scratch);
        return norm(scratch) / nb;
    }
};

using Vec = std::vector<double>;

// krylov.cpp:119-161
int run_cg(Ws& ws, const double* b, double* x, double nb, int limit, int fixed, double tol,
           std::vector<double>& hist, int* bd_iter)
{
    const int64_t n = ws.n;
    Vec r(n), p(n), q(n), scratch(n);
    ws.apply(x, r.data());
    ws.scal(-1.0, r.data());
    ws.axpy(1.0, b, r.data());
    hist.push_back(ws.norm(r.data()) / nb);
    if (!fixed && hist.back() <= tol) return 0;
    p = r;
    double rho = ws.dot(r.data(), r.data());
    bool frozen = false;
    for (int it = 1; it <= limit; ++it) {
        if (frozen) {
            hist.push_back(hist.back());
            continue;
        }
        ws.apply(p.data(), q.data());
        const double pq = ws.dot(p.data(), q.data());
        if (std::abs(pq) < 1e-30) return *bd_iter = it, 3;
        const double alpha = rho / pq;
        ws.axpy(alpha, p.data(), x);
        ws.axpy(-alpha, q.data(), r.data());
        const double rel = ws.true_residual(b, x, scratch.data(), nb);
        hist.push_back(rel);
        if (!fixed && rel <= tol) return 0;
        if (fixed && rel <= 1e-13) {
            frozen = true;
            continue;
        }
        const double rho_next = ws.dot(r.data(), r.data());
        if (std::abs(rho) < 1e-30) return *bd_iter = it, 3;
        const double beta = rho_next / rho;
        rho = rho_next;
        ws.scal(beta, p.data());
        ws.axpy(1.0, r.data(), p.data());
    }
    return 0;
}

// krylov.cpp:164-230
int run_bicgstab(Ws& ws, const double* b, double* x, double nb, int limit, int fixed,
                 double tol, std::vector<double>& hist, int* bd_iter)
{
    const int64_t n = ws.n;
    Vec r(n), rt, p, v(n), s(n), t(n), scratch(n);
    ws.apply(x, r.data());
    ws.scal(-1.0, r.data());
    ws.axpy(1.0, b, r.data());
    hist.push_back(ws.norm(r.data()) / nb);
    if (!fixed && hist.back() <= tol) return 0;
    rt = r;
    p = r;
    double rho = 0.0, alpha = 1.0, omega = 1.0;
    bool frozen = false;
    for (int it = 1; it <= limit; ++it) {
        if (frozen) {
            hist.push_back(hist.back());
            continue;
        }
        const double rho_next = ws.dot(rt.data(), r.data());
        if (it > 1) {
            if (std::abs(rho) < 1e-30) return *bd_iter = it, 3;
            if (std::abs(omega) < 1e-30) return *bd_iter = it, 3;
            const double beta = (rho_next / rho) * (alpha / omega);
            ws.axpy(-omega, v.data(), p.data());
            ws.scal(beta, p.data());
            ws.axpy(1.0, r.data(), p.data());
        }
        rho = rho_next;
        ws.apply(p.data(), v.data());
        const double rtv = ws.dot(rt.data(), v.data());
        if (std::abs(rtv) < 1e-30) return *bd_iter = it, 3;
        alpha = rho / rtv;
        s = r;
        ws.axpy(-alpha, v.data(), s.data());
        const double s_rel = ws.norm(s.data()) / nb;
        ws.apply(s.data(), t.data());
        const double tt = ws.dot(t.data(), t.data());
        if (std::abs(tt) < 1e-30) {
            if (s_rel > 1e-13) return *bd_iter = it, 3;
            omega = 0.0;
        } else {
            omega = ws.dot(t.data(), s.data()) / tt;
        }
        ws.axpy(alpha, p.data(), x);
        ws.axpy(omega, s.data(), x);
        r = s;
        ws.axpy(-omega, t.data(), r.data());
        const double rel = ws.true_residual(b, x, scratch.data(), nb);
        hist.push_back(rel);
        if (!fixed && rel <= tol) return 0;
        if (fixed && rel <= 1e-13) frozen = true;
    }
    return 0;
}

}  // namespace

extern "C" {

double port_xdot(int64_t n, const double* x, const double* y) { return xdot(n, x, y); }

double port_xsum(int64_t n, const double* v)
{
    XAcc a;
    for (int64_t i = 0; i < n; ++i) a.add(v[i]);
    return a.round();
}

// krylov.cpp:446-512 solve_impl (x0 given, zero-b short-circuit) around
// run_cg / run_bicgstab with exact dots.  kind: 0 CG, 1 BiCGSTAB.
// Returns 0 (ran; see *converged) or 3 (BreakdownError at *bd_iter).
int port_xsolve(int kind, int32_t n, const int32_t* rp, const int32_t* ci, const double* vals,
                const double* b, double* x, double tol, int max_iters, int fixed_iters,
                double* hist_out, int64_t hist_cap, int* iterations, int* converged,
                int64_t* flops, int* bd_iter)
{
    Ws ws{Csr{n, rp, ci, vals, rp[n]}, n};
    std::vector<double> hist;
    *bd_iter = -1;
    const double nb = ws.norm(b);
    int st = 0;
    if (nb == 0.0) {
        std::memset(x, 0, sizeof(double) * n);
        hist.push_back(0.0);
    } else {
        const int limit = fixed_iters > 0 ? fixed_iters : max_iters;
        st = kind == 0 ? run_cg(ws, b, x, nb, limit, fixed_iters > 0, tol, hist, bd_iter)
                       : run_bicgstab(ws, b, x, nb, limit, fixed_iters > 0, tol, hist, bd_iter);
    }
    *iterations = static_cast<int>(hist.size()) - 1;
    *converged = !hist.empty() && hist.back() <= tol;
    *flops = ws.flops;
    for (int64_t i = 0; i < static_cast<int64_t>(hist.size()) && i < hist_cap; ++i)
        hist_out[i] = hist[i];
    return st;
}

}  // extern "C"
