// oracle/port.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/port.h).
//
// CPU restatement of the reference's SpMV path and of the SURVEY.md App. B
// specs the reference lacks.  Built FMA-free (-ffp-contract=off) so sums
// reproduce the reference's bit patterns.
//
// Each function cites the reference code it restates (paths relative to
// /root/reference/proj) or the App. B rule it implements.
#include "port.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

// Row-parallel helper (no OpenMP runtime in this toolchain).  Per-row work
// is order-independent, so results do not depend on the thread count.
template <typename F>
void par_rows(int64_t n, F&& f)
{
    unsigned t = std::max(1u, std::thread::hardware_concurrency());
    if (n < 65536) t = 1;
    std::vector<std::thread> th;
    for (unsigned w = 0; w < t; ++w) {
        th.emplace_back([&, w] {
            const int64_t b = n * w / t, e = n * (w + 1) / t;
            for (int64_t i = b; i < e; ++i) f(i);
        });
    }
    for (auto& x : th) x.join();
}

inline int32_t clampi(int64_t v, int64_t lo, int64_t hi)
{
    return static_cast<int32_t>(std::min(std::max(v, lo), hi));
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- generators
// App. B "Stencils": row r = (k*m + i)*m + j (j fastest); entries emitted in
// ascending column order so coo_from_entries is a no-op sort.
int64_t port_stencil_nnz(int kind, int m)
{
    const int64_t mm = m;
    if (kind == 0) return 5 * mm * mm - 4 * mm;
    if (kind == 1) return 7 * mm * mm * mm - 6 * mm * mm;
    return (3 * mm - 2) * (3 * mm - 2) * (3 * mm - 2);
}

void port_stencil_csr(int kind, int m, double gamma, int32_t* row_ptr,
                      int32_t* cols, double* vals)
{
    int64_t k_out = 0;
    row_ptr[0] = 0;
    if (kind == 0) {
        // 2D 5-pt Poisson: diag 4, neighbours -1.
        for (int i = 0; i < m; ++i) {
            for (int j = 0; j < m; ++j) {
                const int64_t r = static_cast<int64_t>(i) * m + j;
                auto put = [&](int64_t c, double v) {
                    cols[k_out] = static_cast<int32_t>(c);
                    vals[k_out] = v;
                    ++k_out;
                };
                if (i > 0) put(r - m, -1.0);
                if (j > 0) put(r - 1, -1.0);
                put(r, 4.0);
                if (j < m - 1) put(r + 1, -1.0);
                if (i < m - 1) put(r + m, -1.0);
                row_ptr[r + 1] = static_cast<int32_t>(k_out);
            }
        }
        return;
    }
    const int64_t plane = static_cast<int64_t>(m) * m;
    for (int k = 0; k < m; ++k) {
        for (int i = 0; i < m; ++i) {
            for (int j = 0; j < m; ++j) {
                const int64_t r = (static_cast<int64_t>(k) * m + i) * m + j;
                auto put = [&](int64_t c, double v) {
                    cols[k_out] = static_cast<int32_t>(c);
                    vals[k_out] = v;
                    ++k_out;
                };
                if (kind == 1) {
                    // 7-pt upwind convection-diffusion: diag 6+3g,
                    // -(1+g) on k-1/i-1/j-1, -1 on k+1/i+1/j+1.
                    const double lo = -1.0 - gamma;
                    if (k > 0) put(r - plane, lo);
                    if (i > 0) put(r - m, lo);
                    if (j > 0) put(r - 1, lo);
                    put(r, 6.0 + 3.0 * gamma);
                    if (j < m - 1) put(r + 1, -1.0);
                    if (i < m - 1) put(r + m, -1.0);
                    if (k < m - 1) put(r + plane, -1.0);
                } else {
                    // 27-pt: diag 26, all 26 in-cube neighbours -1.
                    for (int dk = -1; dk <= 1; ++dk) {
                        if (k + dk < 0 || k + dk >= m) continue;
                        for (int di = -1; di <= 1; ++di) {
                            if (i + di < 0 || i + di >= m) continue;
                            for (int dj = -1; dj <= 1; ++dj) {
                                if (j + dj < 0 || j + dj >= m) continue;
                                const bool d = dk == 0 && di == 0 && dj == 0;
                                put(r + dk * plane + di * m + dj,
                                    d ? 26.0 : -1.0);
                            }
                        }
                    }
                }
                row_ptr[r + 1] = static_cast<int32_t>(k_out);
            }
        }
    }
}

// harness.cpp:90-99 seeded_values: mt19937_64(seed), U(-1,1) in order.
void port_seeded_values(int64_t n, uint64_t seed, double* out)
{
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

struct PowerLaw {
    std::vector<int32_t> row_ptr, cols;
    std::vector<double> vals;
};

// App. B "Power-law (cfg3)": mt19937_64(seed); per row L = clamp(
// floor(8.25/sqrt(1-U)), 1, max_len); L uniform column draws in
// [max(0,r-w), min(N-1,r+w)] until len distinct; values V(-1,1) in column
// order.
void* port_powerlaw_new(int32_t n, uint64_t seed, int32_t max_len,
                        int32_t window, int64_t* nnz)
{
    auto* h = new PowerLaw;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::uniform_real_distribution<double> V(-1.0, 1.0);
    h->row_ptr.resize(static_cast<size_t>(n) + 1);
    h->row_ptr[0] = 0;
    h->cols.reserve(static_cast<size_t>(n) * 17);
    h->vals.reserve(static_cast<size_t>(n) * 17);
    std::vector<int32_t> draw;
    for (int32_t r = 0; r < n; ++r) {
        const double u = U(rng);
        const int64_t len = clampi(
            static_cast<int64_t>(std::floor(8.25 / std::sqrt(1.0 - u))), 1,
            max_len);
        const int32_t lo = std::max<int64_t>(0, static_cast<int64_t>(r) - window);
        const int32_t hi = std::min<int64_t>(n - 1, static_cast<int64_t>(r) + window);
        std::uniform_int_distribution<int32_t> D(lo, hi);
        // Draw until `len` distinct columns are held: whenever the buffer
        // reaches len it is sorted and de-duplicated, and drawing resumes if
        // duplicates were dropped (the survey probe's rule; pins the App. B
        // KAT nnz = 268,195,029 at N = 2^24).
        draw.clear();
        while (static_cast<int64_t>(draw.size()) < len) {
            draw.push_back(D(rng));
            if (static_cast<int64_t>(draw.size()) == len) {
                std::sort(draw.begin(), draw.end());
                draw.erase(std::unique(draw.begin(), draw.end()), draw.end());
            }
        }
        for (auto c : draw) {
            h->cols.push_back(c);
            h->vals.push_back(V(rng));
        }
        h->row_ptr[static_cast<size_t>(r) + 1] =
            static_cast<int32_t>(h->cols.size());
    }
    *nnz = static_cast<int64_t>(h->cols.size());
    return h;
}

void port_powerlaw_fill(void* hp, int32_t* row_ptr, int32_t* cols, double* vals)
{
    auto* h = static_cast<PowerLaw*>(hp);
    std::memcpy(row_ptr, h->row_ptr.data(), h->row_ptr.size() * 4);
    std::memcpy(cols, h->cols.data(), h->cols.size() * 4);
    std::memcpy(vals, h->vals.data(), h->vals.size() * 8);
}

void port_free(void* h) { delete static_cast<PowerLaw*>(h); }

// ------------------------------------------------------------------- SpMV
// reference.cpp:74-89 ref_spmv_csr: per row, sum from 0.0 in ascending k.
void port_spmv_csr_f64(int32_t nrows, const int32_t* row_ptr,
                       const int32_t* cols, const double* vals,
                       const double* x, double* y)
{
    par_rows(nrows, [&](int64_t r_) {
        const int32_t r = static_cast<int32_t>(r_);
        double sum = 0.0;
        for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            sum += vals[k] * x[cols[k]];
        }
        y[r] = sum;
    });
}

// App. B FP32: same order, float accumulation.
void port_spmv_csr_f32(int32_t nrows, const int32_t* row_ptr,
                       const int32_t* cols, const float* vals, const float* x,
                       float* y)
{
    par_rows(nrows, [&](int64_t r_) {
        const int32_t r = static_cast<int32_t>(r_);
        float sum = 0.0f;
        for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            sum += vals[k] * x[cols[k]];
        }
        y[r] = sum;
    });
}

// reference.cpp:59-71 ref_spmv_coo: zero y, then y[row[k]] += v*x[col] in k.
void port_spmv_coo_f64(int32_t nrows, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, const double* vals,
                       const double* x, double* y)
{
    std::memset(y, 0, static_cast<size_t>(nrows) * sizeof(double));
    for (int64_t k = 0; k < nnz; ++k) {
        y[rows[k]] += vals[k] * x[cols[k]];
    }
}

// App. B ELL (Ginkgo column-major): entry (r,j) at j*stride + r; padding
// column -1 is skipped so the per-row order equals CSR's.
void port_spmv_ell_f64(int32_t nrows, int32_t width, int64_t stride,
                       const int32_t* cols, const double* vals,
                       const double* x, double* y)
{
    par_rows(nrows, [&](int64_t r_) {
        const int32_t r = static_cast<int32_t>(r_);
        double sum = 0.0;
        for (int32_t j = 0; j < width; ++j) {
            const int64_t at = static_cast<int64_t>(j) * stride + r;
            const int32_t c = cols[at];
            if (c >= 0) sum += vals[at] * x[c];
        }
        y[r] = sum;
    });
}

// App. B SELL-P: entry (r,j) at (slice_sets[r/S] + j)*S + r%S.
void port_spmv_sellp_f64(int32_t nrows, int32_t S, const int32_t* slice_sets,
                         const int32_t* cols, const double* vals,
                         const double* x, double* y)
{
    par_rows(nrows, [&](int64_t r_) {
        const int32_t r = static_cast<int32_t>(r_);
        const int32_t s = r / S;
        const int32_t len = slice_sets[s + 1] - slice_sets[s];
        double sum = 0.0;
        for (int32_t j = 0; j < len; ++j) {
            const int64_t at =
                (static_cast<int64_t>(slice_sets[s]) + j) * S + r % S;
            const int32_t c = cols[at];
            if (c >= 0) sum += vals[at] * x[c];
        }
        y[r] = sum;
    });
}

// ------------------------------------------------------------ conversions
int32_t port_csr_max_row(int32_t nrows, const int32_t* row_ptr)
{
    int32_t w = 0;
    for (int32_t r = 0; r < nrows; ++r) w = std::max(w, row_ptr[r + 1] - row_ptr[r]);
    return w;
}

void port_csr_to_ell(int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                     const double* vals, int32_t width, int64_t stride,
                     int32_t* ell_cols, double* ell_vals)
{
    par_rows(nrows, [&](int64_t r_) {
        const int32_t r = static_cast<int32_t>(r_);
        const int32_t len = row_ptr[r + 1] - row_ptr[r];
        for (int32_t j = 0; j < width; ++j) {
            const int64_t at = static_cast<int64_t>(j) * stride + r;
            if (j < len) {
                ell_cols[at] = cols[row_ptr[r] + j];
                ell_vals[at] = vals[row_ptr[r] + j];
            } else {
                ell_cols[at] = -1;
                ell_vals[at] = 0.0;
            }
        }
    });
}

int64_t port_sellp_sets(int32_t nrows, const int32_t* row_ptr, int32_t S,
                        int32_t* slice_lengths, int32_t* slice_sets)
{
    const int32_t nslices = (nrows + S - 1) / S;
    int64_t acc = 0;
    for (int32_t s = 0; s < nslices; ++s) {
        int32_t w = 0;
        for (int32_t r = s * S; r < std::min(nrows, (s + 1) * S); ++r) {
            w = std::max(w, row_ptr[r + 1] - row_ptr[r]);
        }
        if (slice_lengths) slice_lengths[s] = w;
        if (slice_sets) slice_sets[s] = static_cast<int32_t>(acc);
        acc += w;
    }
    if (slice_sets) slice_sets[nslices] = static_cast<int32_t>(acc);
    return acc * S;
}

void port_csr_to_sellp(int32_t nrows, const int32_t* row_ptr,
                       const int32_t* cols, const double* vals, int32_t S,
                       const int32_t* slice_sets, int32_t* s_cols,
                       double* s_vals)
{
    const int32_t nslices = (nrows + S - 1) / S;
    par_rows(nslices, [&](int64_t s_) {
        const int32_t s = static_cast<int32_t>(s_);
        const int32_t w = slice_sets[s + 1] - slice_sets[s];
        for (int32_t lane = 0; lane < S; ++lane) {
            const int32_t r = s * S + lane;
            const int32_t len = r < nrows ? row_ptr[r + 1] - row_ptr[r] : 0;
            for (int32_t j = 0; j < w; ++j) {
                const int64_t at =
                    (static_cast<int64_t>(slice_sets[s]) + j) * S + lane;
                if (j < len) {
                    s_cols[at] = cols[row_ptr[r] + j];
                    s_vals[at] = vals[row_ptr[r] + j];
                } else {
                    s_cols[at] = -1;
                    s_vals[at] = 0.0;
                }
            }
        }
    });
}

// formats.cpp:132-155: histogram row_ptr[row+1]++ then inclusive scan.
void port_coo_to_csr(int32_t nrows, int64_t nnz, const int32_t* rows,
                     int32_t* row_ptr)
{
    std::memset(row_ptr, 0, (static_cast<size_t>(nrows) + 1) * 4);
    for (int64_t k = 0; k < nnz; ++k) ++row_ptr[rows[k] + 1];
    for (int32_t i = 1; i <= nrows; ++i) row_ptr[i] += row_ptr[i - 1];
}

// formats.cpp:158-179: expand row_ptr into row indices.
void port_csr_to_coo(int32_t nrows, const int32_t* row_ptr, int32_t* rows)
{
    for (int32_t r = 0; r < nrows; ++r) {
        for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) rows[k] = r;
    }
}

// ------------------------------------------------------ partition + halo
// App. B "Partition maps": rank(r) = min(r / ceil(N/P), P-1).
int32_t port_part_rank_of(int32_t n, int32_t P, int32_t row)
{
    const int64_t chunk = (static_cast<int64_t>(n) + P - 1) / P;
    return static_cast<int32_t>(std::min<int64_t>(row / chunk, P - 1));
}

void port_part_range(int32_t n, int32_t P, int32_t rank, int32_t* begin,
                     int32_t* end)
{
    // Smallest row with rank(row) == rank, and the first row past it.
    const int64_t chunk = (static_cast<int64_t>(n) + P - 1) / P;
    int64_t b = std::min<int64_t>(static_cast<int64_t>(rank) * chunk, n);
    int64_t e = rank == P - 1 ? n : std::min<int64_t>((rank + 1) * chunk, n);
    *begin = static_cast<int32_t>(b);
    *end = static_cast<int32_t>(e);
}

int64_t port_part_ghosts(int32_t n, int32_t P, int32_t rank,
                         const int32_t* row_ptr, const int32_t* cols,
                         int32_t* ghosts, int64_t cap)
{
    int32_t b, e;
    port_part_range(n, P, rank, &b, &e);
    std::vector<int32_t> g;
    for (int32_t r = b; r < e; ++r) {
        for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            if (cols[k] < b || cols[k] >= e) g.push_back(cols[k]);
        }
    }
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    const int64_t m = std::min<int64_t>(cap, static_cast<int64_t>(g.size()));
    if (ghosts && m > 0) std::memcpy(ghosts, g.data(), static_cast<size_t>(m) * 4);
    return static_cast<int64_t>(g.size());
}

void port_part_local_cols(int32_t n, int32_t P, int32_t rank,
                          const int32_t* row_ptr, const int32_t* cols,
                          const int32_t* ghosts, int64_t nghost,
                          int32_t* local_cols)
{
    int32_t b, e;
    port_part_range(n, P, rank, &b, &e);
    const int32_t nlocal = e - b;
    const int32_t base = row_ptr[b];
    for (int32_t r = b; r < e; ++r) {
        for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            const int32_t c = cols[k];
            int32_t lc;
            if (c >= b && c < e) {
                lc = c - b;
            } else {
                auto it = std::lower_bound(ghosts, ghosts + nghost, c);
                lc = nlocal + static_cast<int32_t>(it - ghosts);
            }
            local_cols[k - base] = lc;
        }
    }
}

// reference.cpp:46-56 ref_dot: sequential sum from 0.0.
double port_dot(int64_t n, const double* x, const double* y)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}

}  // extern "C"
