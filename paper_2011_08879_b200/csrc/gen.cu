// gen.cu -- synthetic inputs of the benchmark configurations (SURVEY.md §8d,
// App. B).  Input synthesis only: not on the measured path.
//   stencils    generated on the device (row lengths -> scan -> fill), row
//               r = (k*m + i)*m + j, columns ascending within a row
//   seeded x    std::mt19937_64 + std::uniform_real_distribution(-1,1) in
//               row order: the reference harness's seeded_values
//               (src/bench/harness.cpp:90-99), same libstdc++ => same bits
//   power-law   host generator of App. B (mt19937_64(42), L = clamp(
//               floor(8.25/sqrt(1-U)), 1, 10000), L distinct columns in a
//               +-65536 window, values U(-1,1) in column order)
#include <algorithm>
#include <cmath>
#include <cub/device/device_scan.cuh>
#include <random>
#include <vector>

#include "api_guard.h"

namespace lbk {
namespace {

struct StencilGeo {
    int kind, m;
    double gamma;
};

// Visits the entries of row r in ascending column order.
template <class F>
__device__ void stencil_row(const StencilGeo& g, long long r, F&& put)
{
    const long long m = g.m;
    if (g.kind == 0) {
        const long long i = r / m, j = r % m;
        if (i > 0) put(r - m, -1.0);
        if (j > 0) put(r - 1, -1.0);
        put(r, 4.0);
        if (j < m - 1) put(r + 1, -1.0);
        if (i < m - 1) put(r + m, -1.0);
        return;
    }
    const long long plane = m * m;
    const long long k = r / plane, i = (r / m) % m, j = r % m;
    if (g.kind == 1) {
        const double lo = -1.0 - g.gamma;
        if (k > 0) put(r - plane, lo);
        if (i > 0) put(r - m, lo);
        if (j > 0) put(r - 1, lo);
        put(r, 6.0 + 3.0 * g.gamma);
        if (j < m - 1) put(r + 1, -1.0);
        if (i < m - 1) put(r + m, -1.0);
        if (k < m - 1) put(r + plane, -1.0);
        return;
    }
    for (int dk = -1; dk <= 1; ++dk) {
        if (k + dk < 0 || k + dk >= m) continue;
        for (int di = -1; di <= 1; ++di) {
            if (i + di < 0 || i + di >= m) continue;
            for (int dj = -1; dj <= 1; ++dj) {
                if (j + dj < 0 || j + dj >= m) continue;
                const bool d = dk == 0 && di == 0 && dj == 0;
                put(r + dk * plane + di * m + dj, d ? 26.0 : -1.0);
            }
        }
    }
}

__global__ void stencil_len_kernel(StencilGeo g, long long n, int* __restrict__ len)
{
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        int c = 0;
        stencil_row(g, r, [&](long long, double) { ++c; });
        len[r + 1] = c;
    }
}

__global__ void stencil_fill_kernel(StencilGeo g, long long n, const int* __restrict__ row_ptr,
                                    int* __restrict__ cols, double* __restrict__ vals)
{
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
         r += (long long)gridDim.x * blockDim.x) {
        int k = row_ptr[r];
        stencil_row(g, r, [&](long long c, double v) {
            cols[k] = static_cast<int>(c);
            vals[k] = v;
            ++k;
        });
    }
}

struct PowerLawHost {
    std::vector<int32_t> row_ptr, cols;
    std::vector<double> vals;
};

}  // namespace
}  // namespace lbk

using namespace lbk;

extern "C" {

int64_t lbk_gen_stencil_nnz(int kind, int m)
{
    const int64_t mm = m;
    if (kind == 0) return 5 * mm * mm - 4 * mm;
    if (kind == 1) return 7 * mm * mm * mm - 6 * mm * mm;
    return (3 * mm - 2) * (3 * mm - 2) * (3 * mm - 2);
}

lbk_status lbk_gen_stencil_csr(lbk_ctx ctx, int kind, int m, double gamma, int32_t* row_ptr,
                               int32_t* cols, double* vals)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(kind >= 0 && kind <= 2 && m > 0, LBK_CONFIGURATION_ERROR, "gen_stencil: bad kind/size");
        const long long n = kind == 0 ? 1LL * m * m : 1LL * m * m * m;
        need(n < (1LL << 31) && lbk_gen_stencil_nnz(kind, m) < (1LL << 31), LBK_SHAPE_ERROR,
             "gen_stencil: problem exceeds int32 indices");
        StencilGeo g{kind, m, gamma};
        const int grid = static_cast<int>(std::min<long long>((n + 255) / 256, 1 << 20));
        LBK_CUDA(cudaMemsetAsync(row_ptr, 0, 4, ctx->stream));
        stencil_len_kernel<<<grid, 256, 0, ctx->stream>>>(g, n, row_ptr);
        LBK_LAUNCH_CHECK();
        size_t tb = 0;
        LBK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, row_ptr, row_ptr, n + 1, ctx->stream));
        void* t = nullptr;
        LBK_CUDA(cudaMallocAsync(&t, tb, ctx->stream));
        LBK_CUDA(cub::DeviceScan::InclusiveSum(t, tb, row_ptr, row_ptr, n + 1, ctx->stream));
        LBK_CUDA(cudaFreeAsync(t, ctx->stream));
        stencil_fill_kernel<<<grid, 256, 0, ctx->stream>>>(g, n, row_ptr, cols, vals);
        LBK_LAUNCH_CHECK();
    });
}

void lbk_gen_seeded_values(int64_t n, uint64_t seed, double* out)
{
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (int64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

void* lbk_gen_powerlaw(int32_t n, uint64_t seed, int32_t max_len, int32_t window, int64_t* nnz)
{
    auto* h = new PowerLawHost;
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> U(0.0, 1.0), V(-1.0, 1.0);
    h->row_ptr.assign(static_cast<size_t>(n) + 1, 0);
    h->cols.reserve(static_cast<size_t>(n) * 17);
    h->vals.reserve(static_cast<size_t>(n) * 17);
    std::vector<int32_t> pick;
    for (int32_t r = 0; r < n; ++r) {
        long long len = static_cast<long long>(std::floor(8.25 / std::sqrt(1.0 - U(rng))));
        len = std::min<long long>(std::max<long long>(len, 1), max_len);
        const int32_t lo = static_cast<int32_t>(std::max<long long>(0, 1LL * r - window));
        const int32_t hi = static_cast<int32_t>(std::min<long long>(n - 1, 1LL * r + window));
        std::uniform_int_distribution<int32_t> D(lo, hi);
        pick.clear();
        while (static_cast<long long>(pick.size()) < len) {
            pick.push_back(D(rng));
            if (static_cast<long long>(pick.size()) == len) {
                std::sort(pick.begin(), pick.end());
                pick.erase(std::unique(pick.begin(), pick.end()), pick.end());
            }
        }
        for (int32_t c : pick) {
            h->cols.push_back(c);
            h->vals.push_back(V(rng));
        }
        h->row_ptr[static_cast<size_t>(r) + 1] = static_cast<int32_t>(h->cols.size());
    }
    *nnz = static_cast<int64_t>(h->cols.size());
    return h;
}

void lbk_gen_powerlaw_fill(void* hp, int32_t* row_ptr, int32_t* cols, double* vals)
{
    auto* h = static_cast<PowerLawHost*>(hp);
    std::copy(h->row_ptr.begin(), h->row_ptr.end(), row_ptr);
    std::copy(h->cols.begin(), h->cols.end(), cols);
    std::copy(h->vals.begin(), h->vals.end(), vals);
}

void lbk_gen_powerlaw_free(void* hp) { delete static_cast<PowerLawHost*>(hp); }

}  // extern "C"
