// blas1.cu -- BLAS-1 entry points (reference kernels.hpp:79-91, api.cpp:69-110;
// backends reference.cpp:17-56).  Element-wise ops round exactly like the
// FMA-free reference (products and sums rounded separately), so axpy/scal/
// fill/copy are bit-identical to it.  dot/nrm2 use a deterministic
// two-stage tree (per-block partials summed in block order by the last
// block), so results are reproducible run to run; the order differs from
// the reference's sequential sum (tolerance 1e-12, SPEC.md kernels module).
#include "api_guard.h"

namespace lbk {

namespace {

constexpr int kThreads = 256;

int grid_for(lbk_ctx ctx, long long n, int per_thread)
{
    long long want = (n + (long long)kThreads * per_thread - 1) / ((long long)kThreads * per_thread);
    long long cap = static_cast<long long>(ctx->num_sms) * 8;
    if (want < 1) want = 1;
    return static_cast<int>(want < cap ? want : cap);
}

__global__ void axpy_kernel(long long n, double alpha, const double* __restrict__ x,
                            double* __restrict__ y)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = add_rn(y[i], mul_rn(alpha, x[i]));
}

__global__ void scal_kernel(long long n, double alpha, double* __restrict__ x)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        x[i] = mul_rn(x[i], alpha);
}

__global__ void fill_kernel(long long n, double v, double* __restrict__ x)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        x[i] = v;
}

__global__ void dot_kernel(long long n, const double* __restrict__ x,
                           const double* __restrict__ y, RedWs ws, int take_sqrt)
{
    __shared__ double sh[32];
    double acc[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        acc[0] = add_rn(acc[0], mul_rn(x[i], y[i]));
    block_sum<1>(acc, threadIdx.x, blockDim.x, sh);
    grid_reduce_finish<1>(acc, ws, threadIdx.x, blockDim.x, sh, [&](const double* t) {
        ws.out[0] = take_sqrt ? sqrt(t[0]) : t[0];
    });
}

void dot_launch(lbk_ctx ctx, long long n, const double* x, const double* y, double* dst_dev,
                bool take_sqrt)
{
    RedWs ws = red_ws(ctx, kRedMaxBlocks, 1);
    const int grid = grid_for(ctx, n, 4);
    dot_kernel<<<grid, kThreads, 0, ctx->stream>>>(n, x, y, ws, take_sqrt ? 1 : 0);
    LBK_LAUNCH_CHECK();
    if (dst_dev && dst_dev != ws.out)
        LBK_CUDA(cudaMemcpyAsync(dst_dev, ws.out, sizeof(double), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
}

double dot_to_host(lbk_ctx ctx, long long n, const double* x, const double* y, bool take_sqrt)
{
    RedWs ws = red_ws(ctx, kRedMaxBlocks, 1);
    dot_launch(ctx, n, x, y, ws.out, take_sqrt);
    LBK_CUDA(cudaMemcpyAsync(ctx->host_pinned, ws.out, sizeof(double), cudaMemcpyDeviceToHost,
                             ctx->stream));
    LBK_CUDA(cudaStreamSynchronize(ctx->stream));
    return ctx->host_pinned[0];
}

void check_n(long long n, const char* what)
{
    need(n >= 0, LBK_SHAPE_ERROR, std::string(what) + ": negative length");
}

// BabelStream-style calibration (the reference's measure_peak_bandwidth,
// src/bench/harness.cpp:125-141, and its stream kernels, reference.cpp:92-130):
// 128-bit streaming loads/stores, grid = a whole number of waves.
__global__ void __launch_bounds__(256) stream_copy_kernel(long long n2, const double2* __restrict__ a,
                                                          double2* __restrict__ c)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
         i += (long long)gridDim.x * blockDim.x)
        __stcs(c + i, __ldcs(a + i));
}

__global__ void __launch_bounds__(256) stream_triad_kernel(long long n2, double s,
                                                           const double2* __restrict__ b,
                                                           const double2* __restrict__ c,
                                                           double2* __restrict__ a)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
         i += (long long)gridDim.x * blockDim.x) {
        const double2 x = __ldcs(b + i), y = __ldcs(c + i);
        __stcs(a + i, make_double2(add_rn(x.x, mul_rn(s, y.x)), add_rn(x.y, mul_rn(s, y.y))));
    }
}

}  // namespace
}  // namespace lbk

using namespace lbk;

extern "C" {

lbk_status lbk_axpy_f64(lbk_ctx ctx, int64_t n, double alpha, const double* x, double* y)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "axpy");
        if (n == 0) return;
        axpy_kernel<<<grid_for(ctx, n, 4), kThreads, 0, ctx->stream>>>(n, alpha, x, y);
        LBK_LAUNCH_CHECK();
    });
}

lbk_status lbk_scal_f64(lbk_ctx ctx, int64_t n, double alpha, double* x)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "scal");
        if (n == 0) return;
        scal_kernel<<<grid_for(ctx, n, 4), kThreads, 0, ctx->stream>>>(n, alpha, x);
        LBK_LAUNCH_CHECK();
    });
}

lbk_status lbk_fill_f64(lbk_ctx ctx, int64_t n, double value, double* x)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "fill");
        if (n == 0) return;
        fill_kernel<<<grid_for(ctx, n, 4), kThreads, 0, ctx->stream>>>(n, value, x);
        LBK_LAUNCH_CHECK();
    });
}

lbk_status lbk_copy_f64(lbk_ctx ctx, int64_t n, const double* x, double* y)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "copy");
        if (n) LBK_CUDA(cudaMemcpyAsync(y, x, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    });
}

lbk_status lbk_dot_f64(lbk_ctx ctx, int64_t n, const double* x, const double* y, double* result)
{
    if (!ctx || !result) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "dot");
        *result = n == 0 ? 0.0 : dot_to_host(ctx, n, x, y, false);
    });
}

lbk_status lbk_nrm2_f64(lbk_ctx ctx, int64_t n, const double* x, double* result)
{
    if (!ctx || !result) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "nrm2");
        *result = n == 0 ? 0.0 : dot_to_host(ctx, n, x, x, true);
    });
}

lbk_status lbk_stream_copy_f64(lbk_ctx ctx, int64_t n, const double* a, double* c)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "stream_copy");
        need(n % 2 == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
                 (reinterpret_cast<uintptr_t>(c) & 15) == 0,
             LBK_USAGE_ERROR, "stream_copy: even n and 16-B aligned arrays");
        if (n == 0) return;
        stream_copy_kernel<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(
            n / 2, reinterpret_cast<const double2*>(a), reinterpret_cast<double2*>(c));
        LBK_LAUNCH_CHECK();
    });
}

lbk_status lbk_stream_triad_f64(lbk_ctx ctx, int64_t n, double scalar, const double* b,
                                const double* c, double* a)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "stream_triad");
        need(n % 2 == 0, LBK_USAGE_ERROR, "stream_triad: even n");
        if (n == 0) return;
        stream_triad_kernel<<<ctx->num_sms * 8, 256, 0, ctx->stream>>>(
            n / 2, scalar, reinterpret_cast<const double2*>(b), reinterpret_cast<const double2*>(c),
            reinterpret_cast<double2*>(a));
        LBK_LAUNCH_CHECK();
    });
}

lbk_status lbk_dot_f64_dev(lbk_ctx ctx, int64_t n, const double* x, const double* y,
                           double* result_dev)
{
    if (!ctx || !result_dev) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        check_n(n, "dot");
        if (n == 0) {
            LBK_CUDA(cudaMemsetAsync(result_dev, 0, sizeof(double), ctx->stream));
            return;
        }
        dot_launch(ctx, n, x, y, result_dev, false);
    });
}

}  // extern "C"
