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
