// spmv_launch.cuh -- host-side launchers for the SpMV kernels (plans, grid
// sizing, alignment-driven kernel choice).  Shared by the SpMV entry points
// (spmv.cu) and the fused solver steps (solver.cu).
#pragma once

#include <atomic>
#include <cstdlib>
#include <cstring>

#include "api_guard.h"
#include "spmv_kernels.cuh"

namespace lbk {

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Number of plan tiles (the plan holds ntiles + 1 int32 boundaries).
inline int stream_ntiles(long long nnz, long long nrows, int idx_arrays)
{
    const long long tn = stream_tile_nnz(nnz, nrows, idx_arrays);
    long long t = (nnz + tn - 1) / tn;
    return static_cast<int>(t < 1 ? 1 : t);
}
inline int csr_ntiles(long long nnz, long long nrows) { return stream_ntiles(nnz, nrows, 1); }
inline int coo_ntiles(long long nnz, long long nrows) { return stream_ntiles(nnz, nrows, 2); }

void csr_plan_launch(lbk_ctx ctx, const int* row_ptr, int nrows, long long nnz, int* tile_rows);
// SELL-P tiles are runs of k whole slices, k = slots' worth of mean-size
// slices (a mean-size tile never straddles a slot: the entry-window rule of
// CSR would pair two 27-column slices into an oversize tile).
inline int sellp_slices_per_tile(long long stored, int nslices)
{
    const long long mean = nslices > 0 ? (stored + nslices - 1) / nslices : 1;
    const long long k = (StreamCfg<double, 1>::kCap - 128) / (mean < 1 ? 1 : mean);
    return static_cast<int>(k < 1 ? 1 : (k > 32 ? 32 : k));
}
inline int sellp_ntiles(long long stored, int nslices)
{
    const int k = sellp_slices_per_tile(stored, nslices);
    const long long t = (nslices + k - 1) / k;
    return static_cast<int>(t < 1 ? 1 : t);
}
void sellp_plan_launch(lbk_ctx ctx, const int* slice_sets, int nslices, long long stored,
                       int* tile_slices);
// The warp-pipelined SELL-P kernel is opt-in (LBK_SELLP_ALGO=stream): on
// cfg2 it measured 143 us against 129 us for the 4-rows-per-thread sliced
// kernel, both latency-bound on the gathers (ncu: issue ~30%).
inline bool sellp_force_sliced()
{
    static int v = [] {
        const char* e = std::getenv("LBK_SELLP_ALGO");
        return (e && std::strcmp(e, "stream") == 0) ? 0 : 1;
    }();
    return v != 0;
}
void coo_plan_launch(lbk_ctx ctx, const int* rows, int nrows, long long nnz, int* tile_starts);

// Forces the warp-per-row CSR kernel (diagnostics / A-B comparison).
inline bool csr_force_warp()
{
    static int v = [] {
        const char* e = std::getenv("LBK_CSR_ALGO");
        return (e && std::strcmp(e, "warp") == 0) ? 1 : 0;
    }();
    return v != 0;
}

// Warp-per-row CSR straight from global memory (LBK_CSR_ALGO=warp: A/B
// comparison against the stream kernel).
template <typename T, class Epi>
__global__ void __launch_bounds__(256)
    csr_warp_kernel(CsrView<T> A, const T* __restrict__ x, Epi epi, RedWs ws)
{
    pdl_enter();
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    if constexpr (Epi::NV > 0) red_begin<NV>();
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
    const int lane = threadIdx.x & 31;
    const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long rr = w0; rr < A.nrows; rr += nw) {
        const int r = static_cast<int>(rr);
        const int rs = __ldg(A.row_ptr + r), re = __ldg(A.row_ptr + r + 1);
        T part = T(0);
        if (re - rs <= 32) {
            // short row: lane k holds product k, lane 0 sums them in order
            // (bit-identical to the sequential reference)
            T p = T(0);
            if (rs + lane < re) p = mul_rn(__ldg(A.vals + rs + lane), ldg_nc(x + __ldg(A.cols + rs + lane)));
            T sum = T(0);
            for (int k = 0; k < re - rs; ++k) sum = add_rn(sum, __shfl_sync(0xffffffffu, p, k));
            part = sum;
        } else {
            for (int k = rs + lane; k < re; k += 32)
                part = add_rn(part, mul_rn(__ldg(A.vals + k), ldg_nc(x + __ldg(A.cols + k))));
            part = warp_sum(part);
        }
        if (lane == 0) epi.row(r, part, acc);
    }
    if constexpr (Epi::NV > 0) {
        grid_reduce<NV>(acc, ws, threadIdx.x, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

// Launch with, when the context asks for it, an L2 access-policy window
// over the gathered vector x (persisting) -- the matrix streams already
// carry evict-first hints, so x keeps its place in L2 between launches.
template <typename... KArgs, typename... Args>
void launch_k(lbk_ctx ctx, void (*kernel)(KArgs...), int grid, int block, size_t smem,
              const void* x, size_t x_bytes, Args&&... args)
{
    const bool window = ctx->l2_persist && x && ctx->persist_max;
    if (!window && !ctx->pdl) {
        kernel<<<grid, block, smem, ctx->stream>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (window) {
        attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
        const size_t nb = x_bytes < ctx->persist_max ? x_bytes : ctx->persist_max;
        attr[na].val.accessPolicyWindow.base_ptr = const_cast<void*>(x);
        attr[na].val.accessPolicyWindow.num_bytes = nb;
        attr[na].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        ++na;
    }
    if (ctx->pdl) {  // every kernel launched here opens with pdl_enter()
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    LBK_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

template <class K>
int blocks_per_sm(K kernel, int threads, size_t smem)
{
    int b = 0;
    LBK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem));
    return b < 1 ? 1 : b;
}

template <typename K>
void set_smem(K kernel, size_t bytes)
{
    LBK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(bytes)));
}

// The >48 KB dynamic shared-memory opt-in is a per-device setting: `mask`
// (one static per kernel instantiation at the call site) records the
// devices this process has opted in on, so a second GPU driven from the
// same process (second ctx, thread or peer group) opts in too.
template <typename K>
void smem_optin(std::atomic<unsigned long long>& mask, int device, K kernel, size_t bytes)
{
    const unsigned long long bit = 1ull << (device & 63);
    if (mask.load(std::memory_order_acquire) & bit) return;
    set_smem(kernel, bytes);
    mask.fetch_or(bit, std::memory_order_acq_rel);
}

// Persistent grid: as many CTAs as fit (shared-memory bound), one warp per
// tile at a time.
template <typename T, int NIDX, int G, class K, class View, class Epi>
void stream_launch(lbk_ctx ctx, K kernel, const View& A, const T* x, const Epi& epi, RedWs ws)
{
    using Cfg = StreamCfg<T, NIDX>;
    constexpr size_t smem = Cfg::smem_bytes;
    static std::atomic<unsigned long long> optin{0};
    smem_optin(optin, ctx->device, kernel, smem);
    static int bps = blocks_per_sm(kernel, Cfg::kThreads, smem);
    long long cap = static_cast<long long>(ctx->num_sms) * bps;
    if (cap > kRedMaxBlocks) cap = kRedMaxBlocks;
    const long long want = (A.ntiles + Cfg::kWarps - 1) / Cfg::kWarps;
    const int grid = static_cast<int>(want < cap ? want : cap);
    launch_k(ctx, kernel, grid, Cfg::kThreads, smem, x, size_t(A.ncols) * sizeof(T), A, x, epi, ws);
    LBK_LAUNCH_CHECK();
}

template <typename T, class Epi>
void launch_csr(lbk_ctx ctx, CsrView<T> A, const T* x, const Epi& epi, RedWs ws)
{
    const bool tma_ok = aligned16(A.vals) && aligned16(A.cols);
    if (csr_force_warp() || !tma_ok) {
        auto k = csr_warp_kernel<T, Epi>;
        static int bps = blocks_per_sm(k, 256, 0);
        long long want = (static_cast<long long>(A.nrows) * 32 + 255) / 256;
        long long cap = static_cast<long long>(ctx->num_sms) * bps;
        int grid = static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
        if (Epi::NV > 0 && grid > kRedMaxBlocks) grid = kRedMaxBlocks;
        k<<<grid, 256, 0, ctx->stream>>>(A, x, epi, ws);
        LBK_LAUNCH_CHECK();
        return;
    }
    if (!A.tile_rows) {
        A.ntiles = csr_ntiles(A.nnz, A.nrows);
        int* plan = static_cast<int*>(scratch(ctx, size_t(A.ntiles + 1) * sizeof(int)));
        csr_plan_launch(ctx, A.row_ptr, A.nrows, A.nnz, plan);
        A.tile_rows = plan;
    }
    switch (stream_group(A.nnz, A.nrows)) {
    case 4: stream_launch<T, 1, 4>(ctx, csr_stream_kernel<T, Epi, 4>, A, x, epi, ws); break;
    case 2: stream_launch<T, 1, 2>(ctx, csr_stream_kernel<T, Epi, 2>, A, x, epi, ws); break;
    default: stream_launch<T, 1, 1>(ctx, csr_stream_kernel<T, Epi, 1>, A, x, epi, ws); break;
    }
}

template <typename T, class Epi>
void launch_coo(lbk_ctx ctx, CooView<T> A, const T* x, const Epi& epi, RedWs ws)
{
    need(aligned16(A.vals) && aligned16(A.cols) && aligned16(A.rows), LBK_USAGE_ERROR,
         "COO arrays must be 16-byte aligned");
    if (!A.tile_starts) {
        A.ntiles = coo_ntiles(A.nnz, A.nrows);
        int* plan = static_cast<int*>(scratch(ctx, size_t(A.ntiles + 1) * sizeof(int)));
        coo_plan_launch(ctx, A.rows, A.nrows, A.nnz, plan);
        A.tile_starts = plan;
    }
    switch (stream_group(A.nnz, A.nrows)) {
    case 4: stream_launch<T, 2, 4>(ctx, coo_stream_kernel<T, Epi, 4>, A, x, epi, ws); break;
    case 2: stream_launch<T, 2, 2>(ctx, coo_stream_kernel<T, Epi, 2>, A, x, epi, ws); break;
    default: stream_launch<T, 2, 1>(ctx, coo_stream_kernel<T, Epi, 1>, A, x, epi, ws); break;
    }
}

template <typename T, class Epi>
void launch_sellp_stream(lbk_ctx ctx, SellpView<T> A, const int* plan, int ntiles, long long stored,
                         const T* x, const Epi& epi, RedWs ws)
{
    using Cfg = StreamCfg<T, 1>;
    auto kernel = sellp_stream_kernel<T, Epi>;
    constexpr size_t smem = Cfg::smem_bytes;
    static std::atomic<unsigned long long> optin{0};
    smem_optin(optin, ctx->device, kernel, smem);
    static int bps = blocks_per_sm(kernel, Cfg::kThreads, smem);
    long long cap = static_cast<long long>(ctx->num_sms) * bps;
    if (cap > kRedMaxBlocks) cap = kRedMaxBlocks;
    const long long want = (ntiles + Cfg::kWarps - 1) / Cfg::kWarps;
    const int grid = static_cast<int>(want < cap ? want : cap);
    launch_k(ctx, kernel, grid, Cfg::kThreads, smem, x, size_t(A.ncols) * sizeof(T), A, plan,
             ntiles, stored, x, epi, ws);
    LBK_LAUNCH_CHECK();
}

// ELL (is_ell) or SELL-P over the sliced column-major layout.
template <typename T, class Epi, bool IS_ELL>
void launch_sliced(lbk_ctx ctx, int nrows, int S, const int* slice_sets, int width,
                   long long ell_stride, const int* cols, const T* vals, const T* x,
                   const Epi& epi, RedWs ws, long long x_len = 0)
{
    const int pitch = IS_ELL ? static_cast<int>(ell_stride) : S;
    const bool quad_ok = aligned16(cols) && aligned16(vals) && pitch % 4 == 0 &&
                         (!IS_ELL || ell_stride >= ((static_cast<long long>(nrows) + 3) & ~3LL));
    static const int algo = [] {
        const char* e = std::getenv("LBK_SLICED");
        // quad (4 rows per thread, 128-bit loads) is the default; lane-per-row
        // and scalar row kernels measured within noise of it on cfg2
        if (e && std::strcmp(e, "lane") == 0) return 0;
        if (e && std::strcmp(e, "row") == 0) return 2;
        return 1;
    }();
    if (algo == 0) {
        auto k = sliced_lane_kernel<T, Epi, IS_ELL>;
        static int bps = blocks_per_sm(k, 256, 0);
        long long want = (static_cast<long long>(nrows) + 255) / 256;
        long long cap = static_cast<long long>(ctx->num_sms) * bps;
        if (Epi::NV > 0 && cap > kRedMaxBlocks) cap = kRedMaxBlocks;
        int grid = static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
        launch_k(ctx, k, grid, 256, 0, x, size_t(x_len) * sizeof(T), nrows, pitch, slice_sets, width,
                 cols, vals, x, epi, ws);
        LBK_LAUNCH_CHECK();
        return;
    }
    const long long units = quad_ok && algo == 1 ? (static_cast<long long>(nrows) + 3) / 4 : nrows;
    if (quad_ok && algo == 1) {
        auto k = sliced_quad_kernel<T, Epi, IS_ELL>;
        static int bps = blocks_per_sm(k, 256, 0);
        long long want = (units + 255) / 256, cap = static_cast<long long>(ctx->num_sms) * bps;
        int grid = static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
        launch_k(ctx, k, grid, 256, 0, x, size_t(x_len) * sizeof(T), nrows, pitch, slice_sets, width,
                 cols, vals, x, epi, ws);
    } else {
        auto k = sliced_row_kernel<T, Epi, IS_ELL>;
        static int bps = blocks_per_sm(k, 256, 0);
        long long want = (units + 255) / 256, cap = static_cast<long long>(ctx->num_sms) * bps;
        int grid = static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
        launch_k(ctx, k, grid, 256, 0, x, size_t(x_len) * sizeof(T), nrows, pitch, slice_sets, width,
                 cols, vals, x, epi, ws);
    }
    LBK_LAUNCH_CHECK();
}

}  // namespace lbk
