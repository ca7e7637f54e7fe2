// spmv.cu -- SpMV entry points of the C ABI (include/lbk.h).
//
// Replaces the reference's spmv_csr / spmv_coo typed wrappers
// (src/kernels/api.cpp:113-140) and their host backends
// (src/kernels/reference.cpp:59-89, parallel.cpp:100-143); adds ELL, SELL-P,
// FP32 and the alpha/beta "advanced apply" the reference lacks.
#include "api_guard.h"
#include "spmv_launch.cuh"

namespace lbk {

__global__ void csr_plan_kernel(const int* __restrict__ row_ptr, int nrows, int ntiles,
                                long long tile_nnz, int* __restrict__ tile_rows)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    if (t == 0) { tile_rows[0] = 0; return; }
    if (t == ntiles) { tile_rows[t] = nrows; return; }
    const long long key = static_cast<long long>(t) * tile_nnz;
    int lo = 0, hi = nrows;  // lower_bound over row_ptr[0..nrows]
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (static_cast<long long>(__ldg(row_ptr + mid)) < key) lo = mid + 1; else hi = mid;
    }
    tile_rows[t] = lo;
}

__global__ void coo_plan_kernel(const int* __restrict__ rows, long long nnz, int ntiles,
                                long long tile_nnz, int* __restrict__ tile_starts)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    if (t == 0) { tile_starts[0] = 0; return; }
    if (t == ntiles) { tile_starts[t] = static_cast<int>(nnz); return; }
    const long long at = static_cast<long long>(t) * tile_nnz;
    const int key = __ldg(rows + at);
    long long lo = 0, hi = at;  // first entry of the row holding `at`
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (__ldg(rows + mid) < key) lo = mid + 1; else hi = mid;
    }
    tile_starts[t] = static_cast<int>(lo);
}

__global__ void sellp_plan_kernel(int nslices, int ntiles, int k, int* __restrict__ tile_slices)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t > ntiles) return;
    const long long s = static_cast<long long>(t) * k;
    tile_slices[t] = static_cast<int>(s < nslices ? s : nslices);
}

void sellp_plan_launch(lbk_ctx ctx, const int* slice_sets, int nslices, long long stored,
                       int* tile_slices)
{
    (void)slice_sets;
    const int nt = sellp_ntiles(stored, nslices);
    sellp_plan_kernel<<<ceil_div(nt + 1, 256), 256, 0, ctx->stream>>>(
        nslices, nt, sellp_slices_per_tile(stored, nslices), tile_slices);
    LBK_LAUNCH_CHECK();
}

void csr_plan_launch(lbk_ctx ctx, const int* row_ptr, int nrows, long long nnz, int* tile_rows)
{
    const int nt = csr_ntiles(nnz, nrows);
    csr_plan_kernel<<<ceil_div(nt + 1, 256), 256, 0, ctx->stream>>>(
        row_ptr, nrows, nt, stream_tile_nnz(nnz, nrows, 1), tile_rows);
    LBK_LAUNCH_CHECK();
}

void coo_plan_launch(lbk_ctx ctx, const int* rows, int nrows, long long nnz, int* tile_starts)
{
    const int nt = coo_ntiles(nnz, nrows);
    coo_plan_kernel<<<ceil_div(nt + 1, 256), 256, 0, ctx->stream>>>(
        rows, nnz, nt, stream_tile_nnz(nnz, nrows, 2), tile_starts);
    LBK_LAUNCH_CHECK();
}

namespace {

void check_common(int nrows, int ncols, long long nnz, lbk_dtype got, lbk_dtype want,
                  const char* what)
{
    need(nrows >= 0 && ncols >= 0, LBK_SHAPE_ERROR, std::string(what) + ": negative dimension");
    need(nnz >= 0 && nnz < (1LL << 31), LBK_SHAPE_ERROR,
         std::string(what) + ": nnz outside [0, 2^31) (int32 indices)");
    need(got == want, LBK_TYPE_ERROR,
         std::string(what) + ": matrix value type does not match the entry point");
}

template <typename T>
CsrView<T> csr_view(const lbk_csr* A, lbk_dtype want)
{
    need(A != nullptr, LBK_USAGE_ERROR, "spmv_csr: null matrix");
    check_common(A->nrows, A->ncols, A->nnz, A->dtype, want, "spmv_csr");
    need(A->row_ptr != nullptr || A->nrows == 0, LBK_USAGE_ERROR, "spmv_csr: null row_ptr");
    CsrView<T> v{A->nrows, A->ncols, A->nnz, A->row_ptr, A->col_idx,
                 static_cast<const T*>(A->vals), A->tile_rows, A->ntiles};
    if (v.tile_rows)
        need(v.ntiles == csr_ntiles(v.nnz, v.nrows), LBK_USAGE_ERROR,
             "spmv_csr: stale plan (ntiles does not match lbk_csr_plan_size)");
    return v;
}

template <typename T>
CooView<T> coo_view(const lbk_coo* A, lbk_dtype want)
{
    need(A != nullptr, LBK_USAGE_ERROR, "spmv_coo: null matrix");
    check_common(A->nrows, A->ncols, A->nnz, A->dtype, want, "spmv_coo");
    CooView<T> v{A->nrows, A->ncols, A->nnz, A->row_idx, A->col_idx,
                 static_cast<const T*>(A->vals), A->tile_starts, A->ntiles};
    if (v.tile_starts)
        need(v.ntiles == coo_ntiles(v.nnz, v.nrows), LBK_USAGE_ERROR,
             "spmv_coo: stale plan (ntiles does not match lbk_coo_plan_size)");
    return v;
}

template <typename T, class Epi>
void run_csr(lbk_ctx ctx, const lbk_csr* A, const T* x, const Epi& epi, lbk_dtype dt)
{
    auto v = csr_view<T>(A, dt);
    if (v.nrows == 0) return;
    launch_csr<T>(ctx, v, x, epi, RedWs{});
}

template <typename T, class Epi>
void run_coo(lbk_ctx ctx, const lbk_coo* A, const T* x, const Epi& epi, lbk_dtype dt)
{
    auto v = coo_view<T>(A, dt);
    if (v.nrows == 0) return;
    if (v.nnz == 0) {
        // empty matrix: y = A x = 0 (reference.cpp:67 zero-fill), through
        // the epilogue so alpha/beta semantics hold
        static_assert(Epi::NV == 0, "");
        launch_sliced<T, Epi, true>(ctx, v.nrows, v.nrows, nullptr, 0, v.nrows, nullptr,
                                    nullptr, x, epi, RedWs{});
        return;
    }
    launch_coo<T>(ctx, v, x, epi, RedWs{});
}

template <typename T, class Epi>
void run_ell(lbk_ctx ctx, const lbk_ell* A, const T* x, const Epi& epi, lbk_dtype dt)
{
    need(A != nullptr, LBK_USAGE_ERROR, "spmv_ell: null matrix");
    check_common(A->nrows, A->ncols, A->nnz, A->dtype, dt, "spmv_ell");
    need(A->width >= 0 && A->stride >= A->nrows, LBK_FORMAT_ERROR,
         "spmv_ell: need width >= 0 and stride >= nrows");
    if (A->nrows == 0) return;
    launch_sliced<T, Epi, true>(ctx, A->nrows, 0, nullptr, A->width, A->stride, A->col_idx,
                                static_cast<const T*>(A->vals), x, epi, RedWs{}, A->ncols);
}

template <typename T, class Epi>
void run_sellp(lbk_ctx ctx, const lbk_sellp* A, const T* x, const Epi& epi, lbk_dtype dt)
{
    need(A != nullptr, LBK_USAGE_ERROR, "spmv_sellp: null matrix");
    check_common(A->nrows, A->ncols, A->nnz, A->dtype, dt, "spmv_sellp");
    need(A->slice_size > 0, LBK_FORMAT_ERROR, "spmv_sellp: slice_size must be positive");
    need(A->nslices == (A->nrows + A->slice_size - 1) / A->slice_size, LBK_FORMAT_ERROR,
         "spmv_sellp: nslices != ceil(nrows / slice_size)");
    if (A->nrows == 0) return;
    const T* vals = static_cast<const T*>(A->vals);
    if (A->slice_size == 32 && aligned16(vals) && aligned16(A->col_idx) && !sellp_force_sliced()) {
        // warp pipeline over whole slices (stored count: one host read of
        // slice_sets[nslices] unless a plan is supplied)
        const int* plan = A->tile_slices;
        int ntiles = A->ntiles;
        long long stored = A->stored;
        if (!plan) {
            if (stored <= 0) {
                int last = 0;
                LBK_CUDA(cudaMemcpyAsync(&last, A->slice_sets + A->nslices, sizeof(int),
                                         cudaMemcpyDeviceToHost, ctx->stream));
                LBK_CUDA(cudaStreamSynchronize(ctx->stream));
                stored = static_cast<long long>(last) * 32;
            }
            ntiles = sellp_ntiles(stored, A->nslices);
            int* p = static_cast<int*>(scratch(ctx, size_t(ntiles + 1) * sizeof(int)));
            sellp_plan_launch(ctx, A->slice_sets, A->nslices, stored, p);
            plan = p;
        }
        need(ntiles == sellp_ntiles(stored, A->nslices), LBK_USAGE_ERROR,
             "spmv_sellp: stale plan (ntiles does not match lbk_sellp_plan_size)");
        launch_sellp_stream<T>(ctx,
                               SellpView<T>{A->nrows, A->ncols, 32, A->nslices, A->slice_sets,
                                            A->col_idx, vals},
                               plan, ntiles, stored, x, epi, RedWs{});
        return;
    }
    launch_sliced<T, Epi, false>(ctx, A->nrows, A->slice_size, A->slice_sets, 0, 0,
                                 A->col_idx, vals, x, epi, RedWs{}, A->ncols);
}

}  // namespace
}  // namespace lbk

using namespace lbk;

extern "C" {

#define LBK_SPMV_ENTRY(NAME, DESC, RUN, T, DT)                                         \
    lbk_status NAME(lbk_ctx ctx, const DESC* A, const T* x, T* y)                      \
    {                                                                                  \
        if (!ctx) return LBK_USAGE_ERROR;                                              \
        NvtxRange nvtx_(#NAME);                                                        \
        return guard(ctx, [&] { RUN<T>(ctx, A, x, EpiStore<T>{y}, DT); });             \
    }
#define LBK_SPMV_ADV_ENTRY(NAME, DESC, RUN, T, DT)                                     \
    lbk_status NAME(lbk_ctx ctx, T alpha, const DESC* A, const T* x, T beta, T* y)     \
    {                                                                                  \
        if (!ctx) return LBK_USAGE_ERROR;                                              \
        NvtxRange nvtx_(#NAME);                                                        \
        return guard(ctx, [&] { RUN<T>(ctx, A, x, EpiAxpby<T>{y, alpha, beta}, DT); }); \
    }

LBK_SPMV_ENTRY(lbk_spmv_csr_f64, lbk_csr, run_csr, double, LBK_F64)
LBK_SPMV_ENTRY(lbk_spmv_csr_f32, lbk_csr, run_csr, float, LBK_F32)
LBK_SPMV_ADV_ENTRY(lbk_spmv_csr_adv_f64, lbk_csr, run_csr, double, LBK_F64)
LBK_SPMV_ADV_ENTRY(lbk_spmv_csr_adv_f32, lbk_csr, run_csr, float, LBK_F32)
LBK_SPMV_ENTRY(lbk_spmv_coo_f64, lbk_coo, run_coo, double, LBK_F64)
LBK_SPMV_ENTRY(lbk_spmv_coo_f32, lbk_coo, run_coo, float, LBK_F32)
LBK_SPMV_ADV_ENTRY(lbk_spmv_coo_adv_f64, lbk_coo, run_coo, double, LBK_F64)
LBK_SPMV_ADV_ENTRY(lbk_spmv_coo_adv_f32, lbk_coo, run_coo, float, LBK_F32)
LBK_SPMV_ENTRY(lbk_spmv_ell_f64, lbk_ell, run_ell, double, LBK_F64)
LBK_SPMV_ENTRY(lbk_spmv_ell_f32, lbk_ell, run_ell, float, LBK_F32)
LBK_SPMV_ADV_ENTRY(lbk_spmv_ell_adv_f64, lbk_ell, run_ell, double, LBK_F64)
LBK_SPMV_ADV_ENTRY(lbk_spmv_ell_adv_f32, lbk_ell, run_ell, float, LBK_F32)
LBK_SPMV_ENTRY(lbk_spmv_sellp_f64, lbk_sellp, run_sellp, double, LBK_F64)
LBK_SPMV_ENTRY(lbk_spmv_sellp_f32, lbk_sellp, run_sellp, float, LBK_F32)
LBK_SPMV_ADV_ENTRY(lbk_spmv_sellp_adv_f64, lbk_sellp, run_sellp, double, LBK_F64)
LBK_SPMV_ADV_ENTRY(lbk_spmv_sellp_adv_f32, lbk_sellp, run_sellp, float, LBK_F32)

lbk_status lbk_csr_plan_size(const lbk_csr* A, int32_t* ntiles_out)
{
    if (!A || !ntiles_out) return LBK_USAGE_ERROR;
    *ntiles_out = csr_ntiles(A->nnz, A->nrows);
    return LBK_OK;
}

lbk_status lbk_csr_plan(lbk_ctx ctx, const lbk_csr* A, int32_t* tile_rows_dev)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->nrows > 0, LBK_USAGE_ERROR, "lbk_csr_plan: empty matrix");
        csr_plan_launch(ctx, A->row_ptr, A->nrows, A->nnz, tile_rows_dev);
    });
}

lbk_status lbk_sellp_plan_size(const lbk_sellp* A, int32_t* ntiles_out)
{
    if (!A || !ntiles_out || A->stored < 0) return LBK_USAGE_ERROR;
    *ntiles_out = sellp_ntiles(A->stored, A->nslices);
    return LBK_OK;
}

lbk_status lbk_sellp_plan(lbk_ctx ctx, const lbk_sellp* A, int32_t* tile_slices_dev)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->slice_size == 32 && A->stored > 0, LBK_USAGE_ERROR,
             "lbk_sellp_plan: needs slice_size 32 and the stored entry count");
        sellp_plan_launch(ctx, A->slice_sets, A->nslices, A->stored, tile_slices_dev);
    });
}

lbk_status lbk_coo_plan_size(const lbk_coo* A, int32_t* ntiles_out)
{
    if (!A || !ntiles_out) return LBK_USAGE_ERROR;
    *ntiles_out = coo_ntiles(A->nnz, A->nrows);
    return LBK_OK;
}

lbk_status lbk_coo_plan(lbk_ctx ctx, const lbk_coo* A, int32_t* tile_starts_dev)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->nnz > 0, LBK_USAGE_ERROR, "lbk_coo_plan: matrix has no entries");
        coo_plan_launch(ctx, A->row_idx, A->nrows, A->nnz, tile_starts_dev);
    });
}

}  // extern "C"
