// convert.cu -- device-side format conversions and validation.
//
// Reference: src/matrix/formats.cpp (paths relative to /root/reference/proj)
//   coo_from_entries  :78-116   bounds check, stable (row,col) sort, sum
//                               duplicates in input order, keep zeros
//   coo_to_csr        :132-155  histogram + inclusive scan; col/vals verbatim
//   csr_to_coo        :158-179  expand row_ptr
//   validate          :182-242  invariant checks -> FormatError
// plus ELL / SELL-P builders (absent from the reference).
// All index outputs are integer work and bit-exact with the reference / the
// oracle restatement; duplicate sums are summed sequentially in input
// order, as the reference does.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "api_guard.h"

namespace lbk {

namespace {

// Stream-ordered temporary device buffer.
struct Tmp {
    void* p = nullptr;
    cudaStream_t s;
    Tmp(size_t bytes, cudaStream_t st) : s(st)
    {
        if (bytes) LBK_CUDA(cudaMallocAsync(&p, bytes, s));
    }
    ~Tmp()
    {
        if (p) cudaFreeAsync(p, s);
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

int grid1d(long long n, int threads = 256)
{
    long long g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > (1LL << 30)) g = 1LL << 30;
    return static_cast<int>(g);
}

// ---------------------------------------------------------- coo <-> csr
__global__ void row_hist_kernel(long long nnz, const int* __restrict__ rows, int* __restrict__ counts)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
         k += (long long)gridDim.x * blockDim.x)
        atomicAdd(counts + rows[k] + 1, 1);
}

__global__ void expand_rows_kernel(int nrows, const int* __restrict__ row_ptr, int* __restrict__ rows)
{
    const long long w = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long r = w; r < nrows; r += nw) {
        const int s = row_ptr[r], e = row_ptr[r + 1];
        for (int k = s + lane; k < e; k += 32) rows[k] = static_cast<int>(r);
    }
}

// ------------------------------------------------------------- assembly
__global__ void bounds_kernel(long long n, const int* __restrict__ rows, const int* __restrict__ cols,
                              int nrows, int ncols, unsigned long long* __restrict__ first_bad)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        const int r = rows[k], c = cols[k];
        if (r < 0 || r >= nrows || c < 0 || c >= ncols) atomicMin(first_bad, (unsigned long long)k);
    }
}

__global__ void make_keys_kernel(long long n, const int* __restrict__ rows, const int* __restrict__ cols,
                                 unsigned long long* __restrict__ keys, long long* __restrict__ idx)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        keys[k] = (static_cast<unsigned long long>(static_cast<unsigned>(rows[k])) << 32) |
                  static_cast<unsigned>(cols[k]);
        idx[k] = k;
    }
}

__global__ void head_flags_kernel(long long n, const unsigned long long* __restrict__ keys,
                                  int* __restrict__ flags)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x)
        flags[k] = (k == 0 || keys[k] != keys[k - 1]) ? 1 : 0;
}

// One thread per canonical entry: sums its duplicate run sequentially in
// input order (stable sort keeps it), formats.cpp:99-108.
__global__ void emit_kernel(long long n, const unsigned long long* __restrict__ keys,
                            const long long* __restrict__ idx, const int* __restrict__ flags,
                            const int* __restrict__ pos, const double* __restrict__ vals,
                            int* __restrict__ rows_out, int* __restrict__ cols_out,
                            double* __restrict__ vals_out)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
         k += (long long)gridDim.x * blockDim.x) {
        if (!flags[k]) continue;
        const unsigned long long key = keys[k];
        double v = vals[idx[k]];
        for (long long j = k + 1; j < n && keys[j] == key; ++j) v = add_rn(v, vals[idx[j]]);
        const int o = pos[k];
        rows_out[o] = static_cast<int>(key >> 32);
        cols_out[o] = static_cast<int>(key & 0xffffffffu);
        vals_out[o] = v;
    }
}

// ------------------------------------------------------------ ELL/SELL-P
__global__ void row_len_kernel(int nrows, const int* __restrict__ row_ptr, int* __restrict__ len)
{
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nrows;
         r += (long long)gridDim.x * blockDim.x)
        len[r] = row_ptr[r + 1] - row_ptr[r];
}

template <typename T>
__global__ void to_ell_kernel(int nrows, const int* __restrict__ row_ptr, const int* __restrict__ cols,
                              const T* __restrict__ vals, int width, long long stride,
                              int* __restrict__ ecols, T* __restrict__ evals)
{
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < stride;
         r += (long long)gridDim.x * blockDim.x) {
        int s = 0, len = 0;
        if (r < nrows) {
            s = row_ptr[r];
            len = row_ptr[r + 1] - s;
        }
        for (int j = 0; j < width; ++j) {
            const long long at = static_cast<long long>(j) * stride + r;
            if (j < len) {
                ecols[at] = cols[s + j];
                evals[at] = vals[s + j];
            } else {
                ecols[at] = -1;
                evals[at] = T(0);
            }
        }
    }
}

__global__ void slice_len_kernel(int nrows, int S, int nslices, const int* __restrict__ row_ptr,
                                 int* __restrict__ slice_len)
{
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nslices;
         s += (long long)gridDim.x * blockDim.x) {
        int w = 0;
        const long long r0 = s * S;
        const long long r1 = r0 + S < nrows ? r0 + S : nrows;
        for (long long r = r0; r < r1; ++r) {
            const int l = row_ptr[r + 1] - row_ptr[r];
            w = l > w ? l : w;
        }
        slice_len[s] = w;
    }
}

template <typename T>
__global__ void to_sellp_kernel(int nrows, int S, int nslices, const int* __restrict__ row_ptr,
                                const int* __restrict__ cols, const T* __restrict__ vals,
                                const int* __restrict__ sets, int* __restrict__ scols,
                                T* __restrict__ svals)
{
    const long long total = static_cast<long long>(nslices) * S;
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < total;
         r += (long long)gridDim.x * blockDim.x) {
        const int sl = static_cast<int>(r / S), lane = static_cast<int>(r % S);
        const int w = sets[sl + 1] - sets[sl];
        int s = 0, len = 0;
        if (r < nrows) {
            s = row_ptr[r];
            len = row_ptr[r + 1] - s;
        }
        for (int j = 0; j < w; ++j) {
            const long long at = (static_cast<long long>(sets[sl]) + j) * S + lane;
            if (j < len) {
                scols[at] = cols[s + j];
                svals[at] = vals[s + j];
            } else {
                scols[at] = -1;
                svals[at] = T(0);
            }
        }
    }
}

// ----------------------------------------------------------- validation
// error codes, lowest row/entry index wins (first violation, like the
// sequential reference loop)
__global__ void validate_csr_kernel(int nrows, int ncols, long long nnz, const int* __restrict__ row_ptr,
                                    const int* __restrict__ cols, unsigned long long* __restrict__ bad)
{
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < nrows;
         r += (long long)gridDim.x * blockDim.x) {
        const int s = row_ptr[r], e = row_ptr[r + 1];
        unsigned long long code = 0;
        if (s > e) code = 1;  // decreasing
        else {
            for (int k = s; k < e && !code; ++k) {
                if (k < 0 || k >= nnz) { code = 4; break; }
                const int c = cols[k];
                if (c < 0 || c >= ncols) code = 2;
                else if (k > s && cols[k - 1] >= c) code = 3;
            }
        }
        if (code) atomicMin(bad, (static_cast<unsigned long long>(r) << 3) | code);
    }
}

__global__ void validate_coo_kernel(int nrows, int ncols, long long nnz, const int* __restrict__ rows,
                                    const int* __restrict__ cols, unsigned long long* __restrict__ bad)
{
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nnz;
         k += (long long)gridDim.x * blockDim.x) {
        const int r = rows[k], c = cols[k];
        unsigned long long code = 0;
        if (r < 0 || r >= nrows || c < 0 || c >= ncols) code = 1;
        else if (k > 0) {
            const int pr = rows[k - 1], pc = cols[k - 1];
            if (!(pr < r || (pr == r && pc < c))) code = 2;
        }
        if (code) atomicMin(bad, (static_cast<unsigned long long>(k) << 3) | code);
    }
}

unsigned long long read_u64(lbk_ctx ctx, const unsigned long long* d)
{
    unsigned long long h = 0;
    LBK_CUDA(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    LBK_CUDA(cudaStreamSynchronize(ctx->stream));
    return h;
}

template <typename T>
void csr_to_ell_impl(lbk_ctx ctx, const lbk_csr* A, int width, long long stride, int* cols_out,
                     void* vals_out)
{
    need(width >= 0 && stride >= A->nrows, LBK_FORMAT_ERROR, "csr_to_ell: need stride >= nrows");
    if (stride == 0 || width == 0) return;
    to_ell_kernel<T><<<grid1d(stride), 256, 0, ctx->stream>>>(
        A->nrows, A->row_ptr, A->col_idx, static_cast<const T*>(A->vals), width, stride, cols_out,
        static_cast<T*>(vals_out));
    LBK_LAUNCH_CHECK();
}

template <typename T>
void csr_to_sellp_impl(lbk_ctx ctx, const lbk_csr* A, int S, const int* sets, int* cols_out,
                       void* vals_out)
{
    const int nslices = (A->nrows + S - 1) / S;
    if (nslices == 0) return;
    to_sellp_kernel<T><<<grid1d(static_cast<long long>(nslices) * S), 256, 0, ctx->stream>>>(
        A->nrows, S, nslices, A->row_ptr, A->col_idx, static_cast<const T*>(A->vals), sets, cols_out,
        static_cast<T*>(vals_out));
    LBK_LAUNCH_CHECK();
}

}  // namespace
}  // namespace lbk

using namespace lbk;

extern "C" {

lbk_status lbk_coo_to_csr(lbk_ctx ctx, const lbk_coo* A, int32_t* row_ptr_out)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->nrows >= 0 && A->nnz >= 0, LBK_SHAPE_ERROR, "coo_to_csr: negative size");
        LBK_CUDA(cudaMemsetAsync(row_ptr_out, 0, (size_t(A->nrows) + 1) * sizeof(int), ctx->stream));
        if (A->nnz > 0) {
            row_hist_kernel<<<grid1d(A->nnz), 256, 0, ctx->stream>>>(A->nnz, A->row_idx, row_ptr_out);
            LBK_LAUNCH_CHECK();
        }
        // inclusive scan of counts (row_ptr[0] stays 0)
        size_t tb = 0;
        LBK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, row_ptr_out, row_ptr_out,
                                               A->nrows + 1, ctx->stream));
        Tmp t(tb, ctx->stream);
        LBK_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb, row_ptr_out, row_ptr_out, A->nrows + 1,
                                               ctx->stream));
    });
}

lbk_status lbk_csr_to_coo(lbk_ctx ctx, const lbk_csr* A, int32_t* row_idx_out)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (A->nrows == 0 || A->nnz == 0) return;
        expand_rows_kernel<<<grid1d(static_cast<long long>(A->nrows) * 32), 256, 0, ctx->stream>>>(
            A->nrows, A->row_ptr, row_idx_out);
        LBK_LAUNCH_CHECK();
    });
}

lbk_status lbk_coo_assemble_f64(lbk_ctx ctx, int32_t nrows, int32_t ncols, int64_t n,
                                const int32_t* rows, const int32_t* cols, const double* vals,
                                int32_t* rows_out, int32_t* cols_out, double* vals_out,
                                int64_t* nnz_out)
{
    if (!ctx || !nnz_out) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(nrows >= 0 && ncols >= 0, LBK_FORMAT_ERROR, "negative matrix dimension");
        need(n >= 0 && n < (1LL << 31), LBK_SHAPE_ERROR, "entry count outside [0, 2^31)");
        *nnz_out = 0;
        if (n == 0) return;
        Tmp bad(sizeof(unsigned long long), ctx->stream);
        LBK_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), ctx->stream));
        bounds_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(n, rows, cols, nrows, ncols,
                                                          bad.as<unsigned long long>());
        LBK_LAUNCH_CHECK();
        const unsigned long long first = read_u64(ctx, bad.as<unsigned long long>());
        if (first != ~0ULL) {
            int rc[2];
            LBK_CUDA(cudaMemcpy(&rc[0], rows + first, 4, cudaMemcpyDeviceToHost));
            LBK_CUDA(cudaMemcpy(&rc[1], cols + first, 4, cudaMemcpyDeviceToHost));
            fail(LBK_FORMAT_ERROR, "entry " + std::to_string(first) + " at (" +
                                       std::to_string(rc[0]) + ", " + std::to_string(rc[1]) +
                                       ") is outside a " + std::to_string(nrows) + "x" +
                                       std::to_string(ncols) + " matrix");
        }
        Tmp keys_in(n * 8, ctx->stream), keys(n * 8, ctx->stream), idx_in(n * 8, ctx->stream),
            idx(n * 8, ctx->stream), flags(n * 4, ctx->stream), pos(n * 4, ctx->stream);
        make_keys_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(n, rows, cols,
                                                             keys_in.as<unsigned long long>(),
                                                             idx_in.as<long long>());
        LBK_LAUNCH_CHECK();
        // LSD radix sort is stable: equal (row, col) keep input order
        // (std::stable_sort, formats.cpp:89-92).
        size_t tb = 0;
        LBK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys_in.as<unsigned long long>(),
                                                 keys.as<unsigned long long>(), idx_in.as<long long>(),
                                                 idx.as<long long>(), n, 0, 64, ctx->stream));
        {
            Tmp t(tb, ctx->stream);
            LBK_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tb, keys_in.as<unsigned long long>(),
                                                     keys.as<unsigned long long>(),
                                                     idx_in.as<long long>(), idx.as<long long>(), n,
                                                     0, 64, ctx->stream));
        }
        head_flags_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(n, keys.as<unsigned long long>(),
                                                              flags.as<int>());
        LBK_LAUNCH_CHECK();
        tb = 0;
        LBK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, flags.as<int>(), pos.as<int>(), n,
                                               ctx->stream));
        {
            Tmp t(tb, ctx->stream);
            LBK_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tb, flags.as<int>(), pos.as<int>(), n,
                                                   ctx->stream));
        }
        emit_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(n, keys.as<unsigned long long>(),
                                                        idx.as<long long>(), flags.as<int>(),
                                                        pos.as<int>(), vals, rows_out, cols_out,
                                                        vals_out);
        LBK_LAUNCH_CHECK();
        int lastpos = 0, lastflag = 0;
        LBK_CUDA(cudaMemcpyAsync(&lastpos, pos.as<int>() + n - 1, 4, cudaMemcpyDeviceToHost, ctx->stream));
        LBK_CUDA(cudaMemcpyAsync(&lastflag, flags.as<int>() + n - 1, 4, cudaMemcpyDeviceToHost, ctx->stream));
        LBK_CUDA(cudaStreamSynchronize(ctx->stream));
        *nnz_out = static_cast<int64_t>(lastpos) + lastflag;
    });
}

lbk_status lbk_csr_ell_width(lbk_ctx ctx, const lbk_csr* A, int32_t* width_out)
{
    if (!ctx || !A || !width_out) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        *width_out = 0;
        if (A->nrows == 0) return;
        Tmp len(size_t(A->nrows) * 4, ctx->stream), mx(4, ctx->stream);
        row_len_kernel<<<grid1d(A->nrows), 256, 0, ctx->stream>>>(A->nrows, A->row_ptr, len.as<int>());
        LBK_LAUNCH_CHECK();
        size_t tb = 0;
        LBK_CUDA(cub::DeviceReduce::Max(nullptr, tb, len.as<int>(), mx.as<int>(), A->nrows, ctx->stream));
        Tmp t(tb, ctx->stream);
        LBK_CUDA(cub::DeviceReduce::Max(t.p, tb, len.as<int>(), mx.as<int>(), A->nrows, ctx->stream));
        int w = 0;
        LBK_CUDA(cudaMemcpyAsync(&w, mx.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
        LBK_CUDA(cudaStreamSynchronize(ctx->stream));
        *width_out = w;
    });
}

lbk_status lbk_csr_to_ell(lbk_ctx ctx, const lbk_csr* A, int32_t width, int64_t stride,
                          int32_t* cols_out, void* vals_out)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (A->dtype == LBK_F64) csr_to_ell_impl<double>(ctx, A, width, stride, cols_out, vals_out);
        else csr_to_ell_impl<float>(ctx, A, width, stride, cols_out, vals_out);
    });
}

lbk_status lbk_csr_sellp_plan(lbk_ctx ctx, const lbk_csr* A, int32_t S, int32_t* slice_lengths_out,
                              int32_t* slice_sets_out, int64_t* stored_out)
{
    if (!ctx || !A || !stored_out) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(S > 0, LBK_CONFIGURATION_ERROR, "slice_size must be positive");
        const int nslices = (A->nrows + S - 1) / S;
        LBK_CUDA(cudaMemsetAsync(slice_sets_out, 0, (size_t(nslices) + 1) * 4, ctx->stream));
        *stored_out = 0;
        if (nslices == 0) return;
        slice_len_kernel<<<grid1d(nslices), 256, 0, ctx->stream>>>(A->nrows, S, nslices, A->row_ptr,
                                                                   slice_lengths_out);
        LBK_LAUNCH_CHECK();
        // slice_sets = exclusive prefix sum (length nslices + 1)
        LBK_CUDA(cudaMemcpyAsync(slice_sets_out + 1, slice_lengths_out, size_t(nslices) * 4,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
        size_t tb = 0;
        LBK_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, slice_sets_out, slice_sets_out,
                                               nslices + 1, ctx->stream));
        Tmp t(tb, ctx->stream);
        LBK_CUDA(cub::DeviceScan::InclusiveSum(t.p, tb, slice_sets_out, slice_sets_out, nslices + 1,
                                               ctx->stream));
        int last = 0;
        LBK_CUDA(cudaMemcpyAsync(&last, slice_sets_out + nslices, 4, cudaMemcpyDeviceToHost, ctx->stream));
        LBK_CUDA(cudaStreamSynchronize(ctx->stream));
        *stored_out = static_cast<int64_t>(last) * S;
    });
}

lbk_status lbk_csr_to_sellp(lbk_ctx ctx, const lbk_csr* A, int32_t S, const int32_t* slice_sets,
                            int32_t* cols_out, void* vals_out)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(S > 0, LBK_CONFIGURATION_ERROR, "slice_size must be positive");
        if (A->dtype == LBK_F64) csr_to_sellp_impl<double>(ctx, A, S, slice_sets, cols_out, vals_out);
        else csr_to_sellp_impl<float>(ctx, A, S, slice_sets, cols_out, vals_out);
    });
}

lbk_status lbk_validate_csr(lbk_ctx ctx, const lbk_csr* A)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->nrows >= 0 && A->ncols >= 0 && A->nnz >= 0, LBK_FORMAT_ERROR, "negative size");
        int ends[2] = {0, 0};
        if (A->nrows >= 0) {
            LBK_CUDA(cudaMemcpyAsync(&ends[0], A->row_ptr, 4, cudaMemcpyDeviceToHost, ctx->stream));
            LBK_CUDA(cudaMemcpyAsync(&ends[1], A->row_ptr + A->nrows, 4, cudaMemcpyDeviceToHost,
                                     ctx->stream));
            LBK_CUDA(cudaStreamSynchronize(ctx->stream));
        }
        // formats.cpp:222-225
        need(ends[0] == 0 && ends[1] == A->nnz, LBK_FORMAT_ERROR, "csr row pointers must span [0, nnz]");
        if (A->nrows == 0) return;
        Tmp bad(8, ctx->stream);
        LBK_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, ctx->stream));
        validate_csr_kernel<<<grid1d(A->nrows), 256, 0, ctx->stream>>>(
            A->nrows, A->ncols, A->nnz, A->row_ptr, A->col_idx, bad.as<unsigned long long>());
        LBK_LAUNCH_CHECK();
        const unsigned long long b = read_u64(ctx, bad.as<unsigned long long>());
        if (b == ~0ULL) return;
        const long long row = static_cast<long long>(b >> 3);
        switch (b & 7) {
        case 1: fail(LBK_FORMAT_ERROR, "csr row pointers decrease at row " + std::to_string(row));
        case 2: fail(LBK_FORMAT_ERROR, "csr column index out of range");
        case 3: fail(LBK_FORMAT_ERROR, "csr column indices not strictly increasing in row " +
                                           std::to_string(row));
        default: fail(LBK_FORMAT_ERROR, "csr row pointers out of [0, nnz] at row " + std::to_string(row));
        }
    });
}

lbk_status lbk_validate_coo(lbk_ctx ctx, const lbk_coo* A)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->nrows >= 0 && A->ncols >= 0 && A->nnz >= 0, LBK_FORMAT_ERROR, "negative size");
        if (A->nnz == 0) return;
        Tmp bad(8, ctx->stream);
        LBK_CUDA(cudaMemsetAsync(bad.p, 0xff, 8, ctx->stream));
        validate_coo_kernel<<<grid1d(A->nnz), 256, 0, ctx->stream>>>(
            A->nrows, A->ncols, A->nnz, A->row_idx, A->col_idx, bad.as<unsigned long long>());
        LBK_LAUNCH_CHECK();
        const unsigned long long b = read_u64(ctx, bad.as<unsigned long long>());
        if (b == ~0ULL) return;
        const long long k = static_cast<long long>(b >> 3);
        if ((b & 7) == 1)
            fail(LBK_FORMAT_ERROR, "entry " + std::to_string(k) + " is outside a " +
                                       std::to_string(A->nrows) + "x" + std::to_string(A->ncols) +
                                       " matrix");
        fail(LBK_FORMAT_ERROR, "coo entries not strictly sorted at " + std::to_string(k));
    });
}

}  // extern "C"
