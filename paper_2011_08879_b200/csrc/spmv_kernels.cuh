// spmv_kernels.cuh -- sm_100a SpMV kernels for CSR, COO, ELL and SELL-P.
//
// Reference semantics (paths relative to /root/reference/proj):
//   CSR  src/kernels/reference.cpp:74-89  y[r] = sum_k vals[k]*x[col[k]],
//        summed from 0.0 in ascending k, empty rows -> 0.
//   COO  src/kernels/reference.cpp:59-71  zero y, y[row[k]] += vals[k]*x[col[k]]
//        in k order (== the CSR order on canonical, sorted COO).
//   ELL / SELL-P: SURVEY.md App. B (Ginkgo layouts), same per-row order.
//
// Design:
//   * CSR and COO are TMA-staged, warp-specialised, persistent kernels.  The
//     matrix is cut into nnz-balanced, row-aligned tiles.  One producer warp
//     streams each tile's `vals`/`col_idx` (and COO `row_idx`) into a shared
//     memory ring with 1-D bulk copies (cp.async.bulk, L2 evict-first) that
//     complete on mbarriers; the consumer warps
//       phase A: p_k = vals_k * x[col_k] for every entry of the tile (all
//                gathers of the tile in flight at once; products rounded
//                individually, no FMA),
//       phase B: one thread per row sums its p_k sequentially from 0.0 in
//                ascending k -- exactly the reference's order, so rows of
//                length <= kLongRow are BIT-IDENTICAL to the FMA-free
//                reference; longer rows are reduced by a whole warp
//                (normwise tolerance).
//     Tiles whose padded size exceeds the ring slot (giant rows) are
//     processed straight from global memory by warp-per-row.
//   * ELL / SELL-P are column-major: thread-per-row (4 rows per thread with
//     128-bit value/index loads where alignment allows), streams read with
//     ld.global.nc.L1::no_allocate, x gathered through the read-only path.
//   * Every kernel takes an epilogue functor, so solver steps fuse their
//     dot products / vector updates into the SpMV pass (solver.cu).
#pragma once

#include "lbk_internal.cuh"

namespace lbk {

constexpr int kLongRow = 32;

template <typename T>
struct CsrView {
    int nrows, ncols;
    long long nnz;
    const int* __restrict__ row_ptr;
    const int* __restrict__ cols;
    const T* __restrict__ vals;
    const int* __restrict__ tile_rows;  // ntiles + 1
    int ntiles;
};

template <typename T>
struct CooView {
    int nrows, ncols;
    long long nnz;
    const int* __restrict__ rows;
    const int* __restrict__ cols;
    const T* __restrict__ vals;
    const int* __restrict__ tile_starts;  // ntiles + 1
    int ntiles;
};

template <typename T>
struct EllView {
    int nrows, ncols, width;
    long long stride;
    const int* __restrict__ cols;
    const T* __restrict__ vals;
};

template <typename T>
struct SellpView {
    int nrows, ncols, S, nslices;
    const int* __restrict__ slice_sets;
    const int* __restrict__ cols;
    const T* __restrict__ vals;
};

// ----------------------------------------------------------- epilogues
// An epilogue receives each finished row sum.  NV = number of double
// accumulators it reduces over the grid (0 = none).  skip() lets a solver
// step turn the whole launch into a no-op once the solve has finished.
template <typename T>
struct EpiStore {
    static constexpr int NV = 0;
    T* __restrict__ y;
    __device__ bool skip() const { return false; }
    __device__ void row(int r, T s, double*) const { y[r] = s; }
    __device__ void finish(const double*) const {}
};

template <typename T>
struct EpiAxpby {
    static constexpr int NV = 0;
    T* __restrict__ y;
    T alpha, beta;
    __device__ bool skip() const { return false; }
    __device__ void row(int r, T s, double*) const
    {
        T v = mul_rn(alpha, s);
        if (beta != T(0)) v = add_rn(v, mul_rn(beta, y[r]));
        y[r] = v;
    }
    __device__ void finish(const double*) const {}
};

// -------------------------------------------------------- plan kernels
// CSR tile t = rows [tile_rows[t], tile_rows[t+1]); tile_rows[t] is the
// first row starting at or after entry t*tile_nnz.
__global__ void csr_plan_kernel(const int* __restrict__ row_ptr, int nrows, int ntiles,
                                long long tile_nnz, int* __restrict__ tile_rows);
// COO tile t = entries [tile_starts[t], tile_starts[t+1]); tile_starts[t]
// is the first entry of the row holding entry t*tile_nnz.
__global__ void coo_plan_kernel(const int* __restrict__ rows, long long nnz, int ntiles,
                                long long tile_nnz, int* __restrict__ tile_starts);

// --------------------------------------------------- CSR staged kernel
struct CsrCfg {
    static constexpr int kConsumerWarps = 8;
    static constexpr int kTile = 2048;   // target nnz per tile
    static constexpr int kCap = 3072;    // ring slot capacity (entries)
    static constexpr int kStages = 4;
};

template <typename T, int CAP, int STAGES>
constexpr size_t csr_smem_bytes()
{
    return size_t(STAGES) * CAP * (sizeof(T) + 4) + size_t(CAP) * sizeof(T);
}

__device__ __forceinline__ void consumer_sync(int nthreads)
{
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <typename T, class Epi, int NCW, int CAP, int STAGES>
__global__ void __launch_bounds__((NCW + 1) * 32)
    csr_staged_kernel(CsrView<T> A, const T* __restrict__ x, Epi epi, RedWs ws)
{
    constexpr int NC = NCW * 32;
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    extern __shared__ __align__(128) unsigned char smem[];
    T* s_vals = reinterpret_cast<T*>(smem);
    int* s_cols = reinterpret_cast<int*>(smem + size_t(STAGES) * CAP * sizeof(T));
    T* s_prod = reinterpret_cast<T*>(smem + size_t(STAGES) * CAP * (sizeof(T) + 4));
    __shared__ __align__(8) uint64_t full[STAGES];
    __shared__ __align__(8) uint64_t empty[STAGES];
    __shared__ int4 info[STAGES];
    __shared__ double red_sh[32 * NV];

    if (epi.skip()) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const long long nnz4 = A.nnz & ~3LL;
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;

    if (warp == NCW) {
        // ---------------- producer warp: one elected lane drives the ring
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int j = 0;
            for (int t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++j) {
                const int s = j % STAGES;
                if (j >= STAGES) mbar_wait(&empty[s], ((j / STAGES) - 1) & 1);
                const int rb = __ldg(A.tile_rows + t), re = __ldg(A.tile_rows + t + 1);
                const int k0 = __ldg(A.row_ptr + rb), k1 = __ldg(A.row_ptr + re);
                info[s] = make_int4(rb, re, k0, k1);
                const long long k0a = k0 & ~3, k1a = (static_cast<long long>(k1) + 3) & ~3LL;
                const bool staged = (k1a - k0a) <= CAP;
                const long long ke = k1a < nnz4 ? k1a : nnz4;
                if (staged && ke > k0a) {
                    const uint32_t n = static_cast<uint32_t>(ke - k0a);
                    mbar_arrive_expect_tx(&full[s], n * uint32_t(sizeof(T) + 4));
                    tma_load_1d(s_vals + size_t(s) * CAP, A.vals + k0a, n * sizeof(T), &full[s], pol);
                    tma_load_1d(s_cols + size_t(s) * CAP, A.cols + k0a, n * 4u, &full[s], pol);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
        }
    } else {
        // ---------------- consumer warps
        int j = 0;
        for (int t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++j) {
            const int s = j % STAGES;
            mbar_wait(&full[s], (j / STAGES) & 1);
            const int4 in = info[s];
            const int rb = in.x, re = in.y, k0 = in.z, k1 = in.w;
            const int k0a = k0 & ~3;
            const long long k1a = (static_cast<long long>(k1) + 3) & ~3LL;
            const bool staged = (k1a - k0a) <= CAP;
            if (staged) {
                T* sv = s_vals + size_t(s) * CAP;
                int* sc = s_cols + size_t(s) * CAP;
                if (k1 > nnz4) {  // ragged tail past the last 16-B chunk
                    const int kt = k0 > nnz4 ? k0 : static_cast<int>(nnz4);
                    for (int k = kt + tid; k < k1; k += NC) {
                        sv[k - k0a] = A.vals[k];
                        sc[k - k0a] = A.cols[k];
                    }
                    fence_proxy_async_smem();
                    consumer_sync(NC);
                }
                // phase A: all products of the tile
                for (int k = k0 + tid; k < k1; k += NC) {
                    const int off = k - k0a;
                    s_prod[off] = mul_rn(sv[off], ldg_nc(x + sc[off]));
                }
                consumer_sync(NC);
                if (lane == 0) mbar_arrive(&empty[s]);  // slot free for the producer
                // phase B: rows
                for (int base = rb; base < re; base += NC) {
                    const int r = base + tid;
                    const bool act = r < re;
                    int rs = 0, rl = 0;
                    if (act) {
                        rs = __ldg(A.row_ptr + r);
                        rl = __ldg(A.row_ptr + r + 1) - rs;
                    }
                    const bool lng = act && rl > kLongRow;
                    unsigned lm = __ballot_sync(0xffffffffu, lng);
                    if (act && !lng) {
                        const T* p = s_prod + (rs - k0a);
                        T sum = T(0);
                        for (int k = 0; k < rl; ++k) sum = add_rn(sum, p[k]);
                        epi.row(r, sum, acc);
                    }
                    while (lm) {
                        const int src = __ffs(lm) - 1;
                        lm &= lm - 1;
                        const int rr = __shfl_sync(0xffffffffu, r, src);
                        const int ss = __shfl_sync(0xffffffffu, rs, src);
                        const int ll = __shfl_sync(0xffffffffu, rl, src);
                        T part = T(0);
                        for (int k = lane; k < ll; k += 32) part = add_rn(part, s_prod[ss - k0a + k]);
                        part = warp_sum(part);
                        if (lane == 0) epi.row(rr, part, acc);
                    }
                }
                consumer_sync(NC);  // s_prod is reused by the next tile
            } else {
                if (lane == 0) mbar_arrive(&empty[s]);
                // giant-row tile: warp per row straight from global memory
                for (int r = rb + warp; r < re; r += NCW) {
                    const int rs = __ldg(A.row_ptr + r), rend = __ldg(A.row_ptr + r + 1);
                    T part = T(0);
                    for (int k = rs + lane; k < rend; k += 32)
                        part = add_rn(part, mul_rn(A.vals[k], ldg_nc(x + A.cols[k])));
                    part = warp_sum(part);
                    if (lane == 0) epi.row(r, part, acc);
                }
            }
        }
    }

    if constexpr (Epi::NV > 0) {
        __syncthreads();
        block_sum<NV>(acc, tid, blockDim.x, red_sh);
        grid_reduce_finish<NV>(acc, ws, tid, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

// --------------------------------------------------- COO staged kernel
struct CooCfg {
    static constexpr int kConsumerWarps = 8;
    static constexpr int kTile = 2048;
    static constexpr int kCap = 3072;
    static constexpr int kStages = 3;
};

template <typename T, int CAP, int STAGES>
constexpr size_t coo_smem_bytes()
{
    return size_t(STAGES) * CAP * (sizeof(T) + 8) + size_t(CAP) * sizeof(T);
}

// first index in [lo, hi) with a[i] >= key
template <typename P>
__device__ __forceinline__ int lower_bound_i(P a, int lo, int hi, int key)
{
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <typename T, class Epi, int NCW, int CAP, int STAGES>
__global__ void __launch_bounds__((NCW + 1) * 32)
    coo_staged_kernel(CooView<T> A, const T* __restrict__ x, Epi epi, RedWs ws)
{
    constexpr int NC = NCW * 32;
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    extern __shared__ __align__(128) unsigned char smem[];
    T* s_vals = reinterpret_cast<T*>(smem);
    int* s_cols = reinterpret_cast<int*>(smem + size_t(STAGES) * CAP * sizeof(T));
    int* s_rows = s_cols + size_t(STAGES) * CAP;
    T* s_prod = reinterpret_cast<T*>(smem + size_t(STAGES) * CAP * (sizeof(T) + 8));
    __shared__ __align__(8) uint64_t full[STAGES];
    __shared__ __align__(8) uint64_t empty[STAGES];
    __shared__ int4 info[STAGES];
    __shared__ double red_sh[32 * NV];

    if (epi.skip()) return;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const long long nnz4 = A.nnz & ~3LL;
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;

    if (warp == NCW) {
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            int j = 0;
            for (int t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++j) {
                const int s = j % STAGES;
                if (j >= STAGES) mbar_wait(&empty[s], ((j / STAGES) - 1) & 1);
                const int k0 = __ldg(A.tile_starts + t), k1 = __ldg(A.tile_starts + t + 1);
                const int r0 = t == 0 ? 0 : __ldg(A.rows + k0);
                const int r1 = t + 1 == A.ntiles ? A.nrows : __ldg(A.rows + k1);
                info[s] = make_int4(r0, r1, k0, k1);
                const long long k0a = k0 & ~3, k1a = (static_cast<long long>(k1) + 3) & ~3LL;
                const bool staged = (k1a - k0a) <= CAP;
                const long long ke = k1a < nnz4 ? k1a : nnz4;
                if (staged && ke > k0a) {
                    const uint32_t n = static_cast<uint32_t>(ke - k0a);
                    mbar_arrive_expect_tx(&full[s], n * uint32_t(sizeof(T) + 8));
                    tma_load_1d(s_vals + size_t(s) * CAP, A.vals + k0a, n * sizeof(T), &full[s], pol);
                    tma_load_1d(s_cols + size_t(s) * CAP, A.cols + k0a, n * 4u, &full[s], pol);
                    tma_load_1d(s_rows + size_t(s) * CAP, A.rows + k0a, n * 4u, &full[s], pol);
                } else {
                    mbar_arrive(&full[s]);
                }
            }
        }
    } else {
        int j = 0;
        for (int t = blockIdx.x; t < A.ntiles; t += gridDim.x, ++j) {
            const int s = j % STAGES;
            mbar_wait(&full[s], (j / STAGES) & 1);
            const int4 in = info[s];
            const int r0 = in.x, r1 = in.y, k0 = in.z, k1 = in.w;
            const int k0a = k0 & ~3;
            const long long k1a = (static_cast<long long>(k1) + 3) & ~3LL;
            const bool staged = (k1a - k0a) <= CAP;
            if (staged) {
                T* sv = s_vals + size_t(s) * CAP;
                int* sc = s_cols + size_t(s) * CAP;
                int* sr = s_rows + size_t(s) * CAP;
                if (k1 > nnz4) {
                    const int kt = k0 > nnz4 ? k0 : static_cast<int>(nnz4);
                    for (int k = kt + tid; k < k1; k += NC) {
                        sv[k - k0a] = A.vals[k];
                        sc[k - k0a] = A.cols[k];
                        sr[k - k0a] = A.rows[k];
                    }
                    fence_proxy_async_smem();
                    consumer_sync(NC);
                }
                for (int k = k0 + tid; k < k1; k += NC) {
                    const int off = k - k0a;
                    s_prod[off] = mul_rn(sv[off], ldg_nc(x + sc[off]));
                }
                consumer_sync(NC);
                // phase B needs the row indices, so the slot is released
                // after the row sweep.
                const int lo0 = k0 - k0a, hi0 = k1 - k0a;
                for (int base = r0; base < r1; base += NC) {
                    const int r = base + tid;
                    const bool act = r < r1;
                    int rs = 0, rl = 0;
                    if (act) {
                        rs = lower_bound_i(sr, lo0, hi0, r);
                        rl = lower_bound_i(sr, rs, hi0, r + 1) - rs;
                    }
                    const bool lng = act && rl > kLongRow;
                    unsigned lm = __ballot_sync(0xffffffffu, lng);
                    if (act && !lng) {
                        T sum = T(0);
                        for (int k = 0; k < rl; ++k) sum = add_rn(sum, s_prod[rs + k]);
                        epi.row(r, sum, acc);
                    }
                    while (lm) {
                        const int src = __ffs(lm) - 1;
                        lm &= lm - 1;
                        const int rr = __shfl_sync(0xffffffffu, r, src);
                        const int ss = __shfl_sync(0xffffffffu, rs, src);
                        const int ll = __shfl_sync(0xffffffffu, rl, src);
                        T part = T(0);
                        for (int k = lane; k < ll; k += 32) part = add_rn(part, s_prod[ss + k]);
                        part = warp_sum(part);
                        if (lane == 0) epi.row(rr, part, acc);
                    }
                }
                consumer_sync(NC);
                if (lane == 0) mbar_arrive(&empty[s]);
            } else {
                if (lane == 0) mbar_arrive(&empty[s]);
                for (int r = r0 + warp; r < r1; r += NCW) {
                    int rs = 0, rend = 0;
                    if (lane == 0) {
                        rs = lower_bound_i(A.rows, k0, k1, r);
                        rend = lower_bound_i(A.rows, rs, k1, r + 1);
                    }
                    rs = __shfl_sync(0xffffffffu, rs, 0);
                    rend = __shfl_sync(0xffffffffu, rend, 0);
                    T part = T(0);
                    for (int k = rs + lane; k < rend; k += 32)
                        part = add_rn(part, mul_rn(A.vals[k], ldg_nc(x + A.cols[k])));
                    part = warp_sum(part);
                    if (lane == 0) epi.row(r, part, acc);
                }
            }
        }
    }

    if constexpr (Epi::NV > 0) {
        __syncthreads();
        block_sum<NV>(acc, tid, blockDim.x, red_sh);
        grid_reduce_finish<NV>(acc, ws, tid, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

// ----------------------------------------------------- ELL / SELL-P
__device__ __forceinline__ int4 ld_stream_i4(const int* p)
{
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double* p)
{
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ float4 ld_stream_f4(const float* p)
{
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

template <typename T>
struct Quad;
template <>
struct Quad<double> {
    double v[4];
    __device__ __forceinline__ void load(const double* p)
    {
        double2 a = ld_stream_d2(p), b = ld_stream_d2(p + 2);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
};
template <>
struct Quad<float> {
    float v[4];
    __device__ __forceinline__ void load(const float* p)
    {
        float4 a = ld_stream_f4(p);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    }
};

// Sliced column-major kernel shared by ELL (one slice of height `stride`)
// and SELL-P.  Each thread owns 4 consecutive rows of one slice: per column
// j it issues one 128-bit index load and one (f32) or two (f64) 128-bit
// value loads, then 4 independent gathers.  Row sums keep the reference's
// ascending-j order.  Requires: slice height % 4 == 0 and 16-B aligned
// arrays (checked by the host).
template <typename T, class Epi, bool IS_ELL>
__global__ void __launch_bounds__(256)
    sliced_quad_kernel(int nrows, int S, const int* __restrict__ slice_sets, int ell_width,
                       const int* __restrict__ cols, const T* __restrict__ vals,
                       const T* __restrict__ x, Epi epi, RedWs ws)
{
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;
    const long long nquads = (static_cast<long long>(nrows) + 3) / 4;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nquads;
         q += (long long)gridDim.x * blockDim.x) {
        const int r0 = static_cast<int>(q * 4);
        long long base;
        int len;
        long long pitch;
        if constexpr (IS_ELL) {
            base = r0;
            len = ell_width;
            pitch = S;  // S carries the ELL stride
        } else {
            const int sl = r0 / S;
            const int a = __ldg(slice_sets + sl), b = __ldg(slice_sets + sl + 1);
            base = static_cast<long long>(a) * S + (r0 - sl * S);
            len = b - a;
            pitch = S;
        }
        T sum[4] = {T(0), T(0), T(0), T(0)};
        int j = 0;
        for (; j + 1 < len; j += 2) {
            const long long o0 = base + j * pitch, o1 = o0 + pitch;
            const int4 c0 = ld_stream_i4(cols + o0), c1 = ld_stream_i4(cols + o1);
            Quad<T> v0, v1;
            v0.load(vals + o0);
            v1.load(vals + o1);
            const int cc0[4] = {c0.x, c0.y, c0.z, c0.w}, cc1[4] = {c1.x, c1.y, c1.z, c1.w};
            T g0[4], g1[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                g0[i] = cc0[i] >= 0 ? ldg_nc(x + cc0[i]) : T(0);
                g1[i] = cc1[i] >= 0 ? ldg_nc(x + cc1[i]) : T(0);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (cc0[i] >= 0) sum[i] = add_rn(sum[i], mul_rn(v0.v[i], g0[i]));
                if (cc1[i] >= 0) sum[i] = add_rn(sum[i], mul_rn(v1.v[i], g1[i]));
            }
        }
        if (j < len) {
            const long long o0 = base + j * pitch;
            const int4 c0 = ld_stream_i4(cols + o0);
            Quad<T> v0;
            v0.load(vals + o0);
            const int cc0[4] = {c0.x, c0.y, c0.z, c0.w};
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (cc0[i] >= 0) sum[i] = add_rn(sum[i], mul_rn(v0.v[i], ldg_nc(x + cc0[i])));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (r0 + i < nrows) epi.row(r0 + i, sum[i], acc);
    }
    if constexpr (Epi::NV > 0) {
        block_sum<NV>(acc, threadIdx.x, blockDim.x, red_sh);
        grid_reduce_finish<NV>(acc, ws, threadIdx.x, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

// Scalar fallback (unaligned / odd slice heights): thread per row.
template <typename T, class Epi, bool IS_ELL>
__global__ void __launch_bounds__(256)
    sliced_row_kernel(int nrows, int S, const int* __restrict__ slice_sets, int ell_width,
                      const int* __restrict__ cols, const T* __restrict__ vals,
                      const T* __restrict__ x, Epi epi, RedWs ws)
{
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;
    for (long long rr = blockIdx.x * (long long)blockDim.x + threadIdx.x; rr < nrows;
         rr += (long long)gridDim.x * blockDim.x) {
        const int r = static_cast<int>(rr);
        long long base;
        int len;
        if constexpr (IS_ELL) {
            base = r;
            len = ell_width;
        } else {
            const int sl = r / S;
            const int a = __ldg(slice_sets + sl), b = __ldg(slice_sets + sl + 1);
            base = static_cast<long long>(a) * S + (r - sl * S);
            len = b - a;
        }
        T sum = T(0);
#pragma unroll 4
        for (int j = 0; j < len; ++j) {
            const long long o = base + static_cast<long long>(j) * S;
            const int c = __ldg(cols + o);
            if (c >= 0) sum = add_rn(sum, mul_rn(__ldg(vals + o), ldg_nc(x + c)));
        }
        epi.row(r, sum, acc);
    }
    if constexpr (Epi::NV > 0) {
        block_sum<NV>(acc, threadIdx.x, blockDim.x, red_sh);
        grid_reduce_finish<NV>(acc, ws, threadIdx.x, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

}  // namespace lbk
