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
//   * CSR and COO are warp-pipelined kernels over nnz-balanced, row-aligned
//     tiles: each warp TMA-stages the next tile's arrays into shared memory
//     while it processes the current one lane-per-row (csr_stream_kernel).
//   * ELL / SELL-P are column-major: thread-per-row (4 rows per thread with
//     128-bit value/index loads where alignment allows), streams read with
//     ld.global.nc.L1::no_allocate, x gathered through the read-only path.
//   * Every kernel takes an epilogue functor, so solver steps fuse their
//     dot products / vector updates into the SpMV pass (solver.cu).
#pragma once

#include <type_traits>

#include "lbk_internal.cuh"

namespace lbk {

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
    __device__ void row(int r, T s, auto*) const { y[r] = s; }
    __device__ void finish(const double*) const {}
};

template <typename T>
struct EpiAxpby {
    static constexpr int NV = 0;
    T* __restrict__ y;
    T alpha, beta;
    struct Pre {
        T y;
    };
    __device__ bool skip() const { return false; }
    __device__ void prefetch(int rb, int re) const
    {
        if constexpr (sizeof(T) == 8)
            if (beta != T(0)) l2_prefetch_rows(reinterpret_cast<const double*>(y), rb, re);
    }
    __device__ Pre pre(int r) const { return {beta != T(0) ? y[r] : T(0)}; }
    __device__ void row_pre(int r, T s, const Pre& p, auto*) const
    {
        T v = mul_rn(alpha, s);
        if (beta != T(0)) v = add_rn(v, mul_rn(beta, p.y));
        y[r] = v;
    }
    __device__ void row(int r, T s, auto* acc) const { row_pre(r, s, pre(r), acc); }
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

// ------------------------------------------------ CSR / COO stream kernels
// Warp-pipelined, TMA-staged CSR / COO over nnz-balanced, row-aligned tiles
// (a merge-path split constrained to row boundaries).  Every warp of a
// persistent grid owns whole tiles and runs its own slot pipeline in
// shared memory (warp_tile_loop):
//   * lane 0 issues 1-D bulk copies (cp.async.bulk, L2 evict-first) of a
//     later tile's vals / col_idx (/ row_idx) into a free slot, completing
//     on that slot's mbarrier -- the matrix streams never touch the LSU/L1
//     data path (ncu showed the L1 data pipe, not HBM, bounding an
//     LSU-streamed version at 82% busy);
//   * meanwhile the warp sweeps the current tile (staged_rows): lane-per-row
//     register gathers for short rows (coalesced like ELL on banded
//     matrices), entry-parallel in-place products when a pass holds long
//     rows;
//   * each row of <= kSeqRow entries is summed sequentially from 0.0 in
//     ascending k with individually rounded products (no FMA) -- the
//     reference's order (reference.cpp:82-88), hence BIT-IDENTICAL to the
//     FMA-free reference; longer rows are reduced by the warp (normwise
//     tolerance);
//   * the one row of a tile that can overflow a slot goes from global memory
//     (warp_row_global), the rest of that tile is staged.
// The tile size is chosen per matrix (one warp pass of 32*G rows of mean
// length): see stream_tile_nnz().
#ifndef LBK_CSR_MINB
#define LBK_CSR_MINB 2  // CTAs per SM the CSR stream kernel is register-budgeted for
#endif
#ifndef LBK_CSR_CAP
#define LBK_CSR_CAP 1024
#endif
#ifndef LBK_CSR_SLOTS
#define LBK_CSR_SLOTS 2
#endif
#ifndef LBK_CSR_WARPS
#define LBK_CSR_WARPS 4
#endif
#ifndef LBK_COO_CAP
#define LBK_COO_CAP 768
#endif
#ifndef LBK_COO_SLOTS
#define LBK_COO_SLOTS 2
#endif
#ifndef LBK_COO_WARPS
#define LBK_COO_WARPS 4
#endif
// Per-format pipeline shape (measured on B200, scripts/variants.sh): a warp
// keeps kSlots-1 tiles in flight while it sweeps one.  CSR: 2 slots x 12 KB
// per warp, 4-warp CTAs, 2 CTAs (8 pipelines) per SM -- 3 slots with fewer
// warps, or smaller slots with more warps, were both slower on cfg2 and
// cfg4.  COO stages 16 B/entry: 2 slots x 12 KB (768 entries), 4-warp CTAs.
template <typename T, int NIDX>
struct StreamCfg {
    static constexpr int kCap = NIDX == 1 ? LBK_CSR_CAP : LBK_COO_CAP;  // entries per slot
    static constexpr int kSlots = NIDX == 1 ? LBK_CSR_SLOTS : LBK_COO_SLOTS;
    static constexpr int kWarps = NIDX == 1 ? LBK_CSR_WARPS : LBK_COO_WARPS;
    static constexpr int kThreads = kWarps * 32;
    static constexpr size_t slot_bytes = size_t(kCap) * (sizeof(T) + 4 * NIDX);
    static constexpr size_t smem_bytes = size_t(kWarps) * kSlots * slot_bytes;
};
constexpr int kTileMin = 384;

// Rows per lane per pass (G) from the mean row length: G*CH = 32 gathers
// in flight per lane whichever the row length.
inline int stream_group(long long nnz, long long nrows)
{
    const long long mean = nrows > 0 ? (nnz + nrows - 1) / nrows : 1;
    return mean <= 8 ? 4 : (mean <= 16 ? 2 : 1);
}

// nnz-balanced tile size: one pass of the warp (32*G rows of mean length),
// clamped so the tile plus a straddling row and alignment padding fits a
// slot.
inline long long stream_tile_nnz(long long nnz, long long nrows, int idx_arrays)
{
    const long long tmax =
        (idx_arrays == 1 ? StreamCfg<double, 1>::kCap : StreamCfg<double, 2>::kCap) - 128;
    long long mean = nrows > 0 ? (nnz + nrows - 1) / nrows : 1;
    long long t = 32LL * stream_group(nnz, nrows) * (mean < 1 ? 1 : mean);
    t = t < kTileMin ? kTileMin : (t > tmax ? tmax : t);
    return t;
}

struct int4x2 {
    int4 a, b;
};

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

// One row straight from global memory by a whole warp: rows <= 32 keep the
// sequential order (bit-exact); longer rows keep 16 loads and then 16
// gathers per lane in flight per round, 4 lane partials and a fixed-order
// warp reduction (deterministic).
template <typename T>
__device__ __forceinline__ T warp_row_global(int ks, int ke, const int* __restrict__ cols,
                                             const T* __restrict__ vals, const T* __restrict__ x)
{
    const int lane = threadIdx.x & 31;
    if (ke - ks <= 256) {
        // up to kSeqRow entries (a row that overflowed its tile's slot can be
        // this short): products 32 at a time, summed in ascending k through
        // shuffles -- the reference's order and bits (reference.cpp:82-88)
        T sum = T(0);
        for (int c = ks; c < ke; c += 32) {
            T p = T(0);
            if (c + lane < ke) p = mul_rn(__ldcs(vals + c + lane), ldg_nc(x + __ldcs(cols + c + lane)));
            const int m = ke - c < 32 ? ke - c : 32;
            for (int k = 0; k < m; ++k) sum = add_rn(sum, __shfl_sync(0xffffffffu, p, k));
        }
        return sum;
    }
    // 16 independent loads (and then gathers) per lane in flight per round
    T p[4] = {T(0), T(0), T(0), T(0)};
    int k = ks + lane;
    for (; k + 15 * 32 < ke; k += 16 * 32) {
        int c[16];
        T v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            c[u] = __ldcs(cols + k + u * 32);
            v[u] = __ldcs(vals + k + u * 32);
        }
        T g[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) g[u] = ldg_nc(x + c[u]);
#pragma unroll
        for (int u = 0; u < 16; ++u) p[u & 3] = add_rn(p[u & 3], mul_rn(v[u], g[u]));
    }
    for (; k < ke; k += 32) p[0] = add_rn(p[0], mul_rn(__ldcs(vals + k), ldg_nc(x + __ldcs(cols + k))));
    const T p0 = p[0], p1 = p[1], p2 = p[2], p3 = p[3];
    return warp_sum(add_rn(add_rn(p0, p1), add_rn(p2, p3)));
}

// Register-level operand prefetch (opt-in, -DLBK_EPI_PRE): an epilogue may
// declare `struct Pre`, `Pre pre(int r)` and `row_pre(r, s, pre, acc)`; the
// staged sweep then issues the row's operand loads (b[r], p[r], ...)
// together with its gathers.  Off by default: with the operand streams
// already L2-prefetched when the tile is staged (EpiPf), the extra live
// registers cost more than the latency they hide -- measured on cfg4/cfg5,
// CG 1102 -> 1176 it/s, BiCGSTAB 728 -> 752, CGS 739 -> 764 without it.
template <class Epi, class = void>
struct EpiPre {
    struct type {};
    __device__ static type load(const Epi&, int) { return {}; }
    template <typename T>
    __device__ static void row(const Epi& e, int r, T s, const type&, auto* acc)
    {
        e.row(r, s, acc);
    }
};
#ifdef LBK_EPI_PRE
template <class Epi>
struct EpiPre<Epi, std::void_t<typename Epi::Pre>> {
    using type = typename Epi::Pre;
    __device__ static type load(const Epi& e, int r) { return e.pre(r); }
    template <typename T>
    __device__ static void row(const Epi& e, int r, T s, const type& p, auto* acc)
    {
        e.row_pre(r, s, p, acc);
    }
};
#endif

// Epilogues that read DRAM operand vectors declare
// `void prefetch(int rb, int re) const`; others prefetch nothing.
template <class Epi, class = void>
struct EpiPf {
    __device__ static void run(const Epi&, int, int) {}
};
template <class Epi>
struct EpiPf<Epi, std::void_t<decltype(&Epi::prefetch)>> {
    __device__ static void run(const Epi& e, int rb, int re) { e.prefetch(rb, re); }
};

constexpr int kSeqRow = 256;  // staged rows up to this length stay bit-exact

// Phase B of a staged tile.  A lane owns G rows per pass (rows base +
// g*32 + lane).  Two modes per pass:
//  * every row of the pass has <= 32/G entries (stencils, regular meshes):
//    the lane gathers all entries of its G rows before summing, so 32
//    independent gathers per lane are in flight together with the
//    epilogue's operand loads, and across the warp the gathers hit the
//    j-th column of consecutive rows -- coalesced like ELL;
//  * some row is longer (power-law tiles): the warp first turns the whole
//    entry span of the pass into products in place, entry-parallel with 16
//    gathers per lane in flight per round (row-major order buys nothing on
//    random columns), then every lane sums its rows from the products.
// Every row of <= kSeqRow entries is summed sequentially from 0.0 in
// ascending k with individually rounded products -- the reference's bits
// (reference.cpp:82-88); longer rows are reduced by the warp.
// `starts(base, s)` fills s[q] (q = 0..G) with the slot offset where row
// base + q*32 + lane starts (the tile's entry end for rows >= re); a row's
// extent is then its start and the next row's start, taken from the
// neighbouring lane -- one lookup per row instead of two.
//
// Exact reductions (xred.cuh): the terms of a pass's rows go to `pend` and
// are added into the lane accumulator during the NEXT pass, right after its
// gathers are issued -- the adds overlap the gather latency instead of
// lengthening the pass.  The caller flushes `pend` at the end.
template <typename T, int G, class Epi, class Starts>
__device__ __forceinline__ void staged_rows(int rb, int re, T* sv, const int* sc,
                                            const T* __restrict__ x, const Epi& epi,
                                            RAcc* acc, Terms<Epi::NV>* pend, Starts&& starts)
{
    using EP = EpiPre<Epi>;
    // (NV == 1 only: two values' pending terms cost 2G registers that the
    // 255-register sweep does not have -- B4 spilled, BiCGSTAB 4% slower)
    constexpr bool kPipe = kExactRed && Epi::NV == 1;
    constexpr int CH = 32 / G;
    const int lane = threadIdx.x & 31;
    for (int base = rb; base < re; base += 32 * G) {
        int o[G], len[G];
        typename EP::type pre[G];
        bool any_long = false;
        int hi = 0;
        int st[G + 1];
        starts(base, st);
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const int r = base + q * 32 + lane;
            // next row's start: the neighbouring lane's (lane 31: lane 0 of
            // the next group, or of the group after the pass)
            int nx = __shfl_sync(0xffffffffu, st[q], (lane + 1) & 31);
            const int wrap = __shfl_sync(0xffffffffu, st[q + 1], 0);
            if (lane == 31) nx = wrap;
            int2 e = make_int2(st[q], nx - st[q]);
            if (r >= re) e = make_int2(0, 0);
            o[q] = e.x;
            len[q] = e.y;
            any_long |= e.y > CH;
            if (r < re) {
                pre[q] = EP::load(epi, r);
                hi = hi > e.x + e.y ? hi : e.x + e.y;
            }
        }
#ifdef LBK_NO_FASTPATH
        if (false) {
#else
        if (!__any_sync(0xffffffffu, any_long)) {
#endif
            T v[G][CH], g[G][CH];
#pragma unroll
            for (int q = 0; q < G; ++q) {
#pragma unroll
                for (int j = 0; j < CH; ++j) {
                    if (j < len[q]) {
                        v[q][j] = sv[o[q] + j];
                        g[q][j] = ldg_nc(x + sc[o[q] + j]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < G; ++q) {
                if constexpr (kPipe) {  // the previous pass's terms, under the gathers
                    terms_flush<SqMask<Epi>::value>(acc, pend[q]);
                    terms_zero(pend[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < G; ++q) {
                const int r = base + q * 32 + lane;
                if (r < re) {
                    T sum = T(0);
#pragma unroll
                    for (int j = 0; j < CH; ++j)
                        if (j < len[q]) sum = add_rn(sum, mul_rn(v[q][j], g[q][j]));
                    if constexpr (kPipe) EP::row(epi, r, sum, pre[q], &pend[q]);
                    else EP::row(epi, r, sum, pre[q], acc);
                }
            }
            continue;
        }
        if constexpr (kPipe) {
#pragma unroll
            for (int q = 0; q < G; ++q) {
                terms_flush<SqMask<Epi>::value>(acc, pend[q]);
                terms_zero(pend[q]);
            }
        }
        // products of the pass's whole entry span, in place
        const int lo = __shfl_sync(0xffffffffu, o[0], 0);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const int t = __shfl_xor_sync(0xffffffffu, hi, d);
            hi = hi > t ? hi : t;
        }
        for (int e0 = lo; e0 < hi; e0 += 16 * 32) {
            T gv[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int e = e0 + u * 32 + lane;
                // L2-only: the long-row path serves irregular matrices whose
                // gathers miss L1 anyway (1.4% hit rate at cfg3); skipping
                // the L1 allocation took cfg3 CSR from 1.60 to 1.52 ms
                if (e < hi) gv[u] = __ldcg(x + sc[e]);
            }
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int e = e0 + u * 32 + lane;
                if (e < hi) sv[e] = mul_rn(sv[e], gv[u]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < G; ++q) {
            const int r = base + q * 32 + lane;
            if (r < re && len[q] <= kSeqRow) {
                T sum = T(0);
                for (int k = 0; k < len[q]; ++k) sum = add_rn(sum, sv[o[q] + k]);
                EP::row(epi, r, sum, pre[q], acc);
            }
            unsigned m = __ballot_sync(0xffffffffu, r < re && len[q] > kSeqRow);
            while (m) {
                const int src = __ffs(m) - 1;
                m &= m - 1;
                const int ss = __shfl_sync(0xffffffffu, o[q], src);
                const int ll = __shfl_sync(0xffffffffu, len[q], src);
                T part = T(0);
                for (int k = lane; k < ll; k += 32) part = add_rn(part, sv[ss + k]);
                part = warp_sum(part);
                if (lane == src) EP::row(epi, r, part, pre[q], acc);
            }
        }
        __syncwarp();
    }
}

// Issues the bulk copies of entries [k0, k1) (aligned down/up to 4 entries,
// clamped to the last full 16-B chunk) into a slot; the ragged tail past
// nnz4 is copied by the warp with ordinary loads.  Returns the aligned base.
template <typename T, int NIDX>
__device__ __forceinline__ int stage_tile(int k0, int k1, long long nnz4, T* sv, int* si0,
                                          int* si1, const T* __restrict__ vals,
                                          const int* __restrict__ idx0,
                                          const int* __restrict__ idx1, uint64_t* bar,
                                          uint64_t pol)
{
    const int lane = threadIdx.x & 31;
    const int ka = k0 & ~3;
    const long long kz = (static_cast<long long>(k1) + 3) & ~3LL;
    const long long ke = kz < nnz4 ? kz : nnz4;
    if (lane == 0) {
        if (ke > ka) {
            const uint32_t n = static_cast<uint32_t>(ke - ka);
            mbar_arrive_expect_tx(bar, n * uint32_t(sizeof(T) + 4 * NIDX));
            tma_load_1d(sv, vals + ka, n * sizeof(T), bar, pol);
            tma_load_1d(si0, idx0 + ka, n * 4u, bar, pol);
            if (NIDX == 2) tma_load_1d(si1, idx1 + ka, n * 4u, bar, pol);
        } else {
            mbar_arrive(bar);
        }
    }
    if (k1 > nnz4) {
        const int kt = k0 > nnz4 ? k0 : static_cast<int>(nnz4);
        for (int k = kt + lane; k < k1; k += 32) {
            sv[k - ka] = vals[k];
            si0[k - ka] = idx0[k];
            if (NIDX == 2) si1[k - ka] = idx1[k];
        }
    }
    return ka;
}

// The per-warp tile loop shared by CSR and COO.  Tiles T_j = t0 + j*nw of
// this warp rotate through NS shared-memory slots: at iteration j the warp
// stages T_{j+NS-1} (bulk copies into the slot T_{j-1} just freed) and then
// sweeps T_j, so NS-1 tiles are always in flight.  Tile metadata needs two
// dependent loads (plan entry, then row_ptr / row_idx at it); they are
// software-pipelined two and one tiles ahead of the staging:
//   iteration j:  load m1(T_{j+NS+1});  load m2(T_{j+NS}) from m1(T_{j+NS});
//                 stage T_{j+NS-1} (bounds complete);  sweep T_j.
// meta1(t) / meta2(t, m1) return the lane-0/1 values (lanes >= 2: 0);
// mk(m1, m2) -> int4 (row begin, row end, entry begin, entry end).
// pf(bounds) issues per-lane loads for the first row pass of a tile (CSR:
// its row_ptr entries) when the tile is staged; staged(...) gets them back.
template <typename T, int NIDX, class M1, class M2, class Mk, class Pf, class Split, class Staged,
          class Wide, class L2pf>
__device__ __forceinline__ void warp_tile_loop(int ntiles, long long nnz, const T* vals,
                                               const int* idx0, const int* idx1,
                                               unsigned char* wbase, uint64_t* bar, M1&& meta1,
                                               M2&& meta2, Mk&& mk, Pf&& pf, Split&& split,
                                               Staged&& staged, Wide&& wide, L2pf&& l2pf)
{
    using Cfg = StreamCfg<T, NIDX>;
    constexpr int CAP = Cfg::kCap, NW = Cfg::kWarps, NS = Cfg::kSlots;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto slot_v = [&](int s) { return reinterpret_cast<T*>(wbase + s * Cfg::slot_bytes); };
    auto slot_i0 = [&](int s) {
        return reinterpret_cast<int*>(wbase + s * Cfg::slot_bytes + CAP * sizeof(T));
    };
    if (lane == 0) {
        for (int q = 0; q < NS; ++q) mbar_init(&bar[q], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const long long nnz4 = nnz & ~3LL;
    const uint64_t pol = policy_evict_first();
    const int nw = gridDim.x * NW;
    auto staged_ok = [&](int4 bd) { return (bd.w - (bd.z & ~3) + 3) <= CAP; };

    const int t0 = blockIdx.x * NW + warp;
    if (t0 >= ntiles) return;
    using PfT = decltype(pf(make_int4(0, 0, 0, 0)));
    struct Q {
        int4 bd;    // staged part: rows [x, y), entries [z, w)
        int4 rest;  // rows [x, y), entries [z, w) straight from global (x == y: none)
        int ka;
        bool st;
        PfT pf;
    };
    // stage tile t (if it exists) into slot s.  Only one row of a tile can
    // overflow a slot -- the last one for a CSR plan, the first one for a
    // COO plan (every other row lies inside the tile's T-entry window) -- so
    // an oversize tile is split(bd) -> (staged part, rest): the rest (the
    // giant row) goes straight from global memory.
    auto issue = [&](int t, int4 bd, int s) {
        Q q;
        q.bd = bd;
        q.rest = make_int4(0, 0, 0, 0);
        q.st = false;
        q.ka = 0;
        if (t < ntiles) {
            if (staged_ok(bd)) {
                q.st = true;
            } else {
                const int4x2 sp = split(bd);
                q.bd = sp.a;
                q.rest = sp.b;
                q.st = q.bd.x < q.bd.y && staged_ok(q.bd);
                if (!q.st) q.rest = bd;  // (cannot happen for CSR/COO plans)
            }
        }
        if (q.st) {
            fence_proxy_async_smem();
            int* i0 = slot_i0(s);
            q.ka = stage_tile<T, NIDX>(q.bd.z, q.bd.w, nnz4, slot_v(s), i0, i0 + CAP, vals, idx0,
                                       idx1, &bar[s], pol);
        }
        q.pf = pf(q.st ? q.bd : make_int4(0, 0, 0, 0));
        if (q.st) l2pf(q.bd);
        return q;
    };
    // prologue: T_0 .. T_{NS-2} staged, metadata of T_{NS-1} complete and
    // m1 of T_NS loaded
    Q qs[NS - 1];
#pragma unroll
    for (int i = 0; i < NS - 1; ++i) {
        const int t = t0 + i * nw;
        const int m1 = meta1(t);
        qs[i] = issue(t, mk(m1, meta2(t, m1)), i);
    }
    int m1a = meta1(t0 + (NS - 1) * nw);
    int m2a = meta2(t0 + (NS - 1) * nw, m1a);
    int m1b = meta1(t0 + NS * nw);
    int it = 0;
    for (int t = t0; t < ntiles; t += nw, ++it) {
        const int slot = it % NS;
        const int tn = t + (NS - 1) * nw;          // tile to stage now
        const int m1c = meta1(tn + 2 * nw);        // consumed two iterations later
        const int m2b = meta2(tn + nw, m1b);       // consumed next iteration
        const Q qn = issue(tn, mk(m1a, m2a), (it + NS - 1) % NS);
        const Q qc = qs[0];
#pragma unroll
        for (int i = 0; i + 1 < NS - 1; ++i) qs[i] = qs[i + 1];
        qs[NS - 2] = qn;
        if (!qc.st && lane == 0) mbar_arrive(&bar[slot]);  // keep the phase in step
        mbar_wait(&bar[slot], (it / NS) & 1);
        __syncwarp();
        if (qc.st) {
            int* i0 = slot_i0(slot);
            staged(qc.bd, qc.ka, slot_v(slot), i0, i0 + CAP, qc.pf);
        }
        if (qc.rest.x < qc.rest.y) wide(qc.rest);
        __syncwarp();
        m1a = m1b;
        m2a = m2b;
        m1b = m1c;
    }
    // tiles staged past the end never arrive: nothing to drain (the
    // issue() calls beyond ntiles staged nothing)
}

template <typename T, class Epi, int G>
__global__ void __launch_bounds__((StreamCfg<T, 1>::kThreads), LBK_CSR_MINB)
    csr_stream_kernel(CsrView<T> A, const T* __restrict__ x, Epi epi, RedWs ws)
{
    pdl_enter();
    using Cfg = StreamCfg<T, 1>;
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[Cfg::kWarps][Cfg::kSlots];
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    if constexpr (Epi::NV > 0) red_begin<NV>();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
    Terms<Epi::NV> pend[G];  // exact mode: the last pass's terms (staged_rows)
#pragma unroll
    for (int q = 0; q < G; ++q) terms_zero(pend[q]);

    struct RowPf {
        int v[G + 1];
    };
    warp_tile_loop<T, 1>(
        A.ntiles, A.nnz, A.vals, A.cols, nullptr,
        smem + size_t(warp) * Cfg::kSlots * Cfg::slot_bytes, bars[warp],
        [&](int t) { return (t < A.ntiles && lane < 2) ? __ldg(A.tile_rows + t + lane) : 0; },
        [&](int t, int b) { return (t < A.ntiles && lane < 2) ? __ldg(A.row_ptr + b) : 0; },
        [&](int b, int k) {
            return make_int4(__shfl_sync(0xffffffffu, b, 0), __shfl_sync(0xffffffffu, b, 1),
                             __shfl_sync(0xffffffffu, k, 0), __shfl_sync(0xffffffffu, k, 1));
        },
        [&](int4 bd) {
            // row_ptr of the tile's first pass: lane holds rows rb + q*32 + lane
            RowPf p;
#pragma unroll
            for (int q = 0; q <= G; ++q) {
                const int r = bd.x + q * 32 + lane;
                p.v[q] = __ldg(A.row_ptr + (r < bd.y ? r : bd.y));
            }
            return p;
        },
        [&](int4 bd) {
            const int ks = __ldg(A.row_ptr + bd.y - 1);  // the giant row is the last one
            return int4x2{make_int4(bd.x, bd.y - 1, bd.z, ks), make_int4(bd.y - 1, bd.y, ks, bd.w)};
        },
        [&](int4 bd, int ka, T* sv, const int* sc, const int*, const RowPf& p) {
            staged_rows<T, G>(bd.x, bd.y, sv, sc, x, epi, acc, pend, [&](int base, int* st) {
                if (base == bd.x) {  // prefetched when the tile was staged
#pragma unroll
                    for (int q = 0; q <= G; ++q) st[q] = p.v[q] - ka;
                } else {
#pragma unroll
                    for (int q = 0; q <= G; ++q) {
                        const int r = base + q * 32 + lane;
                        st[q] = __ldg(A.row_ptr + (r < bd.y ? r : bd.y)) - ka;
                    }
                }
            });
        },
        [&](int4 bd) {
            for (int r = bd.x; r < bd.y; ++r) {
                const int ks = __ldg(A.row_ptr + r), ke = __ldg(A.row_ptr + r + 1);
                const T s = warp_row_global<T>(ks, ke, A.cols, A.vals, x);
                if (lane == 0) epi.row(r, s, acc);
            }
        },
        [&](int4 bd) { EpiPf<Epi>::run(epi, bd.x, bd.y); });

    if constexpr (kExactRed && Epi::NV == 1) {
#pragma unroll
        for (int q = 0; q < G; ++q) terms_flush<SqMask<Epi>::value>(acc, pend[q]);
    }
    if constexpr (Epi::NV > 0) {
        __syncthreads();
        grid_reduce<NV>(acc, ws, tid, Cfg::kThreads, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

// SELL-P with 32-row slices on the same warp pipeline: a slice is one
// contiguous column-major block (entry (r, j) at (slice_sets[s] + j)*32 +
// r%32), so a tile of whole slices is one bulk copy per array.  The sweep
// is lane-per-row: column j of a slice is 32 consecutive shared-memory
// words (conflict-free) and its 32 gathers coalesce like ELL; up to 32
// columns' gathers per lane are in flight before the (sequential,
// reference-order) sum.  Tiles: runs of k whole slices (tile_slices[t] =
// t*k, see sellp_slices_per_tile).
template <typename T, class Epi>
__global__ void __launch_bounds__((StreamCfg<T, 1>::kThreads), 2)
    sellp_stream_kernel(SellpView<T> A, const int* __restrict__ tile_slices, int ntiles,
                        long long stored, const T* __restrict__ x, Epi epi, RedWs ws)
{
    pdl_enter();
    using Cfg = StreamCfg<T, 1>;
    using EP = EpiPre<Epi>;
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[Cfg::kWarps][Cfg::kSlots];
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    if constexpr (Epi::NV > 0) red_begin<NV>();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);

    // one slice (its slice set a, length len), its column block read
    // through colv(a, j, v, c)
    auto slice = [&](int s, int a, int len, auto&& colv) {
        const int r = s * 32 + lane;
        typename EP::type pre;
        if (r < A.nrows) pre = EP::load(epi, r);
        T sum = T(0);
        for (int j0 = 0; j0 < len; j0 += 32) {
            int c[32];
            T v[32], g[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                c[j] = -1;
                if (j0 + j < len) colv(a, j0 + j, v[j], c[j]);
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) g[j] = c[j] >= 0 ? ldg_nc(x + c[j]) : T(0);
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (c[j] >= 0) sum = add_rn(sum, mul_rn(v[j], g[j]));
        }
        if (r < A.nrows) EP::row(epi, r, sum, pre, acc);
    };

    struct SetPf {
        int v;  // slice_sets[first slice of the tile + lane] (<= 32 slices per tile)
    };
    warp_tile_loop<T, 1>(
        ntiles, stored, A.vals, A.cols, nullptr,
        smem + size_t(warp) * Cfg::kSlots * Cfg::slot_bytes, bars[warp],
        [&](int t) { return (t < ntiles && lane < 2) ? __ldg(tile_slices + t + lane) : 0; },
        [&](int t, int b) { return (t < ntiles && lane < 2) ? __ldg(A.slice_sets + b) * 32 : 0; },
        [&](int b, int k) {
            return make_int4(__shfl_sync(0xffffffffu, b, 0), __shfl_sync(0xffffffffu, b, 1),
                             __shfl_sync(0xffffffffu, k, 0), __shfl_sync(0xffffffffu, k, 1));
        },
        [&](int4 bd) {
            const int s = bd.x + lane;
            return SetPf{__ldg(A.slice_sets + (s < bd.y ? s : bd.y))};
        },
        [&](int4 bd) {
            const int ks = __ldg(A.slice_sets + bd.y - 1) * 32;  // the giant slice is the last
            return int4x2{make_int4(bd.x, bd.y - 1, bd.z, ks), make_int4(bd.y - 1, bd.y, ks, bd.w)};
        },
        [&](int4 bd, int ka, T* sv, const int* sc, const int*, const SetPf& p) {
            for (int s = bd.x; s < bd.y; ++s) {
                const int i = s - bd.x;
                int a, e;
                if (i < 31) {
                    a = __shfl_sync(0xffffffffu, p.v, i);
                    e = __shfl_sync(0xffffffffu, p.v, i + 1);
                } else {
                    a = __ldg(A.slice_sets + s);
                    e = __ldg(A.slice_sets + s + 1);
                }
                slice(s, a, e - a, [&](int a, int j, T& v, int& c) {
                    const int o = (a + j) * 32 + lane - ka;
                    v = sv[o];
                    c = sc[o];
                });
            }
        },
        [&](int4 bd) {
            for (int s = bd.x; s < bd.y; ++s) {
                const int a = __ldg(A.slice_sets + s);
                slice(s, a, __ldg(A.slice_sets + s + 1) - a, [&](int a, int j, T& v, int& c) {
                    const long long o = (static_cast<long long>(a) + j) * 32 + lane;
                    v = __ldcs(A.vals + o);
                    c = __ldcs(A.cols + o);
                });
            }
        },
        [&](int4) {});

    if constexpr (Epi::NV > 0) {
        __syncthreads();
        grid_reduce<NV>(acc, ws, tid, Cfg::kThreads, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

__global__ void sellp_plan_kernel(int nslices, int ntiles, int k, int* __restrict__ tile_slices);

// COO: warp tiles are row-aligned entry ranges [tile_starts[t],
// tile_starts[t+1]) of the (row, col)-sorted entries; the tile owns rows
// [r0, r1) including empty ones (reference.cpp:67 zero-fills y first).
// row_idx is staged with vals/col_idx; a lane finds its row's extent by
// binary search over the staged row indices.
template <typename T, class Epi, int G>
__global__ void __launch_bounds__((StreamCfg<T, 2>::kThreads), 2)
    coo_stream_kernel(CooView<T> A, const T* __restrict__ x, Epi epi, RedWs ws)
{
    pdl_enter();
    using Cfg = StreamCfg<T, 2>;
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bars[Cfg::kWarps][Cfg::kSlots];
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    if constexpr (Epi::NV > 0) red_begin<NV>();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
    Terms<Epi::NV> pend[G];  // exact mode: the last pass's terms (staged_rows)
#pragma unroll
    for (int q = 0; q < G; ++q) terms_zero(pend[q]);

    struct NoPf {};
    warp_tile_loop<T, 2>(
        A.ntiles, A.nnz, A.vals, A.cols, A.rows,
        smem + size_t(warp) * Cfg::kSlots * Cfg::slot_bytes, bars[warp],
        [&](int t) { return (t < A.ntiles && lane < 2) ? __ldg(A.tile_starts + t + lane) : 0; },
        [&](int t, int k) {
            if (t >= A.ntiles || lane >= 2) return 0;
            if (lane == 0) return t == 0 ? 0 : __ldg(A.rows + k);
            return t + 1 == A.ntiles ? A.nrows : __ldg(A.rows + k);
        },
        [&](int k, int r) {
            return make_int4(__shfl_sync(0xffffffffu, r, 0), __shfl_sync(0xffffffffu, r, 1),
                             __shfl_sync(0xffffffffu, k, 0), __shfl_sync(0xffffffffu, k, 1));
        },
        [&](int4) { return NoPf{}; },
        [&](int4 bd) {
            // the giant row is the first one (it holds entry t*T); the rest
            // of the tile starts at its end
            int ke = 0;
            if (lane == 0) ke = lower_bound_i(A.rows, bd.z, bd.w, bd.x + 1);
            ke = __shfl_sync(0xffffffffu, ke, 0);
            return int4x2{make_int4(bd.x + 1, bd.y, ke, bd.w), make_int4(bd.x, bd.x + 1, bd.z, ke)};
        },
        [&](int4 bd, int ka, T* sv, const int* sc, const int* sr, const NoPf&) {
            const int lo = bd.z - ka, hi = bd.w - ka;
            staged_rows<T, G>(bd.x, bd.y, sv, sc, x, epi, acc, pend, [&](int base, int* st) {
#pragma unroll
                for (int q = 0; q < G; ++q) {
                    const int r = base + q * 32 + lane;
                    st[q] = r < bd.y ? lower_bound_i(sr, lo, hi, r) : hi;
                }
                // start of the row after the pass (used by lane 31 of the last
                // group): the tile's end when the pass reaches it
                const int rn = base + G * 32;
                st[G] = rn < bd.y ? lower_bound_i(sr, lo, hi, rn) : hi;
            });
        },
        [&](int4 bd) {
            for (int r = bd.x; r < bd.y; ++r) {
                int ks = 0, ke = 0;
                if (lane == 0) {
                    ks = lower_bound_i(A.rows, bd.z, bd.w, r);
                    ke = lower_bound_i(A.rows, ks, bd.w, r + 1);
                }
                ks = __shfl_sync(0xffffffffu, ks, 0);
                ke = __shfl_sync(0xffffffffu, ke, 0);
                const T s = warp_row_global<T>(ks, ke, A.cols, A.vals, x);
                if (lane == 0) epi.row(r, s, acc);
            }
        },
        [&](int4 bd) { EpiPf<Epi>::run(epi, bd.x, bd.y); });

    if constexpr (kExactRed && Epi::NV == 1) {
#pragma unroll
        for (int q = 0; q < G; ++q) terms_flush<SqMask<Epi>::value>(acc, pend[q]);
    }
    if constexpr (Epi::NV > 0) {
        __syncthreads();
        grid_reduce<NV>(acc, ws, tid, Cfg::kThreads, red_sh,
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
#ifndef LBK_QUAD_COLS
#define LBK_QUAD_COLS 6
#endif
template <typename T, class Epi, bool IS_ELL>
__global__ void __launch_bounds__(256)
    sliced_quad_kernel(int nrows, int S, const int* __restrict__ slice_sets, int ell_width,
                       const int* __restrict__ cols, const T* __restrict__ vals,
                       const T* __restrict__ x, Epi epi, RedWs ws)
{
    pdl_enter();
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    if constexpr (Epi::NV > 0) red_begin<NV>();
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
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
        // U columns per step: 4U gathers per thread in flight
        constexpr int U = LBK_QUAD_COLS;
        for (; j + U - 1 < len; j += U) {
            int cc[U][4];
            Quad<T> vv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long o = base + (j + u) * pitch;
                const int4 c = ld_stream_i4(cols + o);
                cc[u][0] = c.x;
                cc[u][1] = c.y;
                cc[u][2] = c.z;
                cc[u][3] = c.w;
                vv[u].load(vals + o);
            }
            T g[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int i = 0; i < 4; ++i) g[u][i] = cc[u][i] >= 0 ? ldg_nc(x + cc[u][i]) : T(0);
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (cc[u][i] >= 0) sum[i] = add_rn(sum[i], mul_rn(vv[u].v[i], g[u][i]));
        }
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
        grid_reduce<NV>(acc, ws, threadIdx.x, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

// Lane-per-row variant: consecutive lanes own consecutive rows, so the
// column-j loads of a warp are one contiguous 128 B (indices) / 256 B
// (values) run and the x gathers of a stencil hit 2 lines -- about half the
// L1 wavefronts of the 4-rows-per-thread kernel, whose gathers stride 32 B
// across lanes.  8 columns' loads and then 8 gathers per thread in flight.
template <typename T, class Epi, bool IS_ELL>
__global__ void __launch_bounds__(256)
    sliced_lane_kernel(int nrows, int S, const int* __restrict__ slice_sets, int ell_width,
                       const int* __restrict__ cols, const T* __restrict__ vals,
                       const T* __restrict__ x, Epi epi, RedWs ws)
{
    pdl_enter();
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    constexpr int U = 8;
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    if constexpr (Epi::NV > 0) red_begin<NV>();
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
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
        const long long pitch = S;
        T sum = T(0);
        for (int j0 = 0; j0 < len; j0 += U) {
            int c[U];
            T v[U], g[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                c[u] = -1;
                if (j0 + u < len) {
                    const long long o = base + (j0 + u) * pitch;
                    c[u] = __ldcs(cols + o);
                    v[u] = __ldcs(vals + o);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) g[u] = c[u] >= 0 ? ldg_nc(x + c[u]) : T(0);
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (c[u] >= 0) sum = add_rn(sum, mul_rn(v[u], g[u]));
        }
        epi.row(r, sum, acc);
    }
    if constexpr (Epi::NV > 0) {
        grid_reduce<NV>(acc, ws, threadIdx.x, blockDim.x, red_sh,
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
    pdl_enter();
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    __shared__ double red_sh[32 * NV];
    if (epi.skip()) return;
    if constexpr (Epi::NV > 0) red_begin<NV>();
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
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
        grid_reduce<NV>(acc, ws, threadIdx.x, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

}  // namespace lbk
