// lbk_internal.cuh -- shared host/device plumbing of the B200 sparse backend.
//
// Host side: the context (device + stream + arena accounting + scratch), the
// status/exception bridge behind the C ABI, and launch helpers.
// Device side: mbarrier / 1-D TMA bulk-copy wrappers (sm_100a PTX), cache-
// hinted loads, warp/block reductions and the deterministic two-stage
// grid reduction used by every dot product.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>

#include "lbk.h"
#include "xred.cuh"

namespace lbk {

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
    lbk_status status;
    int iteration = -1;
    Error(lbk_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(lbk_status s, const std::string& m) { throw Error(s, m); }

#define LBK_CUDA(call)                                                          \
    do {                                                                        \
        cudaError_t e_ = (call);                                                \
        if (e_ != cudaSuccess)                                                  \
            ::lbk::fail(LBK_CUDA_ERROR, std::string(#call ": ") +               \
                                            cudaGetErrorString(e_));            \
    } while (0)

#define LBK_LAUNCH_CHECK() LBK_CUDA(cudaGetLastError())

// ----------------------------------------------------------------- context
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
};

}  // namespace lbk

struct lbk_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    size_t smem_optin = 0;
    std::string err;
    size_t arena_capacity = ~size_t{0};
    size_t arena_used = 0;
    // Scratch regions (device).  `scratch` holds per-call temporaries such
    // as on-the-fly SpMV plans; `red` holds reduction partials + counters
    // (counters are left zeroed by every reduction, see GridReduce).
    lbk::DevBuf scratch;
    lbk::DevBuf red;
    double* host_pinned = nullptr;  // 64 doubles for synchronous readbacks
    // L2 access-policy window on the gathered vector x (per launch,
    // cudaLaunchAttributeAccessPolicyWindow): persisting hits for x, streaming
    // misses.  0 off, 1 on; persist_max = the device's window / carve-out.
    int l2_persist = 0;
    size_t persist_max = 0;
    // programmatic dependent launch for the SpMV / solver kernel chain
    // (LBK_PDL=1; off by default since the exact reductions, see ctx.cu): a
    // kernel's CTAs are scheduled while its predecessor drains and wait in
    // griddepcontrol.wait for its results
    int pdl = 0;
};

namespace lbk {

// Ensure the context's scratch buffer holds `bytes`; returns device ptr.
void* scratch(lbk_ctx ctx, size_t bytes);

// Reduction workspace: `slots` partial doubles per block plus one counter.
struct RedWs {
    double* partials;     // [max_blocks * slots]
    unsigned* counter;    // zero between uses
    double* out;          // [64] device results (dist solver: see DistEnv)
    int defer = 0;        // 1: the finisher only stores the grid totals to
                          // `out` (a cross-rank allreduce runs before the
                          // epilogue's finish(), see dist.cu)
    long long* xacc = nullptr;  // exact mode: the grid's limb accumulator
                                // (kXSlot int64, zero between uses)
    long long* xout = nullptr;  // exact mode, defer: the slot the blocks add
                                // their limbs into (consumer rounds + zeroes)
};
// exact-mode deferred slots in the reduction workspace (DistEnv)
constexpr int kXOutSlots = 8;
RedWs red_ws(lbk_ctx ctx, int max_blocks, int slots);

constexpr int kRedMaxBlocks = 4096;

// --------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(count));
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes)
{
    asm volatile(
        "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
            smem_u32(bar)),
        "r"(bytes)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra LAB_WAIT;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// L2 eviction policies for the bulk streams (matrix values / indices are
// read exactly once per SpMV: evict-first keeps the gathered vector in L2).
__device__ __forceinline__ uint64_t policy_evict_first()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last()
{
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// 1-D TMA: global -> shared bulk copy completing on an mbarrier
// (cp.async.bulk; src/dst 16-B aligned, size a multiple of 16).
__device__ __forceinline__ void tma_load_1d(void* dst_smem, const void* src_gmem,
                                            uint32_t bytes, uint64_t* bar,
                                            uint64_t policy)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::"
        "cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// Orders this thread's generic-proxy shared-memory accesses before later
// async-proxy (TMA) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// L2 prefetch of one vector's rows [rb, re) by the warp (one 128-B line per
// lane per step): the epilogue operand streams of a tile are pulled into L2
// when the tile's matrix data is staged, so the sweep's operand loads hit L2
// instead of paying a DRAM round trip next to the gathers.
__device__ __forceinline__ void l2_prefetch_rows(const double* v, int rb, int re)
{
    if (!v || re <= rb) return;
    const char* b = reinterpret_cast<const char*>(v + rb);
    const char* e = reinterpret_cast<const char*>(v + re);
    const char* line = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(b) & ~uintptr_t(127));
    for (const char* p = line + (threadIdx.x & 31) * 128; p < e; p += 32 * 128)
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// Gathers of x.  -DLBK_GATHER_NOALLOC / -DLBK_GATHER_CG select the
// L1::no_allocate or L2-only (.cg) forms for A/B measurements.
template <typename T>
__device__ __forceinline__ T ldg_nc(const T* p)
{
#if defined(LBK_GATHER_NOALLOC)
    if constexpr (sizeof(T) == 8) {
        double v;
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
        return static_cast<T>(v);
    } else {
        float v;
        asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
        return static_cast<T>(v);
    }
#elif defined(LBK_GATHER_CG)
    return __ldcg(p);
#else
    return __ldg(p);
#endif
}

// Exact-rounding arithmetic helpers: products and sums are rounded
// separately (no FMA contraction), which is what the FMA-free reference
// build computes.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = add_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ------------------------------------------------ reduction accumulators
// Every dot/norm of the path accumulates through racc_add.  Default: the
// exact, partition-independent reduction (xred.cuh).  -DLBK_RED_TREE builds
// the previous deterministic tree (per-lane double sums, block tree, block-
// ordered grid sum) for A/B measurements; its results depend on the grid.
#ifdef LBK_RED_TREE
constexpr bool kExactRed = false;
using RAcc = double;
__device__ __forceinline__ void racc_zero(RAcc& a) { a = 0.0; }
__device__ __forceinline__ void racc_add(RAcc* acc, int k, double t)
{
    acc[k] = __dadd_rn(acc[k], t);
}
#else
constexpr bool kExactRed = true;
using RAcc = XLane;
__device__ __forceinline__ void racc_zero(RAcc& a) { xl_zero(a); }
__device__ __forceinline__ void racc_add(RAcc* acc, int k, double t)
{
    xl_add(acc[k], t, xwarp_limbs() + k * kXV);
}
#endif

// One element's (row's) terms, buffered so that their exact adds can run
// off the critical path: after the next element's / pass's loads are issued
// (vec_kernel, staged_rows).  Every epilogue / vec op adds at most one term
// per value and element.
template <int NV>
struct Terms {
    double v[NV > 0 ? NV : 1];
};
template <int NV>
__device__ __forceinline__ void racc_add(Terms<NV>* t, int k, double x)
{
    t->v[k] = x;
}
template <int NV>
__device__ __forceinline__ void terms_zero(Terms<NV>& t)
{
#pragma unroll
    for (int k = 0; k < (NV > 0 ? NV : 1); ++k) t.v[k] = 0.0;
}
// SQ: bit k set when value k is a sum of squares (epilogue / op `kSq`)
template <unsigned SQ = 0, int NV>
__device__ __forceinline__ void terms_flush(RAcc* acc, const Terms<NV>& t)
{
#pragma unroll
    for (int k = 0; k < NV; ++k) {
        if constexpr (kExactRed) {
            if ((SQ >> k) & 1u) xl_add<true>(acc[k], t.v[k], xwarp_limbs() + k * kXV);
            else xl_add<false>(acc[k], t.v[k], xwarp_limbs() + k * kXV);
        } else {
            racc_add(acc, k, t.v[k]);
        }
    }
}
// Epilogues / vector ops whose reduced values are sums of squares declare
// `static constexpr unsigned kSq` (bit k for value k); default none.
template <class E, class = void>
struct SqMask {
    static constexpr unsigned value = 0;
};
template <class E>
struct SqMask<E, std::void_t<decltype(E::kSq)>> {
    static constexpr unsigned value = E::kSq;
};

// Kernel prologue of every reducing kernel (all threads, after any
// block-uniform early exit): zeroes the block accumulator.
template <int NV>
__device__ __forceinline__ void red_begin()
{
    if constexpr (kExactRed) xred_begin<NV>();
}

// Block-wide sum of NV doubles over the first `nthreads` threads (all of
// which must call).  Result valid in thread 0.  Fixed order => deterministic.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], int tid, int nthreads,
                                          double* sh /* >= 32*NV */)
{
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
    const int warp = tid >> 5, lane = tid & 31, nw = (nthreads + 31) >> 5;
    if (lane == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) sh[warp * NV + i] = v[i];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double t = lane < nw ? sh[lane * NV + i] : 0.0;
            v[i] = warp_sum(t);
        }
    }
}

// Second stage of a deterministic grid reduction: called by every block
// with its block total in thread 0.  The last block to arrive sums all
// partials in block order and calls fin(totals) in thread 0.  Returns true
// in the block that ran the finisher.
template <int NV, class Fin>
__device__ __forceinline__ bool grid_reduce_finish(const double (&v)[NV], RedWs ws,
                                                   int tid, int nthreads, double* sh,
                                                   Fin&& fin)
{
    __shared__ unsigned s_last;
    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) ws.partials[blockIdx.x * NV + i] = v[i];
        __threadfence();
        unsigned prev = atomicAdd(ws.counter, 1u);
        s_last = (prev == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return false;
    __threadfence();
    double acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) acc[i] = 0.0;
    for (int b = tid; b < (int)gridDim.x; b += nthreads) {
#pragma unroll
        for (int i = 0; i < NV; ++i)
            acc[i] = add_rn(acc[i], __ldcg(&ws.partials[b * NV + i]));
    }
    __syncthreads();
    block_sum<NV>(acc, tid, nthreads, sh);
    if (tid == 0) {
        if (ws.defer) {
#pragma unroll
            for (int i = 0; i < NV; ++i) ws.out[i] = acc[i];
        } else {
            fin(acc);
        }
        *ws.counter = 0;
    }
    return true;
}

// Kernel epilogue of every reducing kernel (all threads of the block):
// reduces the lanes' accumulators over the grid; the last block calls
// fin(totals) in thread 0 -- or, with ws.defer, leaves the grid totals for
// the distributed consumer (tree: ws.out doubles; exact: ws.xout limbs).
template <int NV, class Fin>
__device__ __forceinline__ bool grid_reduce(RAcc (&acc)[NV], RedWs ws, int tid, int nthreads,
                                            double* sh, Fin&& fin)
{
    if constexpr (!kExactRed) {
        block_sum<NV>(acc, tid, nthreads, sh);
        return grid_reduce_finish<NV>(acc, ws, tid, nthreads, sh, fin);
    } else {
#pragma unroll
        for (int v = 0; v < NV; ++v) xl_warp_flush(acc[v], xwarp_limbs() + v * kXV);
        __syncthreads();
        long long* G = ws.defer ? ws.xout : ws.xacc;
        const int nw = (nthreads + 31) >> 5;
        for (int i = tid; i < NV * kXV; i += nthreads) {
            long long v = 0;
            for (int w = 0; w < nw; ++w) v += g_xsh[w * kXSlot + i];
            if (v) atomicAdd(reinterpret_cast<unsigned long long*>(G + i),
                             static_cast<unsigned long long>(v));
        }
        if (ws.defer) return false;
        __shared__ unsigned s_xlast;
        __threadfence();
        __syncthreads();
        if (tid == 0) s_xlast = (atomicAdd(ws.counter, 1u) == gridDim.x - 1);
        __syncthreads();
        if (!s_xlast) return false;
        __threadfence();
        for (int i = tid; i < NV * kXV; i += nthreads) {
            g_xsh[i] = __ldcg(G + i);
            G[i] = 0;
        }
        __syncthreads();
        if (tid < 32) {  // warp 0 rounds (xred_round_warp), thread 0 finishes
            double tot[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) tot[v] = xred_round_warp(g_xsh + v * kXV);
            if (tid == 0) {
                fin(tot);
                *ws.counter = 0;
            }
        }
        return true;
    }
}

// First statement of every kernel that may be launched with programmatic
// stream serialization: wait for the predecessor grid's completion (and
// memory flush), then let the successor's CTAs be scheduled.  A no-op for
// ordinary launches.
__device__ __forceinline__ void pdl_enter()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
void launch_pdl(lbk_ctx ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                Args&&... args)
{
    if (!ctx->pdl) {
        kernel<<<grid, block, smem, ctx->stream>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...) != cudaSuccess)
        throw std::runtime_error("kernel launch failed");
}

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace lbk
