// ctx.cu -- context, arena accounting, copies (the Executor seam:
// reference include/larch/core/executor.hpp:130-170, device_array.cpp:144-263).
#include <cstdlib>
#include <cstring>

#include "api_guard.h"

namespace lbk {

namespace {
thread_local std::string g_err;
}

void set_error(lbk_ctx ctx, const std::string& msg)
{
    if (ctx)
        ctx->err = msg;
    g_err = msg;
}

void* scratch(lbk_ctx ctx, size_t bytes)
{
    if (ctx->scratch.bytes < bytes) {
        if (ctx->scratch.ptr) {
            LBK_CUDA(cudaStreamSynchronize(ctx->stream));
            LBK_CUDA(cudaFree(ctx->scratch.ptr));
            ctx->scratch = {};
        }
        size_t want = bytes < (1u << 20) ? (1u << 20) : bytes + bytes / 4;
        LBK_CUDA(cudaMalloc(&ctx->scratch.ptr, want));
        ctx->scratch.bytes = want;
    }
    return ctx->scratch.ptr;
}

RedWs red_ws(lbk_ctx ctx, int max_blocks, int slots)
{
    // Layout: [counter (256 B)] [out: 64 doubles] [xacc: kXSlot int64]
    //         [xout: kXOutSlots x kXSlot int64] [partials]
    // counter, xacc and xout are zero between uses (every consumer re-zeroes).
    const size_t xbytes = size_t(1 + kXOutSlots) * kXSlot * sizeof(long long);
    const size_t head = 256 + 64 * sizeof(double) + xbytes;
    const size_t need_bytes = head + size_t(max_blocks) * slots * sizeof(double);
    if (ctx->red.bytes < need_bytes) {
        if (ctx->red.ptr) {
            LBK_CUDA(cudaStreamSynchronize(ctx->stream));
            LBK_CUDA(cudaFree(ctx->red.ptr));
        }
        size_t want = need_bytes < (1u << 20) ? (1u << 20) : need_bytes;
        LBK_CUDA(cudaMalloc(&ctx->red.ptr, want));
        LBK_CUDA(cudaMemsetAsync(ctx->red.ptr, 0, head, ctx->stream));
        ctx->red.bytes = want;
    }
    auto* base = static_cast<char*>(ctx->red.ptr);
    RedWs ws;
    ws.counter = reinterpret_cast<unsigned*>(base);
    ws.out = reinterpret_cast<double*>(base + 256);
    ws.xacc = reinterpret_cast<long long*>(base + 256 + 64 * sizeof(double));
    ws.xout = ws.xacc + kXSlot;
    ws.partials = reinterpret_cast<double*>(base + head);
    return ws;
}

}  // namespace lbk

using namespace lbk;

extern "C" {

static lbk_status ctx_create_impl(int device, void* stream, bool own, lbk_ctx* out)
{
    if (!out) {
        set_error(nullptr, "lbk_ctx_create: null out pointer");
        return LBK_USAGE_ERROR;
    }
    *out = nullptr;
    auto* ctx = new lbk_ctx_s;
    lbk_status st = guard(nullptr, [&] {
        int ndev = 0;
        LBK_CUDA(cudaGetDeviceCount(&ndev));
        need(device >= 0 && device < ndev, LBK_CONFIGURATION_ERROR,
             "device " + std::to_string(device) + " out of range (have " +
                 std::to_string(ndev) + ")");
        LBK_CUDA(cudaSetDevice(device));
        ctx->device = device;
        LBK_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        int optin = 0;
        LBK_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        ctx->smem_optin = static_cast<size_t>(optin);
        int major = 0;
        LBK_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
        need(major == 10, LBK_DISPATCH_ERROR,
             "lbk kernels are built for sm_100a (B200); device has compute capability " +
                 std::to_string(major) + ".x");
        {
            int win = 0, lim = 0;
            cudaDeviceGetAttribute(&win, cudaDevAttrMaxAccessPolicyWindowSize, device);
            cudaDeviceGetAttribute(&lim, cudaDevAttrMaxPersistingL2CacheSize, device);
            ctx->persist_max = static_cast<size_t>(win < lim ? win : lim);
            const char* e = std::getenv("LBK_L2_PERSIST");
            ctx->l2_persist = (e && e[0] == '1') ? 1 : 0;
            if (ctx->l2_persist && ctx->persist_max)
                cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(lim));
            const char* pdl = std::getenv("LBK_PDL");
            // off unless LBK_PDL=1: with exact reductions the kernels' tails
            // (block flush + global limb atomics) are longer, and early-
            // scheduled successor CTAs waiting in griddepcontrol.wait cost
            // more than they save (CG 1,047 -> 1,094 it/s, P = 8 per-rank
            // iteration 157 -> 149 us without it)
            ctx->pdl = (pdl && pdl[0] == '1') ? 1 : 0;
        }
        {
            // solver workspaces come from the stream-ordered pool; keep freed
            // memory in the pool so repeated solves do not remap pages
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
                uint64_t keep = ~uint64_t{0};
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
        }
        if (own) {
            LBK_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
            ctx->own_stream = true;
        } else {
            ctx->stream = static_cast<cudaStream_t>(stream);
        }
        LBK_CUDA(cudaMallocHost(&ctx->host_pinned, 64 * sizeof(double)));
        red_ws(ctx, kRedMaxBlocks, 4);
        LBK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
    if (st != LBK_OK) {
        delete ctx;
        return st;
    }
    *out = ctx;
    return LBK_OK;
}

lbk_status lbk_ctx_create(int device, lbk_ctx* out)
{
    return ctx_create_impl(device, nullptr, true, out);
}

lbk_status lbk_ctx_create_on_stream(int device, void* stream, lbk_ctx* out)
{
    return ctx_create_impl(device, stream, false, out);
}

lbk_status lbk_ctx_set_stream(lbk_ctx ctx, void* stream)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (ctx->own_stream) {
            LBK_CUDA(cudaStreamSynchronize(ctx->stream));
            LBK_CUDA(cudaStreamDestroy(ctx->stream));
            ctx->own_stream = false;
        }
        ctx->stream = static_cast<cudaStream_t>(stream);
    });
}

lbk_status lbk_ctx_set_l2_persist(lbk_ctx ctx, int on)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        ctx->l2_persist = on ? 1 : 0;
        if (on && ctx->persist_max) {
            int lim = 0;
            LBK_CUDA(cudaDeviceGetAttribute(&lim, cudaDevAttrMaxPersistingL2CacheSize, ctx->device));
            LBK_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, static_cast<size_t>(lim)));
        }
    });
}

lbk_status lbk_ctx_destroy(lbk_ctx ctx)
{
    if (!ctx) return LBK_OK;
    lbk_status st = guard(ctx, [&] {
        cudaStreamSynchronize(ctx->stream);
        if (ctx->scratch.ptr) cudaFree(ctx->scratch.ptr);
        if (ctx->red.ptr) cudaFree(ctx->red.ptr);
        if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
        if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    });
    delete ctx;
    return st;
}

const char* lbk_last_error(lbk_ctx ctx)
{
    if (ctx) return ctx->err.c_str();
    return g_err.c_str();
}

lbk_status lbk_sync(lbk_ctx ctx)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] { LBK_CUDA(cudaStreamSynchronize(ctx->stream)); });
}

lbk_status lbk_ctx_info(lbk_ctx ctx, int* device, int* num_sms, size_t* cap, size_t* used)
{
    if (!ctx) return LBK_USAGE_ERROR;
    if (device) *device = ctx->device;
    if (num_sms) *num_sms = ctx->num_sms;
    if (cap) *cap = ctx->arena_capacity;
    if (used) *used = ctx->arena_used;
    return LBK_OK;
}

lbk_status lbk_ctx_set_arena_capacity(lbk_ctx ctx, size_t bytes)
{
    if (!ctx) return LBK_USAGE_ERROR;
    ctx->arena_capacity = bytes;
    return LBK_OK;
}

lbk_status lbk_alloc(lbk_ctx ctx, size_t bytes, void** out)
{
    if (!ctx || !out) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        *out = nullptr;
        // executor.cpp:254-265: reject past the arena capacity.
        if (bytes > ctx->arena_capacity - ctx->arena_used) {
            fail(LBK_OUT_OF_MEMORY,
                 "out of memory on device " + std::to_string(ctx->device) + ": requested " +
                     std::to_string(bytes) + " bytes, available " +
                     std::to_string(ctx->arena_capacity - ctx->arena_used));
        }
        if (bytes == 0) return;
        cudaError_t e = cudaMalloc(out, bytes);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            fail(LBK_OUT_OF_MEMORY, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
        }
        LBK_CUDA(e);
        ctx->arena_used += bytes;
    });
}

lbk_status lbk_free(lbk_ctx ctx, void* ptr, size_t bytes)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (!ptr) return;
        LBK_CUDA(cudaFree(ptr));
        ctx->arena_used -= bytes < ctx->arena_used ? bytes : ctx->arena_used;
    });
}

lbk_status lbk_memcpy_h2d(lbk_ctx ctx, void* dst, const void* src, size_t bytes)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (bytes) LBK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    });
}

lbk_status lbk_memcpy_d2h(lbk_ctx ctx, void* dst, const void* src, size_t bytes)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        // stream-ordered like every other copy: pinned destinations overlap
        // with work on other streams; lbk_sync (or an event) before reading
        if (bytes) LBK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    });
}

lbk_status lbk_memcpy_peer(lbk_ctx ctx, void* dst, int dst_device, const void* src,
                           int src_device, size_t bytes)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (bytes)
            LBK_CUDA(cudaMemcpyPeerAsync(dst, dst_device, src, src_device, bytes, ctx->stream));
    });
}

lbk_status lbk_memcpy_d2d(lbk_ctx ctx, void* dst, const void* src, size_t bytes)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (bytes) LBK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
    });
}

}  // extern "C"
