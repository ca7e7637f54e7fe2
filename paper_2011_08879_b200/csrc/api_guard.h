// api_guard.h -- exception -> lbk_status bridge for every C-ABI entry point.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <string>

#include "lbk_internal.cuh"

namespace lbk {

void set_error(lbk_ctx ctx, const std::string& msg);

// Runs body(); converts lbk::Error / std::bad_alloc / anything else into a
// status + message.  Mirrors how the reference's CLI maps its exception
// taxonomy (tools/larch.cpp:375-394), but at the ABI instead of exit codes.
// NVTX range over a C-ABI call (tracing: nsys / ncu --nvtx attribute
// device time to the reference-level operation).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <typename F>
lbk_status guard(lbk_ctx ctx, F&& body)
{
    try {
        if (ctx) cudaSetDevice(ctx->device);
        body();
        return LBK_OK;
    } catch (const Error& e) {
        set_error(ctx, e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_error(ctx, "host allocation failed");
        return LBK_OUT_OF_MEMORY;
    } catch (const std::exception& e) {
        set_error(ctx, e.what());
        return LBK_INTERNAL;
    }
}

inline void need(bool cond, lbk_status s, const std::string& msg)
{
    if (!cond) fail(s, msg);
}

}  // namespace lbk
