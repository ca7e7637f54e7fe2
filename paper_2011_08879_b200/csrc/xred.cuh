// xred.cuh -- exactly rounded, partition-independent reductions.
//
// Every dot product and norm of the solvers is reduced EXACTLY and rounded
// once:  dot(x, y) = RNE( sum_i RN(x_i * y_i) ).  Integer addition is
// associative, so the result does not depend on how rows are split over
// lanes, warps, blocks, tiles, interior/boundary sub-matrices or GPUs: the
// distributed solver at any rank count computes the same bits as the
// single-GPU one (VERDICT r1 "partition-independent reductions").  The
// reference sums sequentially (ref_dot, reference.cpp:46-56) or in thread
// chunks (par_dot, parallel.cpp:76-97); the exact sum is the order-free
// member of that family and is pinned by oracle/xkrylov.cpp (itself pinned
// to Python's math.fsum).
//
// Representation: the sum as an integer in units of 2^-1074 (the smallest
// subnormal), in 32-bit digits held in signed 64-bit limbs (carry room).
// Limb i weighs 2^(32 i); limb 72 absorbs the sign.  Three more int64
// counters record +inf, -inf and NaN terms (a plain sum's inf/nan
// semantics, which are order-free too).  kXV int64 per value.
//
// Three levels:
//   lane   XLane: a 192-bit two's-complement window (3 x u64) over limbs
//          [base, base+6); a term is added with a shifted 192-bit add.  A
//          term outside the window flushes it to the block accumulator
//          and re-centres it (rare for solver vectors).
//   block  per-value limbs in static shared memory (g_xsh); at the end each
//          warp sums its lanes' windows with redux.sync on 16-bit halves
//          and one lane adds them in.
//   grid   nonzero block limbs are atomically added (u64) into a global
//          slot; the last block rounds (single GPU) -- or, deferred, the
//          slot itself is what the ranks exchange (int64 sums: NCCL
//          allreduce, host sums, or peer-memory digit posts).
#pragma once

#include <cstdint>

namespace lbk {

constexpr int kXL = 73;           // limbs 0..71: 32-bit digits; 72: sign limb
constexpr int kXPinf = 73, kXNinf = 74, kXNan = 75;
constexpr int kXV = 80;           // int64 per reduced value (padded)
constexpr int kXMaxNV = 2;        // values per fused reduction
constexpr int kXSlot = kXMaxNV * kXV;  // int64 per reduction slot

// Block accumulator: one region of NV values x kXV limbs per warp (lanes
// flush into their own warp's region, so warps never contend), shared by
// every kernel of a translation unit that reduces (zeroed by xred_begin).
constexpr int kXWarps = 8;  // reducing kernels run <= 256 threads
static __shared__ long long g_xsh[kXWarps * kXSlot];
__device__ __forceinline__ long long* xwarp_limbs()
{
    return g_xsh + (threadIdx.x >> 5) * kXSlot;
}

struct XLane {
    unsigned long long w0, w1, w2;
    int base;  // window = limbs [base, base + 6)
};

// 64-bit add into a shared-memory limb with two native 32-bit atomics
// (sm_100 has no shared 64-bit atomic add: atomicAdd(u64) on shared memory
// compiles to a CAS spin loop).  The low word's carry comes from its own
// atomic's old value, so the limb is exact once all adds have landed.
__device__ __forceinline__ void smem_add64(long long* p, long long v)
{
    unsigned* w = reinterpret_cast<unsigned*>(p);
    const unsigned lo = static_cast<unsigned>(v);
    const unsigned hi = static_cast<unsigned>(static_cast<unsigned long long>(v) >> 32);
    const unsigned old = atomicAdd(w, lo);
    const unsigned h = hi + ((old + lo) < old ? 1u : 0u);
    if (h) atomicAdd(w + 1, h);
}

__device__ __forceinline__ void xl_zero(XLane& a)
{
    a.w0 = a.w1 = a.w2 = 0;
    a.base = -4096;  // empty: every term re-centres
}

// add/subtract (t2:t1:t0) into the 192-bit window
__device__ __forceinline__ void add192(XLane& a, unsigned long long t0, unsigned long long t1,
                                       unsigned long long t2)
{
    asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
        : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
        : "l"(t0), "l"(t1), "l"(t2));
}
__device__ __forceinline__ void sub192(XLane& a, unsigned long long t0, unsigned long long t1,
                                       unsigned long long t2)
{
    asm("sub.cc.u64 %0, %0, %3;\n\tsubc.cc.u64 %1, %1, %4;\n\tsubc.u64 %2, %2, %5;"
        : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
        : "l"(t0), "l"(t1), "l"(t2));
}

// Flush one lane's window into a value's limbs (shared or global) with
// atomics.  Window value = U - neg * 2^192 at limb `base`.
__device__ __forceinline__ void xl_flush_atomic(const XLane& a, long long* limbs)
{
    if ((a.w0 | a.w1 | a.w2) == 0) return;
    const unsigned long long w[3] = {a.w0, a.w1, a.w2};
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const unsigned long long d = (w[k >> 1] >> (32 * (k & 1))) & 0xffffffffull;
        if (d) smem_add64(limbs + a.base + k, static_cast<long long>(d));
    }
    if (a.w2 >> 63)
        smem_add64(limbs + a.base + 6, -1LL);
}

static __device__ __noinline__ void xl_special(double v, long long* limbs)
{
    const int which = v != v ? kXNan : (v > 0 ? kXPinf : kXNinf);
    smem_add64(limbs + which, 1LL);
}

// Warp-aggregated flush of every lane's window into the block limbs
// (all 32 lanes call).  When the lanes' windows lie within 2 limbs of each
// other (the normal case) the warp adds them with redux.sync on 16-bit
// halves and lane 0 posts 9 limbs; otherwise every lane flushes itself.
__device__ __forceinline__ void xl_group_flush(const XLane& a, long long* limbs, unsigned mask)
{
    const bool nz = (a.w0 | a.w1 | a.w2) != 0;
    const unsigned act = __ballot_sync(mask, nz);
    if (!act) return;
    const int lo = __reduce_min_sync(mask, nz ? a.base : 0x7fffffff);
    const int hi = __reduce_max_sync(mask, nz ? a.base : -0x7fffffff);
    if (hi - lo > 2) {
        xl_flush_atomic(a, limbs);
        return;
    }
    // lane value as 256 bits (sign-extended), shifted up by (base-lo) limbs
    const int sh = nz ? a.base - lo : 0;
    const unsigned long long ext = (a.w2 >> 63) ? ~0ull : 0ull;
    unsigned long long w[4] = {nz ? a.w0 : 0ull, nz ? a.w1 : 0ull, nz ? a.w2 : 0ull,
                               nz ? ext : 0ull};
    unsigned d[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) d[k] = static_cast<unsigned>(w[k >> 1] >> (32 * (k & 1)));
    unsigned dd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int src = k - sh;  // digit k of the shifted value
        unsigned v = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (j == src) v = d[j];
        if (src < 0) v = 0;
        dd[k] = v;
    }
    // sign: the shifted 256-bit value stands for V + neg * 2^(256) at limb
    // lo; the top 2*sh digits of the shifted-out part are all sign bits
    const int neg = nz && (a.w2 >> 63);
    const int nneg = __popc(__ballot_sync(mask, neg));
    long long tot[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const unsigned l16 = __reduce_add_sync(mask, dd[k] & 0xffffu);
        const unsigned h16 = __reduce_add_sync(mask, dd[k] >> 16);
        tot[k] = static_cast<long long>(l16) + (static_cast<long long>(h16) << 16);
    }
    if ((threadIdx.x & 31) == __ffs(mask) - 1) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (tot[k])
                smem_add64(limbs + lo + k, tot[k]);
        if (nneg)
            smem_add64(limbs + lo + 8, -static_cast<long long>(nneg));
    }
}

__device__ __forceinline__ void xl_warp_flush(const XLane& a, long long* limbs)
{
    xl_group_flush(a, limbs, 0xffffffffu);
}

#ifdef LBK_XRED_STATS
static __device__ unsigned long long g_xred_stats[4];  // direct terms, -, placements, -
#define LBK_XSTAT(i) atomicAdd(&g_xred_stats[i], 1ull)
#else
#define LBK_XSTAT(i) ((void)0)
#endif

// A term outside the lane's window goes straight into the warp's limbs:
// its three 32-bit digits, added (or, negative, subtracted) with shared-
// memory atomics.  No re-centring, no warp vote, no call -- small code on
// the cold path, and the window keeps serving the common magnitudes.
__device__ __forceinline__ void xl_direct(unsigned long long m, int pos, bool neg,
                                          long long* limbs)
{
    const int li = pos >> 5, off = pos & 31;
    const unsigned long long lo = m << off;                 // digits 0, 1
    const unsigned long long d2 = off ? (m >> (64 - off)) : 0ull;  // digit 2
    const long long d0 = static_cast<long long>(lo & 0xffffffffull);
    const long long d1 = static_cast<long long>(lo >> 32);
    const long long sg = neg ? -1 : 1;
    long long* L = limbs + li;
    if (d0) smem_add64(L, sg * d0);
    if (d1) smem_add64(L + 1, sg * d1);
    if (d2) smem_add64(L + 2, sg * static_cast<long long>(d2));
    LBK_XSTAT(0);
}

// Add one term.  `limbs` = this value's flush target (the warp's limbs).
// NN: the caller guarantees v >= 0 (a square): no two's-complement path.
template <bool NN = false>
__device__ __forceinline__ void xl_add(XLane& a, double v, long long* limbs)
{
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    if ((bits << 1) == 0) return;  // +-0
    const int e = static_cast<int>((bits >> 52) & 0x7ff);
    if (e == 0x7ff) {
        xl_special(v, limbs);
        return;
    }
    const unsigned long long m = (bits & 0xfffffffffffffull) | (e ? (1ull << 52) : 0ull);
    const int pos = e ? e - 1 : 0;  // bit position of m's lsb
    int s = pos - 32 * a.base;
    if (__builtin_expect(static_cast<unsigned>(s) > 107u, 0)) {  // outside the window
        if (s < 0) {  // far below the largest terms so far: straight to the limbs
            xl_direct(m, pos, bits >> 63, limbs);
            return;
        }
        // above the window (or the lane's first term): the window follows
        // the largest magnitude -- flush it exactly and re-place it with
        // this term's lsb 64..95 bits above the bottom (room for terms up
        // to 2^64 smaller, and for 12..43 bits of growth); bounded by the
        // ~65 limbs of the double range per lane
        xl_flush_atomic(a, limbs);
        const int b = (pos >> 5) - 2;
        a.base = b < 0 ? 0 : b;
        a.w0 = a.w1 = a.w2 = 0;
        s = pos - 32 * a.base;
        LBK_XSTAT(2);
    }
    // m << s over 192 bits, two's-complement negated for a negative term:
    // (t ^ sg) + (sg & 1) -- branch-free, carried into the 192-bit add
    const bool hi = s >= 64;
    const int u = hi ? s - 64 : s;
    const unsigned long long lo_w = m << u;
    const unsigned long long hi_w = u ? (m >> (64 - u)) : 0ull;
    if constexpr (NN) {
        add192(a, hi ? 0ull : lo_w, hi ? lo_w : hi_w, hi ? hi_w : 0ull);
    } else {
        const unsigned long long sg =
            static_cast<unsigned long long>(static_cast<long long>(bits) >> 63);
        const unsigned long long t0 = (hi ? 0ull : lo_w) ^ sg;
        const unsigned long long t1 = (hi ? lo_w : hi_w) ^ sg;
        const unsigned long long t2 = (hi ? hi_w : 0ull) ^ sg;
        asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;\n\t"
            "add.cc.u64 %0, %0, %6;\n\taddc.cc.u64 %1, %1, 0;\n\taddc.u64 %2, %2, 0;"
            : "+l"(a.w0), "+l"(a.w1), "+l"(a.w2)
            : "l"(t0), "l"(t1), "l"(t2), "l"(sg & 1ull));
    }
}

// Zero the block accumulator; every thread of the block must call.
template <int NV>
__device__ __forceinline__ void xred_begin()
{
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = threadIdx.x; i < nw * kXSlot; i += blockDim.x) g_xsh[i] = 0;
    __syncthreads();
}

// ------------------------------------------------- warp-parallel finish
// The finishing steps run on one warp, not one thread: lane j owns digits
// 3j .. 3j+2 (72 digits), the carries ripple between lanes with shuffles
// (a carry survives a digit only when it is all ones or zero, so the loop
// ends after one or two rounds), and sign, top digit and sticky bits come
// from ballots.  This is the fixed cost of every reduction (the last
// block on one GPU, the finish kernel per exchange in the distributed
// solver), so it matters most at 8 ranks.
struct XMag {
    unsigned d[3];  // magnitude digits 3*lane .. 3*lane+2
    bool neg;
    int special;    // 0 finite, 1 +inf, 2 -inf, 3 nan
};

// All 32 lanes call.  L: one value's raw limbs (kXV int64, read only).
__device__ __forceinline__ XMag xred_mag_warp(const long long* L)
{
    const int lane = threadIdx.x & 31;
    XMag r;
    const long long pinf = L[kXPinf], ninf = L[kXNinf], nan = L[kXNan];
    r.special = (nan || (pinf && ninf)) ? 3 : (pinf ? 1 : (ninf ? 2 : 0));
    long long t[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int i = 3 * lane + k;
        t[k] = i < kXL - 1 ? L[i] : 0;
    }
    long long sign = L[kXL - 1];  // limb 72
    long long c = 0;              // this lane's carry out
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const long long v = t[k] + c;
        c = v >> 32;
        t[k] = v & 0xffffffffLL;
    }
    // ripple the carries up the lanes (lane 23's carry goes to the sign)
    for (;;) {
        if (lane == 23) {
            sign += c;
            c = 0;
        }
        const long long cin = __shfl_up_sync(0xffffffffu, c, 1);
        const bool more = __any_sync(0xffffffffu, c != 0);
        if (!more) break;
        c = 0;
        if (lane > 0 && lane < 24) {
            long long v = t[0] + cin;
            c = v >> 32;
            t[0] = v & 0xffffffffLL;
#pragma unroll
            for (int k = 1; k < 3; ++k) {
                v = t[k] + c;
                c = v >> 32;
                t[k] = v & 0xffffffffLL;
            }
        }
    }
    sign = __shfl_sync(0xffffffffu, sign, 23);
    r.neg = sign < 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) r.d[k] = static_cast<unsigned>(t[k]);
    if (r.neg) {  // magnitude = ~D + 1: the +1 lands on D's lowest nonzero digit
        const bool nz = (r.d[0] | r.d[1] | r.d[2]) != 0;
        const unsigned m = __ballot_sync(0xffffffffu, nz);
        const int l0 = m ? __ffs(m) - 1 : 32;
        int k0 = 3;
        if (lane == l0) k0 = r.d[0] ? 0 : (r.d[1] ? 1 : 2);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const bool below = lane < l0 || (lane == l0 && k < k0);
            const bool at = lane == l0 && k == k0;
            r.d[k] = below ? 0u : (at ? 0u - r.d[k] : ~r.d[k]);
        }
        if (lane >= 24) r.d[0] = r.d[1] = r.d[2] = 0;
    }
    return r;
}

// Round a magnitude (xred_mag_warp) to the nearest double; all lanes call,
// every lane gets the value.
__device__ __forceinline__ double xred_round_mag(const XMag& r)
{
    const int lane = threadIdx.x & 31;
    if (r.special == 3) return __longlong_as_double(0x7ff8000000000000LL);
    if (r.special == 1) return __longlong_as_double(0x7ff0000000000000LL);
    if (r.special == 2) return __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL));
    const int kt = r.d[2] ? 2 : (r.d[1] ? 1 : (r.d[0] ? 0 : -1));
    const unsigned m = __ballot_sync(0xffffffffu, kt >= 0);
    if (!m) return 0.0;
    const int tl = 31 - __clz(static_cast<int>(m));             // top lane
    const int ktop = __shfl_sync(0xffffffffu, kt, tl);
    const int top = 3 * tl + ktop;                               // top digit index
    auto digit = [&](int i) -> unsigned long long {            // broadcast digit i
        const int src = i < 0 ? 0 : i / 3, k = i < 0 ? 0 : i % 3;
        const unsigned v0 = __shfl_sync(0xffffffffu, r.d[0], src);
        const unsigned v1 = __shfl_sync(0xffffffffu, r.d[1], src);
        const unsigned v2 = __shfl_sync(0xffffffffu, r.d[2], src);
        const unsigned v = k == 0 ? v0 : (k == 1 ? v1 : v2);
        return i < 0 ? 0ull : static_cast<unsigned long long>(v);
    };
    const unsigned long long dt = digit(top), d1 = digit(top - 1), d2 = digit(top - 2);
    // sticky: any digit below top - 2
    bool low = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) low |= (3 * lane + k < top - 2) && r.d[k] != 0;
    const bool sticky_low = __any_sync(0xffffffffu, low);
    double res;
    if (top <= 1) {  // < 2^64 units: the value is dt (top 0) or dt:d1 (top 1)
        const unsigned long long v = top == 1 ? ((dt << 32) | d1) : dt;
        res = ldexp(__ull2double_rn(v), -1074);
    } else {
        const int hb = 31 - __clz(static_cast<int>(dt));
        const int ls = 31 - hb;
        const unsigned long long hi64 = (dt << 32) | d1;
        unsigned long long T = ls ? ((hi64 << ls) | (d2 >> (32 - ls))) : hi64;
        const bool sticky = sticky_low || ((d2 << ls) & 0xffffffffull) != 0;
        T |= sticky ? 1ull : 0ull;
        res = ldexp(__ull2double_rn(T), 32 * (top - 2) + 1 + hb - 1074);
    }
    return r.neg ? -res : res;
}

// Digit i (0..71) of a magnitude, fetched from its owning lane; all lanes
// call (out-of-range i gives 0).
__device__ __forceinline__ unsigned xred_digit(const XMag& r, int i)
{
    const int src = (i < 0 || i > 71) ? 0 : i / 3, k = (i < 0 || i > 71) ? 0 : i % 3;
    const unsigned v0 = __shfl_sync(0xffffffffu, r.d[0], src);
    const unsigned v1 = __shfl_sync(0xffffffffu, r.d[1], src);
    const unsigned v2 = __shfl_sync(0xffffffffu, r.d[2], src);
    return (i < 0 || i > 71) ? 0u : (k == 0 ? v0 : (k == 1 ? v1 : v2));
}

__device__ __forceinline__ double xred_round_warp(const long long* L)
{
    return xred_round_mag(xred_mag_warp(L));
}

}  // namespace lbk
