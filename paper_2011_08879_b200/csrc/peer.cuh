// peer.cuh -- the NVLink peer-memory communicator.
//
// Each rank owns one device "window" (cudaMalloc, exported as a CUDA IPC
// handle; in-process groups share the pointer).  Every rank maps every
// peer's window, so the two collectives of the distributed solver are plain
// loads and stores over NVLink issued by lbk's own kernels -- no NCCL on
// the iteration path, no host involvement, and CUDA-graph capturable.
//
// Both use LL-style words (as NCCL's low-latency protocol): a double
// travels as two 8-byte stores {epoch:32 | half:32}; a reader spins until
// both halves carry the epoch it expects.  No fences, no separate flags --
// an 8-byte store arrives whole, and the tag says which epoch it belongs to.
//
//   halo     the pack kernel gathers the values a peer needs and stores
//            them, tagged, straight into that peer's staging slot; after
//            the interior rows, the boundary-row kernel (dist.cuh) reads
//            each ghost from the slot as its tag arrives and hands the slot
//            back (`empty` word in the sender's window).
//   scalars  the finishing kernel of each fused reduction posts the rank's
//            totals into every window's mailbox, waits for all P posts and
//            sums them in rank order -- the same bits on every rank -- then
//            advances the solver recurrence (combine + allreduce + finish
//            in one launch).
//
// Epochs are device counters (seq_x, seq_r) so captured graphs replay
// correctly.  Slots are double-buffered by epoch parity: a sender reuses a
// halo slot only once the receiver has consumed the epoch before last
// (`empty`); a mailbox slot of parity p is rewritten two epochs later,
// which every rank can only reach after all ranks have read it.  Waits spin
// with a timeout (LBK_PEER_TIMEOUT seconds, default 300); a timeout raises
// the sticky `error` word that the host reports as LBK_NCCL_ERROR.
#pragma once

#include "lbk_internal.cuh"

namespace lbk {

constexpr int kPeerMax = 16;     // ranks per peer group (one NVSwitch node)
constexpr int kPeerRedMax = 16;  // values per reduction

struct PeerHdr {
    unsigned long long empty[kPeerMax];  // halo epoch rank q consumed from me
    // reduction mailbox, LL-style: each double travels as two 8-byte words
    // {epoch:32 | half:32}, [parity][source rank][value][half]; a word is
    // valid when its epoch tag matches, so no fences or flags are needed
    unsigned long long red_ll[2][kPeerMax][kPeerRedMax][2];
    // exact-reduction mailbox (xred.cuh): per value a header word then its
    // sign-magnitude 32-bit digits, LL-tagged; [parity][source][word]
    unsigned long long xred_ll[2][kPeerMax][kXSlot];
    unsigned long long seq_x, seq_r;     // local epochs (this rank only)
    unsigned int recv_cnt, pad0_;        // last-block counter
    int error;
    int pad_;
    long long err_info[4];  // first timeout: {what (0 halo values, 1 halo
                            // hand-back, 2 reduction), peer, wanted epoch,
                            // seen epoch}
    long long timeout_ns;
    long long cap;  // halo values per (parity, source) slot -- equal on all ranks
    // staging after the header: [parity][source][cap][2] LL words
};

constexpr size_t kPeerHdrBytes = (sizeof(PeerHdr) + 255) / 256 * 256;

// Kernel argument: every rank's window as mapped into this process.
struct PeerDev {
    PeerHdr* win[kPeerMax];
    int P = 0, rank = 0;
    long long cap = 0;
    // staging slot (parity par, source src) inside rank q's window
    __device__ unsigned long long* stage(int q, int par, int src) const
    {
        return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(win[q]) +
                                                     kPeerHdrBytes) +
               (static_cast<size_t>(par) * P + src) * cap * 2;
    }
};

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long global_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin until *f >= e (acquire), the group fails, or the timeout expires.
__device__ __forceinline__ void peer_wait_ge(const unsigned long long* f, unsigned long long e,
                                             PeerHdr* me, int what, int peer)
{
    if (ld_volatile_u64(f) >= e) return;
    const unsigned long long t0 = global_ns();
    unsigned long long seen;
    while ((seen = ld_volatile_u64(f)) < e) {
        if (*reinterpret_cast<volatile int*>(&me->error)) return;
        if (global_ns() - t0 > static_cast<unsigned long long>(me->timeout_ns)) {
            if (atomicExch(&me->error, 1) == 0) {
                me->err_info[0] = what;
                me->err_info[1] = peer;
                me->err_info[2] = static_cast<long long>(e);
                me->err_info[3] = static_cast<long long>(seen);
            }
            return;
        }
        __nanosleep(100);
    }
}


// Read one LL-encoded double posted with epoch tag e32 (spin until both
// halves carry the tag, the group fails, or the timeout expires).
__device__ __forceinline__ double peer_ll_read(const unsigned long long* w, unsigned e32,
                                               PeerHdr* me, int what, int peer,
                                               unsigned long long e)
{
    unsigned long long a = ld_volatile_u64(w), b = ld_volatile_u64(w + 1);
    if (static_cast<unsigned>(a >> 32) != e32 || static_cast<unsigned>(b >> 32) != e32) {
        const unsigned long long t0 = global_ns();
        for (;;) {
            a = ld_volatile_u64(w);
            b = ld_volatile_u64(w + 1);
            if (static_cast<unsigned>(a >> 32) == e32 && static_cast<unsigned>(b >> 32) == e32)
                break;
            if (*reinterpret_cast<volatile int*>(&me->error)) break;
            if (global_ns() - t0 > static_cast<unsigned long long>(me->timeout_ns)) {
                if (atomicExch(&me->error, 1) == 0) {
                    me->err_info[0] = what;
                    me->err_info[1] = peer;
                    me->err_info[2] = static_cast<long long>(e);
                    me->err_info[3] = static_cast<long long>(a >> 32);
                }
                break;
            }
            __nanosleep(32);
        }
    }
    return __longlong_as_double(static_cast<long long>((b << 32) | (a & 0xffffffffull)));
}

// One LL word: spin until its tag is e32; returns the 32-bit payload.
__device__ __forceinline__ unsigned peer_ll_read32(const unsigned long long* w, unsigned e32,
                                                   PeerHdr* me, int what, int peer,
                                                   unsigned long long e)
{
    unsigned long long a = ld_volatile_u64(w);
    if (static_cast<unsigned>(a >> 32) != e32) {
        const unsigned long long t0 = global_ns();
        for (;;) {
            a = ld_volatile_u64(w);
            if (static_cast<unsigned>(a >> 32) == e32) break;
            if (*reinterpret_cast<volatile int*>(&me->error)) break;
            if (global_ns() - t0 > static_cast<unsigned long long>(me->timeout_ns)) {
                if (atomicExch(&me->error, 1) == 0) {
                    me->err_info[0] = what;
                    me->err_info[1] = peer;
                    me->err_info[2] = static_cast<long long>(e);
                    me->err_info[3] = static_cast<long long>(a >> 32);
                }
                break;
            }
            __nanosleep(32);
        }
    }
    return static_cast<unsigned>(a);
}

__device__ __forceinline__ void peer_ll_store(unsigned long long* w, double v,
                                              unsigned long long tag)
{
    const unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(v));
    st_volatile_u64(w, tag | (bits & 0xffffffffull));
    st_volatile_u64(w + 1, tag | (bits >> 32));
}

// rank q of the (<= kPeerMax) segments [off[q], off[q+1]) holding entry i
__device__ __forceinline__ int seg_of(const int* off, int P, int i)
{
    int q = 0;
    while (q + 1 < P && i >= off[q + 1]) ++q;
    return q;
}

inline int peer_grid(long long n)
{
    const long long b = (n + 255) / 256;
    return b < 1 ? 1 : (b > 296 ? 296 : static_cast<int>(b));
}

// One warp.  Lane i < n (1 <= n <= kPeerRedMax) contributes v; returns the
// rank-ordered sum over all ranks in lane i (identical bits on every rank).
// Every rank reads every other rank's post of this epoch before it can
// post the next, so no rank runs two epochs ahead and parity reuse is safe.
__device__ __forceinline__ double peer_allreduce_warp(const PeerDev& pd, double v, int n)
{
    const int lane = threadIdx.x & 31;
    PeerHdr* me = pd.win[pd.rank];
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&me->seq_r) + 1;
    const int par = static_cast<int>(e & 1);
    const unsigned e32 = static_cast<unsigned>(e);
    const unsigned long long tag = static_cast<unsigned long long>(e32) << 32;
    if (lane < n)
        for (int q = 0; q < pd.P; ++q) peer_ll_store(pd.win[q]->red_ll[par][pd.rank][lane], v, tag);
    double t = 0.0;
    if (lane < n)
        for (int q = 0; q < pd.P; ++q)
            t = add_rn(t, peer_ll_read(me->red_ll[par][q][lane], e32, me, 2, q, e));
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&me->seq_r) = e;
    return t;
}

// Exact variant (xred.cuh).  One warp.  L (shared memory) holds nv values
// of raw limbs (kXV int64 each) -- this rank's exact totals; on return it
// holds the exact sum over all ranks (raw limbs, round with xred_round).
// Each rank posts every value as a header {lo:8 | cnt:8 | neg:1 | pinf:1 |
// ninf:1 | nan:1} and cnt sign-magnitude digits; integer sums make the
// result independent of rank order and of the partition.
__device__ __forceinline__ void peer_xallreduce_warp(const PeerDev& pd, long long* L, int nv)
{
    const int lane = threadIdx.x & 31;
    PeerHdr* me = pd.win[pd.rank];
    __shared__ unsigned hdr[kXMaxNV];
    if (lane == 0) {
        for (int v = 0; v < nv; ++v) {
            long long* X = L + v * kXV;
            long long c = 0;
            for (int i = 0; i < kXL; ++i) {
                const long long t = X[i] + c;
                c = t >> 32;
                X[i] = t & 0xffffffffLL;
            }
            const bool neg = c < 0;
            if (neg) {
                long long cy = 1;
                for (int i = 0; i < kXL; ++i) {
                    const long long t = (0xffffffffLL - X[i]) + cy;
                    cy = t >> 32;
                    X[i] = t & 0xffffffffLL;
                }
            }
            int lo = 0, hi = -1;
            for (int i = 0; i < kXL; ++i)
                if (X[i]) {
                    if (hi < 0) lo = i;
                    hi = i;
                }
            const int cnt = hi < 0 ? 0 : hi - lo + 1;
            hdr[v] = static_cast<unsigned>(lo) | (static_cast<unsigned>(cnt) << 8) |
                     (neg ? 1u << 16 : 0u) | (X[kXPinf] ? 1u << 17 : 0u) |
                     (X[kXNinf] ? 1u << 18 : 0u) | (X[kXNan] ? 1u << 19 : 0u);
        }
    }
    __syncwarp();
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&me->seq_r) + 1;
    const int par = static_cast<int>(e & 1);
    const unsigned e32 = static_cast<unsigned>(e);
    const unsigned long long tag = static_cast<unsigned long long>(e32) << 32;
    for (int v = 0; v < nv; ++v) {
        const unsigned h = hdr[v];
        const int lo = h & 0xff, cnt = (h >> 8) & 0xff;
        for (int w = lane; w <= cnt; w += 32) {
            const unsigned pay = w == 0 ? h : static_cast<unsigned>(L[v * kXV + lo + w - 1]);
            for (int q = 0; q < pd.P; ++q)
                st_volatile_u64(&pd.win[q]->xred_ll[par][pd.rank][v * kXV + w], tag | pay);
        }
    }
    __syncwarp();
    for (int i = lane; i < nv * kXV; i += 32) L[i] = 0;
    __syncwarp();
    for (int q = 0; q < pd.P; ++q) {
        for (int v = 0; v < nv; ++v) {
            const unsigned long long* box = me->xred_ll[par][q] + v * kXV;
            const unsigned h = peer_ll_read32(box, e32, me, 2, q, e);
            const int lo = h & 0xff, cnt = (h >> 8) & 0xff;
            const bool neg = (h >> 16) & 1;
            for (int w = lane; w < cnt; w += 32) {
                const long long d = peer_ll_read32(box + 1 + w, e32, me, 2, q, e);
                L[v * kXV + lo + w] += neg ? -d : d;
            }
            if (lane == 0) {
                L[v * kXV + kXPinf] += (h >> 17) & 1;
                L[v * kXV + kXNinf] += (h >> 18) & 1;
                L[v * kXV + kXNan] += (h >> 19) & 1;
            }
            __syncwarp();
        }
    }
    if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&me->seq_r) = e;
    __syncwarp();
}

}  // namespace lbk
