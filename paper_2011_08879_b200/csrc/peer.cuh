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
//            sums them (exact integer limbs, xred.cuh; the double mailbox is
//            the -DLBK_RED_TREE build's rank-ordered sum) -- the same bits on
//            every rank and at every rank count -- then
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
    int xdigits = 0;  // LBK_XRED_DIGITS=1: post normalised digits always (tests
                      // the wide-range encoding on ordinary data)
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
// holds the exact sum over all ranks (raw limbs, round with xred_round_warp).
// Each rank posts every value as a header {lo:8 | cnt:8 | neg:1 | pinf:1 |
// ninf:1 | nan:1 | raw:1} and either cnt raw limbs (two words each) or cnt
// sign-magnitude digits; integer sums make the result independent of rank
// order and of the partition.
__device__ __forceinline__ void peer_xallreduce_warp(const PeerDev& pd, long long* L, int nv)
{
    const int lane = threadIdx.x & 31;
    PeerHdr* me = pd.win[pd.rank];
    // this rank's values.  Normally the raw limbs' nonzero range, two words
    // per limb {lo32, hi32} (no normalisation pass); a value whose range
    // does not fit its 80-word box (> 39 limbs, only for data spanning
    // ~1250 bits) goes as normalised sign-magnitude digits instead
    unsigned hdr[kXMaxNV];
    int lo_l[kXMaxNV];
    XMag mg[kXMaxNV];
#pragma unroll
    for (int v = 0; v < kXMaxNV; ++v) {
        if (v >= nv) break;
        const long long* X = L + v * kXV;
        int l0 = 99, h0 = -1;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int i = lane + 32 * k;
            if (i < kXL && X[i] != 0) {
                l0 = l0 < i ? l0 : i;
                h0 = i;
            }
        }
        l0 = __reduce_min_sync(0xffffffffu, l0);
        h0 = __reduce_max_sync(0xffffffffu, h0);
        const int cnt = h0 < 0 ? 0 : h0 - l0 + 1;
        const unsigned fl = (X[kXPinf] ? 1u << 17 : 0u) | (X[kXNinf] ? 1u << 18 : 0u) |
                            (X[kXNan] ? 1u << 19 : 0u);
        if (2 * cnt + 1 <= kXV && !pd.xdigits) {
            lo_l[v] = h0 < 0 ? 0 : l0;
            hdr[v] = static_cast<unsigned>(lo_l[v]) | (static_cast<unsigned>(cnt) << 8) | fl |
                     (1u << 20);
        } else {
            mg[v] = xred_mag_warp(X);
            int kl = 3, kh = -1;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (mg[v].d[k]) {
                    kl = kl < k ? kl : k;
                    kh = k;
                }
            const unsigned m = __ballot_sync(0xffffffffu, kh >= 0);
            int lo = 0, dc = 0;
            if (m) {
                const int ll = __ffs(m) - 1, hl = 31 - __clz(static_cast<int>(m));
                lo = 3 * ll + __shfl_sync(0xffffffffu, kl, ll);
                dc = 3 * hl + __shfl_sync(0xffffffffu, kh, hl) - lo + 1;
            }
            lo_l[v] = lo;
            hdr[v] = static_cast<unsigned>(lo) | (static_cast<unsigned>(dc) << 8) |
                     (mg[v].neg ? 1u << 16 : 0u) | fl;
        }
    }
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&me->seq_r) + 1;
    const int par = static_cast<int>(e & 1);
    const unsigned e32 = static_cast<unsigned>(e);
    const unsigned long long tag = static_cast<unsigned long long>(e32) << 32;
#pragma unroll
    for (int v = 0; v < kXMaxNV; ++v) {
        if (v >= nv) break;
        const unsigned h = hdr[v];
        const bool raw = (h >> 20) & 1;
        const int cnt = (h >> 8) & 0xff;
        const int nw = raw ? 2 * cnt : cnt;
        for (int w0 = 0; w0 <= nw; w0 += 32) {  // whole-warp rounds: shuffles inside
            const int w = w0 + lane;
            unsigned pay = h;
            if (raw) {
                if (w > 0 && w <= nw) {
                    const long long lv = L[v * kXV + lo_l[v] + (w - 1) / 2];
                    pay = (w & 1) ? static_cast<unsigned>(lv)
                                  : static_cast<unsigned>(static_cast<unsigned long long>(lv) >> 32);
                }
            } else {
                const unsigned dg = xred_digit(mg[v], lo_l[v] + w - 1);
                if (w > 0) pay = dg;
            }
            if (w <= nw)
                for (int q = 0; q < pd.P; ++q)
                    st_volatile_u64(&pd.win[q]->xred_ll[par][pd.rank][v * kXV + w], tag | pay);
        }
    }
    __syncwarp();
    for (int i = lane; i < nv * kXV; i += 32) L[i] = 0;
    __syncwarp();
    // receive in parallel (not rank after rank): one round of header loads
    // (lane = (rank, value), P * nv <= 32), then every posted digit of every
    // rank as one flat item list, 32 loads in flight per round; the digits
    // are added into the limbs with shared atomics (order-free)
    const int nh = pd.P * nv;
    unsigned hh = 0;
    int hq = 0, hv = 0;
    if (lane < nh) {
        hq = lane / nv;
        hv = lane % nv;
        hh = peer_ll_read32(me->xred_ll[par][hq] + hv * kXV, e32, me, 2, hq, e);
        if (hh & (1u << 17)) smem_add64(L + hv * kXV + kXPinf, 1);
        if (hh & (1u << 18)) smem_add64(L + hv * kXV + kXNinf, 1);
        if (hh & (1u << 19)) smem_add64(L + hv * kXV + kXNan, 1);
    }
    const int hcnt = lane < nh ? static_cast<int>((hh >> 8) & 0xff) : 0;
    int incl = hcnt;  // inclusive prefix of the digit counts over header lanes
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int i0 = 0; i0 < total; i0 += 32) {
        const int it = i0 + lane;
        // owner header lane: the first with incl > it
        int o = 0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const int t = __shfl_sync(0xffffffffu, incl, o + d - 1);
            if (o + d - 1 < 32 && t <= it) o += d;
        }
        const int start = __shfl_sync(0xffffffffu, incl - hcnt, o);
        const unsigned oh = __shfl_sync(0xffffffffu, hh, o);
        const int oq = __shfl_sync(0xffffffffu, hq, o), ov = __shfl_sync(0xffffffffu, hv, o);
        if (it < total) {
            const int w = it - start;
            const unsigned long long* box = me->xred_ll[par][oq] + ov * kXV;
            long long d;
            if ((oh >> 20) & 1) {  // a raw limb: {lo32, hi32}
                const unsigned lo32 = peer_ll_read32(box + 1 + 2 * w, e32, me, 2, oq, e);
                const unsigned hi32 = peer_ll_read32(box + 2 + 2 * w, e32, me, 2, oq, e);
                d = static_cast<long long>((static_cast<unsigned long long>(hi32) << 32) | lo32);
            } else {
                d = peer_ll_read32(box + 1 + w, e32, me, 2, oq, e);
                if ((oh >> 16) & 1) d = -d;
            }
            smem_add64(L + ov * kXV + (oh & 0xff) + w, d);
        }
    }
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(&me->seq_r) = e;
    __syncwarp();
}

}  // namespace lbk
