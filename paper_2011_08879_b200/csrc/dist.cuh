// dist.cuh -- row-partitioned distributed CSR (absent from the
// reference, whose only "communication" is in-process copy routing,
// device_array.cpp:144-201).
//
//   partition  contiguous row blocks, rank(r) = min(r / ceil(N/P), P-1)
//   ghosts     sorted unique non-owned columns of the rank's rows; ghost g
//              gets local column id n_local + g; ghosts owned by rank q form
//              one contiguous run (ghost_off[q], ghost_off[q+1])
//   sends      for each peer q, the local ids q needs from us (q's ghosts we
//              own, ascending) -- learned by one all-to-all of ghost lists
//   rows       interior rows (no ghost column) and boundary rows, each kept
//              as a CSR sub-matrix over the extended vector
//              x_ext = [x_local | x_ghost] with a row map back to local rows
//   SpMV       pack send values -> exchange (NCCL send/recv on a comm stream)
//              overlapped with the interior rows -> boundary rows.  Each row
//              keeps the reference's ascending-k order (boundary rows see
//              their columns renumbered, but ghost ids preserve the global
//              column order, so the k order is unchanged).
#pragma once

#include <nccl.h>

#include <vector>

#include "peer.cuh"
#include "spmv_launch.cuh"

struct lbk_dist_map_s {
    int n_global, ncols_global, P, rank, begin, end, n_local;
    long long nnz_local;
    std::vector<int> ghosts;      // sorted global ids
    std::vector<int> ghost_off;   // P + 1
    std::vector<int> local_cols;  // nnz_local
    std::vector<int> interior, boundary;
    std::vector<int> send_off;    // P + 1
    std::vector<int> send_idx;    // local ids
    bool sends_set = false;
};

namespace lbk {

// Cross-rank operations the distributed path needs.
struct Comm {
    int nranks = 1, rank = 0;
    virtual ~Comm() = default;
    // sum `count` doubles at dev over all ranks, result on every rank (same
    // bits everywhere), stream-ordered on s
    virtual void allreduce_sum(double* dev, int count, cudaStream_t s) = 0;
    // sum `count` int64 at dev over all ranks (exact reductions, xred.cuh:
    // integer sums are order-free), stream-ordered on s
    virtual void allreduce_i64(long long* dev, int count, cudaStream_t s) = 0;
    // halo exchange: send_buf[send_off[q] .. send_off[q+1]) goes to rank q;
    // from rank q we receive recv_off[q+1]-recv_off[q] values into
    // recv + recv_off[q].  Stream-ordered on s.
    virtual void exchange(const double* send_buf, const std::vector<int>& send_off,
                          double* recv, const std::vector<int>& recv_off, cudaStream_t s) = 0;
    // true if exchange() is asynchronous on s (can overlap compute on
    // another stream)
    virtual bool async() const = 0;
    // host wait for s; a communicator that can fail asynchronously (NCCL:
    // a dead peer) polls for that instead of blocking forever
    virtual void wait(cudaStream_t s) { LBK_CUDA(cudaStreamSynchronize(s)); }
    // peer-memory group (peer.cuh): the halo and the scalar reductions run
    // in lbk's own kernels over the mapped windows instead of exchange() /
    // allreduce_sum()
    virtual const PeerDev* peer() const { return nullptr; }
};

struct DevArr {
    void* p = nullptr;
    ~DevArr()
    {
        if (p) cudaFree(p);
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    void alloc(size_t bytes)
    {
        LBK_CUDA(cudaMalloc(&p, bytes < 16 ? 16 : bytes));
    }
};

struct SubCsr {
    int nrows = 0, ncols = 0;
    long long nnz = 0;
    DevArr row_ptr, cols, vals, row_map, plan;
    int ntiles = 0;
    int row_off = -1;  // >= 0: rows are contiguous from row_off (no row_map)
    CsrView<double> view() const
    {
        return CsrView<double>{nrows, ncols, nnz, row_ptr.as<int>(), cols.as<int>(),
                               vals.as<double>(), plan.as<int>(), ntiles};
    }
};

// Epilogue adaptors: sub-matrix row -> local row.
// MappedEpi looks the local row up in a row map (boundary rows, which form
// two runs at the ends of a row block).  OffsetEpi serves a contiguous row
// subset (the interior rows of a row-block partition of a banded matrix)
// with a compile-time offset form: it keeps the inner epilogue's own
// prefetch/pre structure, so the interior SpMV runs the same code as the
// single-GPU kernel (a generic runtime map-or-offset adaptor cost 15-19%
// per SpMV in register pressure, ncu at cfg4).
template <class Epi>
struct MappedEpi {
    static constexpr int NV = Epi::NV;
    static constexpr unsigned kSq = SqMask<Epi>::value;
    Epi e;
    const int* __restrict__ map;
    struct Pre {
        int r;
        typename EpiPre<Epi>::type p;
    };
    __device__ bool skip() const { return e.skip(); }
    __device__ Pre pre(int r) const
    {
        const int m = __ldg(map + r);
        return {m, EpiPre<Epi>::load(e, m)};
    }
    __device__ void row_pre(int, double s, const Pre& p, auto* acc) const
    {
        EpiPre<Epi>::row(e, p.r, s, p.p, acc);
    }
    __device__ void row(int r, double s, auto* acc) const { e.row(__ldg(map + r), s, acc); }
    __device__ void finish(const double* t) const { e.finish(t); }
};

template <class Epi>
struct OffsetEpiBase {
    static constexpr int NV = Epi::NV;
    static constexpr unsigned kSq = SqMask<Epi>::value;
    Epi e;
    int off;
    __device__ bool skip() const { return e.skip(); }
    __device__ void prefetch(int rb, int re) const { EpiPf<Epi>::run(e, rb + off, re + off); }
    __device__ void row(int r, double s, auto* acc) const { e.row(r + off, s, acc); }
    __device__ void finish(const double* t) const { e.finish(t); }
};
template <class Epi, class = void>
struct OffsetEpi : OffsetEpiBase<Epi> {
};
template <class Epi>
struct OffsetEpi<Epi, std::void_t<typename Epi::Pre>> : OffsetEpiBase<Epi> {
    using Pre = typename Epi::Pre;
    __device__ Pre pre(int r) const { return this->e.pre(r + this->off); }
    __device__ void row_pre(int r, double s, const Pre& p, auto* acc) const
    {
        this->e.row_pre(r + this->off, s, p, acc);
    }
};

template <class Epi>
void launch_sub(lbk_ctx ctx, const SubCsr& S, const double* x, const Epi& epi, RedWs ws)
{
    if (S.row_off >= 0)
        launch_csr<double>(ctx, S.view(), x, OffsetEpi<Epi>{{epi, S.row_off}}, ws);
    else
        launch_csr<double>(ctx, S.view(), x, MappedEpi<Epi>{epi, S.row_map.as<int>()}, ws);
}

}  // namespace lbk

struct lbk_dist_csr_s {
    int n_local = 0, n_ghost = 0, P = 1, rank = 0;
    long long nnz_local = 0, n_global = 0, nnz_global = 0;
    lbk::SubCsr interior, boundary;
    std::vector<int> send_off, recv_off;
    lbk::DevArr send_idx, send_buf;
    lbk::DevArr send_off_d, recv_off_d;  // P + 1 each (peer-memory kernels)
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_recv = nullptr;
    int device = 0;
};

struct lbk_comm_s {
    lbk::Comm* impl = nullptr;
};

namespace lbk {

void dist_pack(lbk_ctx ctx, const lbk_dist_csr_s* D, const double* x);
// peer-memory halo: gather + remote store into the neighbours' staging
// slots (before the interior rows)
void peer_push(lbk_ctx ctx, const lbk_dist_csr_s* D, const PeerDev& pd, const double* x);

// Peer-memory boundary rows, fused with the halo receive: thread per
// boundary row, summed sequentially in ascending k (the reference's bits
// for every row length); a ghost column is read straight from this rank's
// staging slot, spinning on its LL tag, so no separate receive kernel or
// ghost copy runs.  Every block then counts itself out; the last one hands
// the slots back and advances the halo epoch -- also when the solver is
// done and the rows are skipped, so all ranks' epochs stay in step.
template <class Epi>
__global__ void __launch_bounds__(256)
    peer_boundary_kernel(PeerDev pd, int nrows, const int* __restrict__ rp,
                         const int* __restrict__ cols, const double* __restrict__ vals,
                         const int* __restrict__ row_map, int row_off, int n_local,
                         const int* __restrict__ recv_off, const double* __restrict__ x, Epi epi,
                         RedWs ws)
{
    pdl_enter();
    constexpr int NV = Epi::NV > 0 ? Epi::NV : 1;
    __shared__ double red_sh[32 * NV];
    __shared__ int ro[kPeerMax + 1];
    PeerHdr* me = pd.win[pd.rank];
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&me->seq_x) + 1;
    const int par = static_cast<int>(e & 1);
    if (threadIdx.x <= pd.P) ro[threadIdx.x] = __ldg(recv_off + threadIdx.x);
    __syncthreads();
    if constexpr (Epi::NV > 0) red_begin<NV>();
    const bool skip = epi.skip();
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
    if (!skip) {
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
             i += gridDim.x * blockDim.x) {
            double s = 0.0;
            const int kb = __ldg(rp + i), ke = __ldg(rp + i + 1);
            for (int k = kb; k < ke; ++k) {
                const int c = __ldg(cols + k);
                double xv;
                if (c < n_local) {
                    xv = __ldg(x + c);
                } else {
                    const int g = c - n_local;
                    const int q = seg_of(ro, pd.P, g);
                    xv = peer_ll_read(pd.stage(pd.rank, par, q) + 2 * size_t(g - ro[q]),
                                      static_cast<unsigned>(e), me, 0, q, e);
                }
                s = add_rn(s, mul_rn(__ldg(vals + k), xv));
            }
            epi.row(row_map ? __ldg(row_map + i) : i + row_off, s, acc);
        }
    }
    // every ghost this block needed has been consumed: count out; the last
    // block hands the slots back and advances the halo epoch
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(&me->recv_cnt, 1u) == gridDim.x - 1) {
        me->recv_cnt = 0;
        // hand back epoch e to EVERY peer, not only those we received
        // from: the epoch counter is per communicator, so a peer that sent
        // us nothing this epoch (another matrix sharing the communicator,
        // with a different neighbour set) must still see it consumed
        // (A,B,B,A over one communicator deadlocked)
        for (int q = 0; q < pd.P; ++q)
            if (q != pd.rank) st_volatile_u64(&pd.win[q]->empty[pd.rank], e);
        *reinterpret_cast<volatile unsigned long long*>(&me->seq_x) = e;
    }
    if constexpr (Epi::NV > 0) {
        if (skip) return;
        grid_reduce<NV>(acc, ws, threadIdx.x, blockDim.x, red_sh,
                               [&](const double* tot) { epi.finish(tot); });
    }
}

template <class Epi>
void peer_boundary(lbk_ctx ctx, const lbk_dist_csr_s* D, const PeerDev& pd, const double* x,
                   const Epi& epi, RedWs ws)
{
    const SubCsr& S = D->boundary;
    launch_pdl(ctx, peer_boundary_kernel<Epi>, dim3(peer_grid(S.nrows)), dim3(256), 0, pd,
               S.nrows, S.row_ptr.as<int>(), S.cols.as<int>(), S.vals.as<double>(),
               S.row_off >= 0 ? nullptr : S.row_map.as<int>(), S.row_off >= 0 ? S.row_off : 0,
               D->n_local, D->recv_off_d.as<int>(), x, epi, ws);
    LBK_LAUNCH_CHECK();
}

// y = A x_ext with the halo exchange overlapped with the interior rows.
// `epi` reduces over interior rows into ws_a.out and boundary rows into
// ws_b.out when the RedWs are deferred (the solver path).
template <class Epi>
void dist_apply(lbk_ctx ctx, lbk_dist_csr_s* D, Comm* comm, double* x_ext, const Epi& epi,
                RedWs ws_a, RedWs ws_b)
{
    const bool xchg = comm && comm->nranks > 1;
    if (xchg && comm->peer()) {
        const PeerDev& pd = *comm->peer();
        peer_push(ctx, D, pd, x_ext);
        if (D->interior.nrows > 0) launch_sub(ctx, D->interior, x_ext, epi, ws_a);
        peer_boundary(ctx, D, pd, x_ext, epi, ws_b);  // always: it advances the epoch
        return;
    }
    if (xchg) {
        dist_pack(ctx, D, x_ext);
        if (comm->async()) {
            LBK_CUDA(cudaEventRecord(D->ev_pack, ctx->stream));
            LBK_CUDA(cudaStreamWaitEvent(D->comm_stream, D->ev_pack, 0));
            comm->exchange(D->send_buf.as<double>(), D->send_off, x_ext + D->n_local, D->recv_off,
                           D->comm_stream);
            LBK_CUDA(cudaEventRecord(D->ev_recv, D->comm_stream));
        } else {
            comm->exchange(D->send_buf.as<double>(), D->send_off, x_ext + D->n_local, D->recv_off,
                           ctx->stream);
        }
    }
    if (D->interior.nrows > 0) launch_sub(ctx, D->interior, x_ext, epi, ws_a);
    if (xchg && comm->async()) LBK_CUDA(cudaStreamWaitEvent(ctx->stream, D->ev_recv, 0));
    if (D->boundary.nrows > 0) launch_sub(ctx, D->boundary, x_ext, epi, ws_b);
}

}  // namespace lbk
