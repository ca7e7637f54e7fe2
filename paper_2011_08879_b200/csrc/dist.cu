// dist.cu -- row-partitioned distributed CSR: partition/halo maps (host,
// bit-exact with the App. B restatement in oracle/port.cpp), the two
// communicator back ends, device setup and the overlapped SpMV entry point.
// See dist.cuh for the layout.
#include <dlfcn.h>

#include <algorithm>
#include <barrier>
#include <chrono>
#include <thread>
#include <cstring>
#include <memory>
#include <mutex>

#include "api_guard.h"
#include "dist.cuh"

namespace lbk {
namespace {

void part_range(int n, int P, int rank, int* b, int* e)
{
    const long long chunk = (static_cast<long long>(n) + P - 1) / P;
    long long lo = std::min<long long>(static_cast<long long>(rank) * chunk, n);
    long long hi = rank == P - 1 ? n : std::min<long long>((rank + 1) * chunk, n);
    *b = static_cast<int>(lo);
    *e = static_cast<int>(hi);
}

// NCCL is resolved at run time (dlopen), not linked: inside a PyTorch
// process the already-loaded libnccl.so.2 (torch's bundled build) is reused,
// so the library never drags a second, older NCCL into the process; a pure
// C/C++ caller gets the system one.  Only the stable core API is used.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclCommGetAsyncError) GetAsyncError = nullptr;
    decltype(&ncclCommAbort) CommAbort = nullptr;
};

const NcclApi& nccl()
{
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
        a.Send = reinterpret_cast<decltype(a.Send)>(dlsym(h, "ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(dlsym(h, "ncclRecv"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
        a.GetErrorString =
            reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.GetAsyncError =
            reinterpret_cast<decltype(a.GetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
        a.CommAbort = reinterpret_cast<decltype(a.CommAbort)>(dlsym(h, "ncclCommAbort"));
        return a;
    }();
    need(api.GetUniqueId && api.CommInitRank && api.AllReduce && api.Send && api.Recv &&
             api.GroupStart && api.GroupEnd && api.GetErrorString && api.CommDestroy,
         LBK_NCCL_ERROR, "NCCL (libnccl.so.2) could not be loaded");
    return api;
}

#define LBK_NCCL(call)                                                                     \
    do {                                                                                   \
        ncclResult_t r_ = (call);                                                          \
        if (r_ != ncclSuccess)                                                             \
            ::lbk::fail(LBK_NCCL_ERROR,                                                    \
                        std::string(#call ": ") + ::lbk::nccl().GetErrorString(r_));       \
    } while (0)

// ------------------------------------------------------------ NCCL
// One process per GPU (torchrun); the unique id travels over the caller's
// bootstrap (torch.distributed broadcast).  Halo exchange = grouped
// ncclSend/ncclRecv on the comm stream; dots = ncclAllReduce(sum).
struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    ~NcclComm() override
    {
        if (comm) nccl().CommDestroy(comm);
    }
    void allreduce_sum(double* dev, int count, cudaStream_t s) override
    {
        LBK_NCCL(nccl().AllReduce(dev, dev, count, ncclDouble, ncclSum, comm, s));
    }
    void allreduce_i64(long long* dev, int count, cudaStream_t s) override
    {
        LBK_NCCL(nccl().AllReduce(dev, dev, count, ncclInt64, ncclSum, comm, s));
    }
    void exchange(const double* send_buf, const std::vector<int>& so, double* recv,
                  const std::vector<int>& ro, cudaStream_t s) override
    {
        const NcclApi& N = nccl();
        LBK_NCCL(N.GroupStart());
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            const int ns = so[q + 1] - so[q], nr = ro[q + 1] - ro[q];
            if (ns > 0) LBK_NCCL(N.Send(send_buf + so[q], ns, ncclDouble, q, comm, s));
            if (nr > 0) LBK_NCCL(N.Recv(recv + ro[q], nr, ncclDouble, q, comm, s));
        }
        LBK_NCCL(N.GroupEnd());
    }
    bool async() const override { return true; }
    // Poll instead of blocking: a failed peer surfaces as an NCCL async
    // error (or, past LBK_NCCL_TIMEOUT seconds, default 600, as a timeout);
    // the communicator is then aborted so the call returns instead of
    // hanging in the collective.
    void wait(cudaStream_t s) override
    {
        static const double limit = [] {
            const char* e = std::getenv("LBK_NCCL_TIMEOUT");
            return e ? std::atof(e) : 600.0;
        }();
        const auto t0 = std::chrono::steady_clock::now();
        for (int spin = 0;; ++spin) {
            const cudaError_t q = cudaStreamQuery(s);
            if (q == cudaSuccess) return;
            if (q != cudaErrorNotReady) LBK_CUDA(q);
            ncclResult_t ae = ncclSuccess;
            if (nccl().GetAsyncError) nccl().GetAsyncError(comm, &ae);
            const double el =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if ((ae != ncclSuccess && ae != ncclInProgress) || el > limit) {
                if (nccl().CommAbort) nccl().CommAbort(comm);
                comm = nullptr;
                fail(LBK_NCCL_ERROR, ae != ncclSuccess
                                         ? std::string("NCCL async error: ") +
                                               nccl().GetErrorString(ae)
                                         : "NCCL wait timed out (LBK_NCCL_TIMEOUT)");
            }
            if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
    }
};

// ------------------------------------------------------------ threads
// In-process SPMD group: P host threads, each driving its own lbk_ctx (on
// the same or on different devices), meet at host barriers.  Used for
// P virtual ranks on one GPU (the partition / halo / reduction logic runs
// exactly as with NCCL) and for single-process multi-GPU runs.  Allreduce
// sums the per-rank values on the host (exact int64 limbs for the solver's
// reductions, allreduce_i64; doubles in rank order for the public
// allreduce_sum), so every rank gets the same bits; exchanges are
// device-to-device copies from the peers' send buffers.
struct ThreadShared {
    int P;
    std::barrier<> bar;
    std::vector<double> slots[2];
    std::vector<long long> islots[2];
    std::vector<const double*> send_bufs;
    std::vector<const std::vector<int>*> send_offs;
    explicit ThreadShared(int p) : P(p), bar(p), send_bufs(p), send_offs(p)
    {
        slots[0].resize(size_t(p) * 32);
        slots[1].resize(size_t(p) * 32);
        islots[0].resize(size_t(p) * kXSlot);
        islots[1].resize(size_t(p) * kXSlot);
    }
};

struct ThreadComm final : Comm {
    std::shared_ptr<ThreadShared> sh;
    int parity = 0;
    void allreduce_sum(double* dev, int count, cudaStream_t s) override
    {
        need(count <= 32, LBK_USAGE_ERROR, "thread allreduce: at most 32 values");
        auto& slot = sh->slots[parity];
        parity ^= 1;
        LBK_CUDA(cudaMemcpyAsync(slot.data() + size_t(rank) * 32, dev, count * sizeof(double),
                                 cudaMemcpyDeviceToHost, s));
        LBK_CUDA(cudaStreamSynchronize(s));
        sh->bar.arrive_and_wait();
        double tot[32];
        for (int i = 0; i < count; ++i) tot[i] = 0.0;
        for (int q = 0; q < nranks; ++q)
            for (int i = 0; i < count; ++i) tot[i] += slot[size_t(q) * 32 + i];
        LBK_CUDA(cudaMemcpyAsync(dev, tot, count * sizeof(double), cudaMemcpyHostToDevice, s));
        LBK_CUDA(cudaStreamSynchronize(s));
    }
    void allreduce_i64(long long* dev, int count, cudaStream_t s) override
    {
        need(count <= kXSlot, LBK_USAGE_ERROR, "thread allreduce: too many limbs");
        auto& slot = sh->islots[parity];
        parity ^= 1;
        LBK_CUDA(cudaMemcpyAsync(slot.data() + size_t(rank) * kXSlot, dev,
                                 count * sizeof(long long), cudaMemcpyDeviceToHost, s));
        LBK_CUDA(cudaStreamSynchronize(s));
        sh->bar.arrive_and_wait();
        long long tot[kXSlot];
        for (int i = 0; i < count; ++i) tot[i] = 0;
        for (int q = 0; q < nranks; ++q)
            for (int i = 0; i < count; ++i) tot[i] += slot[size_t(q) * kXSlot + i];
        LBK_CUDA(cudaMemcpyAsync(dev, tot, count * sizeof(long long), cudaMemcpyHostToDevice, s));
        LBK_CUDA(cudaStreamSynchronize(s));
    }
    void exchange(const double* send_buf, const std::vector<int>& so, double* recv,
                  const std::vector<int>& ro, cudaStream_t s) override
    {
        LBK_CUDA(cudaStreamSynchronize(s));  // pack finished
        sh->send_bufs[rank] = send_buf;
        sh->send_offs[rank] = &so;
        sh->bar.arrive_and_wait();
        for (int q = 0; q < nranks; ++q) {
            const int nr = ro[q + 1] - ro[q];
            if (q == rank || nr == 0) continue;
            const auto& pso = *sh->send_offs[q];
            need(pso[rank + 1] - pso[rank] == nr, LBK_INTERNAL,
                 "halo exchange: send/recv counts disagree");
            LBK_CUDA(cudaMemcpyAsync(recv + ro[q], sh->send_bufs[q] + pso[rank],
                                     size_t(nr) * sizeof(double), cudaMemcpyDefault, s));
        }
        LBK_CUDA(cudaStreamSynchronize(s));
        sh->bar.arrive_and_wait();  // peers may reuse their send buffers
    }
    bool async() const override { return false; }
};

// ------------------------------------------------ peer-memory group
// See peer.cuh for the protocol.
struct PeerComm final : Comm {
    int device = 0;
    PeerHdr* local = nullptr;       // this rank's window (owned)
    std::vector<void*> opened;      // IPC-mapped peer windows (closed on destroy)
    PeerDev pd{};
    bool ready = false;
    int* err_host = nullptr;  // pinned
    ~PeerComm() override
    {
        for (void* p : opened) cudaIpcCloseMemHandle(p);
        if (local) cudaFree(local);
        if (err_host) cudaFreeHost(err_host);
    }
    const PeerDev* peer() const override
    {
        need(ready, LBK_USAGE_ERROR, "peer communicator: peers not opened yet");
        return &pd;
    }
    void set_ready() { ready = true; }
    void allreduce_sum(double* dev, int count, cudaStream_t s) override;
    void allreduce_i64(long long*, int, cudaStream_t) override
    {
        fail(LBK_INTERNAL, "peer communicator: exact reductions run in the finish kernels");
    }
    void exchange(const double*, const std::vector<int>&, double*, const std::vector<int>&,
                  cudaStream_t) override
    {
        fail(LBK_INTERNAL, "peer communicator: halo runs in the pack/receive kernels");
    }
    bool async() const override { return true; }
    void wait(cudaStream_t s) override
    {
        // stream-ordered read of the error word: a legacy-stream copy could
        // wait on a peer's stream that is itself waiting for this rank
        LBK_CUDA(cudaMemcpyAsync(err_host, &local->error, sizeof(int), cudaMemcpyDeviceToHost, s));
        LBK_CUDA(cudaStreamSynchronize(s));
        if (*err_host == 0) return;
        long long info[4] = {0, 0, 0, 0};
        cudaMemcpy(info, local->err_info, sizeof(info), cudaMemcpyDeviceToHost);
        static const char* what[] = {"halo values", "halo slot hand-back", "reduction totals"};
        fail(LBK_NCCL_ERROR, "peer communicator: rank " + std::to_string(rank) +
                                 " timed out waiting for " + what[info[0] % 3] + " of rank " +
                                 std::to_string(info[1]) + " (epoch " + std::to_string(info[2]) +
                                 ", seen " + std::to_string(info[3]) +
                                 "; LBK_PEER_TIMEOUT); the group is unusable");
    }
    void create(int P, int r, int dev, long long cap)
    {
        need(P >= 1 && P <= kPeerMax, LBK_USAGE_ERROR,
             "peer communicator: at most " + std::to_string(kPeerMax) + " ranks");
        need(r >= 0 && r < P && cap >= 0, LBK_USAGE_ERROR, "peer communicator: bad rank/cap");
        nranks = P;
        rank = r;
        device = dev;
        LBK_CUDA(cudaSetDevice(dev));
        const size_t bytes = kPeerHdrBytes + size_t(2) * P * size_t(cap) * 2 * sizeof(double);
        LBK_CUDA(cudaMallocHost(&err_host, sizeof(int)));
        *err_host = 0;
        LBK_CUDA(cudaMalloc(&local, bytes));
        LBK_CUDA(cudaMemset(local, 0, bytes));
        PeerHdr h{};
        const char* e = std::getenv("LBK_PEER_TIMEOUT");
        h.timeout_ns = static_cast<long long>((e ? std::atof(e) : 300.0) * 1e9);
        h.cap = cap;
        LBK_CUDA(cudaMemcpy(local, &h, sizeof(h), cudaMemcpyHostToDevice));
        pd.P = P;
        pd.rank = r;
        pd.cap = cap;
        const char* xd = std::getenv("LBK_XRED_DIGITS");
        pd.xdigits = (xd && xd[0] == '1') ? 1 : 0;
        pd.win[r] = local;
    }
    // every window must use the same slot capacity (senders index the
    // receiver's staging area with their own cap)
    void verify_caps() const
    {
        for (int q = 0; q < nranks; ++q) {
            long long c = -1;
            LBK_CUDA(cudaMemcpy(&c, &pd.win[q]->cap, sizeof(c), cudaMemcpyDefault));
            need(c == pd.cap, LBK_USAGE_ERROR,
                 "peer communicator: ranks disagree on the halo capacity");
        }
    }
};

__global__ void peer_allreduce_kernel(PeerDev pd, double* dev, int count)
{
    pdl_enter();
    const int lane = threadIdx.x;
    const double v = lane < count ? dev[lane] : 0.0;
    const double t = peer_allreduce_warp(pd, v, count > 0 ? count : 1);
    if (lane < count) dev[lane] = t;
}

void PeerComm::allreduce_sum(double* dev, int count, cudaStream_t s)
{
    need(count >= 0 && count <= kPeerRedMax, LBK_USAGE_ERROR,
         "peer allreduce: at most " + std::to_string(kPeerRedMax) + " values");
    need(ready, LBK_USAGE_ERROR, "peer communicator: peers not opened yet");
    peer_allreduce_kernel<<<1, 32, 0, s>>>(pd, dev, count);
    LBK_LAUNCH_CHECK();
}

// gather x[send_idx] and store each peer's run, LL-tagged with the halo
// epoch, into its staging slot (parity e & 1, source = this rank) -- once
// the receiver has handed back the slot's previous epoch
__global__ void peer_push_kernel(PeerDev pd, const int* __restrict__ send_off,
                                 const int* __restrict__ send_idx, const double* __restrict__ x)
{
    pdl_enter();
    __shared__ int so[kPeerMax + 1];
    PeerHdr* me = pd.win[pd.rank];
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&me->seq_x) + 1;
    const int par = static_cast<int>(e & 1);
    const unsigned long long tag = (e & 0xffffffffull) << 32;
    if (threadIdx.x <= pd.P) so[threadIdx.x] = send_off[threadIdx.x];
    __syncthreads();
    const int q0 = threadIdx.x;
    if (q0 < pd.P && so[q0 + 1] > so[q0] && e > 2) peer_wait_ge(&me->empty[q0], e - 2, me, 1, q0);
    __syncthreads();
    const int ns = so[pd.P];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
        const int q = seg_of(so, pd.P, i);
        peer_ll_store(pd.stage(q, par, pd.rank) + 2 * size_t(i - so[q]), x[__ldg(send_idx + i)],
                      tag);
    }
}


__global__ void pack_kernel(int n, const int* __restrict__ idx, const double* __restrict__ x,
                            double* __restrict__ out)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        out[i] = x[__ldg(idx + i)];
}

lbk_dist_map_s* map_of(lbk_dist_map m)
{
    need(m != nullptr, LBK_USAGE_ERROR, "null distributed map");
    return m;
}

// Builds one row-subset sub-matrix (rows `rows`, columns already local).
void build_sub(lbk_ctx ctx, SubCsr& S, const std::vector<int>& rows, const int32_t* row_ptr,
               const std::vector<int>& lcols, const double* vals, int ncols)
{
    std::vector<int> rp(rows.size() + 1, 0), cols;
    std::vector<double> v;
    for (size_t i = 0; i < rows.size(); ++i) {
        const int r = rows[i];
        for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            cols.push_back(lcols[k]);
            v.push_back(vals[k]);
        }
        rp[i + 1] = static_cast<int>(cols.size());
    }
    S.nrows = static_cast<int>(rows.size());
    S.row_off = rows.empty() ? 0 : rows.front();
    for (size_t i = 1; i < rows.size() && S.row_off >= 0; ++i)
        if (rows[i] != rows[i - 1] + 1) S.row_off = -1;
    S.ncols = ncols;
    S.nnz = static_cast<long long>(cols.size());
    S.row_ptr.alloc(rp.size() * 4);
    S.cols.alloc(cols.size() * 4);
    S.vals.alloc(v.size() * 8);
    S.row_map.alloc(rows.size() * 4);
    LBK_CUDA(cudaMemcpy(S.row_ptr.p, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice));
    if (!cols.empty()) {
        LBK_CUDA(cudaMemcpy(S.cols.p, cols.data(), cols.size() * 4, cudaMemcpyHostToDevice));
        LBK_CUDA(cudaMemcpy(S.vals.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    }
    if (!rows.empty())
        LBK_CUDA(cudaMemcpy(S.row_map.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    if (S.nrows > 0) {
        S.ntiles = csr_ntiles(S.nnz, S.nrows);
        S.plan.alloc(size_t(S.ntiles + 1) * 4);
        csr_plan_launch(ctx, S.row_ptr.as<int>(), S.nrows, S.nnz, S.plan.as<int>());
    }
}

}  // namespace

void dist_pack(lbk_ctx ctx, const lbk_dist_csr_s* D, const double* x)
{
    const int n = D->send_off.back();
    if (n == 0) return;
    pack_kernel<<<ceil_div(n, 256) < 1184 ? ceil_div(n, 256) : 1184, 256, 0, ctx->stream>>>(
        n, D->send_idx.as<int>(), x, D->send_buf.as<double>());
    LBK_LAUNCH_CHECK();
}

void peer_push(lbk_ctx ctx, const lbk_dist_csr_s* D, const PeerDev& pd, const double* x)
{
    need(pd.P == D->P && pd.rank == D->rank, LBK_USAGE_ERROR,
         "dist spmv: communicator does not match the partition");
    for (int q = 0; q < D->P; ++q)
        need(D->send_off[q + 1] - D->send_off[q] <= pd.cap &&
                 D->recv_off[q + 1] - D->recv_off[q] <= pd.cap,
             LBK_USAGE_ERROR, "peer communicator: halo capacity too small for this matrix");
    launch_pdl(ctx, peer_push_kernel, dim3(peer_grid(D->send_off.back())), dim3(256), 0, pd,
               D->send_off_d.as<int>(), D->send_idx.as<int>(), x);
    LBK_LAUNCH_CHECK();
}


}  // namespace lbk

using namespace lbk;

extern "C" {

lbk_status lbk_part_range(int32_t n, int32_t nparts, int32_t rank, int32_t* begin, int32_t* end)
{
    if (!begin || !end || n < 0 || nparts < 1 || rank < 0 || rank >= nparts)
        return LBK_USAGE_ERROR;
    part_range(n, nparts, rank, begin, end);
    return LBK_OK;
}

lbk_status lbk_dist_map_create(int32_t n_global, int32_t ncols_global, int32_t nparts,
                               int32_t rank, int32_t n_local, const int32_t* row_ptr,
                               const int32_t* cols, lbk_dist_map* out)
{
    if (!out) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        need(nparts >= 1 && rank >= 0 && rank < nparts, LBK_USAGE_ERROR,
             "dist map: rank outside [0, nparts)");
        need(n_global == ncols_global, LBK_SHAPE_ERROR,
             "dist map: the row partition is applied to x, so the matrix must be square");
        auto m = std::make_unique<lbk_dist_map_s>();
        m->n_global = n_global;
        m->ncols_global = ncols_global;
        m->P = nparts;
        m->rank = rank;
        part_range(n_global, nparts, rank, &m->begin, &m->end);
        m->n_local = m->end - m->begin;
        need(n_local == m->n_local, LBK_SHAPE_ERROR,
             "dist map: n_local " + std::to_string(n_local) + " != partition size " +
                 std::to_string(m->n_local));
        need(row_ptr != nullptr && row_ptr[0] == 0, LBK_FORMAT_ERROR,
             "dist map: local row_ptr must start at 0");
        const long long nnz = row_ptr[n_local];
        m->nnz_local = nnz;
        const int b = m->begin, e = m->end;
        for (long long k = 0; k < nnz; ++k) {
            const int c = cols[k];
            need(c >= 0 && c < ncols_global, LBK_FORMAT_ERROR, "dist map: column out of range");
            if (c < b || c >= e) m->ghosts.push_back(c);
        }
        std::sort(m->ghosts.begin(), m->ghosts.end());
        m->ghosts.erase(std::unique(m->ghosts.begin(), m->ghosts.end()), m->ghosts.end());
        m->ghost_off.assign(nparts + 1, 0);
        {
            size_t g = 0;
            for (int q = 0; q < nparts; ++q) {
                int qb, qe;
                part_range(n_global, nparts, q, &qb, &qe);
                m->ghost_off[q] = static_cast<int>(g);
                while (g < m->ghosts.size() && m->ghosts[g] < qe) ++g;
            }
            m->ghost_off[nparts] = static_cast<int>(m->ghosts.size());
        }
        m->local_cols.resize(static_cast<size_t>(nnz));
        for (int r = 0; r < n_local; ++r) {
            bool ghost = false;
            for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
                const int c = cols[k];
                if (c >= b && c < e) {
                    m->local_cols[k] = c - b;
                } else {
                    ghost = true;
                    m->local_cols[k] =
                        n_local + static_cast<int>(std::lower_bound(m->ghosts.begin(), m->ghosts.end(), c) -
                                                   m->ghosts.begin());
                }
            }
            (ghost ? m->boundary : m->interior).push_back(r);
        }
        *out = m.release();
    });
}

lbk_status lbk_dist_map_info(lbk_dist_map m, lbk_dist_map_info_t* info)
{
    if (!m || !info) return LBK_USAGE_ERROR;
    info->begin = m->begin;
    info->end = m->end;
    info->n_local = m->n_local;
    info->n_ghost = static_cast<int32_t>(m->ghosts.size());
    info->n_interior = static_cast<int32_t>(m->interior.size());
    info->n_boundary = static_cast<int32_t>(m->boundary.size());
    info->nnz_local = m->nnz_local;
    info->n_send = m->sends_set ? m->send_off.back() : -1;
    return LBK_OK;
}

lbk_status lbk_dist_map_ghosts(lbk_dist_map m, int32_t* ghosts, int32_t* ghost_off)
{
    if (!m) return LBK_USAGE_ERROR;
    if (ghosts && !m->ghosts.empty())
        std::memcpy(ghosts, m->ghosts.data(), m->ghosts.size() * 4);
    if (ghost_off) std::memcpy(ghost_off, m->ghost_off.data(), m->ghost_off.size() * 4);
    return LBK_OK;
}

lbk_status lbk_dist_map_local_cols(lbk_dist_map m, int32_t* local_cols)
{
    if (!m || !local_cols) return LBK_USAGE_ERROR;
    if (!m->local_cols.empty())
        std::memcpy(local_cols, m->local_cols.data(), m->local_cols.size() * 4);
    return LBK_OK;
}

lbk_status lbk_dist_map_rows(lbk_dist_map m, int32_t* interior, int32_t* boundary)
{
    if (!m) return LBK_USAGE_ERROR;
    if (interior && !m->interior.empty())
        std::memcpy(interior, m->interior.data(), m->interior.size() * 4);
    if (boundary && !m->boundary.empty())
        std::memcpy(boundary, m->boundary.data(), m->boundary.size() * 4);
    return LBK_OK;
}

lbk_status lbk_dist_map_set_sends(lbk_dist_map m, const int32_t* req_off, const int32_t* req_gids)
{
    if (!m || !req_off) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        need(req_off[0] == 0, LBK_FORMAT_ERROR, "send requests: offsets must start at 0");
        m->send_off.assign(req_off, req_off + m->P + 1);
        m->send_idx.resize(static_cast<size_t>(req_off[m->P]));
        for (int q = 0; q < m->P; ++q) {
            need(req_off[q + 1] >= req_off[q], LBK_FORMAT_ERROR, "send requests: offsets decrease");
            need(q != m->rank || req_off[q + 1] == req_off[q], LBK_FORMAT_ERROR,
                 "send requests: a rank cannot request from itself");
            for (int i = req_off[q]; i < req_off[q + 1]; ++i) {
                const int g = req_gids[i];
                need(g >= m->begin && g < m->end, LBK_FORMAT_ERROR,
                     "send requests: global id " + std::to_string(g) + " not owned by rank " +
                         std::to_string(m->rank));
                need(i == req_off[q] || req_gids[i - 1] < g, LBK_FORMAT_ERROR,
                     "send requests: ids must be strictly increasing per peer");
                m->send_idx[i] = g - m->begin;
            }
        }
        m->sends_set = true;
    });
}

lbk_status lbk_dist_map_sends(lbk_dist_map m, int32_t* send_off, int32_t* send_idx)
{
    if (!m || !m->sends_set) return LBK_USAGE_ERROR;
    if (send_off) std::memcpy(send_off, m->send_off.data(), m->send_off.size() * 4);
    if (send_idx && !m->send_idx.empty())
        std::memcpy(send_idx, m->send_idx.data(), m->send_idx.size() * 4);
    return LBK_OK;
}

lbk_status lbk_dist_map_destroy(lbk_dist_map m)
{
    delete m;
    return LBK_OK;
}

// ------------------------------------------------------------ comms
lbk_status lbk_comm_nccl_unique_id(void* id_out)
{
    if (!id_out) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        ncclUniqueId id;
        LBK_NCCL(nccl().GetUniqueId(&id));
        std::memcpy(id_out, &id, sizeof(id));
    });
}

lbk_status lbk_comm_init_nccl(const void* id, int32_t nranks, int32_t rank, int32_t device,
                              lbk_comm* out)
{
    if (!id || !out) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        LBK_CUDA(cudaSetDevice(device));
        auto c = std::make_unique<NcclComm>();
        c->nranks = nranks;
        c->rank = rank;
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof(uid));
        LBK_NCCL(nccl().CommInitRank(&c->comm, nranks, uid, rank));
        auto h = std::make_unique<lbk_comm_s>();
        h->impl = c.release();
        *out = h.release();
    });
}

lbk_status lbk_comm_init_threads(int32_t nranks, lbk_comm* comms_out)
{
    if (!comms_out || nranks < 1) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        auto sh = std::make_shared<ThreadShared>(nranks);
        for (int r = 0; r < nranks; ++r) {
            auto c = std::make_unique<ThreadComm>();
            c->nranks = nranks;
            c->rank = r;
            c->sh = sh;
            auto h = std::make_unique<lbk_comm_s>();
            h->impl = c.release();
            comms_out[r] = h.release();
        }
    });
}

lbk_status lbk_comm_init_peer(int32_t nranks, int32_t rank, int32_t device, int64_t halo_cap,
                              lbk_comm* out)
{
    if (!out) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        auto c = std::make_unique<PeerComm>();
        c->create(nranks, rank, device, halo_cap);
        if (nranks == 1) c->set_ready();
        auto h = std::make_unique<lbk_comm_s>();
        h->impl = c.release();
        *out = h.release();
    });
}

lbk_status lbk_comm_peer_handle(lbk_comm comm, void* handle_out)
{
    if (!comm || !handle_out) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        auto* c = dynamic_cast<PeerComm*>(comm->impl);
        need(c != nullptr, LBK_USAGE_ERROR, "not a peer communicator");
        LBK_CUDA(cudaSetDevice(c->device));
        cudaIpcMemHandle_t h;
        LBK_CUDA(cudaIpcGetMemHandle(&h, c->local));
        std::memcpy(handle_out, &h, sizeof(h));
    });
}

lbk_status lbk_comm_peer_open(lbk_comm comm, const void* handles)
{
    if (!comm || !handles) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        auto* c = dynamic_cast<PeerComm*>(comm->impl);
        need(c != nullptr, LBK_USAGE_ERROR, "not a peer communicator");
        need(!c->ready || c->nranks == 1, LBK_USAGE_ERROR, "peer communicator already open");
        LBK_CUDA(cudaSetDevice(c->device));
        const auto* hs = static_cast<const cudaIpcMemHandle_t*>(handles);
        for (int q = 0; q < c->nranks; ++q) {
            if (q == c->rank) continue;
            void* p = nullptr;
            LBK_CUDA(cudaIpcOpenMemHandle(&p, hs[q], cudaIpcMemLazyEnablePeerAccess));
            c->opened.push_back(p);
            c->pd.win[q] = static_cast<PeerHdr*>(p);
        }
        c->verify_caps();
        c->set_ready();
    });
}

lbk_status lbk_comm_init_peer_group(int32_t nranks, const int32_t* devices, int64_t halo_cap,
                                    lbk_comm* comms_out)
{
    if (!comms_out || !devices || nranks < 1) return LBK_USAGE_ERROR;
    return guard(nullptr, [&] {
        // one context per rank: ranks sharing a device (and so a context)
        // could deadlock -- a kernel spinning on a peer's flag blocks any
        // device-synchronising call (cudaFree, lazy module load, ...) the
        // peer's host thread makes before it posts
        for (int r = 0; r < nranks; ++r)
            for (int q = 0; q < r; ++q)
                need(devices[r] != devices[q], LBK_USAGE_ERROR,
                     "peer group: one device per rank (use one process per rank to fold "
                     "several ranks onto one GPU)");
        std::vector<std::unique_ptr<PeerComm>> cs;
        for (int r = 0; r < nranks; ++r) {
            cs.push_back(std::make_unique<PeerComm>());
            cs.back()->create(nranks, r, devices[r], halo_cap);
        }
        for (int r = 0; r < nranks; ++r)
            for (int q = 0; q < nranks; ++q) {
                cs[r]->pd.win[q] = cs[q]->local;
                if (devices[r] != devices[q]) {
                    int ok = 0;
                    LBK_CUDA(cudaDeviceCanAccessPeer(&ok, devices[r], devices[q]));
                    need(ok, LBK_USAGE_ERROR, "peer group: devices without peer access");
                    LBK_CUDA(cudaSetDevice(devices[r]));
                    const cudaError_t e = cudaDeviceEnablePeerAccess(devices[q], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else LBK_CUDA(e);
                }
            }
        for (int r = 0; r < nranks; ++r) {
            cs[r]->set_ready();
            auto h = std::make_unique<lbk_comm_s>();
            h->impl = cs[r].release();
            comms_out[r] = h.release();
        }
    });
}

lbk_status lbk_comm_sync(lbk_ctx ctx, lbk_comm comm)
{
    if (!ctx) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        if (comm) comm->impl->wait(ctx->stream);
        else LBK_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

lbk_status lbk_comm_destroy(lbk_comm c)
{
    if (c) {
        delete c->impl;
        delete c;
    }
    return LBK_OK;
}

lbk_status lbk_comm_allreduce_sum_f64(lbk_ctx ctx, lbk_comm comm, double* dev, int32_t count)
{
    if (!ctx || !comm) return LBK_USAGE_ERROR;
    return guard(ctx, [&] { comm->impl->allreduce_sum(dev, count, ctx->stream); });
}

// ------------------------------------------------------------ matrix
lbk_status lbk_dist_csr_create(lbk_ctx ctx, lbk_dist_map m, const int32_t* row_ptr,
                               const double* vals, int64_t n_global_nnz, lbk_dist_csr* out)
{
    if (!ctx || !out) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        map_of(m);
        need(m->sends_set, LBK_USAGE_ERROR,
             "dist csr: call lbk_dist_map_set_sends (ghost-list all-to-all) first");
        need(row_ptr != nullptr && row_ptr[m->n_local] == m->nnz_local, LBK_FORMAT_ERROR,
             "dist csr: row_ptr does not match the map");
        auto D = std::make_unique<lbk_dist_csr_s>();
        D->n_local = m->n_local;
        D->n_ghost = static_cast<int>(m->ghosts.size());
        D->P = m->P;
        D->rank = m->rank;
        D->nnz_local = m->nnz_local;
        D->n_global = m->n_global;
        D->nnz_global = n_global_nnz;
        D->device = ctx->device;
        const int next = m->n_local + D->n_ghost;
        build_sub(ctx, D->interior, m->interior, row_ptr, m->local_cols, vals, m->n_local);
        build_sub(ctx, D->boundary, m->boundary, row_ptr, m->local_cols, vals, next);
        D->send_off = m->send_off;
        D->recv_off = m->ghost_off;
        const size_t ns = m->send_idx.size();
        D->send_idx.alloc(ns * 4);
        D->send_buf.alloc(ns * 8);
        if (ns)
            LBK_CUDA(cudaMemcpy(D->send_idx.p, m->send_idx.data(), ns * 4, cudaMemcpyHostToDevice));
        D->send_off_d.alloc(size_t(D->P + 1) * 4);
        D->recv_off_d.alloc(size_t(D->P + 1) * 4);
        LBK_CUDA(cudaMemcpy(D->send_off_d.p, D->send_off.data(), size_t(D->P + 1) * 4,
                            cudaMemcpyHostToDevice));
        LBK_CUDA(cudaMemcpy(D->recv_off_d.p, D->recv_off.data(), size_t(D->P + 1) * 4,
                            cudaMemcpyHostToDevice));
        LBK_CUDA(cudaStreamCreateWithFlags(&D->comm_stream, cudaStreamNonBlocking));
        LBK_CUDA(cudaEventCreateWithFlags(&D->ev_pack, cudaEventDisableTiming));
        LBK_CUDA(cudaEventCreateWithFlags(&D->ev_recv, cudaEventDisableTiming));
        LBK_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = D.release();
    });
}

lbk_status lbk_dist_csr_info(lbk_dist_csr D, int32_t* n_local, int32_t* n_ghost)
{
    if (!D) return LBK_USAGE_ERROR;
    if (n_local) *n_local = D->n_local;
    if (n_ghost) *n_ghost = D->n_ghost;
    return LBK_OK;
}

lbk_status lbk_dist_csr_destroy(lbk_dist_csr D)
{
    if (D) {
        cudaSetDevice(D->device);
        if (D->comm_stream) cudaStreamDestroy(D->comm_stream);
        if (D->ev_pack) cudaEventDestroy(D->ev_pack);
        if (D->ev_recv) cudaEventDestroy(D->ev_recv);
        delete D;
    }
    return LBK_OK;
}

lbk_status lbk_dist_spmv_f64(lbk_ctx ctx, lbk_dist_csr D, lbk_comm comm, double* x_ext, double* y)
{
    if (!ctx || !D) return LBK_USAGE_ERROR;
    NvtxRange nvtx_("lbk_dist_spmv_f64");
    return guard(ctx, [&] {
        need(D->P == 1 || (comm && comm->impl->nranks == D->P && comm->impl->rank == D->rank),
             LBK_USAGE_ERROR, "dist spmv: communicator does not match the partition");
        dist_apply(ctx, D, comm ? comm->impl : nullptr, x_ext, EpiStore<double>{y}, RedWs{},
                   RedWs{});
    });
}

}  // extern "C"
