// solver.cu -- device-resident, fused CG and BiCGSTAB.
//
// Reference: src/solver/krylov.cpp (paths relative to /root/reference/proj)
//   solve_impl      :446-512  validation, zero-b short-circuit, result
//   run_cg          :119-161  CG with true-residual stop every iteration
//   run_bicgstab    :164-230  BiCGSTAB, same stopping rule
//   Workspace       :36-88    flop accounting (apply 2nnz; dot/norm/axpy 2n;
//                             scal n) -- reproduced exactly
//   check_breakdown :91-97    |v| < 1e-30 -> BreakdownError(iteration)
//   machine_floor   :23       fixed-iteration freeze at rel <= 1e-13
//
// Every scalar of the recurrences lives in device memory (SolverState).
// Each fused kernel ends in a deterministic grid reduction whose last block
// ("finisher", one thread) advances the scalar recurrence, records the
// residual history, detects breakdown / convergence / freeze and raises
// `done`; every later kernel of the solve then exits immediately.  The host
// only launches chunks of iterations and polls `done` once per chunk, so
// there is no host round-trip per dot product (the reference synchronises
// on every dot, api.cpp:95-104).
//
// Per-iteration kernels (reference semantics, residual_mode 0):
//   CG        K1  q = A p            | <p,q>
//             K2  x += a p, r -= a q  | <r,r>
//             K3  t = b - A x         | <t,t>
//             P   p = beta p + r      (fused into K3 with -DLBK_FUSED_P)
//   CGS       S1  u, p updates (vec) S2 v = A p | <rt,v>   S3 q, w (vec)
//             S4  t = A w + x, r updates | <rt,r>    S5 true residual
//   BiCGSTAB  B2  v = A p            | <rt,v>
//             B3  s = r - a v         | <s,s>
//             B4  t = A s            | <t,t>, <t,s>
//             B5  x += a p + w s; r = s - w t | <rt,r>
//             B6  t = b - A x         | <t,t>
//             P   next p update       (fused into B6 with -DLBK_FUSED_P)
// residual_mode 1 (CG only) drops K3's SpMV: the stopping test uses the
// recurrence residual sqrt(<r,r>)/||b||, and a true residual is computed
// and must pass before convergence is declared.
#include <chrono>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "api_guard.h"
#include "dist.cuh"
#include "spmv_launch.cuh"

namespace lbk {

namespace {

constexpr double kBreakdownEps = 1e-30;  // krylov.cpp:18
constexpr double kMachineFloor = 1e-13;  // krylov.cpp:23
constexpr double kHappyEps = 1e-14;      // krylov.cpp:24

enum : int { ST_RUNNING = 0, ST_CONVERGED = 1, ST_LIMIT = 2, ST_BREAKDOWN = 3, ST_FROZEN = 4 };

struct SolverState {
    int done;
    int status;
    int iter;
    int breakdown_iter;
    int breakdown_what;  // 0 <p,Ap>, 1 rho, 2 omega, 3 <rt,Ap>, 4 <t,t>
    int hist_len;
    int limit;
    int fixed;
    int verify_pending;  // residual_mode 1: true residual requested
    int res_pending;     // peer two-exchange path: a deferred residual awaits
    double tol, norm_b;
    double rho, rho_next, alpha, beta, omega;
    double s_rel;
    double last_rel;
    long long n, nnz;
    long long flops;
    double* hist;
    struct GmresState* gm;  // GMRES only
};

// Restarted GMRES (krylov.cpp:308-443): the Hessenberg column, Givens
// rotations, rotated rhs and back-substitution are O(restart^2) scalars that
// the reference keeps on the host; here they live in device memory and are
// advanced by the finisher threads, so no host round trip per step.
struct GmresState {
    int restart;
    int steps;        // steps done in this cycle
    int cycle_done;
    int happy;
    int cycle_limit;  // min(restart, limit - iterations)
    int iterations;   // completed steps over all cycles
    double beta, hnext;
    double* H;        // (restart + 1) x restart, row-major [i * restart + j]
    double *gc, *gs, *g, *y;
};

__device__ __forceinline__ bool bd(double v) { return fabs(v) < kBreakdownEps; }

__device__ void push_hist(SolverState* st, double rel)
{
    st->hist[st->hist_len] = rel;
    st->hist_len += 1;
    st->last_rel = rel;
}

__device__ void raise_breakdown(SolverState* st, int what, int iter)
{
    st->status = ST_BREAKDOWN;
    st->breakdown_what = what;
    st->breakdown_iter = iter;
    st->done = 1;
}

// ---------------------------------------------------------- epilogues
// Initial residual r = b - A x (krylov.cpp:108-116: apply, scal(-1),
// axpy(1,b) == b - Ax exactly), copies to p (and rt), <r,r>.
struct EpiInit {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;  // <r,r>
    const double* __restrict__ b;
    double* __restrict__ r;
    double* __restrict__ p;
    double* __restrict__ rt;  // may be null
    SolverState* st;
    int bicg;                 // 1: BiCGSTAB / CGS preamble (iter = 1, rho = <rt,r>)
    double* __restrict__ u;   // CGS: u = r for iteration 1 (krylov.cpp:259-261), may be null
    struct Pre {
        double b;
    };
    __device__ bool skip() const { return false; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(b, rb, re);
    }
    __device__ Pre pre(int i) const { return {b[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        const double v = add_rn(pr.b, -s);
        r[i] = v;
        p[i] = v;
        if (rt) rt[i] = v;
        if (u) u[i] = v;
        racc_add(acc, 0, mul_rn(v, v));
    }
    __device__ void finish(const double* tot) const
    {
        const double rr = tot[0];
        const double rel = sqrt(rr) / st->norm_b;
        st->hist_len = 0;
        push_hist(st, rel);
        const long long n = st->n;
        st->flops += 2 * st->nnz + n + 2 * n + 2 * n;  // apply, scal, axpy, norm
        if (!st->fixed && rel <= st->tol) {
            st->status = ST_CONVERGED;
            st->done = 1;
            return;
        }
        if (!bicg) {
            st->rho = rr;  // rho = dot(r, r)
            st->flops += 2 * n;
        } else {
            // iteration 1 preamble (krylov.cpp:188, 198): rho = dot(rt, r)
            // with rt == r, so it equals <r,r> bit for bit; no p update.
            st->iter = 1;
            st->flops += 2 * n;
            st->rho = rr;
            st->alpha = 1.0;
            st->omega = 1.0;
        }
    }
};

// CG K1: q = A p, <p,q>
struct EpiCgK1 {
    static constexpr int NV = 1;
    double* __restrict__ q;
    const double* __restrict__ p;
    SolverState* st;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    struct Pre {
        double p;
    };
    __device__ Pre pre(int i) const { return {p[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        q[i] = s;
        racc_add(acc, 0, mul_rn(pr.p, s));
    }
    __device__ void finish(const double* tot) const
    {
        const int iter = st->iter + 1;
        st->iter = iter;
        const double pq = tot[0];
        st->flops += 2 * st->nnz + 2 * st->n;
        if (bd(pq)) {
            raise_breakdown(st, 0, iter);
            return;
        }
        st->alpha = st->rho / pq;
    }
};

// CG K3: true residual (+ fused p = beta p + r for the next iteration).
struct EpiCgK3 {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;  // ||t||^2
    const double* __restrict__ b;
    double* __restrict__ p;
    const double* __restrict__ r;
    SolverState* st;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(b, rb, re);
        l2_prefetch_rows(p, rb, re);
        l2_prefetch_rows(r, rb, re);
    }
    struct Pre {
        double b, p, r;
    };
    __device__ Pre pre(int i) const { return {b[i], p[i], r[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        const double t = add_rn(pr.b, -s);
        racc_add(acc, 0, mul_rn(t, t));
        const double beta = st->beta;
        p[i] = add_rn(mul_rn(pr.p, beta), pr.r);
    }
    __device__ void finish(const double* tot) const;
};

__device__ void cg_after_residual(SolverState* st, double rel)
{
    const long long n = st->n;
    push_hist(st, rel);
    if (!st->fixed && rel <= st->tol) {
        st->status = ST_CONVERGED;
        st->done = 1;
        return;
    }
    if (st->fixed && rel <= kMachineFloor) {
        st->status = ST_FROZEN;
        st->done = 1;
        return;
    }
    // rho_next = dot(r, r); check_breakdown(rho); beta; scal; axpy
    st->flops += 2 * n + n + 2 * n;
    if (bd(st->rho)) {
        raise_breakdown(st, 1, st->iter);
        return;
    }
    st->rho = st->rho_next;
    if (st->iter >= st->limit) {
        st->status = ST_LIMIT;
        st->done = 1;
    }
}

__device__ void EpiCgK3::finish(const double* tot) const
{
    st->flops += 2 * st->nnz + st->n + 2 * st->n + 2 * st->n;  // true_residual
    cg_after_residual(st, sqrt(tot[0]) / st->norm_b);
}

// K3 without the fused p update: the true residual alone, then p = beta p
// + r as its own vector pass (OpCgP).  The default on the unmerged paths:
// fusing the p update into the SpMV epilogue (EpiCgK3, -DLBK_FUSED_P) adds
// three operand streams to a latency-bound sweep; split, CG ran 1,115
// against 1,106 it/s (scripts/gpu_r2ao.sh, two repeats).
struct EpiCgK3s {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;  // ||t||^2
    const double* __restrict__ b;
    SolverState* st;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const { l2_prefetch_rows(b, rb, re); }
    struct Pre {
        double b;
    };
    __device__ Pre pre(int i) const { return {b[i]}; }
    __device__ void row(int i, double s, auto* acc) const
    {
        const double t = add_rn(b[i], -s);
        racc_add(acc, 0, mul_rn(t, t));
    }
    __device__ void row_pre(int, double s, const Pre& pr, auto* acc) const
    {
        const double t = add_rn(pr.b, -s);
        racc_add(acc, 0, mul_rn(t, t));
    }
    __device__ void finish(const double* tot) const;
};

__device__ void EpiCgK3s::finish(const double* tot) const
{
    st->flops += 2 * st->nnz + st->n + 2 * st->n + 2 * st->n;  // true_residual
    cg_after_residual(st, sqrt(tot[0]) / st->norm_b);
}

// residual_mode 1: stand-alone true residual check (no p update).
struct EpiTrueRes {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;
    const double* __restrict__ b;
    SolverState* st;
    struct Pre {
        double b;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0 || !st->verify_pending; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(b, rb, re);
    }
    __device__ Pre pre(int i) const { return {b[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int, double s, const Pre& pr, auto* acc) const
    {
        const double t = add_rn(pr.b, -s);
        racc_add(acc, 0, mul_rn(t, t));
    }
    __device__ void finish(const double* tot) const
    {
        st->flops += 2 * st->nnz + st->n + 2 * st->n + 2 * st->n;
        const double rel = sqrt(tot[0]) / st->norm_b;
        st->verify_pending = 0;
        // replace the recurrence estimate of this iteration by the truth
        st->hist[st->hist_len - 1] = rel;
        st->last_rel = rel;
        if (rel <= st->tol) {
            st->status = ST_CONVERGED;
            st->done = 1;
        } else if (st->iter >= st->limit) {
            st->status = ST_LIMIT;
            st->done = 1;
        } else {
            // verification failed: continue the recurrence (rho update that
            // OpCgK2 deferred)
            st->flops += 5 * st->n;
            if (bd(st->rho)) {
                raise_breakdown(st, 1, st->iter);
                return;
            }
            st->rho = st->rho_next;
        }
    }
};

// BiCGSTAB B2: v = A p, <rt,v>
struct EpiBiB2 {
    static constexpr int NV = 1;
    double* __restrict__ v;
    const double* __restrict__ rt;
    SolverState* st;
    struct Pre {
        double rt;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(rt, rb, re);
    }
    __device__ Pre pre(int i) const { return {rt[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        v[i] = s;
        racc_add(acc, 0, mul_rn(pr.rt, s));
    }
    __device__ void finish(const double* tot) const
    {
        st->flops += 2 * st->nnz + 2 * st->n;
        const double rtv = tot[0];
        if (bd(rtv)) {
            raise_breakdown(st, 3, st->iter);
            return;
        }
        st->alpha = st->rho / rtv;
    }
};

// BiCGSTAB B4: t = A s, <t,t>, <t,s>
struct EpiBiB4 {
    static constexpr int NV = 2;
    static constexpr unsigned kSq = 1;  // <t,t> (value 0); <t,s> signed
    double* __restrict__ t;
    const double* __restrict__ s;
    SolverState* st;
    struct Pre {
        double s;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(s, rb, re);
    }
    __device__ Pre pre(int i) const { return {s[i]}; }
    __device__ void row(int i, double sum, auto* acc) const { row_pre(i, sum, pre(i), acc); }
    __device__ void row_pre(int i, double sum, const Pre& pr, auto* acc) const
    {
        t[i] = sum;
        racc_add(acc, 0, mul_rn(sum, sum));
        racc_add(acc, 1, mul_rn(sum, pr.s));
    }
    __device__ void finish(const double* tot) const
    {
        st->flops += 2 * st->nnz + 2 * st->n;
        const double tt = tot[0];
        if (bd(tt)) {
            if (st->s_rel > kMachineFloor) {
                raise_breakdown(st, 4, st->iter);
                return;
            }
            st->omega = 0.0;  // exact half-step convergence
        } else {
            st->flops += 2 * st->n;
            st->omega = tot[1] / tt;
        }
    }
};

// BiCGSTAB B6: true residual + fused p = (p - w v) beta + r for iter+1.
struct EpiBiB6 {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;
    const double* __restrict__ b;
    double* __restrict__ p;
    const double* __restrict__ v;
    const double* __restrict__ r;
    SolverState* st;
    struct Pre {
        double b, p, v, r;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(b, rb, re);
        l2_prefetch_rows(p, rb, re);
        l2_prefetch_rows(v, rb, re);
        l2_prefetch_rows(r, rb, re);
    }
    __device__ Pre pre(int i) const { return {b[i], p[i], v[i], r[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        const double t = add_rn(pr.b, -s);
        racc_add(acc, 0, mul_rn(t, t));
        const double beta = st->beta, omega = st->omega;
        p[i] = add_rn(mul_rn(add_rn(pr.p, mul_rn(-omega, pr.v)), beta), pr.r);
    }
    __device__ void finish(const double* tot) const
    {
        const long long n = st->n;
        st->flops += 2 * st->nnz + n + 2 * n + 2 * n;
        const double rel = sqrt(tot[0]) / st->norm_b;
        push_hist(st, rel);
        if (!st->fixed && rel <= st->tol) {
            st->status = ST_CONVERGED;
            st->done = 1;
            return;
        }
        if (st->fixed && rel <= kMachineFloor) {
            st->status = ST_FROZEN;
            st->done = 1;
            return;
        }
        if (st->iter >= st->limit) {
            st->status = ST_LIMIT;
            st->done = 1;
            return;
        }
        // start of iteration iter+1 (krylov.cpp:188-198): dot(rt, r) was
        // reduced in B5; checks on rho and omega; p update (done in row()).
        const int next = st->iter + 1;
        st->iter = next;
        st->flops += 2 * n;
        if (bd(st->rho)) {
            raise_breakdown(st, 1, next);
            return;
        }
        if (bd(st->omega)) {
            raise_breakdown(st, 2, next);
            return;
        }
        st->flops += 2 * n + n + 2 * n;
        st->rho = st->rho_next;
    }
};

// B6 without the fused p update (the default; see EpiCgK3s): the true
// residual alone, then OpBiP.
struct EpiBiB6s {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;
    const double* __restrict__ b;
    SolverState* st;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const { l2_prefetch_rows(b, rb, re); }
    __device__ void row(int i, double s, auto* acc) const
    {
        const double t = add_rn(b[i], -s);
        racc_add(acc, 0, mul_rn(t, t));
    }
    __device__ void finish(const double* tot) const
    {
        EpiBiB6{b, nullptr, nullptr, nullptr, st}.finish(tot);
    }
};

// BiCGSTAB p = (p - omega v) beta + r (krylov.cpp:199-201), skipped once the
// solve is over
struct OpBiP {
    static constexpr int NV = 1;
    double* __restrict__ p;
    const double* __restrict__ v;
    const double* __restrict__ r;
    SolverState* st;
    double beta, omega;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prologue()
    {
        beta = st->beta;
        omega = st->omega;
    }
    struct In {
        double p, v, r;
    };
    __device__ In load(long long i) const { return {p[i], v[i], r[i]}; }
    __device__ void elem(long long i, const In& in, auto*) const
    {
        p[i] = add_rn(mul_rn(add_rn(in.p, mul_rn(-omega, in.v)), beta), in.r);
    }
    static constexpr bool kNoFinish = true;
    __device__ void finish(const double*) const {}
};

// CGS (krylov.cpp:233-297), reference semantics (true residual each
// iteration).  Per iteration: S1 u/p update (vec), S2 v = A p + <rt,v>,
// S3 q, w (vec), S4 t = A w fused with x += a w, r -= a t and <rt,r> (the
// next iteration's rho), S5 true residual.
struct EpiCgsV {
    static constexpr int NV = 1;
    double* __restrict__ v;
    const double* __restrict__ rt;
    SolverState* st;
    struct Pre {
        double rt;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(rt, rb, re);
    }
    __device__ Pre pre(int i) const { return {rt[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        v[i] = s;
        racc_add(acc, 0, mul_rn(pr.rt, s));
    }
    __device__ void finish(const double* tot) const
    {
        st->flops += 2 * st->nnz + 2 * st->n;  // apply + dot(rt, v)
        const double sigma = tot[0];
        if (bd(sigma)) {
            raise_breakdown(st, 3, st->iter);
            return;
        }
        st->alpha = st->rho / sigma;
    }
};

struct EpiCgsT {
    static constexpr int NV = 1;
    double* __restrict__ t;
    double* __restrict__ x;
    double* __restrict__ r;
    const double* __restrict__ w;
    const double* __restrict__ rt;
    SolverState* st;
    struct Pre {
        double x, r, w, rt;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(x, rb, re);
        l2_prefetch_rows(r, rb, re);
        l2_prefetch_rows(w, rb, re);
        l2_prefetch_rows(rt, rb, re);
    }
    __device__ Pre pre(int i) const { return {x[i], r[i], w[i], rt[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        const double a = st->alpha;
        t[i] = s;
        x[i] = add_rn(pr.x, mul_rn(a, pr.w));
        const double rn = add_rn(pr.r, mul_rn(-a, s));
        r[i] = rn;
        racc_add(acc, 0, mul_rn(pr.rt, rn));
    }
    __device__ void finish(const double* tot) const
    {
        // q axpy, w axpy, apply(w), x axpy, r axpy
        st->flops += 2 * st->n + 2 * st->n + 2 * st->nnz + 2 * st->n + 2 * st->n;
        st->rho_next = tot[0];  // dot(rt, r) at the top of the next iteration
    }
};

struct EpiCgsRes {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;
    const double* __restrict__ b;
    SolverState* st;
    struct Pre {
        double b;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(b, rb, re);
    }
    __device__ Pre pre(int i) const { return {b[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int, double s, const Pre& pr, auto* acc) const
    {
        const double t = add_rn(pr.b, -s);
        racc_add(acc, 0, mul_rn(t, t));
    }
    __device__ void finish(const double* tot) const
    {
        const long long n = st->n;
        st->flops += 2 * st->nnz + n + 2 * n + 2 * n;  // true_residual
        const double rel = sqrt(tot[0]) / st->norm_b;
        push_hist(st, rel);
        if (!st->fixed && rel <= st->tol) {
            st->status = ST_CONVERGED;
            st->done = 1;
            return;
        }
        if (st->fixed && rel <= kMachineFloor) {
            st->status = ST_FROZEN;
            st->done = 1;
            return;
        }
        if (st->iter >= st->limit) {
            st->status = ST_LIMIT;
            st->done = 1;
            return;
        }
        // top of iteration iter+1 (krylov.cpp:257-275): rho_next = dot(rt,
        // r) (reduced in S4), check rho, beta, the u/p updates (9 n flops)
        const int next = st->iter + 1;
        st->iter = next;
        st->flops += 2 * n;
        if (bd(st->rho)) {
            raise_breakdown(st, 1, next);
            return;
        }
        st->beta = st->rho_next / st->rho;
        st->flops += n + 2 * n + n + 2 * n + n + 2 * n;
        st->rho = st->rho_next;
    }
};

// ----------------------------------------------------------- GMRES
__device__ bool gm_step_skip(const SolverState* st, int jj)
{
    const GmresState* G = st->gm;
    return *(volatile const int*)&st->done != 0 || *(volatile const int*)&G->cycle_done != 0 ||
           jj >= *(volatile const int*)&G->cycle_limit;
}

// r = b - A x into V0 and <r,r>: the initial true residual (first = 1,
// krylov.cpp:420-424) or the end-of-cycle true residual (krylov.cpp:397-399);
// either way it is also the next cycle's initial residual (same x, same
// bits), whose flops are counted when that cycle starts.
struct EpiGmRes {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;
    const double* __restrict__ b;
    double* __restrict__ v0;
    SolverState* st;
    int first;
    struct Pre {
        double b;
    };
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(b, rb, re);
    }
    __device__ Pre pre(int i) const { return {b[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        const double t = add_rn(pr.b, -s);
        v0[i] = t;
        racc_add(acc, 0, mul_rn(t, t));
    }
    __device__ void finish(const double* tot) const
    {
        GmresState* G = st->gm;
        const long long n = st->n, nnz = st->nnz;
        const double rr = tot[0];
        const double rel = sqrt(rr) / st->norm_b;
        st->flops += 2 * nnz + n + 2 * n + 2 * n;  // true_residual
        if (first) {
            st->hist_len = 0;
            push_hist(st, rel);
            if (!st->fixed && rel <= st->tol) {
                st->status = ST_CONVERGED;
                st->done = 1;
                return;
            }
        } else {
            G->iterations += G->steps;
            st->hist[st->hist_len - 1] = rel;  // replaces the last estimate
            st->last_rel = rel;
            if (!st->fixed && rel <= st->tol) {
                st->status = ST_CONVERGED;
                st->done = 1;
                return;
            }
            if (st->fixed && rel <= kMachineFloor) {
                st->status = ST_FROZEN;
                st->done = 1;
                return;
            }
            if (G->iterations >= st->limit) {
                st->status = ST_LIMIT;
                st->done = 1;
                return;
            }
        }
        // next cycle: initial_residual + norm (krylov.cpp:315-316)
        st->flops += 2 * nnz + n + 2 * n + 2 * n;
        const double beta = sqrt(rr);
        G->steps = 0;
        G->happy = 0;
        if (beta == 0.0) {
            // zero residual: nothing to iterate on (krylov.cpp:426-433)
            G->cycle_done = 1;
            st->status = st->fixed ? ST_FROZEN : ST_CONVERGED;
            st->done = 1;
            return;
        }
        st->flops += n;  // scal(1 / beta)
        G->beta = beta;
        G->g[0] = beta;
        const int left = st->limit - G->iterations;
        G->cycle_limit = G->restart < left ? G->restart : left;
        G->cycle_done = 0;
    }
};

// S1 of step jj: w = A v_jj, <v_0, w> (the first MGS dot, krylov.cpp:339-344)
struct EpiGmApply {
    static constexpr int NV = 1;
    double* __restrict__ w;
    const double* __restrict__ v0;
    SolverState* st;
    int jj;
    struct Pre {
        double v0;
    };
    __device__ bool skip() const { return gm_step_skip(st, jj); }
    __device__ void prefetch(int rb, int re) const
    {
        l2_prefetch_rows(v0, rb, re);
    }
    __device__ Pre pre(int i) const { return {v0[i]}; }
    __device__ void row(int i, double s, auto* acc) const { row_pre(i, s, pre(i), acc); }
    __device__ void row_pre(int i, double s, const Pre& pr, auto* acc) const
    {
        w[i] = s;
        racc_add(acc, 0, mul_rn(pr.v0, s));
    }
    __device__ void finish(const double* tot) const
    {
        GmresState* G = st->gm;
        st->flops += 2 * st->nnz + 2 * st->n;
        G->H[0 * G->restart + jj] = tot[0];
    }
};

// ------------------------------------------------ element-wise steps
// Ops that reduce nothing declare `static constexpr bool kNoFinish = true`:
// no grid reduction, and no rank exchange on the distributed path.
template <class Op, class = void>
struct NoFinish : std::false_type {
};
template <class Op>
struct NoFinish<Op, std::void_t<decltype(Op::kNoFinish)>> : std::bool_constant<Op::kNoFinish> {
};

// >= 4 CTAs (32 warps) per SM: a streaming pass needs the loads of many
// warps in flight; the exact accumulator must not cost occupancy
template <class Op>
__global__ void __launch_bounds__(256, 4) vec_kernel(long long n, Op op, RedWs ws)
{
    pdl_enter();
    constexpr int NV = Op::NV;
    __shared__ double sh[32 * NV];
    if (op.skip()) return;
    if constexpr (!NoFinish<Op>::value) red_begin<NV>();
    RAcc acc[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) racc_zero(acc[i]);
    op.prologue();
    // U elements per step (4, or 2 for ops with many operands: the 64-
    // register budget of 4 CTAs/SM): all loads of the step first (ahead of
    // any store, so nothing serialises on possible aliasing), then the
    // updates; the exact adds of a step's terms run during the NEXT step,
    // after its loads are issued (software-pipelined like staged_rows)
    constexpr int U = sizeof(typename Op::In) <= 16 ? 4 : 2;
    const long long stride = (long long)gridDim.x * blockDim.x;
    Terms<NV> pend[U];
#pragma unroll
    for (int u = 0; u < U; ++u) terms_zero(pend[u]);
    long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    for (; i0 + (U - 1) * stride < n; i0 += U * stride) {
        typename Op::In in[U];
#pragma unroll
        for (int u = 0; u < U; ++u) in[u] = op.load(i0 + u * stride);
        Terms<NV> t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            terms_zero(t[u]);
            op.elem(i0 + u * stride, in[u], &t[u]);
        }
        if constexpr (!NoFinish<Op>::value) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                terms_flush<SqMask<Op>::value>(acc, pend[u]);
                pend[u] = t[u];
            }
        }
    }
    for (; i0 < n; i0 += stride) {  // the last < U elements
        const typename Op::In in = op.load(i0);
        Terms<NV> t;
        terms_zero(t);
        op.elem(i0, in, &t);
        if constexpr (!NoFinish<Op>::value) terms_flush<SqMask<Op>::value>(acc, t);
    }
    if constexpr (!NoFinish<Op>::value) {
#pragma unroll 1
        for (int u = 0; u < U; ++u) {
            terms_flush<SqMask<Op>::value>(acc, pend[0]);
#pragma unroll
            for (int k = 0; k + 1 < U; ++k) pend[k] = pend[k + 1];
        }
    }
    if constexpr (!NoFinish<Op>::value) {
        grid_reduce<NV>(acc, ws, threadIdx.x, blockDim.x, sh,
                               [&](const double* tot) { op.finish(tot); });
    }
}

// CG K2: x += alpha p; r -= alpha q; <r,r>; beta = <r,r>/rho (for K3).
struct OpCgK2 {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;  // <r,r>
    double* __restrict__ x;
    double* __restrict__ r;
    const double* __restrict__ p;
    const double* __restrict__ q;
    SolverState* st;
    int recurrence;
    double alpha;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prologue() { alpha = st->alpha; }
    struct In {
        double x, p, r, q;
    };
    __device__ In load(long long i) const { return {x[i], p[i], r[i], q[i]}; }
    __device__ void elem(long long i, const In& in, auto* acc) const
    {
        x[i] = add_rn(in.x, mul_rn(alpha, in.p));
        const double rn = add_rn(in.r, mul_rn(-alpha, in.q));
        r[i] = rn;
        racc_add(acc, 0, mul_rn(rn, rn));
    }
    __device__ void finish(const double* tot) const
    {
        st->flops += 4 * st->n;
        st->rho_next = tot[0];
        st->beta = tot[0] / st->rho;
        if (recurrence) {
            // stopping test on the recurrence residual; a true residual
            // must confirm convergence (EpiTrueRes), else iteration goes on
            const double rel = sqrt(tot[0]) / st->norm_b;
            const long long n = st->n;
            st->hist[st->hist_len] = rel;
            st->hist_len += 1;
            st->last_rel = rel;
            if (rel <= st->tol || st->iter >= st->limit) {
                st->verify_pending = 1;
                return;
            }
            st->flops += 2 * n + n + 2 * n;
            if (bd(st->rho)) {
                raise_breakdown(st, 1, st->iter);
                return;
            }
            st->rho = st->rho_next;
        }
    }
};

// residual_mode 1: p = beta p + r (skipped while a verification is pending)
struct OpCgP {
    static constexpr int NV = 1;
    double* __restrict__ p;
    const double* __restrict__ r;
    SolverState* st;
    double beta;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prologue() { beta = st->beta; }
    struct In {
        double p, r;
    };
    __device__ In load(long long i) const { return {p[i], r[i]}; }
    __device__ void elem(long long i, const In& in, auto*) const
    {
        p[i] = add_rn(mul_rn(in.p, beta), in.r);
    }
    static constexpr bool kNoFinish = true;  // nothing to reduce
    __device__ void finish(const double*) const {}
};

// BiCGSTAB B3: s = r - alpha v; <s,s>
struct OpBiB3 {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;  // <s,s>
    double* __restrict__ s;
    const double* __restrict__ r;
    const double* __restrict__ v;
    SolverState* st;
    double alpha;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prologue() { alpha = st->alpha; }
    struct In {
        double r, v;
    };
    __device__ In load(long long i) const { return {r[i], v[i]}; }
    __device__ void elem(long long i, const In& in, auto* acc) const
    {
        const double sv = add_rn(in.r, mul_rn(-alpha, in.v));
        s[i] = sv;
        racc_add(acc, 0, mul_rn(sv, sv));
    }
    __device__ void finish(const double* tot) const
    {
        st->flops += 4 * st->n;  // axpy + norm
        st->s_rel = sqrt(tot[0]) / st->norm_b;
    }
};

// BiCGSTAB B5: x += alpha p; x += omega s; r = s - omega t; <rt, r>
struct OpBiB5 {
    static constexpr int NV = 1;
    double* __restrict__ x;
    double* __restrict__ r;
    const double* __restrict__ p;
    const double* __restrict__ s;
    const double* __restrict__ t;
    const double* __restrict__ rt;
    SolverState* st;
    double alpha, omega;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prologue()
    {
        alpha = st->alpha;
        omega = st->omega;
    }
    struct In {
        double s, x, p, t, rt;
    };
    __device__ In load(long long i) const { return {s[i], x[i], p[i], t[i], rt[i]}; }
    __device__ void elem(long long i, const In& in, auto* acc) const
    {
        x[i] = add_rn(add_rn(in.x, mul_rn(alpha, in.p)), mul_rn(omega, in.s));
        const double rn = add_rn(in.s, mul_rn(-omega, in.t));
        r[i] = rn;
        racc_add(acc, 0, mul_rn(in.rt, rn));
    }
    __device__ void finish(const double* tot) const
    {
        st->flops += 6 * st->n;
        st->rho_next = tot[0];
        // beta for the p update fused into B6 (checked there)
        st->beta = (tot[0] / st->rho) * (st->alpha / st->omega);
    }
};

// CGS S1: u = beta q + r; p = beta (beta p + q) + u (krylov.cpp:264-271,
// the reference's scal/axpy sequence, each step rounded); a no-op in
// iteration 1, where EpiInit already set u = p = r.
struct OpCgsUP {
    static constexpr int NV = 1;
    double* __restrict__ u;
    double* __restrict__ p;
    const double* __restrict__ q;
    const double* __restrict__ r;
    SolverState* st;
    double beta;
    __device__ bool skip() const
    {
        return *(volatile int*)&st->done != 0 || *(volatile int*)&st->iter <= 1;
    }
    __device__ void prologue() { beta = st->beta; }
    struct In {
        double q, r, p;
    };
    __device__ In load(long long i) const { return {q[i], r[i], p[i]}; }
    __device__ void elem(long long i, const In& in, auto*) const
    {
        const double ui = add_rn(mul_rn(in.q, beta), in.r);
        u[i] = ui;
        p[i] = add_rn(mul_rn(add_rn(mul_rn(in.p, beta), in.q), beta), ui);
    }
    // nothing to reduce: the distributed path skips the rank exchange
    static constexpr bool kNoFinish = true;
    __device__ void finish(const double*) const {}
};

// CGS S3: q = u - alpha v; w = u + q
struct OpCgsQW {
    static constexpr int NV = 1;
    double* __restrict__ q;
    double* __restrict__ w;
    const double* __restrict__ u;
    const double* __restrict__ v;
    SolverState* st;
    double alpha;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prologue() { alpha = st->alpha; }
    struct In {
        double u, v;
    };
    __device__ In load(long long i) const { return {u[i], v[i]}; }
    __device__ void elem(long long i, const In& in, auto*) const
    {
        const double qi = add_rn(in.u, mul_rn(-alpha, in.v));
        q[i] = qi;
        w[i] = add_rn(in.u, qi);
    }
    static constexpr bool kNoFinish = true;  // nothing to reduce
    __device__ void finish(const double*) const {}
};

// MGS pass i of step jj (i >= 1): w -= h[i-1][jj] v_{i-1}, then <v_i, w>;
// i == jj + 1 is the closing pass: w -= h[jj][jj] v_jj, then <w, w> = hnext^2
// and the Givens update of column jj (krylov.cpp:340-375).
struct OpGmMgs {
    static constexpr int NV = 1;
    double* __restrict__ w;
    const double* __restrict__ vprev;
    const double* __restrict__ vi;  // null on the closing pass
    SolverState* st;
    int i, jj;
    double h;
    __device__ bool skip() const { return gm_step_skip(st, jj); }
    __device__ void prologue() { h = st->gm->H[(i - 1) * st->gm->restart + jj]; }
    struct In {
        double w, vprev, vi;
    };
    __device__ In load(long long k) const { return {w[k], vprev[k], vi ? vi[k] : 0.0}; }
    __device__ void elem(long long k, const In& in, auto* acc) const
    {
        const double wn = add_rn(in.w, mul_rn(-h, in.vprev));
        w[k] = wn;
        racc_add(acc, 0, mul_rn(vi ? in.vi : wn, wn));
    }
    __device__ void finish(const double* tot) const
    {
        GmresState* G = st->gm;
        const int m = G->restart;
        double* H = G->H;
        st->flops += 2 * st->n + 2 * st->n;  // axpy + dot / norm
        if (vi) {
            H[i * m + jj] = tot[0];
            return;
        }
        const double hnext = sqrt(tot[0]);
        G->hnext = hnext;
        for (int r = 0; r < jj; ++r) {
            const double a = H[r * m + jj], c = H[(r + 1) * m + jj];
            const double upper = add_rn(mul_rn(G->gc[r], a), mul_rn(G->gs[r], c));
            H[(r + 1) * m + jj] = add_rn(mul_rn(-G->gs[r], a), mul_rn(G->gc[r], c));
            H[r * m + jj] = upper;
        }
        const double denom = hypot(H[jj * m + jj], hnext);
        if (bd(denom)) {
            raise_breakdown(st, 5, G->steps + 1);
            return;
        }
        G->gc[jj] = H[jj * m + jj] / denom;
        G->gs[jj] = hnext / denom;
        H[jj * m + jj] = denom;
        G->g[jj + 1] = mul_rn(-G->gs[jj], G->g[jj]);
        G->g[jj] = mul_rn(G->gc[jj], G->g[jj]);
        G->steps += 1;
        push_hist(st, fabs(G->g[jj + 1]) / st->norm_b);  // in-cycle estimate
        G->happy = hnext < kHappyEps;
        if (G->happy) {
            G->cycle_done = 1;
            return;
        }
        st->flops += st->n;  // scal(1 / hnext)
        if ((!st->fixed && st->last_rel <= st->tol) || G->steps >= G->cycle_limit)
            G->cycle_done = 1;
    }
};

// v_{jj+1} = w / hnext (krylov.cpp:369); skipped when the cycle ends here.
struct OpGmScale {
    static constexpr int NV = 1;
    double* __restrict__ v;
    const double* __restrict__ w;  // null: scale v in place by 1 / beta
    SolverState* st;
    int jj;
    double inv;
    __device__ bool skip() const { return gm_step_skip(st, jj); }
    __device__ void prologue() { inv = 1.0 / (w ? st->gm->hnext : st->gm->beta); }
    struct In {
        double a;
    };
    __device__ In load(long long k) const { return {w ? w[k] : v[k]}; }
    __device__ void elem(long long k, const In& in, auto*) const { v[k] = mul_rn(in.a, inv); }
    static constexpr bool kNoFinish = true;  // nothing to reduce
    __device__ void finish(const double*) const {}
};

// Back substitution of the rotated triangle (krylov.cpp:381-391).
__global__ void gmres_backsub_kernel(SolverState* st)
{
    if (st->done) return;
    GmresState* G = st->gm;
    const int m = G->restart, steps = G->steps;
    for (int i = steps - 1; i >= 0; --i) {
        double sum = G->g[i];
        for (int k = i + 1; k < steps; ++k) sum = add_rn(sum, -mul_rn(G->H[i * m + k], G->y[k]));
        if (bd(G->H[i * m + i])) {
            raise_breakdown(st, 6, i + 1);
            return;
        }
        G->y[i] = sum / G->H[i * m + i];
    }
    st->flops += static_cast<long long>(steps) * steps;
}

// gmres_restart_cycle only: the cycle's last basis vector v_steps =
// w / hnext (krylov.cpp:369-370 pushes it; the solver's own cycle skips it,
// nothing reads it).  Not after a happy breakdown.
struct OpGmLast {
    static constexpr int NV = 1;
    double* __restrict__ V;
    long long ld;
    const double* __restrict__ w;
    SolverState* st;
    double inv;
    double* vout;
    __device__ bool skip() const
    {
        return *(volatile int*)&st->done != 0 || *(volatile int*)&st->gm->happy != 0;
    }
    __device__ void prologue()
    {
        inv = 1.0 / st->gm->hnext;
        vout = V + st->gm->steps * ld;
    }
    struct In {
        double w;
    };
    __device__ In load(long long k) const { return {w[k]}; }
    __device__ void elem(long long k, const In& in, auto*) const { vout[k] = mul_rn(in.w, inv); }
    static constexpr bool kNoFinish = true;
    __device__ void finish(const double*) const {}
};

// x += y_0 v_0 + y_1 v_1 + ... in the reference's axpy order (krylov.cpp:392-394)
struct OpGmUpdate {
    static constexpr int NV = 1;
    double* __restrict__ x;
    const double* __restrict__ V;
    long long ld;
    SolverState* st;
    int steps;
    __device__ bool skip() const { return *(volatile int*)&st->done != 0; }
    __device__ void prologue() { steps = st->gm->steps; }
    struct In {};
    __device__ In load(long long) const { return {}; }
    __device__ void elem(long long k, const In&, auto*) const
    {
        const double* y = st->gm->y;
        double v = x[k];
        for (int i = 0; i < steps; ++i) v = add_rn(v, mul_rn(__ldg(y + i), V[i * ld + k]));
        x[k] = v;
    }
    // reads the step count from the state: in the distributed environment
    // finish() runs in a separate kernel on a copy whose prologue never ran
    __device__ void finish(const double*) const { st->flops += 2LL * st->gm->steps * st->n; }
};

// -------------------------------------------------------- operators
struct CsrOp {
    CsrView<double> A;
    template <class Epi>
    void apply(lbk_ctx ctx, const double* x, const Epi& e, RedWs ws) const
    {
        launch_csr<double>(ctx, A, x, e, ws);
    }
};

struct CooOp {
    CooView<double> A;
    template <class Epi>
    void apply(lbk_ctx ctx, const double* x, const Epi& e, RedWs ws) const
    {
        launch_coo<double>(ctx, A, x, e, ws);
    }
};

template <class Op>
void launch_vec(lbk_ctx ctx, long long n, const Op& op, RedWs ws)
{
    auto k = vec_kernel<Op>;
    static int bps = blocks_per_sm(k, 256, 0);
    long long want = (n + 255) / 256;
    long long cap = static_cast<long long>(ctx->num_sms) * bps;
    if (cap > kRedMaxBlocks) cap = kRedMaxBlocks;
    int grid = static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap);
    launch_pdl(ctx, k, dim3(grid), dim3(256), 0, n, op, ws);
    LBK_LAUNCH_CHECK();
}

struct DevBufs {
    std::vector<void*> ptrs;
    cudaStream_t s;
    explicit DevBufs(cudaStream_t st) : s(st) {}
    template <typename T>
    T* get(size_t count)
    {
        void* p = nullptr;
        LBK_CUDA(cudaMallocAsync(&p, count * sizeof(T) + 16, s));
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    ~DevBufs()
    {
        for (auto* p : ptrs) cudaFreeAsync(p, s);
    }
};

const char* breakdown_what(int w)
{
    switch (w) {
    case 0: return "division by vanishing <p, Ap>";
    case 1: return "division by vanishing rho";
    case 2: return "division by vanishing omega";
    case 3: return "division by vanishing <rt, Ap>";
    case 5: return "division by vanishing Givens denominator";
    case 6: return "division by vanishing triangular diagonal";
    default: return "division by vanishing <t, t>";
    }
}

// Single-device environment: the fused kernels reduce and finish in one
// launch (RedWs.defer = 0).
template <class MatOp>
struct LocalEnv {
    static constexpr bool kMergeCg = false;
    lbk_ctx ctx;
    MatOp op;
    RedWs ws;
    long long n, nnz;
    long long n_local() const { return n; }
    long long n_ext() const { return n; }
    long long n_global() const { return n; }
    long long nnz_global() const { return nnz; }
    bool ext_x() const { return false; }
    // chunks after the first replay as a captured CUDA graph (round 2: on by
    // default -- with PDL off the launch gaps show, CG +0.6%, the
    // recurrence stop +1.2%); LBK_SOLVER_GRAPH=0 launches eagerly
    bool graph_ok() const
    {
        const char* e = std::getenv("LBK_SOLVER_GRAPH");
        return !(e && e[0] == '0');
    }
    template <class Epi>
    void apply(const double* x, const Epi& e) { op.apply(ctx, x, e, ws); }
    template <class Op>
    void vec(const Op& o) { launch_vec(ctx, n, o, ws); }
    void sync() { LBK_CUDA(cudaStreamSynchronize(ctx->stream)); }
    double norm(const double* b)
    {
        double v = 0.0;
        if (lbk_nrm2_f64(ctx, n, b, &v) != LBK_OK) fail(LBK_CUDA_ERROR, ctx->err);
        return v;
    }
};

// Distributed environment: every reduction is deferred --
// the fused kernels leave their local totals in ws.out, a one-warp kernel
// combines interior + boundary parts in fixed order, the communicator sums
// over ranks (ncclAllReduce / thread group), and a one-thread kernel runs
// the epilogue's finish() on the global totals, so the scalar recurrence
// advances identically on every rank.
template <int NV>
__global__ void combine_kernel(double* base, int has_a, int has_b)
{
    const int i = threadIdx.x;
    if (i < NV) {
        double v = 0.0;
        if (has_a) v = add_rn(v, base[i]);
        if (has_b) v = add_rn(v, base[8 + i]);
        base[16 + i] = v;
    }
}

template <class E>
__global__ void finish_kernel(E e, const double* tot)
{
    if (e.skip()) return;
    double t[E::NV > 0 ? E::NV : 1];
#pragma unroll
    for (int i = 0; i < E::NV; ++i) t[i] = tot[i];
    e.finish(t);
}

// Peer-memory group: combine + the rank-ordered sum over the peers'
// windows + finish() in one launch (peer.cuh).
template <class E>
__global__ void peer_finish_kernel(E e, const double* base, int has_a, int has_b, PeerDev pd)
{
    pdl_enter();
    if (e.skip()) return;
    static_assert(E::NV <= 8, "peer finish: at most 8 values");
    const int lane = threadIdx.x;
    double v = 0.0;
    if (lane < E::NV) {
        if (has_a) v = add_rn(v, base[lane]);
        if (has_b) v = add_rn(v, base[8 + lane]);
    }
    const double t = peer_allreduce_warp(pd, v, E::NV > 0 ? E::NV : 1);
    __shared__ double tot[8];
    if (lane < E::NV) tot[lane] = t;
    __syncwarp();
    if (lane == 0) e.finish(tot);
}

// CG / BiCGSTAB over the peer group with one exchange fewer per iteration:
// the true residual ||b - Ax||^2 of K3 (CG) / B6 (BiCGSTAB) stays
// rank-local (deferred to out[32], out[40]) and is exchanged together with
// the next K1's <p, Ap> / B2's <rt, v>.  Its finish (history, convergence)
// then runs here, before K1's -- the same totals, bits and order of state
// updates as the unmerged path; only the decision to stop arrives one
// kernel later (that K1's SpMV is wasted work).
template <class E1, class E3>
__global__ void peer_finish_cg_kernel(E1 e1, E3 e3, const double* base, int has_a, int has_b,
                                      PeerDev pd)
{
    pdl_enter();
    if (e1.skip()) return;
    const int lane = threadIdx.x;
    const bool pending = e1.st->res_pending != 0;  // a K3 ran since the last K1
    double v = 0.0;
    if (lane == 0) {
        if (has_a) v = add_rn(v, base[0]);
        if (has_b) v = add_rn(v, base[8]);
    } else if (lane == 1 && pending) {
        if (has_a) v = add_rn(v, base[32]);
        if (has_b) v = add_rn(v, base[40]);
    }
    const double t = peer_allreduce_warp(pd, v, 2);
    __shared__ double tot[2];
    if (lane < 2) tot[lane] = t;
    __syncwarp();
    if (lane == 0) {
        if (pending) {
            e3.finish(&tot[1]);
            if (e1.st->done) return;
        }
        e1.finish(&tot[0]);
        e1.st->res_pending = 1;  // this iteration's K3 follows, deferred
    }
}

// the last K3's deferred residual, when the launch loop ends on it
template <class E3>
__global__ void peer_flush_cg_kernel(E3 e3, const double* base, int has_a, int has_b, PeerDev pd)
{
    pdl_enter();
    if (e3.skip() || !e3.st->res_pending) return;
    const int lane = threadIdx.x;
    double v = 0.0;
    if (lane == 0) {
        if (has_a) v = add_rn(v, base[32]);
        if (has_b) v = add_rn(v, base[40]);
    }
    const double t = peer_allreduce_warp(pd, v, 1);
    __shared__ double tot[1];
    if (lane == 0) {
        tot[0] = t;
        e3.finish(tot);
    }
}

// Exact mode (xred.cuh): the fused kernels of a rank add their limbs into
// one deferred slot (interior and boundary rows alike -- integer sums need
// no combine step); the slot is summed over ranks (NCCL int64 allreduce /
// host sums / peer digit posts) and rounded once, so every rank and every
// rank count sees the same bits as the single-GPU solver.
// Move a deferred slot (n int64, n <= 5 * 32) into shared memory and zero
// it: all loads first (one round trip), then the stores.  One warp.
__device__ __forceinline__ void take_slot(long long* L, long long* slot, int n)
{
    const int lane = threadIdx.x & 31;
    long long v[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        v[k] = i < n ? __ldcg(slot + i) : 0;
    }
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int i = lane + 32 * k;
        if (i < n) {
            L[i] = v[k];
            slot[i] = 0;
        }
    }
}

template <class E>
__global__ void xfinish_kernel(E e, long long* slot)
{
    constexpr int NV = E::NV > 0 ? E::NV : 1;
    __shared__ long long L[NV * kXV];
    if (e.skip()) return;
    take_slot(L, slot, NV * kXV);
    __syncthreads();
    double t[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) t[v] = xred_round_warp(L + v * kXV);
    if (threadIdx.x == 0) e.finish(t);
}

template <class E>
__global__ void peer_xfinish_kernel(E e, long long* slot, PeerDev pd)
{
    pdl_enter();
    constexpr int NV = E::NV > 0 ? E::NV : 1;
    __shared__ long long L[NV * kXV];
    if (e.skip()) return;
    const int lane = threadIdx.x;
    take_slot(L, slot, NV * kXV);
    __syncwarp();
    peer_xallreduce_warp(pd, L, NV);
    double t[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) t[v] = xred_round_warp(L + v * kXV);
    if (lane == 0) e.finish(t);
}

// exact-mode twin of peer_finish_cg_kernel: K1's <p,Ap> (slot s1) and the
// pending K3 residual (slot s3) travel in one exchange
template <class E1, class E3>
__global__ void peer_xfinish_cg_kernel(E1 e1, E3 e3, long long* s1, long long* s3, PeerDev pd)
{
    pdl_enter();
    __shared__ long long L[2 * kXV];
    if (e1.skip()) return;
    const int lane = threadIdx.x;
    const bool pending = e1.st->res_pending != 0;
    take_slot(L, s1, kXV);
    if (pending) take_slot(L + kXV, s3, kXV);
    else
        for (int i = lane; i < kXV; i += 32) L[kXV + i] = 0;
    __syncwarp();
    // the pending residual goes first so its finish runs before K1's
    if (pending) {
        for (int i = lane; i < kXV; i += 32) {
            const long long a = L[i];
            L[i] = L[kXV + i];
            L[kXV + i] = a;
        }
        __syncwarp();
    }
    peer_xallreduce_warp(pd, L, pending ? 2 : 1);
    const double t3 = pending ? xred_round_warp(L) : 0.0;
    const double t1 = xred_round_warp(pending ? L + kXV : L);
    if (lane == 0) {
        if (pending) {
            e3.finish(&t3);
            if (e1.st->done) return;
        }
        e1.finish(&t1);
        e1.st->res_pending = 1;
    }
}

template <class E3>
__global__ void peer_xflush_cg_kernel(E3 e3, long long* s3, PeerDev pd)
{
    pdl_enter();
    __shared__ long long L[kXV];
    if (e3.skip() || !e3.st->res_pending) return;
    const int lane = threadIdx.x;
    take_slot(L, s3, kXV);
    __syncwarp();
    peer_xallreduce_warp(pd, L, 1);
    const double t = xred_round_warp(L);
    if (lane == 0) e3.finish(&t);
}

// ||b|| of the distributed right-hand side (exact mode)
struct OpSelfDot {
    static constexpr int NV = 1;
    static constexpr unsigned kSq = 1;
    const double* __restrict__ b;
    __device__ bool skip() const { return false; }
    __device__ void prologue() {}
    struct In {
        double b;
    };
    __device__ In load(long long i) const { return {b[i]}; }
    __device__ void elem(long long, const In& in, auto* acc) const
    {
        racc_add(acc, 0, mul_rn(in.b, in.b));
    }
    __device__ void finish(const double*) const {}
};
struct EpiSqrtTot {
    static constexpr int NV = 1;
    double* out;
    __device__ bool skip() const { return false; }
    __device__ void finish(const double* t) const { *out = sqrt(t[0]); }
};

struct DistEnv {
    static constexpr bool kMergeCg = true;
    lbk_ctx ctx;
    lbk_dist_csr_s* D;
    Comm* comm;
    RedWs ws;
    long long n_local() const { return D->n_local; }
    long long n_ext() const { return static_cast<long long>(D->n_local) + D->n_ghost; }
    long long n_global() const { return D->n_global; }
    long long nnz_global() const { return D->nnz_global; }
    bool ext_x() const { return true; }
    // asynchronous (NCCL) or no communicator: capturable; the thread group
    // synchronises on the host
    bool graph_ok() const
    {
        const char* e = std::getenv("LBK_SOLVER_GRAPH");
        if (e && e[0] == '0') return false;
        return !comm || comm->async();
    }
    // NCCL reduces even at one rank (keeps the captured path identical)
    bool reduce() const { return comm && (comm->nranks > 1 || comm->async()); }

    template <class E>
    void finish(const E& e, int has_a, int has_b)
    {
        // peer group: combine + the rank sum + finish() in one launch
        if (const PeerDev* pd = comm ? comm->peer() : nullptr) {
            launch_pdl(ctx, peer_finish_kernel<E>, dim3(1), dim3(32), 0, e, ws.out, has_a, has_b,
                       *pd);
            LBK_LAUNCH_CHECK();
            return;
        }
        combine_kernel<E::NV><<<1, 32, 0, ctx->stream>>>(ws.out, has_a, has_b);
        LBK_LAUNCH_CHECK();
        if (reduce()) comm->allreduce_sum(ws.out + 16, E::NV, ctx->stream);
        finish_kernel<E><<<1, 1, 0, ctx->stream>>>(e, ws.out + 16);
        LBK_LAUNCH_CHECK();
    }
    long long* xslot(int k) const { return ws.xout + size_t(k) * kXSlot; }
    // exact mode: sum slot k over the ranks, round, finish()
    template <class E>
    void finish_x(const E& e, int k)
    {
        if (const PeerDev* pd = comm ? comm->peer() : nullptr) {
            launch_pdl(ctx, peer_xfinish_kernel<E>, dim3(1), dim3(32), 0, e, xslot(k), *pd);
            LBK_LAUNCH_CHECK();
            return;
        }
        if (reduce()) comm->allreduce_i64(xslot(k), (E::NV > 0 ? E::NV : 1) * kXV, ctx->stream);
        xfinish_kernel<E><<<1, 32, 0, ctx->stream>>>(e, xslot(k));
        LBK_LAUNCH_CHECK();
    }
    RedWs deferred(int k) const
    {
        RedWs w = ws;
        w.defer = 1;
        w.xout = xslot(k);
        return w;
    }
    template <class Epi>
    void apply(double* x, const Epi& e)
    {
        if constexpr (kExactRed) {
            dist_apply(ctx, D, comm, x, e, deferred(0), deferred(0));
            finish_x(e, 0);
            return;
        }
        RedWs wa = ws, wb = ws;
        wa.defer = wb.defer = 1;
        wb.out = ws.out + 8;
        dist_apply(ctx, D, comm, x, e, wa, wb);
        finish(e, D->interior.nrows > 0, D->boundary.nrows > 0);
    }
    // two-exchange CG (peer group; LBK_CG_MERGE=0 turns it off)
    bool merge_cg() const
    {
        const char* e = std::getenv("LBK_CG_MERGE");
        return comm && comm->peer() && !(e && e[0] == '0');
    }
    template <class E1, class E3>
    void apply_k1_merged(double* x, const E1& e1, const E3& e3)
    {
        if constexpr (kExactRed) {
            dist_apply(ctx, D, comm, x, e1, deferred(0), deferred(0));
            launch_pdl(ctx, peer_xfinish_cg_kernel<E1, E3>, dim3(1), dim3(32), 0, e1, e3,
                       xslot(0), xslot(1), *comm->peer());
            LBK_LAUNCH_CHECK();
            return;
        }
        RedWs wa = ws, wb = ws;
        wa.defer = wb.defer = 1;
        wb.out = ws.out + 8;
        dist_apply(ctx, D, comm, x, e1, wa, wb);
        launch_pdl(ctx, peer_finish_cg_kernel<E1, E3>, dim3(1), dim3(32), 0, e1, e3, ws.out,
                   D->interior.nrows > 0 ? 1 : 0, D->boundary.nrows > 0 ? 1 : 0, *comm->peer());
        LBK_LAUNCH_CHECK();
    }
    template <class E3>
    void apply_k3_deferred(double* x, const E3& e3)
    {
        if constexpr (kExactRed) {
            dist_apply(ctx, D, comm, x, e3, deferred(1), deferred(1));
            return;
        }
        RedWs wa = ws, wb = ws;
        wa.defer = wb.defer = 1;
        wa.out = ws.out + 32;
        wb.out = ws.out + 40;
        dist_apply(ctx, D, comm, x, e3, wa, wb);
    }
    template <class E3>
    void flush_k3(const E3& e3)
    {
        if constexpr (kExactRed) {
            launch_pdl(ctx, peer_xflush_cg_kernel<E3>, dim3(1), dim3(32), 0, e3, xslot(1),
                       *comm->peer());
            LBK_LAUNCH_CHECK();
            return;
        }
        launch_pdl(ctx, peer_flush_cg_kernel<E3>, dim3(1), dim3(32), 0, e3, ws.out,
                   D->interior.nrows > 0 ? 1 : 0, D->boundary.nrows > 0 ? 1 : 0, *comm->peer());
        LBK_LAUNCH_CHECK();
    }
    template <class Op>
    void vec(const Op& o)
    {
        if constexpr (kExactRed) {
            launch_vec(ctx, D->n_local, o, deferred(0));
            if constexpr (!NoFinish<Op>::value) finish_x(o, 0);
            return;
        }
        RedWs wa = ws;
        wa.defer = 1;
        launch_vec(ctx, D->n_local, o, wa);
        if constexpr (!NoFinish<Op>::value) finish(o, 1, 0);
    }
    void sync()
    {
        if (comm) comm->wait(ctx->stream);
        else LBK_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    double norm(const double* b)
    {
        if constexpr (kExactRed) {
            launch_vec(ctx, D->n_local, OpSelfDot{b}, deferred(2));
            finish_x(EpiSqrtTot{ws.out + 24}, 2);
            double v = 0.0;
            LBK_CUDA(cudaMemcpyAsync(&v, ws.out + 24, sizeof(double), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            sync();
            return v;
        }
        double* d = ws.out + 24;
        if (lbk_dot_f64_dev(ctx, D->n_local, b, b, d) != LBK_OK) fail(LBK_CUDA_ERROR, ctx->err);
        if (reduce()) comm->allreduce_sum(d, 1, ctx->stream);
        double v = 0.0;
        LBK_CUDA(cudaMemcpyAsync(&v, d, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        sync();
        return std::sqrt(v);
    }
};

// Result assembly shared by every solver: copy x back, read the state and
// the history, apply the fixed-iteration freeze padding (krylov.cpp:135-137)
// and raise BreakdownError with its iteration.
template <class Env>
void finish_solve(lbk_ctx ctx, Env& env, SolverState* st, double* hist, double* x, double* x_user,
                  long long n, int limit, const lbk_solver_cfg* cfg, lbk_solve_result* res,
                  double* history, int hist_cap, cudaEvent_t ev0, cudaEvent_t ev1)
{
    SolverState h{};
    if (env.ext_x() && n)
        LBK_CUDA(cudaMemcpyAsync(x_user, x, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
    LBK_CUDA(cudaEventRecord(ev1, ctx->stream));
    LBK_CUDA(cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    LBK_CUDA(cudaStreamSynchronize(ctx->stream));
    float ms = 0;
    LBK_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);

    std::vector<double> hv(static_cast<size_t>(h.hist_len));
    if (h.hist_len)
        LBK_CUDA(cudaMemcpy(hv.data(), hist, hv.size() * sizeof(double), cudaMemcpyDeviceToHost));
    if (h.status == ST_FROZEN) {
        // krylov.cpp:135-137: frozen iterations repeat the last entry
        while (static_cast<int>(hv.size()) < limit + 1) hv.push_back(hv.back());
    }
    res->iterations = static_cast<int>(hv.size()) - 1;
    res->history_len = static_cast<int>(hv.size());
    res->final_rel_residual = hv.back();
    res->converged = res->final_rel_residual <= cfg->rel_tol ? 1 : 0;
    res->flop_count = h.flops;
    res->elapsed = ms * 1e-3;
    if (history) {
        const int m = res->history_len < hist_cap ? res->history_len : hist_cap;
        for (int i = 0; i < m; ++i) history[i] = hv[i];
    }
    if (h.status == ST_BREAKDOWN) {
        res->breakdown_iter = h.breakdown_iter;
        Error e(LBK_BREAKDOWN, std::string(breakdown_what(h.breakdown_what)) + " at iteration " +
                                   std::to_string(h.breakdown_iter));
        throw e;
    }
}

// gmres_restart_cycle (krylov.hpp:78-89): one cycle, its outcome, and
// optionally the cycle's orthonormal basis (device, n per vector)
struct CycleOut {
    int steps = 0, happy = 0;
    double rel = 0.0;
    double* basis = nullptr;
    int basis_cap = 0;
    int basis_count = 0;
};

template <class Env>
void solve_impl(lbk_ctx ctx, Env& env, const double* b, double* x_user, const lbk_solver_cfg* cfg,
                lbk_solve_result* res, double* history, int hist_cap, CycleOut* cyc = nullptr)
{
    NvtxRange nvtx_("lbk_solve");
    // krylov.cpp:449-472 validation
    need(cfg != nullptr && res != nullptr, LBK_USAGE_ERROR, "solve: null config/result");
    need(cfg->max_iters >= 1, LBK_CONFIGURATION_ERROR, "max_iters must be positive");
    need(cfg->rel_tol > 0.0, LBK_CONFIGURATION_ERROR, "rel_tol must be positive");
    need(cfg->kind >= 0 && cfg->kind <= 3, LBK_CONFIGURATION_ERROR,
         "solver kind must be 0 (cg), 1 (bicgstab), 2 (cgs) or 3 (gmres)");
    need(cfg->kind != 3 || (cfg->gmres_restart >= 1 && cfg->gmres_restart <= cfg->max_iters),
         LBK_CONFIGURATION_ERROR, "gmres_restart must lie in [1, max_iters]");
    need(cfg->residual_mode == 0 || (cfg->residual_mode == 1 && cfg->kind == 0),
         LBK_CONFIGURATION_ERROR, "residual_mode 1 is implemented for CG only");
    need(cfg->residual_mode == 0 || cfg->fixed_iters <= 0, LBK_CONFIGURATION_ERROR,
         "residual_mode 1 cannot be combined with fixed_iters");
    std::memset(res, 0, sizeof(*res));

    const bool fixed = cfg->fixed_iters > 0;
    const int limit = fixed ? cfg->fixed_iters : cfg->max_iters;
    const bool bicg = cfg->kind == 1;
    const bool cgs = cfg->kind == 2;
    const bool gmres = cfg->kind == 3;
    const bool recurrence = cfg->residual_mode == 1;
    const long long n = env.n_local(), ne = env.n_ext();

    cudaEvent_t ev0, ev1;
    LBK_CUDA(cudaEventCreate(&ev0));
    LBK_CUDA(cudaEventCreate(&ev1));
    LBK_CUDA(cudaEventRecord(ev0, ctx->stream));

    DevBufs bufs(ctx->stream);
    auto* st = bufs.get<SolverState>(1);
    auto* hist = bufs.get<double>(size_t(limit) + 2);
    // norm_b (krylov.cpp:478) -- host value needed for the zero-b rule
    double norm_b = env.norm(b);
    // cycle_entry (krylov.cpp:551-565): a zero b normalises by 1
    if (cyc && norm_b == 0.0) norm_b = 1.0;
    SolverState h{};
    h.limit = limit;
    h.fixed = fixed ? 1 : 0;
    h.tol = cfg->rel_tol;
    h.norm_b = norm_b;
    h.n = env.n_global();
    h.nnz = env.nnz_global();
    h.flops = 2 * h.n;
    h.hist = hist;
    if (norm_b == 0.0) {
        // krylov.cpp:479-482: x = 0, converged, history [0]
        if (n) LBK_CUDA(cudaMemsetAsync(x_user, 0, size_t(n) * sizeof(double), ctx->stream));
        LBK_CUDA(cudaEventRecord(ev1, ctx->stream));
        LBK_CUDA(cudaEventSynchronize(ev1));
        float ms = 0;
        cudaEventElapsedTime(&ms, ev0, ev1);
        res->converged = 1;
        res->iterations = 0;
        res->final_rel_residual = 0.0;
        res->history_len = 1;
        res->flop_count = 2 * h.n;
        res->elapsed = ms * 1e-3;
        if (history && hist_cap > 0) history[0] = 0.0;
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        return;
    }
    LBK_CUDA(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));

    // vectors the operator is applied to (p, s, x) carry room for the halo
    double* x = x_user;
    if (env.ext_x()) {
        x = bufs.get<double>(ne);
        if (n) LBK_CUDA(cudaMemcpyAsync(x, x_user, size_t(n) * sizeof(double),
                                        cudaMemcpyDeviceToDevice, ctx->stream));
    }
    if (gmres) {
        const int m = cfg->gmres_restart;
        auto* G = bufs.get<GmresState>(1);
        GmresState gh{};
        gh.restart = m;
        gh.H = bufs.get<double>(size_t(m + 1) * m);
        gh.gc = bufs.get<double>(m);
        gh.gs = bufs.get<double>(m);
        gh.g = bufs.get<double>(m + 1);
        gh.y = bufs.get<double>(m);
        LBK_CUDA(cudaMemcpyAsync(G, &gh, sizeof(gh), cudaMemcpyHostToDevice, ctx->stream));
        h.gm = G;
        LBK_CUDA(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
        double* V = bufs.get<double>(size_t(m + 1) * ne);
        double* w = bufs.get<double>(n);
        env.apply(x, EpiGmRes{b, V, st, 1});
        env.vec(OpGmScale{V, nullptr, st, 0, 0.0});
        int* done_host = reinterpret_cast<int*>(ctx->host_pinned);
        for (;;) {
            for (int jj = 0; jj < m; ++jj) {
                env.apply(V + size_t(jj) * ne, EpiGmApply{w, V, st, jj});
                for (int i = 1; i <= jj + 1; ++i)
                    env.vec(OpGmMgs{w, V + size_t(i - 1) * ne, i <= jj ? V + size_t(i) * ne : nullptr,
                                    st, i, jj, 0.0});
                env.vec(OpGmScale{V + size_t(jj + 1) * ne, w, st, jj, 0.0});
            }
            gmres_backsub_kernel<<<1, 1, 0, ctx->stream>>>(st);
            LBK_LAUNCH_CHECK();
            env.vec(OpGmUpdate{x, V, ne, st, 0});
            if (cyc) {
                // the cycle's steps and happy flag (before the residual kernel
                // resets them for a next cycle), then its true residual into
                // w (V keeps the basis)
                GmresState gc{};
                SolverState sc{};
                LBK_CUDA(cudaMemcpyAsync(&gc, G, sizeof(gc), cudaMemcpyDeviceToHost, ctx->stream));
                if (cyc->basis) env.vec(OpGmLast{V, ne, w, st, 0.0, nullptr});
                env.apply(x, EpiGmRes{b, w, st, 0});
                LBK_CUDA(cudaMemcpyAsync(&sc, st, sizeof(sc), cudaMemcpyDeviceToHost, ctx->stream));
                env.sync();
                need(sc.status != ST_BREAKDOWN, LBK_BREAKDOWN,
                     std::string(breakdown_what(sc.breakdown_what)) + " at iteration " +
                         std::to_string(sc.breakdown_iter));
                cyc->steps = gc.steps;
                cyc->happy = gc.happy;
                cyc->rel = sc.last_rel;
                int count = gc.happy ? gc.steps : gc.steps + 1;
                if (gc.steps == 0) {  // b - A x == 0: happy, empty basis (krylov.cpp:317-324)
                    cyc->happy = 1;
                    cyc->rel = 0.0;
                    count = 0;
                }
                cyc->basis_count = count;
                if (cyc->basis) {
                    need(count <= cyc->basis_cap, LBK_USAGE_ERROR,
                         "gmres_restart_cycle: basis_out holds fewer than steps + 1 vectors");
                    for (int i = 0; i < count && n; ++i)
                        LBK_CUDA(cudaMemcpyAsync(cyc->basis + size_t(i) * n, V + size_t(i) * ne,
                                                 size_t(n) * sizeof(double),
                                                 cudaMemcpyDeviceToDevice, ctx->stream));
                }
                if (env.ext_x() && n)
                    LBK_CUDA(cudaMemcpyAsync(x_user, x, size_t(n) * sizeof(double),
                                             cudaMemcpyDeviceToDevice, ctx->stream));
                env.sync();
                cudaEventDestroy(ev0);
                cudaEventDestroy(ev1);
                return;
            }
            env.apply(x, EpiGmRes{b, V, st, 0});
            env.vec(OpGmScale{V, nullptr, st, 0, 0.0});
            LBK_CUDA(cudaMemcpyAsync(done_host, &st->done, sizeof(int), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            env.sync();
            if (*done_host) break;
        }
        finish_solve(ctx, env, st, hist, x, x_user, n, limit, cfg, res, history, hist_cap, ev0, ev1);
        return;
    }

    double* r = bufs.get<double>(n);
    double* p = bufs.get<double>(ne);
    double* q = bufs.get<double>(n);  // CG q / BiCGSTAB v
    double* rt = (bicg || cgs) ? bufs.get<double>(n) : nullptr;
    double* s = bicg ? bufs.get<double>(ne) : nullptr;
    double* t = (bicg || cgs) ? bufs.get<double>(n) : nullptr;
    double* u = cgs ? bufs.get<double>(n) : nullptr;
    double* w = cgs ? bufs.get<double>(ne) : nullptr;

    env.apply(x, EpiInit{b, r, p, rt, st, (bicg || cgs) ? 1 : 0, u});

    bool merge = false;
    if constexpr (Env::kMergeCg) merge = !cgs && !gmres && !recurrence && env.merge_cg();
    auto iteration = [&] {
        if (cgs) {
            // v and t share storage: v is dead once S3 has formed q, w
            env.vec(OpCgsUP{u, p, q, r, st, 0.0});
            env.apply(p, EpiCgsV{t, rt, st});
            env.vec(OpCgsQW{q, w, u, t, st, 0.0});
            env.apply(w, EpiCgsT{t, x, r, w, rt, st});
            env.apply(x, EpiCgsRes{b, st});
        } else if (!bicg) {
            if constexpr (Env::kMergeCg) {
                if (merge && !recurrence) {
                    env.apply_k1_merged(p, EpiCgK1{q, p, st}, EpiCgK3{b, p, r, st});
                    env.vec(OpCgK2{x, r, p, q, st, 0, 0.0});
                    env.apply_k3_deferred(x, EpiCgK3{b, p, r, st});
                    return;
                }
            }
            env.apply(p, EpiCgK1{q, p, st});
            env.vec(OpCgK2{x, r, p, q, st, recurrence ? 1 : 0, 0.0});
            if (!recurrence) {
#ifdef LBK_FUSED_P
                env.apply(x, EpiCgK3{b, p, r, st});
#else
                env.apply(x, EpiCgK3s{b, st});
                env.vec(OpCgP{p, r, st, 0.0});
#endif
            } else {
                env.apply(x, EpiTrueRes{b, st});
                env.vec(OpCgP{p, r, st, 0.0});
            }
        } else {
            if constexpr (Env::kMergeCg) {
                if (merge) {
                    env.apply_k1_merged(p, EpiBiB2{q, rt, st}, EpiBiB6{b, p, q, r, st});
                    env.vec(OpBiB3{s, r, q, st, 0.0});
                    env.apply(s, EpiBiB4{t, s, st});
                    env.vec(OpBiB5{x, r, p, s, t, rt, st, 0.0, 0.0});
                    env.apply_k3_deferred(x, EpiBiB6{b, p, q, r, st});
                    return;
                }
            }
            env.apply(p, EpiBiB2{q, rt, st});
            env.vec(OpBiB3{s, r, q, st, 0.0});
            env.apply(s, EpiBiB4{t, s, st});
            env.vec(OpBiB5{x, r, p, s, t, rt, st, 0.0, 0.0});
#ifdef LBK_FUSED_P
            env.apply(x, EpiBiB6{b, p, q, r, st});
#else
            env.apply(x, EpiBiB6s{b, st});
            env.vec(OpBiP{p, q, r, st, 0.0, 0.0});
#endif
        }
    };
    // Chunked launch loop; `done` is polled once per chunk.  Where the
    // environment allows (no host-synchronous communicator), chunks after
    // the first are captured once into a CUDA graph and replayed: the whole
    // chunk -- SpMV/vector kernels, deferred-reduction kernels, NCCL halo
    // send/recv on the comm stream and ncclAllReduce -- becomes one launch.
    int* done_host = reinterpret_cast<int*>(ctx->host_pinned);
    const int chunk = 16;
    const bool use_graph = env.graph_ok();
    cudaGraphExec_t gexec = nullptr;
    int launched = 0;
    for (;;) {
        const int todo = limit - launched < chunk ? limit - launched : chunk;
        if (use_graph && launched > 0 && todo == chunk) {
            if (!gexec) {
                // capture on a private stream (the context's stream may be the
                // legacy default stream, which cannot be captured); the
                // graph is then launched on the context's stream
                cudaStream_t home = ctx->stream, cap = nullptr;
                LBK_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
                cudaGraph_t graph = nullptr;
                ctx->stream = cap;
                cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed);
                if (e == cudaSuccess) {
                    try {
                        for (int c = 0; c < chunk; ++c) iteration();
                    } catch (...) {
                        cudaStreamEndCapture(cap, &graph);
                        ctx->stream = home;
                        cudaStreamDestroy(cap);
                        throw;
                    }
                    e = cudaStreamEndCapture(cap, &graph);
                }
                ctx->stream = home;
                cudaStreamDestroy(cap);
                LBK_CUDA(e);
                LBK_CUDA(cudaGraphInstantiate(&gexec, graph, 0));
                cudaGraphDestroy(graph);
            }
            LBK_CUDA(cudaGraphLaunch(gexec, ctx->stream));
        } else {
            for (int c = 0; c < todo; ++c) iteration();
        }
        launched += todo;
        LBK_CUDA(cudaMemcpyAsync(done_host, &st->done, sizeof(int), cudaMemcpyDeviceToHost,
                                 ctx->stream));
        env.sync();
        if (*done_host || launched >= limit) break;
    }
    if (gexec) cudaGraphExecDestroy(gexec);
    if constexpr (Env::kMergeCg) {
        // the launch loop ends on a deferred residual
        if (merge && bicg) env.flush_k3(EpiBiB6{b, p, q, r, st});
        if (merge && !bicg) env.flush_k3(EpiCgK3{b, p, r, st});
    }
    finish_solve(ctx, env, st, hist, x, x_user, n, limit, cfg, res, history, hist_cap, ev0, ev1);
}

}  // namespace
}  // namespace lbk

using namespace lbk;

extern "C" {

lbk_status lbk_solve_csr(lbk_ctx ctx, const lbk_csr* A, const double* b, double* x,
                         const lbk_solver_cfg* cfg, lbk_solve_result* result, double* history,
                         int32_t history_cap)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->dtype == LBK_F64, LBK_TYPE_ERROR, "solve: FP64 matrices only");
        need(A->nrows == A->ncols, LBK_SHAPE_ERROR,
             "solve requires a square matrix, got " + std::to_string(A->nrows) + "x" +
                 std::to_string(A->ncols));
        CsrOp op{CsrView<double>{A->nrows, A->ncols, A->nnz, A->row_ptr, A->col_idx,
                                 static_cast<const double*>(A->vals), A->tile_rows, A->ntiles}};
        if (!op.A.tile_rows && A->nrows > 0 && aligned16(A->vals) && aligned16(A->col_idx)) {
            // build the plan once for the whole solve
            op.A.ntiles = csr_ntiles(A->nnz, A->nrows);
            int* plan = static_cast<int*>(scratch(ctx, size_t(op.A.ntiles + 1) * sizeof(int)));
            csr_plan_launch(ctx, A->row_ptr, A->nrows, A->nnz, plan);
            op.A.tile_rows = plan;
        }
        LocalEnv<CsrOp> env{ctx, op, red_ws(ctx, kRedMaxBlocks, 2), A->nrows, A->nnz};
        solve_impl(ctx, env, b, x, cfg, result, history, history_cap);
    });
}

lbk_status lbk_gmres_restart_cycle_csr(lbk_ctx ctx, const lbk_csr* A, const double* b, double* x,
                                       int32_t restart, double* basis_out, int32_t basis_cap,
                                       lbk_gmres_cycle_result* result)
{
    if (!ctx || !A || !result) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(restart >= 1, LBK_CONFIGURATION_ERROR, "restart must be positive");
        need(A->dtype == LBK_F64, LBK_TYPE_ERROR, "gmres_restart_cycle: FP64 matrices only");
        need(A->nrows == A->ncols, LBK_SHAPE_ERROR,
             "solve requires a square matrix, got " + std::to_string(A->nrows) + "x" +
                 std::to_string(A->ncols));
        CsrOp op{CsrView<double>{A->nrows, A->ncols, A->nnz, A->row_ptr, A->col_idx,
                                 static_cast<const double*>(A->vals), A->tile_rows, A->ntiles}};
        if (!op.A.tile_rows && A->nrows > 0 && aligned16(A->vals) && aligned16(A->col_idx)) {
            op.A.ntiles = csr_ntiles(A->nnz, A->nrows);
            int* plan = static_cast<int*>(scratch(ctx, size_t(op.A.ntiles + 1) * sizeof(int)));
            csr_plan_launch(ctx, A->row_ptr, A->nrows, A->nnz, plan);
            op.A.tile_rows = plan;
        }
        LocalEnv<CsrOp> env{ctx, op, red_ws(ctx, kRedMaxBlocks, 2), A->nrows, A->nnz};
        // one cycle of `restart` steps, no in-cycle stop (cycle_entry,
        // krylov.cpp:551-565: CycleControl tol = -1)
        lbk_solver_cfg cfg{};
        cfg.kind = 3;
        cfg.max_iters = restart;
        cfg.rel_tol = 1.0;
        cfg.fixed_iters = restart;
        cfg.gmres_restart = restart;
        lbk_solve_result res{};
        CycleOut cyc;
        cyc.basis = basis_out;
        cyc.basis_cap = basis_cap;
        solve_impl(ctx, env, b, x, &cfg, &res, nullptr, 0, &cyc);
        result->rel_residual = cyc.rel;
        result->steps = cyc.steps;
        result->happy_breakdown = cyc.happy;
        result->basis_count = cyc.basis_count;
    });
}

lbk_status lbk_solve_coo(lbk_ctx ctx, const lbk_coo* A, const double* b, double* x,
                         const lbk_solver_cfg* cfg, lbk_solve_result* result, double* history,
                         int32_t history_cap)
{
    if (!ctx || !A) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(A->dtype == LBK_F64, LBK_TYPE_ERROR, "solve: FP64 matrices only");
        need(A->nrows == A->ncols, LBK_SHAPE_ERROR,
             "solve requires a square matrix, got " + std::to_string(A->nrows) + "x" +
                 std::to_string(A->ncols));
        need(A->nnz > 0, LBK_USAGE_ERROR, "solve: COO matrix without entries");
        CooOp op{CooView<double>{A->nrows, A->ncols, A->nnz, A->row_idx, A->col_idx,
                                 static_cast<const double*>(A->vals), A->tile_starts, A->ntiles}};
        if (!op.A.tile_starts) {
            op.A.ntiles = coo_ntiles(A->nnz, A->nrows);
            int* plan = static_cast<int*>(scratch(ctx, size_t(op.A.ntiles + 1) * sizeof(int)));
            coo_plan_launch(ctx, A->row_idx, A->nrows, A->nnz, plan);
            op.A.tile_starts = plan;
        }
        LocalEnv<CooOp> env{ctx, op, red_ws(ctx, kRedMaxBlocks, 2), A->nrows, A->nnz};
        solve_impl(ctx, env, b, x, cfg, result, history, history_cap);
    });
}

lbk_status lbk_dist_solve(lbk_ctx ctx, lbk_dist_csr D, lbk_comm comm, const double* b, double* x,
                          const lbk_solver_cfg* cfg, lbk_solve_result* result, double* history,
                          int32_t history_cap)
{
    if (!ctx || !D) return LBK_USAGE_ERROR;
    return guard(ctx, [&] {
        need(D->P == 1 || (comm && comm->impl->nranks == D->P && comm->impl->rank == D->rank),
             LBK_USAGE_ERROR, "dist solve: communicator does not match the partition");
        DistEnv env{ctx, D, comm ? comm->impl : nullptr, red_ws(ctx, kRedMaxBlocks, 2)};
        if constexpr (kExactRed)  // the deferred slots start every solve at zero
            LBK_CUDA(cudaMemsetAsync(env.ws.xout, 0, size_t(kXOutSlots) * kXSlot * sizeof(long long),
                                     ctx->stream));
        solve_impl(ctx, env, b, x, cfg, result, history, history_cap);
    });
}

}  // extern "C"

#ifdef LBK_XRED_STATS
// dev builds only (scripts/variants.sh LBK_XRED_STATS): exact-reduction
// lane statistics of the solver kernels {flushes, slides, re-centres, -}
extern "C" int lbk_dbg_xred_stats(unsigned long long* out, int reset)
{
    cudaMemcpyFromSymbol(out, lbk::g_xred_stats, sizeof(unsigned long long) * 4);
    if (reset) {
        unsigned long long z[4] = {0, 0, 0, 0};
        cudaMemcpyToSymbol(lbk::g_xred_stats, z, sizeof(z));
    }
    return 0;
}
#endif
