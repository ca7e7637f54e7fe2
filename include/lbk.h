/* include/lbk.h -- C ABI of the B200 sparse backend ("lbk").
 *
 * This is the drop-in boundary for the reference's SpMV/Krylov hot path
 * (reference = /root/reference/proj, "larch").  Every entry point names the
 * reference interface it replaces (file:line, relative to that tree).
 *
 * Conventions
 *  - C linkage, plain pointers and sizes, no C++ or torch types.
 *  - Every function returns an lbk_status; lbk_last_error(ctx) gives the
 *    message (ctx may be NULL for errors raised before a context exists).
 *    Status codes map 1:1 onto the reference's exception taxonomy
 *    (include/larch/core/error.hpp:16-131).  No exception crosses the ABI.
 *  - Matrix descriptors are plain structs of DEVICE pointers borrowed (not
 *    owned) by the call.  Vectors are device pointers.  Kernels never
 *    allocate their outputs (reference kernels.hpp:76-97 contract).
 *  - One lbk_ctx is bound to one device and one CUDA stream; calls on a ctx
 *    are stream-ordered and not re-entrant across threads.  SpMV / BLAS-1 /
 *    conversion calls are asynchronous on that stream; calls that return a
 *    host value (dot/nrm2 to host, solve, ell_width, sellp_plan, validate)
 *    synchronise the stream before returning.  The reference's wrappers are
 *    synchronous (dispatch.cpp:112-117); lbk_sync(ctx) restores that.
 *  - Indices are int32 (reference SPEC.md:359); nnz is int64 in the
 *    descriptors so sizes above 2^31 are rejected cleanly, not wrapped.
 */
#ifndef LBK_H
#define LBK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------- status */
/* error.hpp:16-131 -> status codes */
typedef enum lbk_status {
    LBK_OK = 0,
    LBK_SHAPE_ERROR = 1,           /* ShapeError           error.hpp:49 */
    LBK_PLACEMENT_ERROR = 2,       /* PlacementError       error.hpp:63 */
    LBK_TYPE_ERROR = 3,            /* TypeError            error.hpp:56 */
    LBK_DISPATCH_ERROR = 4,        /* DispatchError        error.hpp:78 */
    LBK_USAGE_ERROR = 5,           /* UsageError           error.hpp:71 */
    LBK_CONFIGURATION_ERROR = 6,   /* ConfigurationError   error.hpp:23 */
    LBK_OUT_OF_MEMORY = 7,         /* OutOfMemoryError     error.hpp:30 */
    LBK_FORMAT_ERROR = 8,          /* FormatError          error.hpp:100 */
    LBK_BREAKDOWN = 9,             /* BreakdownError       error.hpp:115 */
    LBK_BENCHMARK_INTEGRITY = 10,  /* BenchmarkIntegrityError error.hpp:128 */
    LBK_UNSUPPORTED_FORMAT = 11,   /* UnsupportedFormatError (a FormatError) error.hpp:108 */
    LBK_CUDA_ERROR = 20,           /* device/runtime failure (new) */
    LBK_NCCL_ERROR = 21,           /* collective failure (new) */
    LBK_INTERNAL = 99
} lbk_status;

typedef enum lbk_dtype { LBK_F64 = 0, LBK_F32 = 1 } lbk_dtype;

/* ------------------------------------------------------------ context */
/* Replaces the Executor seam: executor.hpp:130-170 (kind/synchronize/
 * raw_alloc with arena capacity -> OutOfMemoryError) and create_executor
 * executor.hpp:261-262. */
typedef struct lbk_ctx_s* lbk_ctx;

lbk_status lbk_ctx_create(int device, lbk_ctx* out);
/* Bind to an existing cudaStream_t (e.g. torch.cuda.current_stream()). */
lbk_status lbk_ctx_create_on_stream(int device, void* cuda_stream, lbk_ctx* out);
lbk_status lbk_ctx_set_stream(lbk_ctx ctx, void* cuda_stream);
lbk_status lbk_ctx_destroy(lbk_ctx ctx);
const char* lbk_last_error(lbk_ctx ctx);
/* Executor::synchronize (executor.hpp:146). */
lbk_status lbk_sync(lbk_ctx ctx);
/* Number of SMs, device id, arena accounting (executor.hpp:150-160). */
lbk_status lbk_ctx_info(lbk_ctx ctx, int* device, int* num_sms,
                        size_t* arena_capacity, size_t* arena_used);
lbk_status lbk_ctx_set_arena_capacity(lbk_ctx ctx, size_t bytes);
/* L2 access-policy window over the SpMV's gathered vector x (persisting,
 * per launch via cudaLaunchAttributeAccessPolicyWindow).  Default off
 * (env LBK_L2_PERSIST=1 turns it on at context creation). */
lbk_status lbk_ctx_set_l2_persist(lbk_ctx ctx, int on);
/* Executor::raw_alloc / raw_free (executor.cpp:254-279): device memory,
 * 256-B aligned, LBK_OUT_OF_MEMORY past the arena capacity. */
lbk_status lbk_alloc(lbk_ctx ctx, size_t bytes, void** out);
lbk_status lbk_free(lbk_ctx ctx, void* ptr, size_t bytes);
/* copy()/array_from_host/array_to_host (device_array.cpp:144-263); device
 * to device across GPUs is a direct peer copy, not 3-hop master staging.
 * All copies are stream-ordered on the context's stream (asynchronous with
 * pinned host memory): lbk_sync before reading a host destination. */
lbk_status lbk_memcpy_h2d(lbk_ctx ctx, void* dst, const void* src, size_t bytes);
lbk_status lbk_memcpy_d2h(lbk_ctx ctx, void* dst, const void* src, size_t bytes);
lbk_status lbk_memcpy_d2d(lbk_ctx ctx, void* dst, const void* src, size_t bytes);
/* explicit GPU -> GPU copy (NVLink P2P where enabled), stream-ordered */
lbk_status lbk_memcpy_peer(lbk_ctx ctx, void* dst, int dst_device, const void* src,
                           int src_device, size_t bytes);

/* ---------------------------------------------------------- matrices */
/* CsrMatrix (formats.hpp:65-76).  `tile_rows` is an optional load-balance
 * plan from lbk_csr_plan(); when NULL the SpMV builds it per call. */
typedef struct lbk_csr {
    int32_t nrows, ncols;
    int64_t nnz;
    lbk_dtype dtype;
    const int32_t* row_ptr;  /* nrows + 1 */
    const int32_t* col_idx;  /* nnz */
    const void* vals;        /* nnz, double or float */
    const int32_t* tile_rows; /* optional plan, see lbk_csr_plan */
    int32_t ntiles;
} lbk_csr;

/* CooMatrix (formats.hpp:49-60): sorted by (row, col), unique. */
typedef struct lbk_coo {
    int32_t nrows, ncols;
    int64_t nnz;
    lbk_dtype dtype;
    const int32_t* row_idx;
    const int32_t* col_idx;
    const void* vals;
    const int32_t* tile_starts; /* optional plan, see lbk_coo_plan */
    int32_t ntiles;
} lbk_coo;

/* ELL, Ginkgo column-major (new): entry (r, j) at
 * j*stride + r, padding column -1 / value 0. */
typedef struct lbk_ell {
    int32_t nrows, ncols;
    int64_t nnz;      /* logical nonzeros (flop accounting) */
    lbk_dtype dtype;
    int32_t width;
    int64_t stride;   /* >= nrows */
    const int32_t* col_idx;  /* width * stride */
    const void* vals;
} lbk_ell;

/* SELL-P (new; App. B): slice size S, entry (r, j) at
 * (slice_sets[r/S] + j)*S + r%S, padding column -1 / value 0. */
typedef struct lbk_sellp {
    int32_t nrows, ncols;
    int64_t nnz;
    lbk_dtype dtype;
    int32_t slice_size;
    int32_t nslices;
    const int32_t* slice_lengths; /* nslices */
    const int32_t* slice_sets;    /* nslices + 1 */
    const int32_t* col_idx;       /* slice_sets[nslices] * S */
    const void* vals;
    int64_t stored;               /* slice_sets[nslices] * S, or 0 (read on demand) */
    const int32_t* tile_slices;   /* optional plan (S == 32), see lbk_sellp_plan */
    int32_t ntiles;
} lbk_sellp;

/* ------------------------------------------------------------- SpMV */
/* spmv_csr / spmv_coo (kernels.hpp:94-97, api.cpp:113-140): y <- A x,
 * overwrite, empty rows -> 0.  Shape checks raise LBK_SHAPE_ERROR
 * (api.cpp:27-33); a descriptor dtype that does not match the entry point
 * raises LBK_TYPE_ERROR.  The _adv variants are the north star's "advanced
 * apply" y <- alpha A x + beta y (absent from the reference; beta == 0 does
 * not read y). */
lbk_status lbk_spmv_csr_f64(lbk_ctx, const lbk_csr* A, const double* x, double* y);
lbk_status lbk_spmv_csr_f32(lbk_ctx, const lbk_csr* A, const float* x, float* y);
lbk_status lbk_spmv_csr_adv_f64(lbk_ctx, double alpha, const lbk_csr* A,
                                const double* x, double beta, double* y);
lbk_status lbk_spmv_csr_adv_f32(lbk_ctx, float alpha, const lbk_csr* A,
                                const float* x, float beta, float* y);
lbk_status lbk_spmv_coo_f64(lbk_ctx, const lbk_coo* A, const double* x, double* y);
lbk_status lbk_spmv_coo_f32(lbk_ctx, const lbk_coo* A, const float* x, float* y);
lbk_status lbk_spmv_coo_adv_f64(lbk_ctx, double alpha, const lbk_coo* A,
                                const double* x, double beta, double* y);
lbk_status lbk_spmv_coo_adv_f32(lbk_ctx, float alpha, const lbk_coo* A,
                                const float* x, float beta, float* y);
lbk_status lbk_spmv_ell_f64(lbk_ctx, const lbk_ell* A, const double* x, double* y);
lbk_status lbk_spmv_ell_f32(lbk_ctx, const lbk_ell* A, const float* x, float* y);
lbk_status lbk_spmv_ell_adv_f64(lbk_ctx, double alpha, const lbk_ell* A,
                                const double* x, double beta, double* y);
lbk_status lbk_spmv_ell_adv_f32(lbk_ctx, float alpha, const lbk_ell* A,
                                const float* x, float beta, float* y);
lbk_status lbk_spmv_sellp_f64(lbk_ctx, const lbk_sellp* A, const double* x, double* y);
lbk_status lbk_spmv_sellp_f32(lbk_ctx, const lbk_sellp* A, const float* x, float* y);
lbk_status lbk_spmv_sellp_adv_f64(lbk_ctx, double alpha, const lbk_sellp* A,
                                  const double* x, double beta, double* y);
lbk_status lbk_spmv_sellp_adv_f32(lbk_ctx, float alpha, const lbk_sellp* A,
                                  const float* x, float beta, float* y);

/* Load-balance plans (Ginkgo's "strategy" objects; the reference has none).
 * CSR: nnz-balanced row tiles; tile_rows needs lbk_csr_plan_size() int32s.
 * COO: row-aligned entry tiles. */
lbk_status lbk_csr_plan_size(const lbk_csr* A, int32_t* ntiles_out);
lbk_status lbk_csr_plan(lbk_ctx, const lbk_csr* A, int32_t* tile_rows_dev);
lbk_status lbk_coo_plan_size(const lbk_coo* A, int32_t* ntiles_out);
/* SELL-P (slice_size 32): tiles of whole slices for the warp-pipelined
 * kernel; tile_slices needs ntiles + 1 int32s; A->stored must be set. */
lbk_status lbk_sellp_plan_size(const lbk_sellp* A, int32_t* ntiles_out);
lbk_status lbk_sellp_plan(lbk_ctx, const lbk_sellp* A, int32_t* tile_slices_dev);
lbk_status lbk_coo_plan(lbk_ctx, const lbk_coo* A, int32_t* tile_starts_dev);

/* ------------------------------------------------------------ BLAS-1 */
/* kernels.hpp:79-91, api.cpp:69-110.  Reductions are exactly rounded:
 * dot = RNE(sum_i RN(x_i y_i)), accumulated as integers (csrc/xred.cuh),
 * so the result depends on neither the launch configuration nor, in the
 * distributed solver, the partition -- bitwise reproducible everywhere
 * (the reference's sequential and chunked sums, reference.cpp:46-56 /
 * parallel.cpp:76-97, are two roundings of the same exact value). */
lbk_status lbk_axpy_f64(lbk_ctx, int64_t n, double alpha, const double* x, double* y);
lbk_status lbk_scal_f64(lbk_ctx, int64_t n, double alpha, double* x);
lbk_status lbk_fill_f64(lbk_ctx, int64_t n, double value, double* x);
lbk_status lbk_copy_f64(lbk_ctx, int64_t n, const double* x, double* y);
/* result to HOST (synchronises) */
lbk_status lbk_dot_f64(lbk_ctx, int64_t n, const double* x, const double* y, double* result);
lbk_status lbk_nrm2_f64(lbk_ctx, int64_t n, const double* x, double* result);
/* result to DEVICE memory (stream-ordered, no sync) */
lbk_status lbk_dot_f64_dev(lbk_ctx, int64_t n, const double* x, const double* y, double* result_dev);

/* Bandwidth calibration (the reference's stream kernels, reference.cpp:92-130,
 * and measure_peak_bandwidth, harness.cpp:125-141): c <- a (16 n bytes),
 * a <- b + s c (24 n bytes).  n even, arrays 16-B aligned. */
lbk_status lbk_stream_copy_f64(lbk_ctx, int64_t n, const double* a, double* c);
lbk_status lbk_stream_triad_f64(lbk_ctx, int64_t n, double scalar, const double* b,
                                const double* c, double* a);
/* the rest of the reference's StreamOp set (kernels.hpp:58-68,
 * reference.cpp:104-120): b <- s c (16 n bytes), c <- a + b (24 n bytes),
 * sum a_i b_i to HOST (16 n bytes; exactly rounded, synchronises). */
lbk_status lbk_stream_mul_f64(lbk_ctx, int64_t n, double scalar, const double* c, double* b);
lbk_status lbk_stream_add_f64(lbk_ctx, int64_t n, const double* a, const double* b, double* c);
lbk_status lbk_stream_dot_f64(lbk_ctx, int64_t n, const double* a, const double* b,
                              double* result);
/* flops_sweep (kernels.hpp:70-73, reference.cpp:124-130, fma_chain.hpp):
 * x_i <- fma_chain(x_i, fma_per_element), bit-identical to the reference
 * (2 flops per step, 16 n bytes per call). */
lbk_status lbk_flops_sweep_f64(lbk_ctx, int64_t n, int32_t fma_per_element, double* x);

/* ------------------------------------------------------- conversions */
/* coo_to_csr (formats.cpp:132-155): row histogram + scan; col/vals are
 * identical to the COO arrays (CSR inherits COO order), so only row_ptr is
 * produced. */
lbk_status lbk_coo_to_csr(lbk_ctx, const lbk_coo* A, int32_t* row_ptr_out);
/* csr_to_coo (formats.cpp:158-179): expand row_ptr into row indices. */
lbk_status lbk_csr_to_coo(lbk_ctx, const lbk_csr* A, int32_t* row_idx_out);
/* coo_from_entries (formats.cpp:78-116): bounds check (FormatError),
 * stable sort by (row, col), duplicates summed in input order, explicit
 * zeros kept.  Inputs/outputs are device arrays of length n; *nnz_out
 * (host) receives the canonical count.  Synchronises. */
lbk_status lbk_coo_assemble_f64(lbk_ctx, int32_t nrows, int32_t ncols, int64_t n,
                                const int32_t* rows, const int32_t* cols,
                                const double* vals, int32_t* rows_out,
                                int32_t* cols_out, double* vals_out,
                                int64_t* nnz_out);
/* ELL: width = max row length (synchronises). */
lbk_status lbk_csr_ell_width(lbk_ctx, const lbk_csr* A, int32_t* width_out);
lbk_status lbk_csr_to_ell(lbk_ctx, const lbk_csr* A, int32_t width, int64_t stride,
                          int32_t* cols_out, void* vals_out);
/* SELL-P: slice_lengths[nslices], slice_sets[nslices+1] (device), stored
 * element count to host (synchronises); then the fill. */
lbk_status lbk_csr_sellp_plan(lbk_ctx, const lbk_csr* A, int32_t slice_size,
                              int32_t* slice_lengths_out, int32_t* slice_sets_out,
                              int64_t* stored_out);
lbk_status lbk_csr_to_sellp(lbk_ctx, const lbk_csr* A, int32_t slice_size,
                            const int32_t* slice_sets, int32_t* cols_out,
                            void* vals_out);
/* validate(Csr/Coo) (formats.cpp:182-242): LBK_FORMAT_ERROR on violation. */
lbk_status lbk_validate_csr(lbk_ctx, const lbk_csr* A);
lbk_status lbk_validate_coo(lbk_ctx, const lbk_coo* A);

/* MatrixMarket ingestion (read_matrix_market, reference io.hpp:25-28 /
 * io.cpp:71-191): host parse with the reference's acceptance rules and
 * messages; the entry list (symmetric files expanded, 0-based) is then
 * assembled on the device with lbk_coo_assemble_f64.  lbk_mm_read returns
 * LBK_FORMAT_ERROR / LBK_UNSUPPORTED_FORMAT with lbk_mm_last_error(). */
typedef struct lbk_mm_s* lbk_mm;
lbk_status lbk_mm_read(const char* path, lbk_mm* out);
const char* lbk_mm_last_error(void);
lbk_status lbk_mm_info(lbk_mm m, int32_t* nrows, int32_t* ncols, int64_t* n_entries);
/* host pointers owned by the handle, valid until lbk_mm_free */
lbk_status lbk_mm_entries(lbk_mm m, const int32_t** rows, const int32_t** cols, const double** vals);
lbk_status lbk_mm_free(lbk_mm m);

/* ----------------------------------------------------------- solvers */
/* SolverConfig / SolveResult (krylov.hpp:22-44).  kind: 0 = CG, 1 =
 * BiCGSTAB, 2 = CGS, 3 = restarted GMRES (krylov.hpp:17).
 * residual_mode 0 = reference semantics: true residual ||b - A x||/||b||
 * recomputed every iteration (krylov.cpp:77-84, 145, 221); 1 = recurrence
 * residual for the stopping test, with the true residual verified before
 * convergence is declared (iteration continues if verification fails). */
typedef struct lbk_solver_cfg {
    int32_t kind;
    int32_t max_iters;     /* default 1000 */
    double rel_tol;        /* default 1e-10 */
    int32_t fixed_iters;   /* <= 0: unset */
    int32_t residual_mode; /* 0 true residual each iteration, 1 recurrence */
    int32_t gmres_restart; /* kind 3: Krylov basis per cycle, [1, max_iters] (krylov.hpp:28) */
} lbk_solver_cfg;

typedef struct lbk_solve_result {
    int32_t converged;
    int32_t iterations;
    double final_rel_residual;
    double elapsed;          /* seconds, device-timed */
    int64_t flop_count;      /* reference accounting, krylov.cpp:41-69 */
    int32_t breakdown_iter;  /* >0 when LBK_BREAKDOWN is returned */
    int32_t history_len;     /* iterations + 1 */
} lbk_solve_result;

/* solve(A, b, x, cfg) (krylov.hpp:53-56, krylov.cpp:446-512, 587-598).
 * x is the initial guess on entry and the solution on exit (device).
 * history (HOST, may be NULL) receives min(history_len, history_cap)
 * entries.  Validation errors as solve_impl (krylov.cpp:449-472).
 * Breakdown -> LBK_BREAKDOWN with result->breakdown_iter set. */
lbk_status lbk_solve_csr(lbk_ctx, const lbk_csr* A, const double* b, double* x,
                         const lbk_solver_cfg* cfg, lbk_solve_result* result,
                         double* history, int32_t history_cap);
lbk_status lbk_solve_coo(lbk_ctx, const lbk_coo* A, const double* b, double* x,
                         const lbk_solver_cfg* cfg, lbk_solve_result* result,
                         double* history, int32_t history_cap);

/* gmres_restart_cycle (krylov.hpp:62-89, krylov.cpp:308-406, 551-565): one
 * restarted-GMRES cycle of `restart` steps from the x passed in (updated in
 * place), no in-cycle stopping test; a subdiagonal below 1e-14 ends the
 * cycle early (happy breakdown).  rel_residual = ||b - A x|| / ||b|| after
 * the cycle (||b|| = 1 when b = 0).  basis_out (DEVICE, may be NULL)
 * receives the cycle's orthonormal basis, basis_count vectors of nrows
 * (steps + 1, or steps after a happy breakdown); basis_cap = vectors it
 * holds. */
typedef struct lbk_gmres_cycle_result {
    double rel_residual;
    int32_t steps;
    int32_t happy_breakdown;
    int32_t basis_count;
} lbk_gmres_cycle_result;
lbk_status lbk_gmres_restart_cycle_csr(lbk_ctx, const lbk_csr* A, const double* b, double* x,
                                       int32_t restart, double* basis_out, int32_t basis_cap,
                                       lbk_gmres_cycle_result* result);

/* ------------------------------------------------- distributed (new) */
/* Row-partitioned CSR over P ranks (the reference has no
 * distributed matrix).  Partition: contiguous row blocks,
 * rank(r) = min(r / ceil(N/P), P-1).  Host-side maps (no device needed):
 * build the map from the rank's own rows (global column ids), exchange
 * ghost lists with the peers (an all-to-all the caller runs over its own
 * bootstrap, e.g. torch.distributed), hand the requests back with
 * lbk_dist_map_set_sends, then create the device matrix.  Vectors the
 * operator is applied to must hold n_local + n_ghost doubles (the halo
 * lands behind the owned part). */
typedef struct lbk_dist_map_s* lbk_dist_map;
typedef struct lbk_dist_csr_s* lbk_dist_csr;
typedef struct lbk_comm_s* lbk_comm;
typedef struct lbk_dist_map_info_t {
    int32_t begin, end, n_local, n_ghost, n_interior, n_boundary;
    int64_t nnz_local;
    int32_t n_send; /* -1 until lbk_dist_map_set_sends */
} lbk_dist_map_info_t;

lbk_status lbk_part_range(int32_t n, int32_t nparts, int32_t rank, int32_t* begin, int32_t* end);
/* row_ptr: local, n_local + 1 entries starting at 0; cols: GLOBAL ids. */
lbk_status lbk_dist_map_create(int32_t n_global, int32_t ncols_global, int32_t nparts,
                               int32_t rank, int32_t n_local, const int32_t* row_ptr,
                               const int32_t* cols, lbk_dist_map* out);
lbk_status lbk_dist_map_info(lbk_dist_map m, lbk_dist_map_info_t* info);
/* ghosts: sorted global ids [n_ghost]; ghost_off [nparts+1]: the ghosts
 * owned by rank q are ghosts[ghost_off[q] .. ghost_off[q+1]). */
lbk_status lbk_dist_map_ghosts(lbk_dist_map m, int32_t* ghosts, int32_t* ghost_off);
/* local column ids: owned c -> c - begin, ghost -> n_local + ghost index. */
lbk_status lbk_dist_map_local_cols(lbk_dist_map m, int32_t* local_cols);
lbk_status lbk_dist_map_rows(lbk_dist_map m, int32_t* interior, int32_t* boundary);
/* req_off[nparts+1], req_gids: the global ids peer q requested from this
 * rank (q's ghost_off run for this rank), strictly increasing per peer. */
lbk_status lbk_dist_map_set_sends(lbk_dist_map m, const int32_t* req_off, const int32_t* req_gids);
lbk_status lbk_dist_map_sends(lbk_dist_map m, int32_t* send_off, int32_t* send_idx);
lbk_status lbk_dist_map_destroy(lbk_dist_map m);

/* Communicators: NCCL (one process per GPU; the 128-byte unique id comes
 * from rank 0 over the caller's bootstrap) or an in-process thread group
 * (P host threads, each with its own lbk_ctx; used for P virtual ranks on
 * one device and for single-process multi-GPU). */
lbk_status lbk_comm_nccl_unique_id(void* id_out /* 128 bytes */);
lbk_status lbk_comm_init_nccl(const void* id, int32_t nranks, int32_t rank, int32_t device,
                              lbk_comm* out);
lbk_status lbk_comm_init_threads(int32_t nranks, lbk_comm* comms_out /* [nranks] */);
/* Peer-memory group (new; csrc/peer.cuh): every rank maps every peer's
 * device window, and the halo exchange and the solver's scalar reductions
 * run as lbk's own kernels storing over NVLink -- no NCCL on the iteration
 * path, CUDA-graph capturable, the solver's reductions exactly rounded
 * over all ranks (same bits on every rank and at every rank count).  halo_cap = the largest per-peer ghost count of any rank
 * (equal on all ranks).  One process per GPU: init, publish the 64-byte
 * IPC handle over the caller's bootstrap, open all handles (nranks x 64
 * bytes, in rank order).  In-process: lbk_comm_init_peer_group, one
 * distinct device per rank (ranks sharing a context could deadlock: a
 * kernel spinning on a peer's flag blocks device-synchronising calls of
 * the peer's host thread).  Several ranks on one GPU need one process
 * each.  At most 16 ranks.  Destroying a peer communicator is collective
 * (peers may still be storing into its window until they finish). */
lbk_status lbk_comm_init_peer(int32_t nranks, int32_t rank, int32_t device, int64_t halo_cap,
                              lbk_comm* out);
lbk_status lbk_comm_peer_handle(lbk_comm comm, void* handle_out /* 64 bytes */);
lbk_status lbk_comm_peer_open(lbk_comm comm, const void* handles /* nranks * 64 bytes */);
lbk_status lbk_comm_init_peer_group(int32_t nranks, const int32_t* devices, int64_t halo_cap,
                                    lbk_comm* comms_out /* [nranks] */);
/* Wait for the context's stream and report a communicator failure (NCCL
 * async error, peer timeout) as LBK_NCCL_ERROR. */
lbk_status lbk_comm_sync(lbk_ctx ctx, lbk_comm comm);
lbk_status lbk_comm_destroy(lbk_comm c);
lbk_status lbk_comm_allreduce_sum_f64(lbk_ctx ctx, lbk_comm comm, double* dev, int32_t count);

/* Device matrix from the map + this rank's row_ptr (local) and values
 * (HOST arrays); n_global_nnz feeds the reference flop accounting. */
lbk_status lbk_dist_csr_create(lbk_ctx ctx, lbk_dist_map m, const int32_t* row_ptr,
                               const double* vals, int64_t n_global_nnz, lbk_dist_csr* out);
lbk_status lbk_dist_csr_info(lbk_dist_csr D, int32_t* n_local, int32_t* n_ghost);
lbk_status lbk_dist_csr_destroy(lbk_dist_csr D);
/* y[n_local] <- A x; x_ext[n_local + n_ghost] (halo filled by the call).
 * Peer communicator: pack + store into the neighbours' windows -> interior
 * rows -> wait + unpack -> boundary rows, all on the context's stream.
 * NCCL: pack -> ncclSend/ncclRecv on a comm stream overlapped with the
 * interior rows -> boundary rows.  Collective: every rank calls it, on the
 * same context stream every time (the peer epochs are per stream order). */
lbk_status lbk_dist_spmv_f64(lbk_ctx ctx, lbk_dist_csr D, lbk_comm comm, double* x_ext, double* y);
/* Distributed solve (CG / BiCGSTAB / CGS / GMRES, lbk_solver_cfg as
 * lbk_solve_csr): b, x are the rank's n_local parts.  Dot products are
 * exactly rounded over all ranks, so every rank sees the same iterations,
 * history and result -- and they are the single-GPU lbk_solve_csr bits for
 * any number of ranks and any row partition.  Collective. */
lbk_status lbk_dist_solve(lbk_ctx ctx, lbk_dist_csr D, lbk_comm comm, const double* b, double* x,
                          const lbk_solver_cfg* cfg, lbk_solve_result* result, double* history,
                          int32_t history_cap);

/* ------------------------------------------------ synthetic inputs */
/* Benchmark configurations; input synthesis, not
 * part of the measured path.  kind 0 = 2D 5-pt (m x m), 1 = 3D 7-pt
 * (m^3, upwind gamma), 2 = 3D 27-pt (m^3); rows r = (k*m + i)*m + j,
 * ascending columns.  Device arrays sized by lbk_gen_stencil_nnz. */
int64_t lbk_gen_stencil_nnz(int kind, int m);
lbk_status lbk_gen_stencil_csr(lbk_ctx, int kind, int m, double gamma, int32_t* row_ptr,
                               int32_t* cols, double* vals);
/* seeded_values (reference src/bench/harness.cpp:90-99): mt19937_64(seed),
 * uniform_real_distribution(-1,1), HOST output. */
void lbk_gen_seeded_values(int64_t n, uint64_t seed, double* out);
/* App. B power-law generator (HOST); handle -> fill -> free. */
void* lbk_gen_powerlaw(int32_t n, uint64_t seed, int32_t max_len, int32_t window, int64_t* nnz);
void lbk_gen_powerlaw_fill(void* h, int32_t* row_ptr, int32_t* cols, double* vals);
void lbk_gen_powerlaw_free(void* h);

#ifdef __cplusplus
}
#endif
#endif /* LBK_H */
