/* oracle/port.h -- TEST INFRASTRUCTURE ONLY (see oracle/README.md).
 *
 * CPU restatement of the SpMV/Krylov hot path of the reference
 * (/root/reference/proj) plus the pieces the reference does not contain and
 * SURVEY.md App. B specifies (ELL, SELL-P, FP32, row partition + halo maps,
 * synthetic generators).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this; the product never links it.
 *
 * Parity status: CSR/COO SpMV and the conversions are pinned against the
 * reference library itself (oracle/_ref, tests/test_oracle.py).  ELL,
 * SELL-P, FP32 and the partition maps have no reference implementation
 * ("parity unpinned" in the reference sense); they are pinned to the App. B
 * integer KATs and cross-checked bit-for-bit against the reference CSR SpMV.
 */
#ifndef LBK_ORACLE_PORT_H
#define LBK_ORACLE_PORT_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- generators ---- */
/* kind: 0 = 2D 5-pt Poisson (m x m), 1 = 3D 7-pt (m^3, gamma), 2 = 3D 27-pt */
int64_t port_stencil_nnz(int kind, int m);
void port_stencil_csr(int kind, int m, double gamma, int32_t* row_ptr,
                      int32_t* cols, double* vals);
/* mt19937_64(seed) + uniform_real_distribution<double>(-1,1), drawn in order
 * (reference src/bench/harness.cpp:90-99). */
void port_seeded_values(int64_t n, uint64_t seed, double* out);
/* power-law generator; returns an opaque handle, nnz via *nnz. */
void* port_powerlaw_new(int32_t n, uint64_t seed, int32_t max_len,
                        int32_t window, int64_t* nnz);
void port_powerlaw_fill(void* h, int32_t* row_ptr, int32_t* cols, double* vals);
void port_free(void* h);

/* ---- SpMV restatements: per row, sum from 0 in ascending k, no FMA ---- */
void port_spmv_csr_f64(int32_t nrows, const int32_t* row_ptr,
                       const int32_t* cols, const double* vals,
                       const double* x, double* y);
void port_spmv_csr_f32(int32_t nrows, const int32_t* row_ptr,
                       const int32_t* cols, const float* vals, const float* x,
                       float* y);
void port_spmv_coo_f64(int32_t nrows, int64_t nnz, const int32_t* rows,
                       const int32_t* cols, const double* vals,
                       const double* x, double* y);
void port_spmv_ell_f64(int32_t nrows, int32_t width, int64_t stride,
                       const int32_t* cols, const double* vals,
                       const double* x, double* y);
void port_spmv_sellp_f64(int32_t nrows, int32_t slice_size,
                         const int32_t* slice_sets, const int32_t* cols,
                         const double* vals, const double* x, double* y);

/* ---- conversions ---- */
int32_t port_csr_max_row(int32_t nrows, const int32_t* row_ptr);
void port_csr_to_ell(int32_t nrows, const int32_t* row_ptr, const int32_t* cols,
                     const double* vals, int32_t width, int64_t stride,
                     int32_t* ell_cols, double* ell_vals);
/* returns stored element count; fills slice_lengths[nslices],
 * slice_sets[nslices+1] when the pointers are non-null. */
int64_t port_sellp_sets(int32_t nrows, const int32_t* row_ptr,
                        int32_t slice_size, int32_t* slice_lengths,
                        int32_t* slice_sets);
void port_csr_to_sellp(int32_t nrows, const int32_t* row_ptr,
                       const int32_t* cols, const double* vals,
                       int32_t slice_size, const int32_t* slice_sets,
                       int32_t* s_cols, double* s_vals);
void port_coo_to_csr(int32_t nrows, int64_t nnz, const int32_t* rows,
                     int32_t* row_ptr);
void port_csr_to_coo(int32_t nrows, const int32_t* row_ptr, int32_t* rows);

/* ---- row partition + halo maps (App. B "Partition maps") ---- */
int32_t port_part_rank_of(int32_t n, int32_t nparts, int32_t row);
void port_part_range(int32_t n, int32_t nparts, int32_t rank, int32_t* begin,
                     int32_t* end);
/* ghosts of `rank`: sorted unique columns outside [begin,end) referenced by
 * its rows.  Returns the ghost count; writes up to cap entries. */
int64_t port_part_ghosts(int32_t n, int32_t nparts, int32_t rank,
                         const int32_t* row_ptr, const int32_t* cols,
                         int32_t* ghosts, int64_t cap);
/* local column ids of the rank's rows: owned c -> c-begin, ghost -> n_local +
 * position in the sorted ghost list. */
void port_part_local_cols(int32_t n, int32_t nparts, int32_t rank,
                          const int32_t* row_ptr, const int32_t* cols,
                          const int32_t* ghosts, int64_t nghost,
                          int32_t* local_cols);

/* ---- BLAS-1 (reference order: sequential) ---- */
double port_dot(int64_t n, const double* x, const double* y);

/* ---- exactly rounded reductions (oracle/xkrylov.cpp) ----
 * RNE(sum of RN(x_i*y_i)): the product's partition-independent reduction. */
double port_xdot(int64_t n, const double* x, const double* y);
double port_xsum(int64_t n, const double* v);
/* krylov.cpp CG (kind 0) / BiCGSTAB (kind 1) with exactly rounded dots.
 * Returns 0, or 3 on BreakdownError (iteration in *bd_iter). */
int port_xsolve(int kind, int32_t n, const int32_t* rp, const int32_t* ci, const double* vals,
                const double* b, double* x, double tol, int max_iters, int fixed_iters,
                double* hist_out, int64_t hist_cap, int* iterations, int* converged,
                int64_t* flops, int* bd_iter);

#ifdef __cplusplus
}
#endif
#endif
