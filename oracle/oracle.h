/*
 * oracle.h - CPU restatement of the reference's block-Toeplitz matvec and
 * restarted GMRES. TEST INFRASTRUCTURE ONLY: imported by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs, always as the checker or the timed CPU baseline, never as the
 * product path.
 *
 * Every function restates the reference file:line named beside it
 * (/root/reference/proj/...). Pinning status:
 *  - fftInPlace: PINNED bit-exactly against the reference's own fft.cpp,
 *    compiled into oracle/_ref (tests/test_oracle.py, tests/golden/).
 *  - applyA / gmres: PARITY UNPINNED against reference outputs -- the
 *    reference linsolve.cpp needs Eigen3, which is absent here, and no
 *    golden vectors exist; checked instead against SPEC.md's known-answer
 *    properties with an independent dense numpy product / LU solve.
 * The synthetic nine-component correction is not reference code; it is the
 * BASELINE.json perturbation, defined in include/tbt_gen.h.
 */
#ifndef TBT_ORACLE_H
#define TBT_ORACLE_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_op orc_op;

/* nextPow2 (proj/src/fft.cpp:22-26). */
size_t orc_next_pow2(size_t n);
/* fftInPlace (proj/src/fft.cpp:28-53); returns 1 for non-power-of-two. */
int orc_fft(double* a, size_t n, int inverse);

/* Operator over canonical Sparse generator blocks (toeplitz.hpp:72-74,
 * order toeplitz.cpp:305-312), m x m column-major complex each. The blocks
 * are copied. */
orc_op* orc_create(int nx, int ny, int m, const double* blocks);
/* FULL generator layout (every shift, non-reciprocal): (2ny-1)(2nx-1)
 * blocks, i = 1-ny..ny-1 outer, j = 1-nx..nx-1 inner, m x m column-major. */
orc_op* orc_create_full(int nx, int ny, int m, const double* blocks);
void orc_destroy(orc_op* op);

/* buildASpectra (proj/src/linsolve.cpp:239-258), optionally threaded over
 * (m, n) entries (the reference is serial; results are identical). */
int orc_precompute(orc_op* op, int nthreads);
/* Copies ahat in the reference layout [(m*e5+n)*L + f] (linsolve.cpp:147). */
int orc_ahat(const orc_op* op, double* out);
long long orc_bins(const orc_op* op); /* L = L1*L0 */

/* Nine-component correction: 40 slots (see tbt_gen.h), rank r. */
int orc_set_correction(orc_op* op, int rank, const double* d, const double* u,
                       const double* v);

/* applyA (linsolve.cpp:260-290): pure two-level Toeplitz product. */
/* Margin coupling B/B^T/C (row f1), tbt_gen.h layouts; apply, diagonal and
 * gmres then act on nA + nM unknowns (orc_size). */
int orc_set_margin(orc_op* op, const int* e, const double* bside, const double* brow, const double* bcorner,
                   const double* c);
/* SemiSparse margin coupling (linsolve.cpp:294,318,338): dense B (nM x nA)
 * and C (nM x nM), column-major. */
int orc_set_margin_dense(orc_op* op, const int* e, const double* bfull, const double* c);
long long orc_size(const orc_op* op);

int orc_apply_a(const orc_op* op, const double* x, double* y);
/* Full synthetic operator y = A x + correction (the role of
 * ToeplitzMatvec::apply, linsolve.cpp:373-388). */
int orc_apply(const orc_op* op, const double* x, double* y);
/* ncols independent applies (apply, or applyA when a_only) split over
 * nthreads std::threads, one column per task (the reference's per-column
 * parallelFor, linsolve.cpp:572). X, Y are n x ncols column-major. */
int orc_apply_cols(const orc_op* op, const double* x, double* y, int ncols,
                   int nthreads, int a_only);
/* Direct spatial product for selected target elements, no FFT:
 * y[k*m ..] = sum_e' Z(e_k, e') x(e') (+ correction). Works without
 * orc_precompute at any size. */
int orc_apply_rows(const orc_op* op, const double* x, const long long* elems,
                   long long count, double* y);
/* Dense Z (N x N column-major); only for small N. */
/* Bounded CPU sample of applyA at sizes whose spectra do not fit host memory:
 * the forward transforms of x and the per-row work of nrows output rows whose
 * block row / column lines (tbtgen_block_lines) are given; timed sections in
 * seconds (single thread), y[r * nx*ny + e]. */
int orc_sampled_apply(int nx, int ny, int m, int nrows, const double* const* row_lines,
                      const double* const* col_lines, const double* x, double* y, double* t_fwd, double* t_rows,
                      int nthreads);
int orc_dense(const orc_op* op, double* z);
/* Diagonal of the operator (ToeplitzMatvec::diagonal, linsolve.cpp:390-408,
 * plus the correction's diagonal). */
int orc_diagonal(const orc_op* op, double* d);

/* iterativeSolve (linsolve.cpp:551-593) over gmres (linsolve.cpp:425-515),
 * without the throw: per column iterations / final relative residual /
 * converged flag, and a history of (kind, value) pairs:
 * kind 0 = true relative residual at a restart (linsolve.cpp:447-448),
 * kind 1 = |g_{j+1}| / beta_0 after inner iteration (linsolve.cpp:489-492;
 *          beta_0 = first cycle's preconditioned residual, so late cycles
 *          are not rescaled by their own small beta),
 * kind 2 = final true residual once maxIter is exhausted (linsolve.cpp:512).
 * hist has hist_cap pairs per column; hist_len gets the count per column.
 * use_a_only selects applyA as the operator (schurSolve's inner solve,
 * linsolve.cpp:644). nthreads splits columns (parallelFor, mesh.cpp:27-53). */
int orc_gmres(const orc_op* op, const double* b, double* x, int ncols,
              double tol, int max_iter, int restart, int precondition,
              int use_a_only, int nthreads, int* iterations, double* residual,
              int* converged, double* hist, int hist_cap, int* hist_len);

/* schurSolve (linsolve.cpp:595-682) on the margin representation: A-only
 * GMRES for [V1, B^T], S = C - B F, partial-pivot LU with the pivot-ratio
 * check, I2 = -S^-1 B U, I1 = U - F I2. b, x: (nA+nM) x ncols column-major.
 * Returns 0, 1 (user error) or 2 (numeric error), message in err. */
int orc_schur(const orc_op* op, const double* b, double* x, int ncols, double tol, int max_iter, int restart,
              int precondition, int nthreads, int* iterations, double* residual, char* err, int errcap);

/* portNetwork (postproc.cpp:186-230) and arrayFarfield /
 * embeddedElementPatterns (:134-184), restated for row f4. */
int orc_port_network(const double* current, long long ld, int p, const long long* feed, double len,
                     const double* z0, double* y, double* z, double* s);
int orc_array_farfield(int nx, int ny, const int* e, const double* const* tco, const double* const* tcx, int ndir,
                       const double* dirs, double dx, double dy, double k, double eta, const double* current, int p,
                       const double* weights, int q, double* co, double* cx);

#ifdef __cplusplus
}
#endif

#endif /* TBT_ORACLE_H */
