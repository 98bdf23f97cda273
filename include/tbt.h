/*
 * tbt.h - C ABI of the B200 multilevel block-Toeplitz matvec + GMRES
 * (hot path of arXiv 2506.04710, reference "arraymom").
 *
 * Each entry point replaces a reference interface (paths relative to
 * /root/reference/proj):
 *   tbt_create / tbt_set_generators / tbt_precompute
 *       ToeplitzMatvec::ToeplitzMatvec(rep, model)  include/arraymom/linsolve.hpp:61
 *       -> Impl ctor + buildASpectra                  src/linsolve.cpp:160-216,239-258
 *       (generators in the ToeplitzRep Sparse order   include/arraymom/toeplitz.hpp:72-74,
 *        src/toeplitz.cpp:305-312)
 *   tbt_set_correction
 *       the non-Toeplitz edge/corner terms of Z^part (ToeplitzMatvec::apply's
 *       B/B^T/C part, src/linsolve.cpp:384-386); here the BASELINE.json
 *       nine-component diag+rank-r perturbation (include/tbt_gen.h)
 *   tbt_apply        ToeplitzMatvec::apply        linsolve.hpp:64, linsolve.cpp:373-388
 *   tbt_apply_a      ToeplitzMatvec::applyA       linsolve.hpp:65, linsolve.cpp:260-290
 *   tbt_diagonal     ToeplitzMatvec::diagonal     linsolve.hpp:69, linsolve.cpp:390-408
 *   tbt_size_a       ToeplitzMatvec::sizeA        linsolve.hpp:71
 *   tbt_gmres        iterativeSolve / gmres       linsolve.hpp:88-89, linsolve.cpp:425-515,551-593
 *                    (use_a_only = the schurSolve inner A-solve, linsolve.cpp:640-657)
 *   tbt_status codes UserError (exit 1) / NumericError (exit 2),
 *                    include/arraymom/common.hpp:38-50
 *
 * Conventions: complex values are interleaved (re, im) doubles, binary
 * compatible with std::complex<double> (common.hpp:28). Vectors use the
 * reference's unknown order, element-major / basis-minor:
 * index (r*nx + c)*m + k (src/array_model.cpp:219-220,230-235). Several
 * right-hand sides are stored column-major (n x nrhs), like Eigen's MatrixXc.
 * One context is bound to one CUDA device and one stream. Every entry point
 * takes the context's lock, so concurrent calls on one context are
 * serialised by the library (use one context per thread for concurrency;
 * the reference's apply is const and re-entrant per thread, and the batched
 * nrhs entry points replace its per-column threads, linsolve.cpp:572).
 *
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point returns TBT_CUDA_ERROR.
 */
#ifndef TBT_H
#define TBT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TBT_OK = 0,
  TBT_USER_ERROR = 1,    /* UserError: bad sizes, missing inputs, bad order */
  TBT_NUMERIC_ERROR = 2, /* NumericError: GMRES did not converge */
  TBT_CUDA_ERROR = 3     /* device failure / no device */
} tbt_status;

typedef enum { TBT_HOST = 0, TBT_DEVICE = 1 } tbt_where;

typedef struct tbt_ctx tbt_ctx;

typedef struct {
  int nx, ny;    /* element grid (level 0 = x columns, level 1 = y rows)  */
  int m;         /* basis functions per element (reference e5)            */
  int max_nrhs;  /* largest nrhs later passed to apply/gmres (>= 1)        */
  int device;    /* CUDA device ordinal                                    */
  int flags;     /* TBT_EMBED_SMOOTH or 0                                 */
} tbt_desc;

/* Embedding choice: 0 = the reference's next power of two >= 2n-1 per level
 * (linsolve.cpp:240-242); TBT_EMBED_SMOOTH = the smallest 2^a 3^b length
 * >= 2n-1 (mixed-radix transforms), e.g. 36 x 18 bins instead of 64 x 32. */
#define TBT_EMBED_SMOOTH 1

typedef struct {
  double tol;       /* relative residual target (reference default 1e-8)   */
  int max_iter;     /* inner iterations per column (default 2000)          */
  int restart;      /* GMRES(restart) (default 60)                         */
  int precondition; /* left Jacobi (default 1, linsolve.hpp:51)            */
  int use_a_only;   /* 1: operator = applyA (schurSolve's inner solves)    */
  int hist_cap;     /* history entries kept per column (0 = none)          */
  int orthog;       /* Arnoldi orthogonalisation, both modified Gram-Schmidt
                       (linsolve.cpp:465-468): 0 = the projection sweep, one
                       grid barrier per projection; 1 = low-synchronisation
                       form h = (I+L)^-1 V^H w, 3 barriers per step (single
                       column, n <= 4096 * SMs; else falls back to 0)     */
} tbt_gmres_opts;

typedef struct {
  int* iterations;   /* [nrhs] inner iterations                            */
  double* residual;  /* [nrhs] final true relative residual                */
  int* converged;    /* [nrhs] 1 / 0                                       */
  double* history;   /* [nrhs][hist_cap][2] (kind, value) pairs or NULL:
                        kind 0 restart true residual, 1 |g_{j+1}|/beta_0
                        (beta_0: first cycle's preconditioned residual),
                        2 final true residual after max_iter               */
  int* history_len;  /* [nrhs] entries produced (may exceed hist_cap)      */
  int matvecs;       /* batched operator applications issued               */
} tbt_gmres_stats;

tbt_status tbt_create(const tbt_desc* desc, tbt_ctx** out);
void tbt_destroy(tbt_ctx* ctx);

/* Thread-local message of the last failing call on this thread. */
const char* tbt_last_error(void);

/* Binds the context to an existing cudaStream_t (NULL = its own stream). */
tbt_status tbt_set_stream(tbt_ctx* ctx, void* stream);
void* tbt_get_stream(tbt_ctx* ctx);

/* Canonical A generators, nx*ny + (nx-1)*(ny-1) blocks of m x m
 * column-major complex, ToeplitzRep Sparse order (see above). Host memory. */
tbt_status tbt_set_generators(tbt_ctx* ctx, const double* blocks,
                              long long nblocks);
/* FULL generator layout (non-reciprocal operators, which the reference's
 * Sparse ToeplitzRep cannot hold, toeplitz.hpp:72-74): the block of EVERY
 * shift, (2ny-1)(2nx-1) of them, shift i = 1-ny..ny-1 (level 1, outer) by
 * j = 1-nx..nx-1 (level 0, inner), each m x m column-major; block (i, j)
 * couples source element (r, c) to target (r+i, c+j). Internally split into
 * a reciprocal part (the usual half spectrum) and an anti-reciprocal part
 * (a second half spectrum with the partner product negated); when the
 * input is reciprocal the second part is empty. Such contexts take the
 * multi-launch apply path and cannot be distributed or spectrum-cached. */
tbt_status tbt_set_generators_full(tbt_ctx* ctx, const double* blocks, long long nblocks);

/* 40 diag + rank-r terms (8 edge/corner components x 5 relations, layout of
 * tbtgen_correction in tbt_gen.h). rank 0 with d = NULL clears. Host memory. */
tbt_status tbt_set_correction(tbt_ctx* ctx, int rank, const double* d,
                              const double* u, const double* v);

/* Fourier-domain blocks in bin-pair-major layout (kernel K1); cached until
 * destroy or the next set_generators. */
tbt_status tbt_precompute(tbt_ctx* ctx);

/* y = Z x (full synthetic operator) for nrhs columns. Device-resident
 * single-column applies are replayed from a CUDA graph cached per
 * (x, y) pointer pair. */
tbt_status tbt_apply(tbt_ctx* ctx, const double* x, double* y, int nrhs,
                     int where);
/* y_i = Z x_i for `count` independent single-column vectors in HOST
 * memory (x: count consecutive length-n vectors, y likewise), e.g. a batch
 * of excitations or a stream of requests. The host-to-device copy of
 * x_{i+1}, the apply of x_i and the device-to-host copy of y_{i-1} overlap
 * (two device slots, copy streams next to the context stream); returns
 * when every y_i is in host memory. Same results as count calls of
 * tbt_apply(ctx, x_i, y_i, 1, TBT_HOST); overlap needs pinned host memory
 * (pageable memory works but serialises). Single-GPU contexts without
 * margin parts. */
tbt_status tbt_apply_many(tbt_ctx* ctx, const double* x, double* y, long long count);
/* y = A x (pure two-level block-Toeplitz part). */
tbt_status tbt_apply_a(tbt_ctx* ctx, const double* x, double* y, int nrhs,
                       int where);
/* Diagonal of Z (length n + n_m, host memory). */
tbt_status tbt_diagonal(tbt_ctx* ctx, double* d);
long long tbt_size_a(const tbt_ctx* ctx);
/* Margin unknowns n_m (0 until tbt_set_margin). */
long long tbt_size_m(const tbt_ctx* ctx);

/* Margin coupling B / B^T / C, replacing the margin half
 * of ToeplitzMatvec (linsolve.cpp:179-216 build, :292-349 applyB / applyBT /
 * applyC, :373-388 composition). e[9]: edges per part of components 1..9
 * (e[4] must equal m). Layouts (include/tbt_gen.h, tbtgen_margin):
 *   bside   ToeplitzRep::bSideGen[2][2ny-1], each e_c x (nx*m) column-major
 *   brow    ToeplitzRep::bRowGen[2][ny][2nx-1], each e_c x m column-major
 *   bcorner ToeplitzRep::bCorner[4] (corners 3, 9, 1, 7), e_c x (nx*ny*m)
 *   cmat    the n_m x n_m margin block C (the reference's cBlocks assembled,
 *           partBlock of every margin part pair), column-major
 * Afterwards tbt_apply / tbt_diagonal / tbt_gmres act on n + n_m unknowns in
 * the reference order [elements; margin parts 2, 8, 6, 4, 3, 9, 1, 7]
 * (array_model.cpp:218-228); tbt_apply_a and use_a_only solves keep n. */
tbt_status tbt_set_margin(tbt_ctx* ctx, const int* e, const double* bside, const double* brow,
                          const double* bcorner, const double* cmat);
/* SemiSparse representations (the reference's aLevel1 + bFull + cFull,
 * toeplitz.hpp:90-93): A as generators through tbt_set_generators (read
 * out of aLevel1 by aEntry's SemiSparse rule, linsolve.cpp:220-224), B as
 * one dense nM x nA and C as one dense nM x nM matrix, both column-major;
 * B, B^T and C are applied as dense products (linsolve.cpp:294,318,338). */
tbt_status tbt_set_margin_dense(tbt_ctx* ctx, const int* e, const double* b_full, const double* c);
/* The margin blocks alone (ToeplitzMatvec::applyB / applyBT / applyC,
 * linsolve.hpp:66-68; linsolve.cpp:292-314, 316-334, 336-349):
 *   tbt_apply_b   yM = B xA      x: n   x nrhs, y: n_m x nrhs
 *   tbt_apply_bt  yA = B^T xM    x: n_m x nrhs, y: n   x nrhs
 *   tbt_apply_c   yM = C xM      x: n_m x nrhs, y: n_m x nrhs
 * column-major in `where` memory; user error without margin parts. */
tbt_status tbt_apply_b(tbt_ctx* ctx, const double* x, double* y, int nrhs, int where);
tbt_status tbt_apply_bt(tbt_ctx* ctx, const double* x, double* y, int nrhs, int where);
tbt_status tbt_apply_c(tbt_ctx* ctx, const double* x, double* y, int nrhs, int where);

/* Restarted GMRES with x0 = 0 for nrhs columns in lockstep. b, x are
 * n x nrhs column-major in `where` memory. Returns TBT_NUMERIC_ERROR when a
 * column did not converge, with x, stats and the message still filled in. */
tbt_status tbt_gmres(tbt_ctx* ctx, const double* b, double* x, int nrhs,
                     const tbt_gmres_opts* opts, tbt_gmres_stats* stats,
                     int where);

/* schurSolve (linsolve.cpp:595-682), the reference's
 * default solver: A [U F] = [V1 B^T] by A-only GMRES (opts, batches of
 * max_nrhs columns), S = C - B F, LU with partial pivoting and the
 * pivot-ratio check (:517-528), I2 = -S^-1 B U, I1 = U - F I2. b, x are
 * (n + n_m) x nrhs column-major; b must vanish on the margin rows
 * (TBT_USER_ERROR otherwise). TBT_NUMERIC_ERROR on an unconverged inner
 * solve or a singular S. stats: iterations of the inner solve of each
 * column, residual = |Z x - b| / |b| for Z = [A B^T; B C]. */
tbt_status tbt_schur_solve(tbt_ctx* ctx, const double* b, double* x, int nrhs,
                           const tbt_gmres_opts* opts, tbt_gmres_stats* stats,
                           int where);

/* Row f3: a reference ZTOE1 block cache (saveBlockCache,
 * proj/src/toeplitz.cpp:700-743) straight into a precomputed context.
 * Sparse mode: AGen -> generators, BSide/BRow/BCorner -> margin B, the C
 * records assembled into the margin block by partBlock's rules (:506-573).
 * SemiSparse mode: generators read out of ALevel1, BFullM / CFullM ->
 * tbt_set_margin_dense. Full-mode caches are rejected (user error).
 * tbt_ztoe1_dims reads only the header (e: 9 ints). */
tbt_status tbt_load_ztoe1(const char* path, int max_nrhs, int device,
                          int flags, tbt_ctx** ctx);
tbt_status tbt_ztoe1_dims(const char* path, int* nx, int* ny, int* e);
/* Host-only parse of a Sparse ZTOE1 cache into the tbt_set_generators /
 * tbt_set_margin layouts (any pointer may be NULL; sizes from
 * tbt_ztoe1_dims and tbtgen_margin_lengths). */
tbt_status tbt_ztoe1_read(const char* path, double* gen, double* bside,
                          double* brow, double* bcorner, double* c);
/* Storage mode byte of a ZTOE1 file (0 Full, 1 SemiSparse, 2 Sparse), and
 * the host parse of a SemiSparse cache: generators (Sparse order, read out
 * of aLevel1), bFull (nM x nA) and cFull (nM x nM), column-major. */
tbt_status tbt_ztoe1_mode(const char* path, int* mode);
tbt_status tbt_ztoe1_read_dense(const char* path, double* gen, double* b_full, double* c);
/* Persisted bin-major half spectrum (+ the self block): tbt_load_spectra
 * replaces tbt_set_generators + tbt_precompute on a context of the same
 * nx, ny, m and embedding (K1 skipped across runs). tbt_set_cache_key
 * (<= 32 bytes, e.g. a digest of the generator blocks) names the generator
 * set: tbt_save_spectra stores it, and tbt_load_spectra into a context with
 * a key rejects (user error) a file written under another key or none. A
 * context without a key loads any cache of its shape (explicit opt-in for
 * callers that no longer hold the generators). */
tbt_status tbt_set_cache_key(tbt_ctx* ctx, const unsigned char* key, int len);
tbt_status tbt_save_spectra(tbt_ctx* ctx, const char* path);
tbt_status tbt_load_spectra(tbt_ctx* ctx, const char* path);

/* Row f4, contractions on solved currents (proj/src/postproc.cpp).
 * portNetwork (:186-230): current is ld x p column-major (ld = n or
 * n + n_m), feed_rows the port rows (ExcitationSet::feedRows), edge_len the
 * feed edge length; y, z, s are p x p column-major: Y = I/len^2, Z = Y^-1
 * (TBT_NUMERIC_ERROR when singular), S = (Z - Z0)(Z + Z0)^-1 with the
 * sqrt(z0_j / z0_i) power-wave scaling. */
tbt_status tbt_port_network(tbt_ctx* ctx, const double* current, long long ld,
                            int p, const long long* feed_rows, double edge_len,
                            const double* z0, double* y, double* z, double* s,
                            int where);
/* arrayFarfield / embeddedElementPatterns (:134-184): tensors_co/cx[c] are
 * the component far-field tensors (ndir x e[c], column-major; NULL for
 * empty components), dirs ndir x 3 (row-major unit vectors), parts placed
 * as in array_model.cpp:218-228 with pitch dx, dy; current (n + n_m) x p,
 * weights p x q (q = 1: one excitation; the identity: embedded element
 * patterns); co, cx: ndir x q column-major, already scaled by -j k eta. */
tbt_status tbt_array_farfield(tbt_ctx* ctx, const double* const* tensors_co,
                              const double* const* tensors_cx, const int* e,
                              int ndir, const double* dirs, double dx,
                              double dy, double k, double eta,
                              const double* current, int p,
                              const double* weights, int q, double* co,
                              double* cx, int where);

/* Introspection for tests and the bench. */
typedef struct {
  long long n;          /* nx*ny*m                                        */
  long long bins;       /* L = L1*L0                                      */
  long long pairs;      /* stored Fourier blocks (bin pairs + self bins)  */
  int L0, L1;
  long long spectra_bytes;     /* device bytes of the stored blocks       */
  int binprod_kernel;          /* K3 variant id                           */
  int kernels_per_apply;       /* launches of one tbt_apply (nrhs = 1)    */
  int has_antisym;             /* Z(0,0) not symmetric: block-diag fixup  */
  int apply_path;              /* 3 distributed, 2 persistent single kernel,
                                  1 cluster-fused transforms, 0 line passes */
} tbt_info;
tbt_status tbt_get_info(const tbt_ctx* ctx, tbt_info* info);

/* Copies the stored Fourier block of bin f (m x m row-major: [a][b] =
 * the reference's ahat[(a*m+b)*L + f], linsolve.cpp:147,256) to host. For a
 * bin stored as the transposed partner the transpose is returned. */
tbt_status tbt_get_spectrum_bin(tbt_ctx* ctx, long long f, double* out);

/* Per-launch timing of the bin-product kernel (K3). While enabled, every
 * apply records CUDA events around K3 on the context stream (and is not
 * replayed from a CUDA graph); tbt_timing_read synchronises and returns the
 * summed K3 milliseconds and the number of timed launches since enabling.
 * On a distributed context (tbt_dist_init) the timed sections are instead
 * the exchanges of every apply (forward all-to-all, all-to-all back, and
 * the one-row halo exchange of the edge/corner correction). */
tbt_status tbt_set_timing(tbt_ctx* ctx, int on);
tbt_status tbt_timing_read(tbt_ctx* ctx, double* binprod_ms_total, int* count);

/* ---- Multi-GPU: one process per GPU, the operator sharded over nranks ----
 * Element rows are split in contiguous slabs (vectors); level-0 bin columns
 * in groups closed under s0 -> L0-s0 (Fourier blocks, ~1/nranks each); the
 * two FFT transposes are grouped ncclSend/ncclRecv all-to-alls. No
 * reference counterpart. Call sequence on every rank:
 * tbt_create -> tbt_set_generators (all blocks) -> [tbt_set_correction] ->
 * tbt_dist_init -> tbt_precompute; tbt_apply/tbt_apply_a/tbt_diagonal/
 * tbt_gmres then take and return this rank's row slab (tbt_dist_rows). The
 * distributed tbt_gmres runs the low-synchronisation Arnoldi (orthog = 1
 * whatever opts->orthog says) with two ncclAllReduce calls per iteration;
 * every rank returns the same stats. Requires nranks <= min(ny, L0). */
tbt_status tbt_dist_unique_id(char* id /* NCCL_UNIQUE_ID_BYTES = 128 */);
tbt_status tbt_dist_init(tbt_ctx* ctx, int nranks, int rank, const char* id);
/* The same sharded operator with an in-process transport: nranks contexts
 * of ONE process (any device, normally all on one GPU) that share the same
 * 128-byte id form a group; every rank's calls must be issued concurrently
 * from its own host thread (as the ranks of a multi-process job would be).
 * Exchanges synchronise the calling rank's stream, meet the other ranks at a
 * host barrier and copy device to device; all-reduce sums run in fixed rank
 * order. The pack / exchange / unpack code is the NCCL path's. Used to run
 * and test the P > 1 partition on a single GPU. A failed call on one rank
 * aborts the group (the others fail instead of waiting). */
tbt_status tbt_dist_init_loopback(tbt_ctx* ctx, int nranks, int rank, const char* id);
/* 0 not distributed, 1 NCCL, 2 loopback. */
tbt_status tbt_dist_transport(const tbt_ctx* ctx, int* kind);
tbt_status tbt_dist_rows(const tbt_ctx* ctx, int* row_begin, int* row_end);
/* The partition itself (host only, no device needed). */
tbt_status tbt_dist_plan(int ny, int L0, int nranks, int rank, int* row_begin,
                         int* row_end, int* ncols, int* cols);

/* Phase timing of the persistent single-kernel apply: `on` arms
 * %globaltimer stamps (CTA 0) at its phase boundaries for later applies;
 * out_us (may be NULL) receives the phases of the last armed apply:
 * [0] row FFTs + correction, [1] column FFTs, [2] bin products,
 * [3] inverse column FFTs, [4] inverse row FFTs (microseconds);
 * [5..8] latest and [9..12] earliest CTA arrival at barriers 0..3, relative
 * to the start of the phase the barrier ends. out_us holds 13 doubles. */
tbt_status tbt_phase_times(tbt_ctx* ctx, int on, double* out_us);

/* Per-CTA trace of the persistent apply (diagnostics; needs TBT_CTATRACE=1
 * in the environment when the context is created): the last 8 launches,
 * slot = launch index mod 8, each [16 events][256 CTAs] of u64:
 * %globaltimer ns at 0 CTA start, 1 after the programmatic-launch wait,
 * 2..5 arrival at / 6..9 release from grid barriers 0..3, 10 end of the
 * inverse row phase, and for a fused GMRES step 12 after its y barrier,
 * 13 after its dot barrier, 14 at its end; event 11 holds %smid.
 * cap >= 8*16*256. */
tbt_status tbt_cta_trace(tbt_ctx* ctx, unsigned long long* out, long long cap, long long* launches);

/* Times `iters` back-to-back device-resident applies (nrhs columns) with
 * CUDA events on the context stream; out_ms = mean ms per apply and
 * out_binprod_ms = mean ms of the bin-product kernel (events around it). */
tbt_status tbt_bench_apply(tbt_ctx* ctx, const double* x_dev, double* y_dev,
                           int nrhs, int iters, int use_graph, double* out_ms,
                           double* out_binprod_ms);

#ifdef __cplusplus
}
#endif

#endif /* TBT_H */
