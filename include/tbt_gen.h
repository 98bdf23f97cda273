/*
 * tbt_gen.h - seeded synthetic inputs for the multilevel block-Toeplitz path.
 *
 * BASELINE.json configs C1..C5 replace the reference's EFIE blocks
 * (proj/src/kernel.cpp:309 computeBlock) with a seeded generator. This header
 * is the single definition of that generator; the CUDA path, the CPU oracle
 * and the benches all consume its output, so "identical seeded inputs" holds
 * by construction.
 *
 * Complex data is interleaved (re, im) double, binary compatible with
 * std::complex<double> (reference proj/include/arraymom/common.hpp:28) and
 * with the ZTOE1 payload (proj/src/toeplitz.cpp:676).
 *
 * Generator blocks are emitted in the reference's canonical Sparse order
 * (proj/src/toeplitz.cpp:305-312): level-1 shift i = 0..ny-1 (y), level-0
 * shift j = (i == 0 ? 0 : 1-nx) .. nx-1 (x); each block is m x m column-major
 * (SPEC.md:376). Entry (a, b) of block (i, j) is
 *     exp(-j*pi*R)/(1+R) * (u + j v)/sqrt(m),  R = sqrt(i^2 + j^2),
 * u, v ~ N(0,1) from a counter-based RNG (SplitMix64 finaliser + Box-Muller),
 * so every value depends only on (seed, block, entry) and not on threading.
 * The self block (0,0) is drawn on its upper triangle and mirrored (MoM
 * reciprocity), then gets +(2+2j) on the diagonal.
 */
#ifndef TBT_GEN_H
#define TBT_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Number of canonical A generator blocks, nx*ny + (nx-1)*(ny-1)
 * (reference ToeplitzRep::aBlockCount, proj/src/toeplitz.cpp:636-639). */
long long tbtgen_num_blocks(int nx, int ny);

/* Shifts (i = level-1/y, j = level-0/x) of canonical block t. Returns 0 or 1
 * when t is out of range. */
int tbtgen_block_shift(int nx, int ny, long long t, int* i, int* j);

/* Fills out[t * m*m*2 ...] for every canonical block t (see above).
 * nthreads <= 0 means hardware concurrency. Returns 0 on success. */
int tbtgen_blocks(int nx, int ny, int m, uint64_t seed, double* out,
                  int nthreads);

/* Row a and column a of every canonical block (t-major, m entries each):
 * rows[t*m + b] = Z_t(a, b), cols[t*m + b] = Z_t(b, a), the same values as
 * tbtgen_blocks without materialising the blocks (the C5 CPU sample needs a
 * few output rows of the 19 GB generator set). Returns 0 on success. */
int tbtgen_block_lines(int nx, int ny, int m, uint64_t seed, int a, double* rows, double* cols,
                       int nthreads);

/* Nine-component edge/corner perturbations. For component c in
 * {1,2,3,4,6,7,8,9} (reference numbering, proj/include/arraymom/
 * array_model.hpp:26-29) and relation rel in {0 self, 1 +x, 2 -x, 3 +y, 4 -y}
 * the perturbation is P = diag(d) + U V^T with
 *     d = scale * CN(0,1),  U = scale * CN(0,1)/sqrt(m),  V = CN(0,1)/sqrt(m)
 * (CN(0,1) = (u + j v)/sqrt(2)). Output slot s = slot(c)*5 + rel where
 * slot maps 1,2,3,4,6,7,8,9 -> 0..7: d[s*m], U[s*m*rank] and V[s*m*rank]
 * (m x rank column-major). */
int tbtgen_correction(int m, int rank, uint64_t seed, double scale, double* d,
                      double* u, double* v);

/* n x ncols column-major complex N(0,1) (u + j v, u, v ~ N(0,1)). */
int tbtgen_rhs_normal(long long n, int ncols, uint64_t seed, double* out);

/* Delta-gap excitation, one seeded basis index k_e in [0, m) per element
 * e = r*nx + c, value exp(-j*pi*c*sin(steer_deg)); all other entries 0. */
int tbtgen_rhs_delta_steered(int nx, int ny, int m, uint64_t seed,
                             double steer_deg, double* out);

/* nx*ny unit columns (one port per element, mirrors buildExcitation
 * proj/src/linsolve.cpp:45-47): column e has 1 at row e*m + k_e.
 * out is (nx*ny*m) x (nx*ny) column-major. port_rows (optional) gets k_e. */
int tbtgen_rhs_ports(int nx, int ny, int m, uint64_t seed, double* out,
                     long long* port_rows);

/* Margin coupling: synthetic stand-ins for the
 * reference's margin generators (ToeplitzRep::bSideGen / bRowGen / bCorner,
 * proj/include/arraymom/toeplitz.hpp:76-84) and the margin-against-margin
 * blocks ToeplitzMatvec caches as cBlocks (proj/src/linsolve.cpp:210-215).
 * e[9] = edges per part of components 1..9 (e[4] = m). Margin unknowns follow
 * the part order of proj/src/array_model.cpp:218-228: ny parts of component
 * 2, ny of 8, nx of 6, nx of 4, then the corners 3, 9, 1, 7.
 *   bside  : regions (comp 2, comp 8) x (2ny-1) shifts s = idx + 1 - ny,
 *            each e_c x (nx*m) column-major: B block (margin row a, element
 *            row b) = G(a - b)                      (linsolve.cpp:179-185)
 *   brow   : regions (comp 6, comp 4) x ny element rows j x (2nx-1) shifts
 *            k = idx + 1 - nx, each e_c x m column-major: block (margin
 *            column a, element (j, b)) = G_j(a - b)  (linsolve.cpp:187-194)
 *   bcorner: corners (3, 9, 1, 7), each e_c x (nx*ny*m) column-major
 *   c      : nM x nM column-major, symmetric (reciprocity)
 * Regions are concatenated in the order above. Entries are
 * scale*exp(-j*pi*R)/(1+R)*CN(0,1)/sqrt(m) with R the distance between the
 * two parts on the (ny+2) x (nx+2) part grid; C adds (2+2j) on its diagonal
 * (the self-term of a margin part). Returns 0 on success. */
long long tbtgen_margin_size(int nx, int ny, const int* e);
long long tbtgen_margin_lengths(int nx, int ny, const int* e, long long* n_bside, long long* n_brow,
                                long long* n_bcorner);
int tbtgen_margin(int nx, int ny, const int* e, uint64_t seed, double scale, double* bside, double* brow,
                  double* bcorner, double* c);

/* Component (1..9) of element (r, c), r = row (y), c = column (x). Corners
 * win over edges; for 1-wide arrays left/bottom win over right/top. */
int tbtgen_component(int nx, int ny, int r, int c);

#ifdef __cplusplus
}
#endif

#endif /* TBT_GEN_H */
