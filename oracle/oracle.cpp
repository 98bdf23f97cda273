// CPU oracle: a restatement of the reference's multilevel block-Toeplitz
// matvec and restarted GMRES (see oracle.h). TEST INFRASTRUCTURE ONLY.
//
// Built with the reference's flags (-std=c++20 -O3 -DNDEBUG, no fast-math;
// proj/CMakeLists.txt:3,11-13,32) by oracle/Makefile.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <chrono>
#include <cstring>
#include <limits>
#include <string>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

using cplx = std::complex<double>;
using cvec = std::vector<cplx>;

namespace {

// --- Foundation --------------------------------------------------------

// parallelFor / resolveThreads (proj/src/mesh.cpp:27-59): static contiguous
// split of [0, count) over std::threads; 0 means hardware concurrency.
int threadsFor(int requested) {
  if (requested > 0) return requested;
  unsigned hc = std::thread::hardware_concurrency();
  return hc ? static_cast<int>(hc) : 1;
}

template <typename Fn>
void forkJoin(long count, int nthreads, Fn&& fn) {
  nthreads = threadsFor(nthreads);
  if (nthreads <= 1 || count <= 1) {
    fn(0L, count);
    return;
  }
  const long workers = std::min<long>(nthreads, count);
  const long chunk = (count + workers - 1) / workers;
  std::vector<std::thread> pool;
  for (long w = 0; w < workers; ++w) {
    const long lo = w * chunk, hi = std::min(count, lo + chunk);
    if (lo < hi) pool.emplace_back([&fn, lo, hi] { fn(lo, hi); });
  }
  for (auto& t : pool) t.join();
}

// --- FFT (proj/src/fft.cpp) ---------------------------------------------

size_t pow2AtLeast(size_t n) {  // fft.cpp:22-26
  size_t p = 1;
  while (p < n) p *= 2;
  return p;
}

// fft.cpp:28-53: iterative radix-2 decimation in time. Bit-reversal
// permutation first, then butterflies of growing span whose twiddle is
// advanced by repeated multiplication with polar(1, sign*2*pi/len).
// Forward sign is -1; the inverse is unscaled.
bool radix2(cplx* a, size_t n, bool inverse) {
  if (n == 0 || (n & (n - 1)) != 0) return false;
  size_t rev = 0;
  for (size_t k = 1; k < n; ++k) {
    size_t mask = n >> 1;
    while (rev & mask) {
      rev ^= mask;
      mask >>= 1;
    }
    rev ^= mask;
    if (k < rev) std::swap(a[k], a[rev]);
  }
  const double sgn = inverse ? 1.0 : -1.0;
  for (size_t span = 2; span <= n; span *= 2) {
    const cplx step = std::polar(1.0, sgn * 2.0 * M_PI / static_cast<double>(span));
    const size_t half = span / 2;
    for (size_t base = 0; base < n; base += span) {
      cplx tw{1.0, 0.0};
      for (size_t q = 0; q < half; ++q) {
        const cplx even = a[base + q];
        const cplx odd = a[base + q + half] * tw;
        a[base + q] = even + odd;
        a[base + q + half] = even - odd;
        tw *= step;
      }
    }
  }
  return true;
}

// Eigen conventions the reference relies on (linsolve.cpp:466, :429 ...):
// a.dot(b) = sum conj(a_i) b_i, norm = sqrt(sum |v_i|^2).
cplx cdot(const cvec& a, const cvec& b) {
  cplx s{0.0, 0.0};
  for (size_t i = 0; i < a.size(); ++i) s += std::conj(a[i]) * b[i];
  return s;
}
double cnorm(const cvec& a) {
  double s = 0.0;
  for (const cplx& v : a) s += std::norm(v);
  return std::sqrt(s);
}

const int kSlotOfComp[10] = {-1, 0, 1, 2, 3, -1, 4, 5, 6, 7};

int componentOf(int nx, int ny, int r, int c) {  // include/tbt_gen.h
  const bool left = c == 0, right = c == nx - 1;
  const bool bottom = r == 0, top = r == ny - 1;
  if (left && bottom) return 1;
  if (left && top) return 3;
  if (right && bottom) return 7;
  if (right && top) return 9;
  if (left) return 2;
  if (right) return 8;
  if (bottom) return 4;
  if (top) return 6;
  return 5;
}

// Toe1D (linsolve.cpp:54-134): a one-level block-Toeplitz operator with
// nr x nc blocks of size p x q, block (a, b) = gen(a - b), applied through a
// circulant embedding of length nextPow2(nr + nc - 1): entry sequences
// transformed once (build), x transformed per source column j, per-bin
// products summed over j, inverse transform, crop to nr, 1/L. applyT uses
// the frequency-reversed spectrum (the transposed circulant).
struct Toe1D {
  long p = 0, q = 0;
  int nr = 0, nc = 0;
  long L = 0;
  cvec ghat;  // [(i*q + j)*L + f]

  bool emptyOp() const { return p == 0 || q == 0 || nr == 0 || nc == 0; }

  // gen(s) -> column-major p x q block for s in [1-nc, nr-1].
  template <typename Gen>
  void build(long pIn, long qIn, int nrIn, int ncIn, Gen&& gen) {
    p = pIn;
    q = qIn;
    nr = nrIn;
    nc = ncIn;
    if (emptyOp()) return;
    L = static_cast<long>(pow2AtLeast(static_cast<size_t>(nr + nc - 1)));
    ghat.assign(static_cast<size_t>(p) * q * L, cplx{0.0, 0.0});
    cvec seq(static_cast<size_t>(L));
    for (long i = 0; i < p; ++i)
      for (long j = 0; j < q; ++j) {
        std::fill(seq.begin(), seq.end(), cplx{0.0, 0.0});
        for (int s = 0; s < nr; ++s) seq[s] = gen(s)[j * p + i];
        for (int s = 1; s < nc; ++s) seq[L - s] = gen(-s)[j * p + i];
        radix2(seq.data(), static_cast<size_t>(L), false);
        std::copy(seq.begin(), seq.end(), ghat.begin() + (i * q + j) * L);
      }
  }

  // y += T x (x: nc*q, y: nr*p).
  void apply(const cplx* x, cplx* y) const {
    if (emptyOp()) return;
    cvec xhat(static_cast<size_t>(q) * L, cplx{0.0, 0.0});
    for (long j = 0; j < q; ++j) {
      cplx* row = xhat.data() + j * L;
      for (int b = 0; b < nc; ++b) row[b] = x[static_cast<long>(b) * q + j];
      radix2(row, static_cast<size_t>(L), false);
    }
    cvec acc(static_cast<size_t>(L));
    const double scale = 1.0 / static_cast<double>(L);
    for (long i = 0; i < p; ++i) {
      std::fill(acc.begin(), acc.end(), cplx{0.0, 0.0});
      for (long j = 0; j < q; ++j) {
        const cplx* g = ghat.data() + (i * q + j) * L;
        const cplx* xr = xhat.data() + j * L;
        for (long f = 0; f < L; ++f) acc[f] += g[f] * xr[f];
      }
      radix2(acc.data(), static_cast<size_t>(L), true);
      for (int a = 0; a < nr; ++a) y[static_cast<long>(a) * p + i] += acc[a] * scale;
    }
  }

  // y += T^T x (x: nr*p, y: nc*q).
  void applyT(const cplx* x, cplx* y) const {
    if (emptyOp()) return;
    cvec xhat(static_cast<size_t>(p) * L, cplx{0.0, 0.0});
    for (long i = 0; i < p; ++i) {
      cplx* row = xhat.data() + i * L;
      for (int a = 0; a < nr; ++a) row[a] = x[static_cast<long>(a) * p + i];
      radix2(row, static_cast<size_t>(L), false);
    }
    cvec acc(static_cast<size_t>(L));
    const double scale = 1.0 / static_cast<double>(L);
    for (long j = 0; j < q; ++j) {
      std::fill(acc.begin(), acc.end(), cplx{0.0, 0.0});
      for (long i = 0; i < p; ++i) {
        const cplx* g = ghat.data() + (i * q + j) * L;
        const cplx* xr = xhat.data() + i * L;
        for (long f = 0; f < L; ++f) acc[f] += g[(L - f) % L] * xr[f];
      }
      radix2(acc.data(), static_cast<size_t>(L), true);
      for (int b = 0; b < nc; ++b) y[static_cast<long>(b) * q + j] += acc[b] * scale;
    }
  }
};

}  // namespace

struct orc_op {
  int nx = 0, ny = 0, e5 = 0;
  long nA = 0;
  std::vector<cplx> gen;  // canonical blocks, column-major each
  std::vector<cplx> genFull;  // FULL layout (tbt_set_generators_full): every shift
  long L0 = 1, L1 = 1, L = 1;
  std::vector<cplx> ahat;  // [(m*e5+n)*L + f], f = s1*L0 + s0
  bool haveSpectra = false;

  int rank = 0;
  std::vector<cplx> pDense;  // 40 dense m x m perturbations, column-major

  // Margin coupling (row f1; ToeplitzMatvec::Impl, linsolve.cpp:160-216):
  // B1/B2 Toeplitz over y (components 2, 8), B3/B4 per element row
  // Toeplitz over x (components 6, 4), dense corners B5..B8 (3, 9, 1, 7),
  // C dense margin x margin. Margin order: array_model.cpp:218-228.
  bool haveMargin = false;
  int e[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
  long nM = 0;
  cvec bSideRaw, bRowRaw, bCornerRaw, cDense;  // tbt_gen.h layouts
  // SemiSparse (linsolve.cpp:294, :318): B is one dense nM x nA matrix.
  bool denseB = false;
  cvec bDense;  // nM x nA column-major
  Toe1D bSide[2];
  std::vector<Toe1D> bRow[2];
  long sideStart[2] = {0, 0}, rowStart[2] = {0, 0}, cornerStart[4] = {0, 0, 0, 0};
  long cornerOff[4] = {0, 0, 0, 0};  // offsets into bCornerRaw

  long nTot() const { return nA + (haveMargin ? nM : 0); }

  // applyB (linsolve.cpp:292-314): yM = B xA.
  void applyB(const cplx* xA, cplx* yM) const {
    for (long k = 0; k < nM; ++k) yM[k] = 0.0;
    if (denseB) {  // rep.bFull * xA
      for (long q = 0; q < nA; ++q)
        for (long k = 0; k < nM; ++k) yM[k] += bDense[q * nM + k] * xA[q];
      return;
    }
    for (int r = 0; r < 2; ++r) bSide[r].apply(xA, yM + sideStart[r]);
    for (int r = 0; r < 2; ++r)
      for (int j = 0; j < ny && !bRow[r].empty(); ++j)
        bRow[r][j].apply(xA + static_cast<long>(j) * nx * e5, yM + rowStart[r]);
    static const int cc[4] = {3, 9, 1, 7};
    for (int c = 0; c < 4; ++c) {
      const long em = e[cc[c] - 1];
      const cplx* bc = bCornerRaw.data() + cornerOff[c];  // em x nA column-major
      for (long i = 0; i < em; ++i) {
        cplx acc{0.0, 0.0};
        for (long q = 0; q < nA; ++q) acc += bc[q * em + i] * xA[q];
        yM[cornerStart[c] + i] += acc;
      }
    }
  }

  // applyBT (linsolve.cpp:316-334): yA += B^T xM.
  void applyBT(const cplx* xM, cplx* yA) const {
    if (denseB) {  // rep.bFull.transpose() * xM
      for (long q = 0; q < nA; ++q) {
        cplx acc{0.0, 0.0};
        for (long k = 0; k < nM; ++k) acc += bDense[q * nM + k] * xM[k];
        yA[q] += acc;
      }
      return;
    }
    for (int r = 0; r < 2; ++r) bSide[r].applyT(xM + sideStart[r], yA);
    for (int r = 0; r < 2; ++r)
      for (int j = 0; j < ny && !bRow[r].empty(); ++j)
        bRow[r][j].applyT(xM + rowStart[r], yA + static_cast<long>(j) * nx * e5);
    static const int cc[4] = {3, 9, 1, 7};
    for (int c = 0; c < 4; ++c) {
      const long em = e[cc[c] - 1];
      const cplx* bc = bCornerRaw.data() + cornerOff[c];
      for (long q = 0; q < nA; ++q) {
        cplx acc{0.0, 0.0};
        for (long i = 0; i < em; ++i) acc += bc[q * em + i] * xM[cornerStart[c] + i];
        yA[q] += acc;
      }
    }
  }

  // applyC (linsolve.cpp:336-349) with the blocks assembled: yM += C xM.
  void applyC(const cplx* xM, cplx* yM) const {
    for (long k = 0; k < nM; ++k) {
      cplx acc{0.0, 0.0};
      for (long l = 0; l < nM; ++l) acc += cDense[l * nM + k] * xM[l];
      yM[k] += acc;
    }
  }

  // Canonical block index of shift (i >= 0, j), reference storage order
  // aGen[0][j] / aGen[i][j-(1-nx)] (toeplitz.hpp:72-74, toeplitz.cpp:305-312).
  long blockIndex(int i, int j) const {
    if (i == 0) return j;
    return nx + static_cast<long>(i - 1) * (2 * nx - 1) + (j - (1 - nx));
  }

  // aEntry (linsolve.cpp:218-227), Sparse branch: negative half through the
  // block symmetry A(-i,-j) = A(i,j)^T.
  cplx aEntry(int i, int j, int m, int n) const {
    if (!genFull.empty())  // FULL layout: every shift stored (non-reciprocal operators)
      return genFull[(static_cast<size_t>(i + ny - 1) * (2 * nx - 1) + static_cast<size_t>(j + nx - 1)) * e5 * e5 +
                     static_cast<size_t>(n) * e5 + m];
    if (i < 0 || (i == 0 && j < 0)) return aEntry(-i, -j, n, m);
    const long t = blockIndex(i, j);
    return gen[static_cast<size_t>(t) * e5 * e5 + static_cast<size_t>(n) * e5 + m];
  }

  // fft2 (linsolve.cpp:229-237): length-L0 transforms of the L1 rows, then
  // length-L1 transforms of the L0 columns through a gathered copy.
  void fft2(cplx* g, bool inverse) const {
    for (long r = 0; r < L1; ++r) radix2(g + r * L0, static_cast<size_t>(L0), inverse);
    cvec col(static_cast<size_t>(L1));
    for (long c = 0; c < L0; ++c) {
      for (long r = 0; r < L1; ++r) col[r] = g[r * L0 + c];
      radix2(col.data(), static_cast<size_t>(L1), inverse);
      for (long r = 0; r < L1; ++r) g[r * L0 + c] = col[r];
    }
  }

  // buildASpectra (linsolve.cpp:239-258): each (m, n) entry sequence over
  // the 2-D shifts is scattered to (i mod L1, j mod L0) and transformed.
  void buildSpectra(int nthreads) {
    ahat.assign(static_cast<size_t>(e5) * e5 * L, cplx{0.0, 0.0});
    forkJoin(static_cast<long>(e5) * e5, nthreads, [&](long lo, long hi) {
      cvec grid(static_cast<size_t>(L));
      for (long mn = lo; mn < hi; ++mn) {
        const int m = static_cast<int>(mn / e5), n = static_cast<int>(mn % e5);
        std::fill(grid.begin(), grid.end(), cplx{0.0, 0.0});
        for (int i = 1 - ny; i <= ny - 1; ++i)
          for (int j = 1 - nx; j <= nx - 1; ++j) {
            const long s1 = i >= 0 ? i : L1 + i;
            const long s0 = j >= 0 ? j : L0 + j;
            grid[s1 * L0 + s0] = aEntry(i, j, m, n);
          }
        fft2(grid.data(), false);
        std::copy(grid.begin(), grid.end(), ahat.begin() + mn * L);
      }
    });
    haveSpectra = true;
  }

  // applyA (linsolve.cpp:260-290).
  void applyA(const cplx* x, cplx* y) const {
    cvec xhat(static_cast<size_t>(e5) * L);
    cvec grid(static_cast<size_t>(L));
    for (int n = 0; n < e5; ++n) {
      std::fill(grid.begin(), grid.end(), cplx{0.0, 0.0});
      for (int r = 0; r < ny; ++r)
        for (int c = 0; c < nx; ++c)
          grid[static_cast<long>(r) * L0 + c] = x[(static_cast<long>(r) * nx + c) * e5 + n];
      fft2(grid.data(), false);
      std::copy(grid.begin(), grid.end(), xhat.begin() + static_cast<long>(n) * L);
    }
    const double scale = 1.0 / static_cast<double>(L);
    for (int m = 0; m < e5; ++m) {
      std::fill(grid.begin(), grid.end(), cplx{0.0, 0.0});
      for (int n = 0; n < e5; ++n) {
        const cplx* g = ahat.data() + (static_cast<size_t>(m) * e5 + n) * L;
        const cplx* xr = xhat.data() + static_cast<size_t>(n) * L;
        for (long f = 0; f < L; ++f) grid[f] += g[f] * xr[f];
      }
      fft2(grid.data(), true);
      for (int r = 0; r < ny; ++r)
        for (int c = 0; c < nx; ++c)
          y[(static_cast<long>(r) * nx + c) * e5 + m] = grid[static_cast<long>(r) * L0 + c] * scale;
    }
  }

  // Synthetic nine-component correction (tbt_gen.h): for every element e
  // of a non-interior component and every relation with an in-array
  // neighbour e', y_e += P x_e' and y_e' += P^T x_e.
  template <typename Visit>
  void forEachCorrection(Visit&& visit) const {
    if (pDense.empty()) return;
    static const int dr[5] = {0, 0, 0, 1, -1};
    static const int dc[5] = {0, 1, -1, 0, 0};
    for (int r = 0; r < ny; ++r)
      for (int c = 0; c < nx; ++c) {
        const int comp = componentOf(nx, ny, r, c);
        if (comp == 5) continue;
        for (int rel = 0; rel < 5; ++rel) {
          const int r2 = r + dr[rel], c2 = c + dc[rel];
          if (r2 < 0 || r2 >= ny || c2 < 0 || c2 >= nx) continue;
          const cplx* P = pDense.data() + static_cast<size_t>(kSlotOfComp[comp] * 5 + rel) * e5 * e5;
          visit(static_cast<long>(r) * nx + c, static_cast<long>(r2) * nx + c2, P);
        }
      }
  }

  void addCorrection(const cplx* x, cplx* y) const {
    forEachCorrection([&](long e, long e2, const cplx* P) {
      for (int a = 0; a < e5; ++a) {
        cplx s1{0.0, 0.0}, s2{0.0, 0.0};
        for (int b = 0; b < e5; ++b) {
          s1 += P[static_cast<size_t>(b) * e5 + a] * x[e2 * e5 + b];  // (P x_e')_a
          s2 += P[static_cast<size_t>(a) * e5 + b] * x[e * e5 + b];   // (P^T x_e)_a
        }
        y[e * e5 + a] += s1;
        y[e2 * e5 + a] += s2;
      }
    });
  }

  // ToeplitzMatvec::apply (linsolve.cpp:373-388): [A xA + B^T xM; B xA + C xM].
  void apply(const cplx* x, cplx* y) const {
    applyA(x, y);
    addCorrection(x, y);
    if (!haveMargin || nM == 0) return;
    applyBT(x + nA, y);
    applyB(x, y + nA);
    applyC(x + nA, y + nA);
  }

  // Z(e, e') block entry (a, b) from the generators (partBlock Sparse
  // branch, toeplitz.cpp:436-447): shift = target - source.
  cplx zEntry(long e, long e2, int a, int b) const {
    const int r = static_cast<int>(e / nx), c = static_cast<int>(e % nx);
    const int r2 = static_cast<int>(e2 / nx), c2 = static_cast<int>(e2 % nx);
    return aEntry(r - r2, c - c2, a, b);
  }
};

extern "C" {

size_t orc_next_pow2(size_t n) { return pow2AtLeast(n); }

int orc_fft(double* a, size_t n, int inverse) {
  return radix2(reinterpret_cast<cplx*>(a), n, inverse != 0) ? 0 : 1;
}

orc_op* orc_create(int nx, int ny, int m, const double* blocks) {
  if (nx < 1 || ny < 1 || m < 1 || blocks == nullptr) return nullptr;
  auto* op = new orc_op;
  op->nx = nx;
  op->ny = ny;
  op->e5 = m;
  op->nA = static_cast<long>(nx) * ny * m;
  const size_t nb = static_cast<size_t>(nx) * ny + static_cast<size_t>(nx - 1) * (ny - 1);
  op->gen.resize(nb * m * m);
  std::memcpy(static_cast<void*>(op->gen.data()), blocks, nb * m * m * sizeof(cplx));
  op->L1 = static_cast<long>(pow2AtLeast(static_cast<size_t>(2 * ny - 1)));
  op->L0 = static_cast<long>(pow2AtLeast(static_cast<size_t>(2 * nx - 1)));
  op->L = op->L1 * op->L0;
  return op;
}

// FULL layout: (2ny-1)(2nx-1) blocks, shift i = 1-ny..ny-1 outer, j inner.
// aEntry reads every shift directly (no A(-s) = A(s)^T mirror).
orc_op* orc_create_full(int nx, int ny, int m, const double* blocks) {
  if (nx < 1 || ny < 1 || m < 1 || blocks == nullptr) return nullptr;
  auto* op = new orc_op;
  op->nx = nx;
  op->ny = ny;
  op->e5 = m;
  op->nA = static_cast<long>(nx) * ny * m;
  const size_t nb = static_cast<size_t>(2 * nx - 1) * (2 * ny - 1);
  op->genFull.resize(nb * m * m);
  std::memcpy(static_cast<void*>(op->genFull.data()), blocks, nb * m * m * sizeof(cplx));
  op->L1 = static_cast<long>(pow2AtLeast(static_cast<size_t>(2 * ny - 1)));
  op->L0 = static_cast<long>(pow2AtLeast(static_cast<size_t>(2 * nx - 1)));
  op->L = op->L1 * op->L0;
  return op;
}

void orc_destroy(orc_op* op) { delete op; }

int orc_precompute(orc_op* op, int nthreads) {
  if (!op) return 1;
  op->buildSpectra(nthreads);
  return 0;
}

long long orc_bins(const orc_op* op) { return op ? op->L : 0; }

int orc_ahat(const orc_op* op, double* out) {
  if (!op || !op->haveSpectra) return 1;
  std::memcpy(out, op->ahat.data(), op->ahat.size() * sizeof(cplx));
  return 0;
}

int orc_set_correction(orc_op* op, int rank, const double* d, const double* u,
                       const double* v) {
  if (!op || rank < 0 || !d) return 1;
  const int m = op->e5;
  op->rank = rank;
  op->pDense.assign(static_cast<size_t>(40) * m * m, cplx{0.0, 0.0});
  const cplx* D = reinterpret_cast<const cplx*>(d);
  const cplx* U = reinterpret_cast<const cplx*>(u);
  const cplx* V = reinterpret_cast<const cplx*>(v);
  for (int s = 0; s < 40; ++s) {
    cplx* P = op->pDense.data() + static_cast<size_t>(s) * m * m;
    for (int b = 0; b < m; ++b)
      for (int a = 0; a < m; ++a) {
        cplx acc = (a == b) ? D[static_cast<size_t>(s) * m + a] : cplx{0.0, 0.0};
        for (int q = 0; q < rank; ++q)
          acc += U[(static_cast<size_t>(s) * rank + q) * m + a] *
                 V[(static_cast<size_t>(s) * rank + q) * m + b];
        P[static_cast<size_t>(b) * m + a] = acc;
      }
  }
  return 0;
}

int orc_set_margin(orc_op* op, const int* e, const double* bside, const double* brow, const double* bcorner,
                   const double* c) {
  if (!op || !e || e[4] != op->e5) return 1;
  const int nx = op->nx, ny = op->ny, m = op->e5;
  for (int q = 0; q < 9; ++q) op->e[q] = e[q];
  op->nM = static_cast<long>(ny) * (e[1] + e[7]) + static_cast<long>(nx) * (e[5] + e[3]) + e[2] + e[8] + e[0] + e[6];
  const long nA = op->nA, nM = op->nM;
  const long nSide = (2L * ny - 1) * (e[1] + e[7]) * nx * m;
  const long nRow = static_cast<long>(ny) * (2 * nx - 1) * (e[5] + e[3]) * m;
  const long nCorner = (static_cast<long>(e[2]) + e[8] + e[0] + e[6]) * nA;
  const cplx* bs = reinterpret_cast<const cplx*>(bside);
  const cplx* br = reinterpret_cast<const cplx*>(brow);
  const cplx* bc = reinterpret_cast<const cplx*>(bcorner);
  const cplx* cc = reinterpret_cast<const cplx*>(c);
  op->bSideRaw.assign(bs, bs + nSide);
  op->bRowRaw.assign(br, br + nRow);
  op->bCornerRaw.assign(bc, bc + nCorner);
  op->cDense.assign(cc, cc + nM * nM);
  // Group offsets (linsolve.cpp:196-205).
  op->sideStart[0] = 0;
  op->sideStart[1] = static_cast<long>(ny) * e[1];
  op->rowStart[0] = static_cast<long>(ny) * (e[1] + e[7]);
  op->rowStart[1] = op->rowStart[0] + static_cast<long>(nx) * e[5];
  long cs = op->rowStart[1] + static_cast<long>(nx) * e[3];
  static const int cornerComps[4] = {3, 9, 1, 7};
  long co = 0;
  for (int q = 0; q < 4; ++q) {
    op->cornerStart[q] = cs;
    op->cornerOff[q] = co;
    cs += e[cornerComps[q] - 1];
    co += static_cast<long>(e[cornerComps[q] - 1]) * nA;
  }
  // B1/B2 (linsolve.cpp:179-186) and B3/B4 (:187-195).
  static const int sideComp[2] = {2, 8}, rowComp[2] = {6, 4};
  long off = 0;
  for (int r = 0; r < 2; ++r) {
    const long em = e[sideComp[r] - 1];
    const cplx* base = op->bSideRaw.data() + off;
    const long bsz = em * nx * m;
    op->bSide[r] = Toe1D{};
    op->bSide[r].build(em, static_cast<long>(nx) * m, ny, ny,
                       [&](int sft) { return base + static_cast<long>(sft - (1 - ny)) * bsz; });
    off += (2L * ny - 1) * bsz;
  }
  off = 0;
  for (int r = 0; r < 2; ++r) {
    const long em = e[rowComp[r] - 1];
    const long bsz = em * m;
    op->bRow[r].assign(ny, Toe1D{});
    for (int j = 0; j < ny; ++j) {
      const cplx* base = op->bRowRaw.data() + off + static_cast<long>(j) * (2 * nx - 1) * bsz;
      op->bRow[r][j].build(em, m, nx, nx, [&](int sft) { return base + static_cast<long>(sft - (1 - nx)) * bsz; });
    }
    off += static_cast<long>(ny) * (2 * nx - 1) * bsz;
  }
  op->haveMargin = true;
  return 0;
}

// SemiSparse margin coupling: dense B (nM x nA) and C (nM x nM), column-major.
int orc_set_margin_dense(orc_op* op, const int* e, const double* bfull, const double* c) {
  if (!op || !e || e[4] != op->e5) return 1;
  const int nx = op->nx, ny = op->ny;
  for (int q = 0; q < 9; ++q) op->e[q] = e[q];
  op->nM = static_cast<long>(ny) * (e[1] + e[7]) + static_cast<long>(nx) * (e[5] + e[3]) + e[2] + e[8] + e[0] + e[6];
  const cplx* bf = reinterpret_cast<const cplx*>(bfull);
  const cplx* cc = reinterpret_cast<const cplx*>(c);
  op->bDense.assign(bf, bf + op->nM * op->nA);
  op->cDense.assign(cc, cc + op->nM * op->nM);
  op->denseB = true;
  op->haveMargin = true;
  return 0;
}

long long orc_size(const orc_op* op) { return op ? op->nTot() : 0; }

int orc_apply_a(const orc_op* op, const double* x, double* y) {
  if (!op || !op->haveSpectra) return 1;
  op->applyA(reinterpret_cast<const cplx*>(x), reinterpret_cast<cplx*>(y));
  return 0;
}

int orc_apply(const orc_op* op, const double* x, double* y) {
  if (!op || !op->haveSpectra) return 1;
  op->apply(reinterpret_cast<const cplx*>(x), reinterpret_cast<cplx*>(y));
  return 0;
}

int orc_apply_cols(const orc_op* op, const double* x, double* y, int ncols,
                   int nthreads, int a_only) {
  if (!op || !op->haveSpectra || ncols < 0) return 1;
  const cplx* X = reinterpret_cast<const cplx*>(x);
  cplx* Y = reinterpret_cast<cplx*>(y);
  forkJoin(ncols, nthreads, [&](long lo, long hi) {
    for (long c = lo; c < hi; ++c) {
      if (a_only)
        op->applyA(X + c * op->nA, Y + c * op->nA);
      else
        op->apply(X + c * op->nTot(), Y + c * op->nTot());
    }
  });
  return 0;
}

int orc_apply_rows(const orc_op* op, const double* xd, const long long* elems,
                   long long count, double* yd) {
  if (!op) return 1;
  const cplx* x = reinterpret_cast<const cplx*>(xd);
  cplx* y = reinterpret_cast<cplx*>(yd);
  const int m = op->e5;
  const long ne = static_cast<long>(op->nx) * op->ny;
  for (long long k = 0; k < count; ++k) {
    const long e = static_cast<long>(elems[k]);
    if (e < 0 || e >= ne) return 1;
    cplx* out = y + k * m;
    for (int a = 0; a < m; ++a) out[a] = cplx{0.0, 0.0};
    for (long e2 = 0; e2 < ne; ++e2)
      for (int b = 0; b < m; ++b) {
        const cplx xv = x[e2 * m + b];
        for (int a = 0; a < m; ++a) out[a] += op->zEntry(e, e2, a, b) * xv;
      }
    op->forEachCorrection([&](long ea, long eb, const cplx* P) {
      if (ea == e)
        for (int a = 0; a < m; ++a)
          for (int b = 0; b < m; ++b) out[a] += P[static_cast<size_t>(b) * m + a] * x[eb * m + b];
      if (eb == e)
        for (int a = 0; a < m; ++a)
          for (int b = 0; b < m; ++b) out[a] += P[static_cast<size_t>(a) * m + b] * x[ea * m + b];
    });
  }
  return 0;
}

int orc_dense(const orc_op* op, double* zd) {
  if (!op) return 1;
  const int m = op->e5;
  const long ne = static_cast<long>(op->nx) * op->ny;
  const long N = ne * m;
  cplx* z = reinterpret_cast<cplx*>(zd);
  for (long e = 0; e < ne; ++e)
    for (long e2 = 0; e2 < ne; ++e2)
      for (int b = 0; b < m; ++b)
        for (int a = 0; a < m; ++a)
          z[(e2 * m + b) * N + e * m + a] = op->zEntry(e, e2, a, b);
  op->forEachCorrection([&](long e, long e2, const cplx* P) {
    for (int b = 0; b < m; ++b)
      for (int a = 0; a < m; ++a) {
        z[(e2 * m + b) * N + e * m + a] += P[static_cast<size_t>(b) * m + a];
        z[(e * m + b) * N + e2 * m + a] += P[static_cast<size_t>(a) * m + b];
      }
  });
  return 0;
}

int orc_diagonal(const orc_op* op, double* dd) {
  if (!op) return 1;
  const int m = op->e5;
  const long ne = static_cast<long>(op->nx) * op->ny;
  cplx* d = reinterpret_cast<cplx*>(dd);
  // ToeplitzMatvec::diagonal (linsolve.cpp:397-399): aEntry(0,0,m,m).
  for (long p = 0; p < ne; ++p)
    for (int a = 0; a < m; ++a) d[p * m + a] = op->aEntry(0, 0, a, a);
  op->forEachCorrection([&](long e, long e2, const cplx* P) {
    if (e != e2) return;
    for (int a = 0; a < m; ++a) d[e * m + a] += 2.0 * P[static_cast<size_t>(a) * m + a];
  });
  // Margin diagonal: the C blocks' diagonal (linsolve.cpp:400-406).
  if (op->haveMargin)
    for (long k = 0; k < op->nM; ++k) d[op->nA + k] = op->cDense[k * op->nM + k];
  return 0;
}

}  // extern "C"

namespace {

struct Outcome {
  int iterations = 0;
  double residual = 0.0;
  bool converged = false;
};

struct History {
  double* buf;
  int cap;
  int len = 0;
  void push(double kind, double v) {
    if (buf && len < cap) {
      buf[2 * len] = kind;
      buf[2 * len + 1] = v;
    }
    ++len;
  }
};

// gmres (linsolve.cpp:425-515): restarted GMRES(restart), x0 = 0, left
// Jacobi, modified Gram-Schmidt with the conjugated inner product, complex
// Givens rotations, inner exit at |g_{j+1}|/beta < 0.1 tol, lucky breakdown,
// back substitution; maxIter counts inner iterations.
template <typename Op>
Outcome gmresColumn(const Op& op, const cvec& b, cvec& x, const cvec* invDiag,
                    double tol, int maxIter, int restart, History& hist) {
  const size_t n = b.size();
  const double bnorm = cnorm(b);
  Outcome out;
  x.assign(n, cplx{0.0, 0.0});
  if (bnorm == 0.0) {
    out.converged = true;
    return out;
  }
  auto precond = [&](cvec& v) {
    if (!invDiag) return;
    for (size_t k = 0; k < n; ++k) v[k] *= (*invDiag)[k];
  };

  std::vector<cvec> basis;
  std::vector<cplx> h(static_cast<size_t>(restart + 1) * restart);
  auto H = [&](int i, int j) -> cplx& { return h[static_cast<size_t>(j) * (restart + 1) + i]; };
  std::vector<cplx> cs(restart), sn(restart), g(restart + 1);
  cvec ax(n), w(n);

  double beta0 = 0.0;  // history scale: first cycle's preconditioned residual
  while (out.iterations < maxIter) {
    op(x, ax);
    cvec r(n);
    for (size_t k = 0; k < n; ++k) r[k] = b[k] - ax[k];
    out.residual = cnorm(r) / bnorm;
    hist.push(0.0, out.residual);
    if (out.residual < tol) {
      out.converged = true;
      return out;
    }
    precond(r);
    const double beta = cnorm(r);
    if (beta == 0.0) {
      out.converged = true;
      return out;
    }
    if (beta0 == 0.0) beta0 = beta;
    basis.assign(1, r);
    for (auto& v : basis[0]) v /= beta;
    std::fill(g.begin(), g.end(), cplx{0.0, 0.0});
    std::fill(h.begin(), h.end(), cplx{0.0, 0.0});
    g[0] = beta;
    int j = 0;
    for (; j < restart && out.iterations < maxIter; ++j, ++out.iterations) {
      op(basis[j], w);
      precond(w);
      for (int i = 0; i <= j; ++i) {
        H(i, j) = cdot(basis[i], w);
        const cplx hij = H(i, j);
        for (size_t k = 0; k < n; ++k) w[k] -= hij * basis[i][k];
      }
      H(j + 1, j) = cnorm(w);
      if (std::abs(H(j + 1, j)) > 0.0) {
        const cplx hn = H(j + 1, j);
        cvec v(n);
        for (size_t k = 0; k < n; ++k) v[k] = w[k] / hn;
        basis.push_back(std::move(v));
      }
      for (int i = 0; i < j; ++i) {
        const cplx t = cs[i] * H(i, j) + sn[i] * H(i + 1, j);
        H(i + 1, j) = -std::conj(sn[i]) * H(i, j) + std::conj(cs[i]) * H(i + 1, j);
        H(i, j) = t;
      }
      const double den = std::sqrt(std::norm(H(j, j)) + std::norm(H(j + 1, j)));
      if (den == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = std::conj(H(j, j)) / den;
        sn[j] = std::conj(H(j + 1, j)) / den;
      }
      H(j, j) = cs[j] * H(j, j) + sn[j] * H(j + 1, j);
      H(j + 1, j) = 0.0;
      const cplx gj = g[j];
      g[j] = cs[j] * gj;
      g[j + 1] = -std::conj(sn[j]) * gj;
      hist.push(1.0, std::abs(g[j + 1]) / beta0);
      if (std::abs(g[j + 1]) / beta < 0.1 * tol) {
        ++j;
        ++out.iterations;
        break;
      }
      if (basis.size() == static_cast<size_t>(j) + 1) {
        ++j;
        ++out.iterations;
        break;
      }
    }
    std::vector<cplx> yv(j);
    for (int i = j - 1; i >= 0; --i) {
      cplx s = g[i];
      for (int k2 = i + 1; k2 < j; ++k2) s -= H(i, k2) * yv[k2];
      yv[i] = s / H(i, i);
    }
    for (int i = 0; i < j; ++i)
      for (size_t k = 0; k < n; ++k) x[k] += yv[i] * basis[i][k];
  }
  // maxIter exhausted: final true residual (linsolve.cpp:512-513).
  op(x, ax);
  cvec r(n);
  for (size_t k = 0; k < n; ++k) r[k] = b[k] - ax[k];
  out.residual = cnorm(r) / bnorm;
  out.converged = out.residual < tol;
  hist.push(2.0, out.residual);
  return out;
}

}  // namespace

extern "C" int orc_gmres(const orc_op* op, const double* b, double* x,
                         int ncols, double tol, int max_iter, int restart,
                         int precondition, int use_a_only, int nthreads,
                         int* iterations, double* residual, int* converged,
                         double* hist, int hist_cap, int* hist_len) {
  if (!op || !op->haveSpectra || ncols < 0 || restart < 1) return 1;
  const long n = use_a_only ? op->nA : op->nTot();
  cvec invDiag;
  if (precondition) {
    // iterativeSolve (linsolve.cpp:556-563): 1/d, or 1 where d == 0.
    invDiag.resize(op->nTot());
    orc_diagonal(op, reinterpret_cast<double*>(invDiag.data()));
    invDiag.resize(n);
    if (use_a_only)
      for (long p = 0; p < n; ++p) invDiag[p] = op->aEntry(0, 0, static_cast<int>(p % op->e5), static_cast<int>(p % op->e5));
    for (auto& d : invDiag) d = (std::abs(d) > 0.0) ? 1.0 / d : cplx{1.0, 0.0};
  }
  auto opFull = [op](const cvec& in, cvec& out) { op->apply(in.data(), out.data()); };
  auto opA = [op](const cvec& in, cvec& out) { op->applyA(in.data(), out.data()); };
  forkJoin(ncols, nthreads, [&](long lo, long hi) {
    for (long c = lo; c < hi; ++c) {
      cvec bc(reinterpret_cast<const cplx*>(b) + c * n, reinterpret_cast<const cplx*>(b) + (c + 1) * n);
      cvec xc;
      History h{hist ? hist + 2L * hist_cap * c : nullptr, hist_cap};
      const Outcome o = use_a_only
                            ? gmresColumn(opA, bc, xc, precondition ? &invDiag : nullptr, tol, max_iter, restart, h)
                            : gmresColumn(opFull, bc, xc, precondition ? &invDiag : nullptr, tol, max_iter, restart, h);
      std::memcpy(x + 2 * c * n, xc.data(), n * sizeof(cplx));
      if (iterations) iterations[c] = o.iterations;
      if (residual) residual[c] = o.residual;
      if (converged) converged[c] = o.converged ? 1 : 0;
      if (hist_len) hist_len[c] = h.len;
    }
  });
  return 0;
}

namespace {

// Eigen::PartialPivLU restated (row interchanges on the largest |a| of the
// column, unit lower L, U in place); perm[k] = original row of row k.
void luPartialPivot(std::vector<cplx>& a, long n, std::vector<long>& perm) {
  perm.resize(n);
  for (long i = 0; i < n; ++i) perm[i] = i;
  auto A = [&](long i, long j) -> cplx& { return a[j * n + i]; };  // column-major
  for (long k = 0; k < n; ++k) {
    long p = k;
    double best = std::abs(A(k, k));
    for (long i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > best) {
        best = std::abs(A(i, k));
        p = i;
      }
    if (p != k) {
      for (long j = 0; j < n; ++j) std::swap(A(k, j), A(p, j));
      std::swap(perm[k], perm[p]);
    }
    if (A(k, k) == cplx{0.0, 0.0}) continue;
    for (long i = k + 1; i < n; ++i) A(i, k) /= A(k, k);
    for (long j = k + 1; j < n; ++j) {
      const cplx akj = A(k, j);
      for (long i = k + 1; i < n; ++i) A(i, j) -= A(i, k) * akj;
    }
  }
}

void luSolve(const std::vector<cplx>& lu, const std::vector<long>& perm, long n, cvec& rhs) {
  cvec y(n);
  for (long i = 0; i < n; ++i) y[i] = rhs[perm[i]];
  for (long i = 0; i < n; ++i)
    for (long k = 0; k < i; ++k) y[i] -= lu[k * n + i] * y[k];
  for (long i = n - 1; i >= 0; --i) {
    for (long k = i + 1; k < n; ++k) y[i] -= lu[k * n + i] * y[k];
    y[i] /= lu[i * n + i];
  }
  rhs = y;
}

}  // namespace

// schurSolve (linsolve.cpp:595-682): A [U F] = [V1 B^T] by A-only GMRES
// columns (Jacobi of A's diagonal), S = C - B F, PartialPivLU of S with the
// pivot-ratio check (:517-528), I2 = -S^{-1} B U, I1 = U - F I2, residual of
// the full operator per column. Returns 0, 1 (user error) or 2 (numeric).
extern "C" int orc_schur(const orc_op* op, const double* b, double* x, int ncols, double tol, int max_iter,
                         int restart, int precondition, int nthreads, int* iterations, double* residual, char* err,
                         int errcap) {
  auto fail = [&](int code, const std::string& msg) {
    if (err && errcap > 0) std::snprintf(err, static_cast<size_t>(errcap), "%s", msg.c_str());
    return code;
  };
  if (!op || !op->haveSpectra || ncols < 1) return fail(1, "schurSolve: bad arguments");
  const long nA = op->nA, nM = op->haveMargin ? op->nM : 0, n = nA + nM;
  const cplx* B = reinterpret_cast<const cplx*>(b);
  for (int c = 0; c < ncols; ++c)
    for (long k = nA; k < n; ++k)
      if (B[c * n + k] != cplx{0.0, 0.0}) return fail(1, "schurSolve: excitation must vanish on margin rows");
  cvec invDiagA;
  if (precondition) {
    invDiagA.resize(nA);
    for (long i = 0; i < nA; ++i) {
      const cplx d = op->aEntry(0, 0, static_cast<int>(i % op->e5), static_cast<int>(i % op->e5));
      invDiagA[i] = std::abs(d) > 0.0 ? 1.0 / d : cplx{1.0, 0.0};
    }
  }
  // Dense B^T (nA x nM) column by column: B^T e_k.
  std::vector<cplx> bt(static_cast<size_t>(nA) * nM, cplx{0.0, 0.0});
  for (long k = 0; k < nM; ++k) {
    cvec e(nM, cplx{0.0, 0.0});
    e[k] = 1.0;
    op->applyBT(e.data(), bt.data() + k * nA);
  }
  const long p = ncols, cols = p + nM;
  std::vector<cplx> uf(static_cast<size_t>(nA) * cols);
  std::vector<int> its(cols, 0);
  std::vector<double> res(cols, 0.0);
  std::vector<int> conv(cols, 0);
  auto opA = [op](const cvec& in, cvec& out) { op->applyA(in.data(), out.data()); };
  forkJoin(cols, nthreads, [&](long lo, long hi) {
    for (long c = lo; c < hi; ++c) {
      cvec rhs(nA);
      if (c < p)
        for (long i = 0; i < nA; ++i) rhs[i] = B[c * n + i];
      else
        std::copy(bt.begin() + (c - p) * nA, bt.begin() + (c - p + 1) * nA, rhs.begin());
      cvec xc;
      History h{nullptr, 0};
      const Outcome o = gmresColumn(opA, rhs, xc, precondition ? &invDiagA : nullptr, tol, max_iter, restart, h);
      std::copy(xc.begin(), xc.end(), uf.begin() + c * nA);
      its[c] = o.iterations;
      res[c] = o.residual;
      conv[c] = o.converged ? 1 : 0;
    }
  });
  for (long c = 0; c < cols; ++c)
    if (!conv[c])
      return fail(2, "schur inner solve did not converge (column " + std::to_string(c) + ", best residual " +
                         std::to_string(res[c]) + ")");
  cplx* X = reinterpret_cast<cplx*>(x);
  for (long c = 0; c < p; ++c) {
    for (long i = 0; i < nA; ++i) X[c * n + i] = uf[c * nA + i];
    for (long k = 0; k < nM; ++k) X[c * n + nA + k] = 0.0;
  }
  if (nM > 0) {
    // S = C - B F with B = (B^T)^T (plain transpose).
    std::vector<cplx> S(static_cast<size_t>(nM) * nM);
    forkJoin(nM, nthreads, [&](long lo, long hi) {
      for (long l = lo; l < hi; ++l)
        for (long k = 0; k < nM; ++k) {
          cplx acc{0.0, 0.0};
          const cplx* bk = bt.data() + k * nA;
          const cplx* fl = uf.data() + (p + l) * nA;
          for (long q = 0; q < nA; ++q) acc += bk[q] * fl[q];
          S[l * nM + k] = op->cDense[l * nM + k] - acc;
        }
    });
    std::vector<long> perm;
    luPartialPivot(S, nM, perm);
    double maxAbs = 0.0, minAbs = std::numeric_limits<double>::infinity();
    for (long i = 0; i < nM; ++i) {
      maxAbs = std::max(maxAbs, std::abs(S[i * nM + i]));
      minAbs = std::min(minAbs, std::abs(S[i * nM + i]));
    }
    if (!(minAbs > 1e-14 * maxAbs))
      return fail(2, "singular matrix in schur complement (pivot ratio " +
                         std::to_string(minAbs / (maxAbs > 0 ? maxAbs : 1.0)) + ")");
    for (long c = 0; c < p; ++c) {
      cvec r(nM);
      for (long k = 0; k < nM; ++k) {
        cplx acc{0.0, 0.0};
        for (long q = 0; q < nA; ++q) acc += bt[k * nA + q] * uf[c * nA + q];
        r[k] = acc;
      }
      luSolve(S, perm, nM, r);
      for (long k = 0; k < nM; ++k) r[k] = -r[k];  // I2
      for (long i = 0; i < nA; ++i) {
        cplx acc{0.0, 0.0};
        for (long k = 0; k < nM; ++k) acc += uf[(p + k) * nA + i] * r[k];
        X[c * n + i] = uf[c * nA + i] - acc;
      }
      for (long k = 0; k < nM; ++k) X[c * n + nA + k] = r[k];
    }
  }
  for (long c = 0; c < p; ++c) {
    cvec xc(X + c * n, X + (c + 1) * n), yc(n);
    op->apply(xc.data(), yc.data());
    double num = 0.0, bn = 0.0;
    for (long i = 0; i < n; ++i) {
      num += std::norm(yc[i] - B[c * n + i]);
      bn += std::norm(B[c * n + i]);
    }
    if (residual) residual[c] = std::sqrt(num) / (bn > 0 ? std::sqrt(bn) : 1.0);
    if (iterations) iterations[c] = its[c];
  }
  return 0;
}

namespace {

// Eigen PartialPivLU(...).inverse() restated: LU with partial pivoting,
// then solve against the identity; returns the pivot ratio.
double luInverse(const std::vector<cplx>& a, long n, std::vector<cplx>& inv) {
  std::vector<cplx> lu = a;
  std::vector<long> perm;
  luPartialPivot(lu, n, perm);
  double maxAbs = 0.0, minAbs = std::numeric_limits<double>::infinity();
  for (long i = 0; i < n; ++i) {
    maxAbs = std::max(maxAbs, std::abs(lu[i * n + i]));
    minAbs = std::min(minAbs, std::abs(lu[i * n + i]));
  }
  inv.assign(static_cast<size_t>(n) * n, cplx{0.0, 0.0});
  for (long c = 0; c < n; ++c) {
    cvec e(n, cplx{0.0, 0.0});
    e[c] = 1.0;
    luSolve(lu, perm, n, e);
    std::copy(e.begin(), e.end(), inv.begin() + c * n);
  }
  return minAbs / (maxAbs > 0 ? maxAbs : 1.0);
}

}  // namespace

// portNetwork (postproc.cpp:186-230). Returns 0, 1 (user) or 2 (singular Y).
extern "C" int orc_port_network(const double* current, long long ld, int p, const long long* feed, double len,
                                const double* z0, double* y, double* z, double* s) {
  if (!(len > 0.0) || p < 1) return 1;
  for (int i = 0; i < p; ++i)
    if (!(z0[i] > 0.0) || feed[i] < 0 || feed[i] >= ld) return 1;
  const cplx* cur = reinterpret_cast<const cplx*>(current);
  std::vector<cplx> Y(static_cast<size_t>(p) * p);
  const double inv = 1.0 / len;
  for (int c = 0; c < p; ++c)
    for (int i = 0; i < p; ++i) Y[c * p + i] = inv * cur[feed[i] + c * ld] * inv;
  std::vector<cplx> Z;
  if (!(luInverse(Y, p, Z) > 1e-14)) return 2;
  std::vector<cplx> zm = Z, zp = Z, zpi;
  for (int i = 0; i < p; ++i) {
    zm[i * p + i] -= z0[i];
    zp[i * p + i] += z0[i];
  }
  luInverse(zp, p, zpi);
  std::vector<cplx> S(static_cast<size_t>(p) * p);
  for (int j = 0; j < p; ++j)
    for (int i = 0; i < p; ++i) {
      cplx acc{0.0, 0.0};
      for (int k = 0; k < p; ++k) acc += zm[k * p + i] * zpi[j * p + k];
      S[j * p + i] = acc * std::sqrt(z0[j] / z0[i]);
    }
  std::memcpy(y, Y.data(), Y.size() * sizeof(cplx));
  std::memcpy(z, Z.data(), Z.size() * sizeof(cplx));
  std::memcpy(s, S.data(), S.size() * sizeof(cplx));
  return 0;
}

// arrayFarfield (postproc.cpp:134-170) for the q columns of current * W
// (q = 1: one excitation; W = I: embeddedElementPatterns, :172-184). Parts
// in the order and at the offsets of array_model.cpp:218-228.
extern "C" int orc_array_farfield(int nx, int ny, const int* e, const double* const* tco, const double* const* tcx,
                                  int ndir, const double* dirs, double dx, double dy, double k, double eta,
                                  const double* current, int p, const double* weights, int q, double* co,
                                  double* cx) {
  struct Part {
    int comp;
    long start;
    double ox, oy;
  };
  std::vector<Part> parts;
  long row = 0;
  auto place = [&](int cmp, double ox, double oy) {
    parts.push_back({cmp, row, ox, oy});
    row += e[cmp - 1];
  };
  for (int r = 1; r <= ny; ++r)
    for (int c = 1; c <= nx; ++c) place(5, (c - 1) * dx, (r - 1) * dy);
  for (int r = 1; r <= ny; ++r) place(2, 0.0, (r - 1) * dy);
  for (int r = 1; r <= ny; ++r) place(8, (nx - 1) * dx, (r - 1) * dy);
  for (int c = 1; c <= nx; ++c) place(6, (c - 1) * dx, (ny - 1) * dy);
  for (int c = 1; c <= nx; ++c) place(4, (c - 1) * dx, 0.0);
  place(3, 0.0, (ny - 1) * dy);
  place(9, (nx - 1) * dx, (ny - 1) * dy);
  place(1, 0.0, 0.0);
  place(7, (nx - 1) * dx, 0.0);
  const long ntot = row;
  const cplx* cur = reinterpret_cast<const cplx*>(current);
  const cplx* W = reinterpret_cast<const cplx*>(weights);
  cplx* CO = reinterpret_cast<cplx*>(co);
  cplx* CX = reinterpret_cast<cplx*>(cx);
  const cplx front(0.0, -k * eta);
  for (int j = 0; j < q; ++j) {
    cvec comb(ntot, cplx{0.0, 0.0});  // current * excitation (:145)
    for (int c = 0; c < p; ++c)
      for (long r = 0; r < ntot; ++r) comb[r] += cur[r + c * ntot] * W[c + static_cast<long>(j) * p];
    for (int i = 0; i < ndir; ++i) {
      cplx fco{0.0, 0.0}, fcx{0.0, 0.0};
      const double* d = dirs + 3 * i;
      for (const Part& pt : parts) {
        const int n = e[pt.comp - 1];
        if (n == 0) continue;
        const cplx* Tco = reinterpret_cast<const cplx*>(tco[pt.comp - 1]);
        const cplx* Tcx = reinterpret_cast<const cplx*>(tcx[pt.comp - 1]);
        cplx sco{0.0, 0.0}, scx{0.0, 0.0};
        for (int t = 0; t < n; ++t) {
          sco += Tco[i + static_cast<long>(t) * ndir] * comb[pt.start + t];
          scx += Tcx[i + static_cast<long>(t) * ndir] * comb[pt.start + t];
        }
        const cplx phase = std::polar(1.0, k * (d[0] * pt.ox + d[1] * pt.oy));
        fco += phase * sco;
        fcx += phase * scx;
      }
      CO[i + static_cast<long>(j) * ndir] = front * fco;
      CX[i + static_cast<long>(j) * ndir] = front * fcx;
    }
  }
  return 0;
}

// ---------------------------------------------------------------------------
// Bounded CPU sample of applyA (linsolve.cpp:260-290) at sizes whose spectra
// do not fit host memory (C5: 38.65 GB): the whole forward half (e5 padded
// 2-D FFTs of x, :264-274) and, for `nrows` output rows m, the reference's
// per-row work (accumulate sum_n ahat_{m,n} * xhat_n over all bins, inverse
// 2-D FFT, crop and scale, :276-288). The spectra of those rows are built
// first (untimed) from row m / column m of every canonical block
// (tbtgen_block_lines), so aEntry's mirrored half (:219) is available.
// Returns the two timed sections in seconds; y[r * ne + e] is the r-th
// sampled output row (the row whose lines were passed) of element e, comparable with a full apply at those rows.
extern "C" int orc_sampled_apply(int nx, int ny, int m, int nrows, const double* const* row_lines,
                                 const double* const* col_lines, const double* xd, double* yd, double* t_fwd,
                                 double* t_rows, int nthreads) {
  if (nx < 1 || ny < 1 || m < 1 || nrows < 1) return 1;
  const long L1 = static_cast<long>(pow2AtLeast(static_cast<size_t>(2 * ny - 1)));
  const long L0 = static_cast<long>(pow2AtLeast(static_cast<size_t>(2 * nx - 1)));
  const long L = L1 * L0;
  const long ne = static_cast<long>(nx) * ny;
  auto blockIndex = [&](int i, int j) -> long {
    if (i == 0) return j;
    return nx + static_cast<long>(i - 1) * (2 * nx - 1) + (j - (1 - nx));
  };
  auto fft2 = [&](cplx* g, bool inverse, cvec& col) {
    for (long r = 0; r < L1; ++r) radix2(g + r * L0, static_cast<size_t>(L0), inverse);
    for (long c = 0; c < L0; ++c) {
      for (long r = 0; r < L1; ++r) col[r] = g[r * L0 + c];
      radix2(col.data(), static_cast<size_t>(L1), inverse);
      for (long r = 0; r < L1; ++r) g[r * L0 + c] = col[r];
    }
  };
  // Spectra of the sampled rows: ahat[(r * m + n) * L + f].
  std::vector<cplx> ahat(static_cast<size_t>(nrows) * m * L);
  forkJoin(static_cast<long>(nrows) * m, nthreads, [&](long lo, long hi) {
    cvec grid(static_cast<size_t>(L)), col(static_cast<size_t>(L1));
    for (long rn = lo; rn < hi; ++rn) {
      const int r = static_cast<int>(rn / m), n = static_cast<int>(rn % m);
      const cplx* rl = reinterpret_cast<const cplx*>(row_lines[r]);
      const cplx* cl = reinterpret_cast<const cplx*>(col_lines[r]);
      std::fill(grid.begin(), grid.end(), cplx{0.0, 0.0});
      for (int i = 1 - ny; i <= ny - 1; ++i)
        for (int j = 1 - nx; j <= nx - 1; ++j) {
          const long s1 = i >= 0 ? i : L1 + i;
          const long s0 = j >= 0 ? j : L0 + j;
          // aEntry(i, j, row, n) = Z_t(row, n); the mirrored half is
          // aEntry(-i, -j, n, row) = Z_t'(n, row) = column `row` of t'.
          const bool mirrored = i < 0 || (i == 0 && j < 0);
          grid[s1 * L0 + s0] = mirrored ? cl[blockIndex(-i, -j) * m + n] : rl[blockIndex(i, j) * m + n];
        }
      fft2(grid.data(), false, col);
      std::copy(grid.begin(), grid.end(), ahat.begin() + rn * L);
    }
  });
  const cplx* x = reinterpret_cast<const cplx*>(xd);
  cplx* y = reinterpret_cast<cplx*>(yd);
  using clk = std::chrono::steady_clock;
  // Timed, single thread, as the reference's applyA: the forward half.
  auto t0 = clk::now();
  cvec xhat(static_cast<size_t>(m) * L), grid(static_cast<size_t>(L)), col(static_cast<size_t>(L1));
  for (int n = 0; n < m; ++n) {
    std::fill(grid.begin(), grid.end(), cplx{0.0, 0.0});
    for (int r = 0; r < ny; ++r)
      for (int c = 0; c < nx; ++c) grid[static_cast<long>(r) * L0 + c] = x[(static_cast<long>(r) * nx + c) * m + n];
    fft2(grid.data(), false, col);
    std::copy(grid.begin(), grid.end(), xhat.begin() + static_cast<long>(n) * L);
  }
  auto t1 = clk::now();
  const double scale = 1.0 / static_cast<double>(L);
  for (int r = 0; r < nrows; ++r) {
    std::fill(grid.begin(), grid.end(), cplx{0.0, 0.0});
    for (int n = 0; n < m; ++n) {
      const cplx* g = ahat.data() + (static_cast<size_t>(r) * m + n) * L;
      const cplx* xr = xhat.data() + static_cast<size_t>(n) * L;
      for (long f = 0; f < L; ++f) grid[f] += g[f] * xr[f];
    }
    fft2(grid.data(), true, col);
    for (int rr = 0; rr < ny; ++rr)
      for (int c = 0; c < nx; ++c)
        y[r * ne + static_cast<long>(rr) * nx + c] = grid[static_cast<long>(rr) * L0 + c] * scale;
  }
  auto t2 = clk::now();
  *t_fwd = std::chrono::duration<double>(t1 - t0).count();
  *t_rows = std::chrono::duration<double>(t2 - t1).count();
  return 0;
}
