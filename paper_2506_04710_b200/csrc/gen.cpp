// Seeded synthetic inputs (see include/tbt_gen.h for the contract).
#include "tbt_gen.h"

#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {

constexpr uint64_t kStreamBlock = 1ULL << 40;
constexpr uint64_t kStreamCorr = 2ULL << 40;
constexpr uint64_t kStreamRhs = 3ULL << 40;
constexpr uint64_t kStreamPort = 4ULL << 40;
constexpr uint64_t kStreamMargin = 5ULL << 40;

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// Key of one (seed, stream) pair; draws are mix64(key + k * golden).
inline uint64_t streamKey(uint64_t seed, uint64_t stream) {
  return mix64(mix64(seed) ^ (stream * 0xD1B54A32D192ED03ULL));
}

inline double uniform(uint64_t key, uint64_t k) {
  const uint64_t b = mix64(key + k * 0x9E3779B97F4A7C15ULL);
  return (static_cast<double>(b >> 11) + 0.5) * 0x1.0p-53;  // (0, 1)
}

// Draw k of a stream: one Box-Muller pair -> two independent N(0,1).
inline void normalPair(uint64_t key, uint64_t k, double* u, double* v) {
  const double u1 = uniform(key, 2 * k);
  const double u2 = uniform(key, 2 * k + 1);
  const double rad = std::sqrt(-2.0 * std::log(u1));
  const double th = 2.0 * M_PI * u2;
  *u = rad * std::cos(th);
  *v = rad * std::sin(th);
}

int resolveThreads(int n) {
  if (n > 0) return n;
  const unsigned hc = std::thread::hardware_concurrency();
  return hc == 0 ? 1 : static_cast<int>(hc);
}

template <typename Fn>
void parallelRange(long long count, int nthreads, Fn fn) {
  nthreads = resolveThreads(nthreads);
  if (nthreads <= 1 || count < 2) {
    fn(0LL, count);
    return;
  }
  if (nthreads > count) nthreads = static_cast<int>(count);
  std::vector<std::thread> pool;
  const long long chunk = (count + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    const long long lo = t * chunk;
    const long long hi = lo + chunk < count ? lo + chunk : count;
    if (lo >= hi) break;
    pool.emplace_back([=] { fn(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

const int kSlotComp[8] = {1, 2, 3, 4, 6, 7, 8, 9};

}  // namespace

extern "C" {

long long tbtgen_num_blocks(int nx, int ny) {
  if (nx < 1 || ny < 1) return 0;
  return static_cast<long long>(nx) * ny +
         static_cast<long long>(nx - 1) * (ny - 1);
}

int tbtgen_block_shift(int nx, int ny, long long t, int* i, int* j) {
  if (t < 0 || t >= tbtgen_num_blocks(nx, ny)) return 1;
  if (t < nx) {
    *i = 0;
    *j = static_cast<int>(t);
    return 0;
  }
  const long long u = t - nx;
  const long long w = 2LL * nx - 1;
  *i = static_cast<int>(1 + u / w);
  *j = static_cast<int>(u % w) + (1 - nx);
  return 0;
}

// Entry (a, b) of canonical block t (shift i, j): the definition in tbt_gen.h.
static inline void blockEntry(int i, int j, int m, uint64_t key, int a, int b, double* re, double* im) {
  const double R = std::sqrt(static_cast<double>(i) * i + static_cast<double>(j) * j);
  const double amp = 1.0 / (1.0 + R);
  const double wr = std::cos(M_PI * R) * amp;
  const double wi = -std::sin(M_PI * R) * amp;
  const double inv = 1.0 / std::sqrt(static_cast<double>(m));
  const bool self = (i == 0 && j == 0);
  // Column-major draw counter; the self block reuses the upper triangle's
  // draw for (a, b) and (b, a).
  long long k = static_cast<long long>(b) * m + a;
  if (self && a > b) k = static_cast<long long>(a) * m + b;
  double u, v;
  normalPair(key, static_cast<uint64_t>(k), &u, &v);
  u *= inv;
  v *= inv;
  *re = wr * u - wi * v;
  *im = wr * v + wi * u;
  if (self && a == b) {
    *re += 2.0;
    *im += 2.0;
  }
}

int tbtgen_blocks(int nx, int ny, int m, uint64_t seed, double* out,
                  int nthreads) {
  if (nx < 1 || ny < 1 || m < 1 || out == nullptr) return 1;
  const long long nb = tbtgen_num_blocks(nx, ny);
  const long long bsz = static_cast<long long>(m) * m;
  parallelRange(nb, nthreads, [&](long long lo, long long hi) {
    for (long long t = lo; t < hi; ++t) {
      int i = 0, j = 0;
      tbtgen_block_shift(nx, ny, t, &i, &j);
      const uint64_t key = streamKey(seed, kStreamBlock + static_cast<uint64_t>(t));
      double* blk = out + 2 * t * bsz;
      for (int b = 0; b < m; ++b)
        for (int a = 0; a < m; ++a) {
          const long long o = 2 * (static_cast<long long>(b) * m + a);
          blockEntry(i, j, m, key, a, b, blk + o, blk + o + 1);
        }
    }
  });
  return 0;
}

int tbtgen_block_lines(int nx, int ny, int m, uint64_t seed, int a, double* rows, double* cols, int nthreads) {
  if (nx < 1 || ny < 1 || m < 1 || a < 0 || a >= m || rows == nullptr || cols == nullptr) return 1;
  const long long nb = tbtgen_num_blocks(nx, ny);
  parallelRange(nb, nthreads, [&](long long lo, long long hi) {
    for (long long t = lo; t < hi; ++t) {
      int i = 0, j = 0;
      tbtgen_block_shift(nx, ny, t, &i, &j);
      const uint64_t key = streamKey(seed, kStreamBlock + static_cast<uint64_t>(t));
      for (int b = 0; b < m; ++b) {
        const long long o = 2 * (t * m + b);
        blockEntry(i, j, m, key, a, b, rows + o, rows + o + 1);
        blockEntry(i, j, m, key, b, a, cols + o, cols + o + 1);
      }
    }
  });
  return 0;
}

int tbtgen_correction(int m, int rank, uint64_t seed, double scale, double* d,
                      double* u, double* v) {
  if (m < 1 || rank < 0 || d == nullptr) return 1;
  if (rank > 0 && (u == nullptr || v == nullptr)) return 1;
  const double isq2 = 1.0 / std::sqrt(2.0);
  const double ism = 1.0 / std::sqrt(static_cast<double>(m));
  for (int s = 0; s < 8; ++s)
    for (int rel = 0; rel < 5; ++rel) {
      const int slot = s * 5 + rel;
      const uint64_t base = kStreamCorr + static_cast<uint64_t>(kSlotComp[s]) * 64 +
                            static_cast<uint64_t>(rel) * 4;
      const uint64_t kd = streamKey(seed, base + 0);
      const uint64_t ku = streamKey(seed, base + 1);
      const uint64_t kv = streamKey(seed, base + 2);
      for (int a = 0; a < m; ++a) {
        double x, y;
        normalPair(kd, static_cast<uint64_t>(a), &x, &y);
        d[2 * (static_cast<long long>(slot) * m + a)] = scale * x * isq2;
        d[2 * (static_cast<long long>(slot) * m + a) + 1] = scale * y * isq2;
      }
      const long long off = static_cast<long long>(slot) * m * rank;
      for (long long q = 0; q < static_cast<long long>(m) * rank; ++q) {
        double x, y;
        normalPair(ku, static_cast<uint64_t>(q), &x, &y);
        u[2 * (off + q)] = scale * x * isq2 * ism;
        u[2 * (off + q) + 1] = scale * y * isq2 * ism;
        normalPair(kv, static_cast<uint64_t>(q), &x, &y);
        v[2 * (off + q)] = x * isq2 * ism;
        v[2 * (off + q) + 1] = y * isq2 * ism;
      }
    }
  return 0;
}

int tbtgen_rhs_normal(long long n, int ncols, uint64_t seed, double* out) {
  if (n < 0 || ncols < 0 || out == nullptr) return 1;
  for (int c = 0; c < ncols; ++c) {
    const uint64_t key = streamKey(seed, kStreamRhs + static_cast<uint64_t>(c));
    for (long long k = 0; k < n; ++k) {
      double x, y;
      normalPair(key, static_cast<uint64_t>(k), &x, &y);
      out[2 * (static_cast<long long>(c) * n + k)] = x;
      out[2 * (static_cast<long long>(c) * n + k) + 1] = y;
    }
  }
  return 0;
}

static long long portIndex(uint64_t seed, long long e, int m) {
  const uint64_t key = streamKey(seed, kStreamPort + static_cast<uint64_t>(e));
  long long k = static_cast<long long>(uniform(key, 0) * m);
  return k >= m ? m - 1 : k;
}

int tbtgen_rhs_delta_steered(int nx, int ny, int m, uint64_t seed,
                             double steer_deg, double* out) {
  if (nx < 1 || ny < 1 || m < 1 || out == nullptr) return 1;
  const long long n = static_cast<long long>(nx) * ny * m;
  for (long long k = 0; k < 2 * n; ++k) out[k] = 0.0;
  const double s = std::sin(steer_deg * M_PI / 180.0);
  for (int r = 0; r < ny; ++r)
    for (int c = 0; c < nx; ++c) {
      const long long e = static_cast<long long>(r) * nx + c;
      const long long row = e * m + portIndex(seed, e, m);
      out[2 * row] = std::cos(M_PI * c * s);
      out[2 * row + 1] = -std::sin(M_PI * c * s);
    }
  return 0;
}

int tbtgen_rhs_ports(int nx, int ny, int m, uint64_t seed, double* out,
                     long long* port_rows) {
  if (nx < 1 || ny < 1 || m < 1 || out == nullptr) return 1;
  const long long ne = static_cast<long long>(nx) * ny;
  const long long n = ne * m;
  for (long long k = 0; k < 2 * n * ne; ++k) out[k] = 0.0;
  for (long long e = 0; e < ne; ++e) {
    const long long row = e * m + portIndex(seed, e, m);
    out[2 * (e * n + row)] = 1.0;
    if (port_rows) port_rows[e] = row;
  }
  return 0;
}

long long tbtgen_margin_size(int nx, int ny, const int* e) {
  if (nx < 1 || ny < 1 || e == nullptr) return 0;
  return static_cast<long long>(ny) * (e[1] + e[7]) + static_cast<long long>(nx) * (e[5] + e[3]) + e[2] + e[8] +
         e[0] + e[6];
}

long long tbtgen_margin_lengths(int nx, int ny, const int* e, long long* n_bside, long long* n_brow,
                                long long* n_bcorner) {
  if (nx < 1 || ny < 1 || e == nullptr) return -1;
  const long long m = e[4], nA = static_cast<long long>(nx) * ny * m;
  const long long sside = (2LL * ny - 1) * (e[1] + e[7]) * nx * m;
  const long long srow = static_cast<long long>(ny) * (2LL * nx - 1) * (e[5] + e[3]) * m;
  const long long scorner = (static_cast<long long>(e[2]) + e[8] + e[0] + e[6]) * nA;
  if (n_bside) *n_bside = sside;
  if (n_brow) *n_brow = srow;
  if (n_bcorner) *n_bcorner = scorner;
  return tbtgen_margin_size(nx, ny, e);
}

namespace {

// Part-grid position (row, col) of margin unknown k (array_model.cpp:218-228:
// component 2 at column -1, 8 at column nx, 6 at row ny, 4 at row -1;
// corners 3 (ny,-1), 9 (ny,nx), 1 (-1,-1), 7 (-1,nx)).
void marginPart(int nx, int ny, const int* e, long long k, int* row, int* col) {
  const long long g2 = static_cast<long long>(ny) * e[1], g8 = static_cast<long long>(ny) * e[7];
  const long long g6 = static_cast<long long>(nx) * e[5], g4 = static_cast<long long>(nx) * e[3];
  if (k < g2) { *row = static_cast<int>(k / e[1]); *col = -1; return; }
  k -= g2;
  if (k < g8) { *row = static_cast<int>(k / e[7]); *col = nx; return; }
  k -= g8;
  if (k < g6) { *row = ny; *col = static_cast<int>(k / e[5]); return; }
  k -= g6;
  if (k < g4) { *row = -1; *col = static_cast<int>(k / e[3]); return; }
  k -= g4;
  const int cc[4] = {3, 9, 1, 7};
  const int cr[4] = {ny, ny, -1, -1}, ccol[4] = {-1, nx, -1, nx};
  for (int q = 0; q < 4; ++q) {
    if (k < e[cc[q] - 1]) { *row = cr[q]; *col = ccol[q]; return; }
    k -= e[cc[q] - 1];
  }
  *row = *col = 0;
}

// One entry: scale * exp(-j pi R)/(1+R) * CN(0,1)/sqrt(m).
void marginEntry(uint64_t key, uint64_t k, double R, double scale, double ism, double* re, double* im) {
  double u, v;
  normalPair(key, k, &u, &v);
  const double amp = scale * ism / (1.0 + R) / std::sqrt(2.0);
  const double wr = std::cos(M_PI * R) * amp, wi = -std::sin(M_PI * R) * amp;
  *re = wr * u - wi * v;
  *im = wr * v + wi * u;
}

}  // namespace

int tbtgen_margin(int nx, int ny, const int* e, uint64_t seed, double scale, double* bside, double* brow,
                  double* bcorner, double* c) {
  if (nx < 1 || ny < 1 || e == nullptr || e[4] < 1) return 1;
  for (int q = 0; q < 9; ++q)
    if (e[q] < 0) return 1;
  const int m = e[4];
  const long long nA = static_cast<long long>(nx) * ny * m;
  const double ism = 1.0 / std::sqrt(static_cast<double>(m));
  // B sides: region r (comp 2 at column -1, comp 8 at column nx), shift s:
  // distance between margin part (a, col) and element (a - s, c).
  const int sideComp[2] = {2, 8};
  double* out = bside;
  for (int r = 0; r < 2; ++r) {
    const int em = e[sideComp[r] - 1];
    const int colM = r == 0 ? -1 : nx;
    for (int idx = 0; idx < 2 * ny - 1; ++idx) {
      const int s = idx + 1 - ny;
      const uint64_t key = streamKey(seed, kStreamMargin + static_cast<uint64_t>(r) * 4096 + idx);
      for (long long q = 0; q < static_cast<long long>(nx) * m; ++q) {
        const int cEl = static_cast<int>(q / m);
        const double R = std::hypot(static_cast<double>(s), static_cast<double>(colM - cEl));
        for (int i = 0; i < em; ++i) {
          const long long o = q * em + i;  // column-major em x (nx*m)
          if (out) marginEntry(key, static_cast<uint64_t>(o), R, scale, ism, out + 2 * o, out + 2 * o + 1);
        }
      }
      if (out) out += 2LL * em * nx * m;
    }
  }
  // B rows: region r (comp 6 at row ny, comp 4 at row -1), element row j,
  // shift k: margin part (rowM, a) vs element (j, a - k).
  const int rowComp[2] = {6, 4};
  out = brow;
  for (int r = 0; r < 2; ++r) {
    const int em = e[rowComp[r] - 1];
    const int rowM = r == 0 ? ny : -1;
    for (int j = 0; j < ny; ++j)
      for (int idx = 0; idx < 2 * nx - 1; ++idx) {
        const int k = idx + 1 - nx;
        const double R = std::hypot(static_cast<double>(rowM - j), static_cast<double>(k));
        const uint64_t key = streamKey(seed, kStreamMargin + (2 + static_cast<uint64_t>(r)) * 4096 * 4096 +
                                                 static_cast<uint64_t>(j) * 4096 + idx);
        for (long long o = 0; o < static_cast<long long>(em) * m; ++o)
          if (out) marginEntry(key, static_cast<uint64_t>(o), R, scale, ism, out + 2 * o, out + 2 * o + 1);
        if (out) out += 2LL * em * m;
      }
  }
  // Corners 3, 9, 1, 7 against every element.
  const int cc[4] = {3, 9, 1, 7};
  const int cr[4] = {ny, ny, -1, -1}, ccol[4] = {-1, nx, -1, nx};
  out = bcorner;
  for (int q = 0; q < 4; ++q) {
    const int em = e[cc[q] - 1];
    const uint64_t key = streamKey(seed, kStreamMargin + 7ULL * 4096 * 4096 + q);
    for (long long col = 0; col < nA; ++col) {
      const long long el = col / m;
      const int er = static_cast<int>(el / nx), ec = static_cast<int>(el % nx);
      const double R = std::hypot(static_cast<double>(cr[q] - er), static_cast<double>(ccol[q] - ec));
      for (int i = 0; i < em; ++i) {
        const long long o = col * em + i;
        if (out) marginEntry(key, static_cast<uint64_t>(o), R, scale, ism, out + 2 * o, out + 2 * o + 1);
      }
    }
    if (out) out += 2LL * em * nA;
  }
  // C: symmetric, drawn on the upper triangle, (2+2j) on the diagonal.
  if (c) {
    const long long nM = tbtgen_margin_size(nx, ny, e);
    const uint64_t key = streamKey(seed, kStreamMargin + 8ULL * 4096 * 4096);
    for (long long l = 0; l < nM; ++l) {
      int rl, cl;
      marginPart(nx, ny, e, l, &rl, &cl);
      for (long long k = 0; k <= l; ++k) {
        int rk, ck;
        marginPart(nx, ny, e, k, &rk, &ck);
        const double R = std::hypot(static_cast<double>(rl - rk), static_cast<double>(cl - ck));
        double re, im;
        marginEntry(key, static_cast<uint64_t>(l * nM + k), R, scale, ism, &re, &im);
        if (k == l) {
          re += 2.0;
          im += 2.0;
        }
        c[2 * (l * nM + k)] = re;  // column l, row k
        c[2 * (l * nM + k) + 1] = im;
        c[2 * (k * nM + l)] = re;
        c[2 * (k * nM + l) + 1] = im;
      }
    }
  }
  return 0;
}

int tbtgen_component(int nx, int ny, int r, int c) {
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

}  // extern "C"
