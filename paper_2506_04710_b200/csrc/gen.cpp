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

int tbtgen_blocks(int nx, int ny, int m, uint64_t seed, double* out,
                  int nthreads) {
  if (nx < 1 || ny < 1 || m < 1 || out == nullptr) return 1;
  const long long nb = tbtgen_num_blocks(nx, ny);
  const long long bsz = static_cast<long long>(m) * m;
  const double inv = 1.0 / std::sqrt(static_cast<double>(m));
  parallelRange(nb, nthreads, [&](long long lo, long long hi) {
    for (long long t = lo; t < hi; ++t) {
      int i = 0, j = 0;
      tbtgen_block_shift(nx, ny, t, &i, &j);
      const double R = std::sqrt(static_cast<double>(i) * i +
                                 static_cast<double>(j) * j);
      const double amp = 1.0 / (1.0 + R);
      const double wr = std::cos(M_PI * R) * amp;
      const double wi = -std::sin(M_PI * R) * amp;
      const uint64_t key = streamKey(seed, kStreamBlock + static_cast<uint64_t>(t));
      double* blk = out + 2 * t * bsz;
      const bool self = (i == 0 && j == 0);
      for (int b = 0; b < m; ++b)
        for (int a = 0; a < m; ++a) {
          // Column-major draw counter; the self block reuses the upper
          // triangle's draw for (a, b) and (b, a).
          long long k = static_cast<long long>(b) * m + a;
          if (self && a > b) k = static_cast<long long>(a) * m + b;
          double u, v;
          normalPair(key, static_cast<uint64_t>(k), &u, &v);
          u *= inv;
          v *= inv;
          double re = wr * u - wi * v;
          double im = wr * v + wi * u;
          if (self && a == b) {
            re += 2.0;
            im += 2.0;
          }
          blk[2 * (static_cast<long long>(b) * m + a)] = re;
          blk[2 * (static_cast<long long>(b) * m + a) + 1] = im;
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
