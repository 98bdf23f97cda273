// Row f3: inputs from files.
//
//  * ZTOE1 block caches written by the reference (saveBlockCache,
//    proj/src/toeplitz.cpp:700-743; format restated from the reader
//    loadBlockCache, :745-815): "ZTOE1", u8 storage mode, i32 nx, ny, e[9],
//    then records {u8 tag, i32 i0, i1, i2, i64 rows, cols, rows*cols
//    complex128 column-major} up to tag 255. Sparse-mode records map onto
//    the device operator: AGen -> generators, BSide / BRow / BCorner -> the
//    margin B generators, and the C records (CToe, CFullRect, C5x, C55) are
//    assembled into the dense margin block with partBlock's rules
//    (:506-573). SemiSparse-mode caches (ALevel1 / BFullM / CFullM) map too:
//    the reference's SemiSparse ToeplitzMatvec runs the same FFT applyA on
//    generators read out of aLevel1 (aEntry, linsolve.cpp:220-224) and
//    applies B, B^T, C as dense products (:294, :318, :338). Full-mode
//    caches hold only the dense matrix and are rejected.
//  * A persisted bin-major spectrum ("TBTS1"), so repeated runs on the same
//    operator (frequency sweeps re-solving many excitations) skip K1.
#include <algorithm>
#include <array>
#include <complex>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <map>
#include <tuple>

#include "tbt_internal.cuh"

namespace tbt {

namespace {

using cplx = std::complex<double>;

struct Mat {
  int64_t rows = 0, cols = 0;
  std::vector<cplx> v;  // column-major
  cplx at(int64_t r, int64_t c) const { return v[static_cast<size_t>(c * rows + r)]; }
};

template <typename T>
T readVal(std::ifstream& in) {
  T v;
  in.read(reinterpret_cast<char*>(&v), sizeof v);
  TBT_USER_CHECK(static_cast<bool>(in), "block cache: truncated file");
  return v;
}

enum Tag : uint8_t {
  kAGen = 1, kBSide = 2, kBRow = 3, kBCorner = 4, kCToe = 5, kCFullRect = 6, kC5x = 7, kC55 = 8,
  kALevel1 = 9, kBFullM = 10, kCFullM = 11, kZFullM = 12, kEnd = 255
};

constexpr int kEdgeComps[4] = {2, 8, 6, 4};    // margin groups 1..4
constexpr int kCornerComps[4] = {3, 9, 1, 7};  // group 5 order

}  // namespace

void readZtoe1(const std::string& path, Ztoe1Data& out) {
  std::ifstream in(path, std::ios::binary);
  TBT_USER_CHECK(static_cast<bool>(in), "cannot open block cache: " + path);
  char magic[5];
  in.read(magic, 5);
  TBT_USER_CHECK(in && std::string(magic, 5) == "ZTOE1", "not a ZTOE1 block cache: " + path);
  const uint8_t mode = readVal<uint8_t>(in);
  out.nx = readVal<int32_t>(in);
  out.ny = readVal<int32_t>(in);
  TBT_USER_CHECK(out.nx >= 1 && out.ny >= 1, "block cache: bad dimensions");
  for (int c = 0; c < 9; ++c) {
    out.e[c] = readVal<int32_t>(in);
    TBT_USER_CHECK(out.e[c] >= 0, "block cache: negative edge count");
  }
  // StorageMode {Full, SemiSparse, Sparse} (toeplitz.hpp:27).
  TBT_USER_CHECK(mode == 2 || mode == 1,
                 "block cache: Full-mode caches hold no block-Toeplitz generators (mode " + std::to_string(mode) +
                     "); use a Sparse or SemiSparse cache");
  out.mode = mode;
  const int nx = out.nx, ny = out.ny, m = out.e[4];
  std::map<std::tuple<int, int, int, int>, Mat> rec;
  for (;;) {
    const uint8_t tag = readVal<uint8_t>(in);
    if (tag == kEnd) break;
    const int i0 = readVal<int32_t>(in), i1 = readVal<int32_t>(in), i2 = readVal<int32_t>(in);
    Mat mt;
    mt.rows = readVal<int64_t>(in);
    mt.cols = readVal<int64_t>(in);
    TBT_USER_CHECK(mt.rows >= 0 && mt.cols >= 0 && mt.rows * mt.cols < (int64_t{1} << 36),
                   "block cache: bad record dimensions");
    TBT_USER_CHECK(tag >= kAGen && tag <= kZFullM, "block cache: unknown record tag");
    // Records the mode's layout has no slot for (initLayout, :181-238): the
    // reference's reader fails on them (index out of range / dimensions).
    const bool sparseTag = tag <= kC55;
    TBT_USER_CHECK(tag != kZFullM && (mode == 2 ? sparseTag : !sparseTag),
                   "block cache: record does not belong to a " + std::string(mode == 2 ? "Sparse" : "SemiSparse") +
                       "-mode layout");
    mt.v.resize(static_cast<size_t>(mt.rows * mt.cols));
    in.read(reinterpret_cast<char*>(mt.v.data()), static_cast<std::streamsize>(mt.v.size() * sizeof(cplx)));
    TBT_USER_CHECK(static_cast<bool>(in), "block cache: truncated file");
    rec[{tag, i0, i1, i2}] = std::move(mt);
  }
  // Record lookup with the layout's dimensions (initLayout, :181-238);
  // absent records are zero, as initLayout leaves them.
  auto get = [&](int tag, int i0, int i1, int i2, int64_t rows, int64_t cols) -> Mat {
    auto it = rec.find({tag, i0, i1, i2});
    Mat z;
    z.rows = rows;
    z.cols = cols;
    if (it == rec.end()) {
      z.v.assign(static_cast<size_t>(rows * cols), cplx{0.0, 0.0});
      return z;
    }
    TBT_USER_CHECK(it->second.rows == rows && it->second.cols == cols,
                   "block cache: record dimensions do not match layout");
    return it->second;
  };
  auto append = [](std::vector<double2>& dst, const Mat& mt) {
    for (const cplx& z : mt.v) dst.push_back(make_double2(z.real(), z.imag()));
  };
  const long long nA = static_cast<long long>(nx) * ny * m;
  out.nM = static_cast<long long>(ny) * (out.e[1] + out.e[7]) + static_cast<long long>(nx) * (out.e[5] + out.e[3]) +
           out.e[2] + out.e[8] + out.e[0] + out.e[6];
  if (mode == 1) {
    // aLevel1[i] is the (nx m)^2 block row of element row i against element
    // row 0 (initLayout :193-196); generator (i, j) is its block
    // (max(j, 0), max(-j, 0)) — aEntry's SemiSparse branch (linsolve.cpp:
    // 220-224) — taken in the canonical Sparse order.
    const int64_t w = static_cast<int64_t>(nx) * m;
    out.gen.clear();
    for (int i = 0; i < ny; ++i) {
      const Mat a1 = get(kALevel1, i, 0, 0, w, w);
      for (int j = (i == 0 ? 0 : 1 - nx); j <= nx - 1; ++j) {
        const int64_t r0 = static_cast<int64_t>(std::max(j, 0)) * m, c0 = static_cast<int64_t>(std::max(-j, 0)) * m;
        for (int b = 0; b < m; ++b)
          for (int a = 0; a < m; ++a) {
            const cplx z = a1.at(r0 + a, c0 + b);
            out.gen.push_back(make_double2(z.real(), z.imag()));
          }
      }
    }
    out.bside.clear();
    out.brow.clear();
    out.bcorner.clear();
    out.bfull.clear();
    out.c.clear();
    if (out.nM > 0) {
      const Mat bf = get(kBFullM, 0, 0, 0, out.nM, nA);
      const Mat cf = get(kCFullM, 0, 0, 0, out.nM, out.nM);
      for (const cplx& z : bf.v) out.bfull.push_back(make_double2(z.real(), z.imag()));
      for (const cplx& z : cf.v) out.c.push_back(make_double2(z.real(), z.imag()));
    }
    return;
  }
  // A generators in canonical order: aGen[0][j], then aGen[i][j - (1-nx)].
  out.gen.clear();
  for (int j = 0; j < nx; ++j) append(out.gen, get(kAGen, 0, j, 0, m, m));
  for (int i = 1; i < ny; ++i)
    for (int j = 0; j < 2 * nx - 1; ++j) append(out.gen, get(kAGen, i, j, 0, m, m));
  out.bside.clear();
  out.brow.clear();
  out.bcorner.clear();
  for (int r = 0; r < 2; ++r) {
    const int em = out.e[kEdgeComps[r] - 1];
    for (int j = 0; j < 2 * ny - 1; ++j) append(out.bside, get(kBSide, r, j, 0, em, static_cast<int64_t>(nx) * m));
  }
  for (int r = 0; r < 2; ++r) {
    const int em = out.e[kEdgeComps[2 + r] - 1];
    for (int j = 0; j < ny; ++j)
      for (int k = 0; k < 2 * nx - 1; ++k) append(out.brow, get(kBRow, r, j, k, em, m));
  }
  for (int c = 0; c < 4; ++c) append(out.bcorner, get(kBCorner, c, 0, 0, out.e[kCornerComps[c] - 1], nA));
  // Dense C from the C records, part by part (partBlock, :506-573).
  const int e2 = out.e[1], e8 = out.e[7], e6 = out.e[5], e4 = out.e[3];
  std::vector<Mat> c11(ny), c21(2 * ny - 1), c22(ny), c33(nx), c43(2 * nx - 1), c44(nx);
  for (int k = 0; k < ny; ++k) {
    c11[k] = get(kCToe, 0, k, 0, e2, e2);
    c22[k] = get(kCToe, 2, k, 0, e8, e8);
  }
  for (int k = 0; k < 2 * ny - 1; ++k) c21[k] = get(kCToe, 1, k, 0, e8, e2);
  for (int k = 0; k < nx; ++k) {
    c33[k] = get(kCToe, 3, k, 0, e6, e6);
    c44[k] = get(kCToe, 5, k, 0, e4, e4);
  }
  for (int k = 0; k < 2 * nx - 1; ++k) c43[k] = get(kCToe, 4, k, 0, e4, e6);
  const Mat c31 = get(kCFullRect, 0, 0, 0, static_cast<int64_t>(nx) * e6, static_cast<int64_t>(ny) * e2);
  const Mat c41 = get(kCFullRect, 1, 0, 0, static_cast<int64_t>(nx) * e4, static_cast<int64_t>(ny) * e2);
  const Mat c32 = get(kCFullRect, 2, 0, 0, static_cast<int64_t>(nx) * e6, static_cast<int64_t>(ny) * e8);
  const Mat c42 = get(kCFullRect, 3, 0, 0, static_cast<int64_t>(nx) * e4, static_cast<int64_t>(ny) * e8);
  int cornerTotal = 0;
  int cornerRowStart[4];
  for (int a = 0; a < 4; ++a) {
    cornerRowStart[a] = cornerTotal;
    cornerTotal += out.e[kCornerComps[a] - 1];
  }
  const int64_t groupCols[4] = {static_cast<int64_t>(ny) * e2, static_cast<int64_t>(ny) * e8,
                                static_cast<int64_t>(nx) * e6, static_cast<int64_t>(nx) * e4};
  std::array<Mat, 4> c5x;
  for (int g = 0; g < 4; ++g) c5x[g] = get(kC5x, g, 0, 0, cornerTotal, groupCols[g]);
  std::array<std::array<Mat, 4>, 4> c55;
  for (int a = 0; a < 4; ++a)
    for (int b = a; b < 4; ++b)
      c55[a][b] = get(kC55, a, b, 0, out.e[kCornerComps[a] - 1], out.e[kCornerComps[b] - 1]);
  // Margin parts: (group, position a (1-based), size, offset).
  struct Part {
    int g, a, size;
    long long off;
  };
  std::vector<Part> parts;
  long long off = 0;
  const int gCount[4] = {ny, ny, nx, nx};
  for (int g = 1; g <= 4; ++g)
    for (int a = 1; a <= gCount[g - 1]; ++a) {
      const int sz = out.e[kEdgeComps[g - 1] - 1];
      parts.push_back({g, a, sz, off});
      off += sz;
    }
  for (int a = 1; a <= 4; ++a) {
    const int sz = out.e[kCornerComps[a - 1] - 1];
    parts.push_back({5, a, sz, off});
    off += sz;
  }
  const long long nM = off;
  out.nM = nM;
  out.c.assign(static_cast<size_t>(nM * nM), make_double2(0.0, 0.0));
  auto eOf = [&](int group) { return out.e[kEdgeComps[group - 1] - 1]; };
  // Entry (r, s) of the (pi, pj) block.
  auto blockEntry = [&](const Part& pi, const Part& pj, int r, int s) -> cplx {
    const int gi = pi.g, gj = pj.g, a = pi.a, b = pj.a;
    auto toe = [&](const std::vector<Mat>& st) { return a - b >= 0 ? st[a - b].at(r, s) : st[b - a].at(s, r); };
    auto rect = [&](const Mat& mt, int ar, int bc, int er, int ec, bool tr) {
      // block (ar, bc) of size er x ec; tr: entry of its transpose
      return tr ? mt.at(static_cast<int64_t>(ar - 1) * er + s, static_cast<int64_t>(bc - 1) * ec + r)
                : mt.at(static_cast<int64_t>(ar - 1) * er + r, static_cast<int64_t>(bc - 1) * ec + s);
    };
    if (gi == 1 && gj == 1) return toe(c11);
    if (gi == 2 && gj == 2) return toe(c22);
    if (gi == 3 && gj == 3) return toe(c33);
    if (gi == 4 && gj == 4) return toe(c44);
    if (gi == 2 && gj == 1) return c21[(a - b) + (ny - 1)].at(r, s);
    if (gi == 1 && gj == 2) return c21[(b - a) + (ny - 1)].at(s, r);
    if (gi == 4 && gj == 3) return c43[(a - b) + (nx - 1)].at(r, s);
    if (gi == 3 && gj == 4) return c43[(b - a) + (nx - 1)].at(s, r);
    if (gi == 3 && gj == 1) return rect(c31, a, b, eOf(3), eOf(1), false);
    if (gi == 1 && gj == 3) return rect(c31, b, a, eOf(3), eOf(1), true);
    if (gi == 4 && gj == 1) return rect(c41, a, b, eOf(4), eOf(1), false);
    if (gi == 1 && gj == 4) return rect(c41, b, a, eOf(4), eOf(1), true);
    if (gi == 3 && gj == 2) return rect(c32, a, b, eOf(3), eOf(2), false);
    if (gi == 2 && gj == 3) return rect(c32, b, a, eOf(3), eOf(2), true);
    if (gi == 4 && gj == 2) return rect(c42, a, b, eOf(4), eOf(2), false);
    if (gi == 2 && gj == 4) return rect(c42, b, a, eOf(4), eOf(2), true);
    if (gi == 5 && gj != 5) return c5x[gj - 1].at(cornerRowStart[a - 1] + r, static_cast<int64_t>(b - 1) * eOf(gj) + s);
    if (gi != 5 && gj == 5) return c5x[gi - 1].at(cornerRowStart[b - 1] + s, static_cast<int64_t>(a - 1) * eOf(gi) + r);
    return a <= b ? c55[a - 1][b - 1].at(r, s) : c55[b - 1][a - 1].at(s, r);
  };
  for (const Part& pi : parts)
    for (const Part& pj : parts)
      for (int s = 0; s < pj.size; ++s)
        for (int r = 0; r < pi.size; ++r) {
          const cplx v = blockEntry(pi, pj, r, s);
          out.c[static_cast<size_t>((pj.off + s) * nM + pi.off + r)] = make_double2(v.real(), v.imag());
        }
}

// ---- persisted spectrum -----------------------------------------------
namespace {
struct SpecHeader {
  char magic[5];
  uint8_t version;  // 2: + the generator key
  int32_t nx, ny, m, L0, L1;
  int64_t npairs;
  uint8_t hasKey;
  uint8_t key[32];  // tbt_set_cache_key of the context that wrote the file
};

// Two pinned staging buffers with an event each.
struct PinnedPair {
  char* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  void alloc(size_t bytes) {
    for (int b = 0; b < 2; ++b) {
      TBT_CUDA_CHECK(cudaMallocHost(&p[b], bytes));
      TBT_CUDA_CHECK(cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming));
    }
  }
  ~PinnedPair() {
    for (int b = 0; b < 2; ++b) {
      if (ev[b]) cudaEventDestroy(ev[b]);
      if (p[b]) cudaFreeHost(p[b]);
    }
  }
};
}  // namespace

void saveSpectra(Ctx& c, const std::string& path) {
  TBT_USER_CHECK(c.havePrecompute && !c.dist, "tbt_save_spectra: needs a precomputed single-GPU context");
  TBT_USER_CHECK(!c.fullMode, "tbt_save_spectra: FULL (non-reciprocal) generators are not cached");
  const long long mm = static_cast<long long>(c.m) * c.m;
  std::ofstream out(path, std::ios::binary);
  TBT_USER_CHECK(static_cast<bool>(out), "cannot write spectra cache: " + path);
  SpecHeader h{};
  std::memcpy(h.magic, "TBTS1", 5);
  h.version = 2;
  h.nx = c.nx;
  h.ny = c.ny;
  h.m = c.m;
  h.L0 = c.L0;
  h.L1 = c.L1;
  h.npairs = c.npairs;
  h.hasKey = c.haveCacheKey ? 1 : 0;
  std::memcpy(h.key, c.cacheKey, sizeof h.key);
  out.write(reinterpret_cast<const char*>(&h), sizeof h);
  out.write(reinterpret_cast<const char*>(c.genHost.data()), static_cast<std::streamsize>(mm * sizeof(double2)));
  // device -> pinned chunk -> file, the copy of the next chunk under the write of this one
  PinnedPair pin;
  const size_t total = static_cast<size_t>(c.npairs * mm) * sizeof(double2);
  const size_t chunk = std::min<size_t>(total, 64u << 20);
  if (chunk > 0) pin.alloc(chunk);
  auto fetch = [&](size_t off, int b) {
    TBT_CUDA_CHECK(cudaMemcpyAsync(pin.p[b], reinterpret_cast<const char*>(c.dSpectra) + off, std::min(chunk, total - off),
                                   cudaMemcpyDeviceToHost, c.stream));
    TBT_CUDA_CHECK(cudaEventRecord(pin.ev[b], c.stream));
  };
  if (total > 0) fetch(0, 0);
  int b = 0;
  for (size_t off = 0; off < total; off += chunk, b ^= 1) {
    if (off + chunk < total) fetch(off + chunk, b ^ 1);
    TBT_CUDA_CHECK(cudaEventSynchronize(pin.ev[b]));
    out.write(pin.p[b], static_cast<std::streamsize>(std::min(chunk, total - off)));
  }
  TBT_USER_CHECK(static_cast<bool>(out), "failed writing spectra cache: " + path);
}

void loadSpectra(Ctx& c, const std::string& path) {
  TBT_USER_CHECK(!c.dist, "tbt_load_spectra: not available on a distributed context");
  std::ifstream in(path, std::ios::binary);
  TBT_USER_CHECK(static_cast<bool>(in), "cannot open spectra cache: " + path);
  SpecHeader h{};
  in.read(reinterpret_cast<char*>(&h), sizeof h);
  TBT_USER_CHECK(in && std::string(h.magic, 5) == "TBTS1" && h.version == 2, "not a TBTS1 spectra cache: " + path);
  TBT_USER_CHECK(h.nx == c.nx && h.ny == c.ny && h.m == c.m && h.L0 == c.L0 && h.L1 == c.L1,
                 "spectra cache: dimensions / embedding do not match the context");
  // A cache of another generator set with the same shape (another frequency
  // of a sweep, another seed) would silently give a wrong operator.
  if (c.haveCacheKey)
    TBT_USER_CHECK(h.hasKey && std::memcmp(h.key, c.cacheKey, sizeof h.key) == 0,
                   "spectra cache: generator key does not match the context (written for other generators)");
  const long long mm = static_cast<long long>(c.m) * c.m;
  c.genHost.resize(static_cast<size_t>(mm));
  in.read(reinterpret_cast<char*>(c.genHost.data()), static_cast<std::streamsize>(mm * sizeof(double2)));
  TBT_USER_CHECK(static_cast<bool>(in), "spectra cache: truncated file");
  splitSelfBlock(c);
  std::vector<int> pairFGlobal;
  planPairs(c, pairFGlobal);
  TBT_USER_CHECK(c.npairs == h.npairs, "spectra cache: pair count mismatch");
  // The spectrum goes file -> pinned chunk -> device, the copy of one chunk
  // under the read of the next (one pageable multi-GB vector, zero-filled,
  // read and then staged by the driver, took 3.7 s at C4 against 0.22 s for
  // generators + K1).
  PinnedPair pin;
  const size_t total = static_cast<size_t>(c.npairs * mm) * sizeof(double2);
  const size_t chunk = std::min<size_t>(total, 64u << 20);
  if (chunk > 0) pin.alloc(chunk);
  int b = 0;
  for (size_t off = 0; off < total; off += chunk, b ^= 1) {
    const size_t n = std::min(chunk, total - off);
    TBT_CUDA_CHECK(cudaEventSynchronize(pin.ev[b]));  // the copy that last used this buffer
    in.read(pin.p[b], static_cast<std::streamsize>(n));
    if (!in) {
      cudaStreamSynchronize(c.stream);
      TBT_USER_CHECK(false, "spectra cache: truncated file");
    }
    TBT_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(c.dSpectra) + off, pin.p[b], n, cudaMemcpyHostToDevice,
                                   c.stream));
    TBT_CUDA_CHECK(cudaEventRecord(pin.ev[b], c.stream));
  }
  TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

}  // namespace tbt
