// Kernel K1: one-time Fourier transform of the translation blocks into the
// bin-pair-major layout streamed by the bin product (K3).
//
// Replaces buildASpectra + aEntry + fft2 (proj/src/linsolve.cpp:218-258).
// The reference stores ahat entry-major / bin-minor, [(m*e5+n)*L + f]
// (linsolve.cpp:147,256); K3 wants each bin's m x m block contiguous, so the
// shift grid is laid out [s1][s0][(a,b)] with the (a,b) entry as the
// contiguous batch index of the FFT line passes: after the 2-D transform,
// bin f's block is already one contiguous row-major m x m run.
//
// Half-spectrum storage. The reference's A obeys A(-i,-j) = A(i,j)^T for
// every shift except (0,0) (aEntry, linsolve.cpp:219). Writing
// Z(0,0) = S0 + K with S0 symmetric and K antisymmetric, the operator is
//   A = Toeplitz(S0 at shift 0) + blockdiag(K),
// and the first term's spectrum satisfies Ahat(-f) = Ahat(f)^T exactly.
// Only one block per bin pair {f, -f} is stored (plus the self-paired bins);
// K3 applies it as Ahat and as Ahat^T. K (zero for reciprocal data, i.e. all
// MoM data) is applied in the spatial domain.
#include <algorithm>
#include <cmath>

#include "tbt_internal.cuh"

namespace tbt {
namespace {

__device__ __forceinline__ int shiftOf(int s, int L, int n) {
  if (s < n) return s;           // non-negative shifts 0..n-1
  if (s >= L - (n - 1)) return s - L;  // negative shifts -(n-1)..-1
  return INT_MIN;                // zero padding
}

// G[s1][s0][ab] = Z(shift)(a, b) for rows a in [a0, a0 + rows); the
// mirrored half is mir * Z(-shift)^T (mir = 1: reciprocal generators; -1:
// the anti-reciprocal part of a FULL generator set, tbt_set_generators_full).
__global__ void gatherShiftGrid(const double2* __restrict__ gen, const double2* __restrict__ s0blk,
                                double2* __restrict__ G, int nx, int ny, int m, int L0, int L1,
                                int a0, int rows, double mir) {
  const long long B = static_cast<long long>(rows) * m;
  const long long total = static_cast<long long>(L0) * L1 * B;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long ab = q % B;
    const long long s = q / B;
    const int s0 = static_cast<int>(s % L0), s1 = static_cast<int>(s / L0);
    const int i = shiftOf(s1, L1, ny), j = shiftOf(s0, L0, nx);
    double2 v = make_double2(0.0, 0.0);
    if (i != INT_MIN && j != INT_MIN) {
      const int a = a0 + static_cast<int>(ab / m), b = static_cast<int>(ab % m);
      const long long mm = static_cast<long long>(m) * m;
      if (i == 0 && j == 0) {
        v = s0blk[static_cast<long long>(b) * m + a];
      } else if (i > 0 || (i == 0 && j > 0)) {
        const long long t = (i == 0) ? j : nx + static_cast<long long>(i - 1) * (2 * nx - 1) + (j - (1 - nx));
        v = gen[t * mm + static_cast<long long>(b) * m + a];
      } else {  // mirrored half: A(-i,-j)^T
        const int ii = -i, jj = -j;
        const long long t = (ii == 0) ? jj : nx + static_cast<long long>(ii - 1) * (2 * nx - 1) + (jj - (1 - nx));
        v = gen[t * mm + static_cast<long long>(a) * m + b];
        v = make_double2(mir * v.x, mir * v.y);
      }
    }
    G[q] = v;
  }
}

// spectra[p][a][b] = G[F_p][(a - a0) * m + b] for a in the chunk.
__global__ void scatterPairs(const double2* __restrict__ G, const int* __restrict__ pairF,
                             double2* __restrict__ spectra, long long npairs, int m, int a0,
                             int rows) {
  const long long B = static_cast<long long>(rows) * m;
  const long long total = npairs * B;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long p = q / B, ab = q % B;
    spectra[p * m * m + static_cast<long long>(a0) * m + ab] = G[static_cast<long long>(pairF[p]) * B + ab];
  }
}

}  // namespace

// The self block's antisymmetric part K = (Z0 - Z0^T)/2 (applied in space);
// returns the symmetric part S0 (column-major) for the gather.
std::vector<double2> splitSelfBlock(Ctx& c) {
  const int m = c.m;
  const long long mm = static_cast<long long>(m) * m;
  std::vector<double2> s0(mm), kk(mm);
  c.hasAntisym = false;
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) {
      const double2 zab = c.genHost[static_cast<size_t>(b) * m + a];  // (a,b) col-major
      const double2 zba = c.genHost[static_cast<size_t>(a) * m + b];
      // (z + z^T)/2 is exactly z when z is symmetric.
      s0[static_cast<size_t>(b) * m + a] = make_double2(0.5 * (zab.x + zba.x), 0.5 * (zab.y + zba.y));
      const double2 k = make_double2(0.5 * (zab.x - zba.x), 0.5 * (zab.y - zba.y));
      kk[static_cast<size_t>(a) * m + b] = k;  // row-major K[a][b]
      if (k.x != 0.0 || k.y != 0.0) c.hasAntisym = true;
    }
  if (c.dAntisym) {
    cudaFree(c.dAntisym);
    c.dAntisym = nullptr;
  }
  if (c.hasAntisym) {
    TBT_CUDA_CHECK(cudaMalloc(&c.dAntisym, mm * sizeof(double2)));
    uploadSync(c.dAntisym, kk.data(), mm * sizeof(double2), c.stream);
  }
  return s0;
}

// Bin pairs f and its partner -f (representatives f <= partner), the
// device pair tables and the spectrum allocation. Distributed: only the
// columns this rank owns (closed under s0 -> -s0, dist.cu), bins
// renumbered to the rank's local [s1][j] layout. pairFGlobal gets the
// global representative bins.
void planPairs(Ctx& c, std::vector<int>& pairFGlobal) {
  const long long mm = static_cast<long long>(c.m) * c.m;
  std::vector<int> colPos(c.L0, -1);
  int nLocalCols = c.L0;
  if (c.dist) {
    nLocalCols = static_cast<int>(c.myColList.size());
    for (int j = 0; j < nLocalCols; ++j) colPos[c.myColList[j]] = j;
  } else {
    for (int j = 0; j < c.L0; ++j) colPos[j] = j;
  }
  auto localBin = [&](long long f) {
    return static_cast<int>((f / c.L0) * nLocalCols + colPos[f % c.L0]);
  };
  c.pairF.clear();
  c.pairG.clear();
  pairFGlobal.clear();
  c.pairOfBin.assign(static_cast<size_t>(c.L), 0);
  for (long long f = 0; f < c.L; ++f) {
    const int s1 = static_cast<int>(f / c.L0), s0i = static_cast<int>(f % c.L0);
    if (colPos[s0i] < 0) continue;
    const long long g = static_cast<long long>((c.L1 - s1) % c.L1) * c.L0 + (c.L0 - s0i) % c.L0;
    if (f <= g) {
      c.pairOfBin[f] = static_cast<long long>(c.pairF.size());
      if (g != f) c.pairOfBin[g] = -(static_cast<long long>(c.pairF.size()) + 1);
      c.pairF.push_back(localBin(f));
      c.pairG.push_back(localBin(g));
      pairFGlobal.push_back(static_cast<int>(f));
    }
  }
  c.npairs = static_cast<long long>(c.pairF.size());
  if (c.dSpectra) cudaFree(c.dSpectra);
  if (c.dPairF) cudaFree(c.dPairF);
  if (c.dPairG) cudaFree(c.dPairG);
  c.dSpectra = nullptr;
  c.dPairF = c.dPairG = nullptr;
  TBT_CUDA_CHECK(cudaMalloc(&c.dSpectra, std::max<long long>(c.npairs, 1) * mm * sizeof(double2)));
  TBT_CUDA_CHECK(cudaMalloc(&c.dPairF, std::max<long long>(c.npairs, 1) * sizeof(int)));
  TBT_CUDA_CHECK(cudaMalloc(&c.dPairG, std::max<long long>(c.npairs, 1) * sizeof(int)));
  uploadSync(c.dPairF, c.pairF.data(), c.npairs * sizeof(int), c.stream);
  uploadSync(c.dPairG, c.pairG.data(), c.npairs * sizeof(int), c.stream);
}

namespace {
// K1 for one generator set (canonical Sparse order on the device, self
// block S0 column-major) into spectra [pair][a][b] (bin-pair-major).
void transformGenerators(Ctx& c, const double2* dGen, const std::vector<double2>& s0, double mir, double2* spectra,
                         const int* dPairFGlobal) {
  const int m = c.m, nx = c.nx, ny = c.ny;
  const long long mm = static_cast<long long>(m) * m;
  cudaStream_t s = c.stream;
  double2 *dS0 = nullptr, *dG = nullptr;
  TBT_CUDA_CHECK(cudaMalloc(&dS0, mm * sizeof(double2)));
  uploadSync(dS0, s0.data(), mm * sizeof(double2), s);
  // Row chunks bounded to ~4 GiB of transform workspace.
  const long long budget = 4LL << 30;
  int rows = static_cast<int>(std::max<long long>(1, std::min<long long>(m, budget / (c.L * m * 16))));
  TBT_CUDA_CHECK(cudaMalloc(&dG, c.L * rows * m * sizeof(double2)));
  const int sms = smCount(c.device);
  for (int a0 = 0; a0 < m; a0 += rows) {
    const int r = std::min(rows, m - a0);
    const long long B = static_cast<long long>(r) * m;
    gatherShiftGrid<<<sms * 8, 256, 0, s>>>(dGen, dS0, dG, nx, ny, m, c.L0, c.L1, a0, r, mir);
    TBT_CUDA_CHECK(cudaGetLastError());
    FftPass pa;  // along s0 (level 0), one line per s1 row, in place
    pa.in = dG;
    pa.out = dG;
    pa.lines = c.L1;
    pa.in_line_stride = pa.out_line_stride = static_cast<long long>(c.L0) * B;
    pa.in_point_stride = pa.out_point_stride = B;
    pa.n = pa.n_in = pa.n_out = c.L0;
    pa.batch = static_cast<int>(B);
    pa.tw = c.dTw0;
    launchFftPass(pa, s);
    FftPass pb;  // along s1 (level 1), one line per s0 column, in place
    pb.in = dG;
    pb.out = dG;
    pb.lines = c.L0;
    pb.in_line_stride = pb.out_line_stride = B;
    pb.in_point_stride = pb.out_point_stride = static_cast<long long>(c.L0) * B;
    pb.n = pb.n_in = pb.n_out = c.L1;
    pb.batch = static_cast<int>(B);
    pb.tw = c.dTw1;
    launchFftPass(pb, s);
    if (c.npairs > 0) scatterPairs<<<sms * 8, 256, 0, s>>>(dG, dPairFGlobal, spectra, c.npairs, m, a0, r);
    TBT_CUDA_CHECK(cudaGetLastError());
  }
  TBT_CUDA_CHECK(cudaStreamSynchronize(s));
  cudaFree(dG);
  cudaFree(dS0);
}
}  // namespace

void buildSpectra(Ctx& c) {
  const long long mm = static_cast<long long>(c.m) * c.m;
  cudaStream_t s = c.stream;
  const std::vector<double2> s0 = splitSelfBlock(c);
  std::vector<int> pairFGlobal;
  planPairs(c, pairFGlobal);
  int* dPairFGlobal = nullptr;
  TBT_CUDA_CHECK(cudaMalloc(&dPairFGlobal, std::max<long long>(c.npairs, 1) * sizeof(int)));
  uploadSync(dPairFGlobal, pairFGlobal.data(), c.npairs * sizeof(int), s);
  transformGenerators(c, c.dGen, s0, 1.0, c.dSpectra, dPairFGlobal);
  if (c.dSpectraAnti) cudaFree(c.dSpectraAnti);
  c.dSpectraAnti = nullptr;
  if (c.fullMode) {
    // The anti-reciprocal part (FULL generators): Ahat_a(-f) = -Ahat_a(f)^T,
    // the same half storage with the partner's product negated by K3.
    TBT_CUDA_CHECK(cudaMalloc(&c.dSpectraAnti, std::max<long long>(c.npairs, 1) * mm * sizeof(double2)));
    const std::vector<double2> zero(static_cast<size_t>(mm), make_double2(0.0, 0.0));
    transformGenerators(c, c.dGenAnti, zero, -1.0, c.dSpectraAnti, dPairFGlobal);
  }
  cudaFree(dPairFGlobal);
}

}  // namespace tbt
