// Row f4: contractions on the solved currents (proj/src/postproc.cpp).
//
//  * portNetwork (:186-230): port currents I(i, c) = current(feedRow_i, c),
//    Y = I / len^2, Z = Y^-1 (partial-pivot LU with the pivot-ratio check),
//    power-wave S = (Z - Z0)(Z + Z0)^-1 scaled by sqrt(z0_j / z0_i).
//  * arrayFarfield / embeddedElementPatterns (:134-184): for excitation
//    weights W (p x q), combined = current W, then per direction i
//        F(i, j) = -j k eta sum_parts e^{j k d_i . o_part} T_comp(part)(i, :) combined(part rows, j)
//    with T the component far-field tensors (co and cross polarisation).
//    One CTA per (direction, column): the phase table per (direction, part)
//    is built first, the contraction streams the combined currents once per
//    direction with fixed-order reductions.
#include <algorithm>
#include <cmath>
#include <limits>

#include "dense.cuh"

namespace tbt {
namespace {

int gridFor(long long n) { return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 8192))); }

// out (M x N, column-major) = A (M x K, lda) * B (K x N, ldb).
__global__ void zgemmNN(const double2* __restrict__ A, long long lda, const double2* __restrict__ B, long long ldb,
                        double2* __restrict__ out, long long ldo, long long M, int N, int K) {
  const long long total = M * N;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = o % M;
    const int j = static_cast<int>(o / M);
    double2 acc = make_double2(0.0, 0.0);
    for (int k = 0; k < K; ++k) cfma(acc, A[i + k * lda], B[k + static_cast<long long>(j) * ldb]);
    out[i + static_cast<long long>(j) * ldo] = acc;
  }
}

// Port currents scaled: Y(i, c) = current(feed_i, c) / len^2.
__global__ void gatherPorts(const double2* __restrict__ cur, long long ldc, const long long* __restrict__ feed,
                            int p, double inv2, double2* __restrict__ Y) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < p * p; o += gridDim.x * blockDim.x) {
    const int i = o % p, c = o / p;
    const double2 v = cur[feed[i] + c * ldc];
    Y[o] = make_double2(v.x * inv2, v.y * inv2);
  }
}

__global__ void identity(double2* __restrict__ M, int p) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < p * p; o += gridDim.x * blockDim.x)
    M[o] = make_double2((o % p) == (o / p) ? 1.0 : 0.0, 0.0);
}

// zm = Z - diag(z0), zp = Z + diag(z0).
__global__ void zShift(const double2* __restrict__ Z, const double* __restrict__ z0, double2* __restrict__ zm,
                       double2* __restrict__ zp, int p) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < p * p; o += gridDim.x * blockDim.x) {
    const int i = o % p, j = o / p;
    double2 v = Z[o];
    double2 a = v, b = v;
    if (i == j) {
      a.x -= z0[i];
      b.x += z0[i];
    }
    zm[o] = a;
    zp[o] = b;
  }
}

__global__ void scaleS(double2* __restrict__ S, const double* __restrict__ z0, int p) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < p * p; o += gridDim.x * blockDim.x) {
    const int i = o % p, j = o / p;
    const double f = sqrt(z0[j] / z0[i]);
    S[o] = make_double2(S[o].x * f, S[o].y * f);
  }
}

struct Parts {
  int nparts;
  const int* comp;        // [nparts] component 1..9
  const long long* start; // [nparts] first row in the current vector
  const double* off;      // [nparts][3] part offsets
  const double2* co[9];   // [ndir][e_c] column-major (ndir rows)
  const double2* cx[9];
  int e[9];
};

// phase[i][part] = exp(j k d_i . o_part)
__global__ void phaseTable(const double* __restrict__ dirs, Parts P, int ndir, double k, double2* __restrict__ ph) {
  const long long total = static_cast<long long>(ndir) * P.nparts;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int part = static_cast<int>(o % P.nparts), i = static_cast<int>(o / P.nparts);
    const double* d = dirs + 3 * i;
    const double* q = P.off + 3 * part;
    double sn, cs;
    sincos(k * (d[0] * q[0] + d[1] * q[1] + d[2] * q[2]), &sn, &cs);
    ph[o] = make_double2(cs, sn);
  }
}

// CTA per (direction i, column j): F(i, j) for both polarisations.
__global__ void __launch_bounds__(256) farfieldKernel(Parts P, const double2* __restrict__ ph,
                                                      const double2* __restrict__ comb, long long ldc, int ndir,
                                                      double2 front, double2* __restrict__ co,
                                                      double2* __restrict__ cx) {
  __shared__ double2 rco[256], rcx[256];
  const int i = blockIdx.x, j = blockIdx.y;
  const double2* cj = comb + static_cast<long long>(j) * ldc;
  double2 aco = make_double2(0.0, 0.0), acx = aco;
  for (int part = 0; part < P.nparts; ++part) {
    const int c = P.comp[part] - 1;
    const int n = P.e[c];
    if (n == 0) continue;
    const double2 phs = ph[static_cast<long long>(i) * P.nparts + part];
    const double2* seg = cj + P.start[part];
    double2 sco = make_double2(0.0, 0.0), scx = sco;
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
      const double2 v = seg[t];
      cfma(sco, P.co[c][i + static_cast<long long>(t) * ndir], v);
      cfma(scx, P.cx[c][i + static_cast<long long>(t) * ndir], v);
    }
    cfma(aco, phs, sco);
    cfma(acx, phs, scx);
  }
  rco[threadIdx.x] = aco;
  rcx[threadIdx.x] = acx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      rco[threadIdx.x] = cadd(rco[threadIdx.x], rco[threadIdx.x + s]);
      rcx[threadIdx.x] = cadd(rcx[threadIdx.x], rcx[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    co[i + static_cast<long long>(j) * ndir] = cmul(front, rco[0]);
    cx[i + static_cast<long long>(j) * ndir] = cmul(front, rcx[0]);
  }
}

struct Dev {
  void* p = nullptr;
  explicit Dev(size_t bytes) { TBT_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
  ~Dev() { cudaFree(p); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

// LU-invert a p x p column-major matrix in place (dst = M^-1); returns the
// pivot ratio min|u_kk| / max|u_kk|.
double luInvert(double2* M, double2* dst, int p, cudaStream_t s) {
  Dev perm(static_cast<size_t>(p) * sizeof(int)), scratch(static_cast<size_t>(p) * p * sizeof(double2));
  std::vector<int> id(p);
  for (int i = 0; i < p; ++i) id[i] = i;
  uploadSync(perm.p, id.data(), p * sizeof(int), s);
  if (p <= 512) {  // one CTA, barriers between steps
    dense::luFactorSmall<<<1, 1024, 0, s>>>(M, p, perm.as<int>());
  } else {
    for (int k = 0; k < p; ++k) {
      dense::luPivot<<<1, 256, 0, s>>>(M, p, k, perm.as<int>());
      if (k + 1 < p) dense::luUpdate<<<gridFor(static_cast<long long>(p - k - 1) * (p - k - 1)), 256, 0, s>>>(M, p, k);
    }
  }
  std::vector<double2> diag(p);
  TBT_CUDA_CHECK(cudaMemcpy2DAsync(diag.data(), sizeof(double2), M, (p + 1) * sizeof(double2), sizeof(double2), p,
                                   cudaMemcpyDeviceToHost, s));
  identity<<<gridFor(static_cast<long long>(p) * p), 256, 0, s>>>(dst, p);
  dense::luSolveCols<<<p, 256, 0, s>>>(M, perm.as<int>(), p, dst, scratch.as<double2>());
  TBT_CUDA_CHECK(cudaGetLastError());
  TBT_CUDA_CHECK(cudaStreamSynchronize(s));
  double maxAbs = 0.0, minAbs = std::numeric_limits<double>::infinity();
  for (const double2& d : diag) {
    const double a = std::hypot(d.x, d.y);
    maxAbs = std::max(maxAbs, a);
    minAbs = std::min(minAbs, a);
  }
  return minAbs / (maxAbs > 0 ? maxAbs : 1.0);
}

}  // namespace

// Device pointers throughout; y, z, s: p x p column-major.
void portNetwork(Ctx& c, const double2* current, long long ldc, int p, const long long* feedDev, double len,
                 const double* z0Dev, double2* y, double2* z, double2* sOut) {
  cudaStream_t s = c.stream;
  gatherPorts<<<gridFor(static_cast<long long>(p) * p), 256, 0, s>>>(current, ldc, feedDev, p, 1.0 / (len * len), y);
  Dev work(static_cast<size_t>(p) * p * sizeof(double2));
  TBT_CUDA_CHECK(cudaMemcpyAsync(work.p, y, static_cast<size_t>(p) * p * sizeof(double2), cudaMemcpyDeviceToDevice, s));
  const double ratio = luInvert(work.as<double2>(), z, p, s);
  if (!(ratio > 1e-14)) throw Error{TBT_NUMERIC_ERROR, "portNetwork: singular admittance matrix"};
  Dev zm(static_cast<size_t>(p) * p * sizeof(double2)), zp(static_cast<size_t>(p) * p * sizeof(double2)),
      zpi(static_cast<size_t>(p) * p * sizeof(double2));
  zShift<<<gridFor(static_cast<long long>(p) * p), 256, 0, s>>>(z, z0Dev, zm.as<double2>(), zp.as<double2>(), p);
  luInvert(zp.as<double2>(), zpi.as<double2>(), p, s);
  zgemmNN<<<gridFor(static_cast<long long>(p) * p), 256, 0, s>>>(zm.as<double2>(), p, zpi.as<double2>(), p, sOut, p, p,
                                                                  p, p);
  scaleS<<<gridFor(static_cast<long long>(p) * p), 256, 0, s>>>(sOut, z0Dev, p);
  TBT_CUDA_CHECK(cudaGetLastError());
}

void arrayFarfield(Ctx& c, const double2* const* tco, const double2* const* tcx, const int* e, int ndir,
                   const double* dirsDev, double dx, double dy, double k, double eta, const double2* current,
                   long long ntot, int p, const double2* W, int q, double2* co, double2* cx) {
  cudaStream_t s = c.stream;
  const int nx = c.nx, ny = c.ny;
  // Parts in the reference order (array_model.cpp:218-228) with offsets.
  std::vector<int> comp;
  std::vector<long long> start;
  std::vector<double> off;
  long long row = 0;
  auto place = [&](int cmp, double ox, double oy) {
    comp.push_back(cmp);
    start.push_back(row);
    off.insert(off.end(), {ox, oy, 0.0});
    row += e[cmp - 1];
  };
  for (int r = 1; r <= ny; ++r)
    for (int col = 1; col <= nx; ++col) place(5, (col - 1) * dx, (r - 1) * dy);
  for (int r = 1; r <= ny; ++r) place(2, 0.0, (r - 1) * dy);
  for (int r = 1; r <= ny; ++r) place(8, (nx - 1) * dx, (r - 1) * dy);
  for (int col = 1; col <= nx; ++col) place(6, (col - 1) * dx, (ny - 1) * dy);
  for (int col = 1; col <= nx; ++col) place(4, (col - 1) * dx, 0.0);
  place(3, 0.0, (ny - 1) * dy);
  place(9, (nx - 1) * dx, (ny - 1) * dy);
  place(1, 0.0, 0.0);
  place(7, (nx - 1) * dx, 0.0);
  TBT_USER_CHECK(row == ntot, "arrayFarfield: current vector size mismatch");
  const int nparts = static_cast<int>(comp.size());
  Dev dComp(nparts * sizeof(int)), dStart(nparts * sizeof(long long)), dOff(off.size() * sizeof(double));
  uploadSync(dComp.p, comp.data(), nparts * sizeof(int), s);
  uploadSync(dStart.p, start.data(), nparts * sizeof(long long), s);
  uploadSync(dOff.p, off.data(), off.size() * sizeof(double), s);
  Parts P{};
  P.nparts = nparts;
  P.comp = dComp.as<int>();
  P.start = dStart.as<long long>();
  P.off = dOff.as<double>();
  for (int i = 0; i < 9; ++i) {
    P.co[i] = tco[i];
    P.cx[i] = tcx[i];
    P.e[i] = e[i];
  }
  // combined = current W (ntot x q).
  Dev comb(static_cast<size_t>(ntot) * q * sizeof(double2));
  zgemmNN<<<gridFor(ntot * q), 256, 0, s>>>(current, ntot, W, p, comb.as<double2>(), ntot, ntot, q, p);
  Dev ph(static_cast<size_t>(ndir) * nparts * sizeof(double2));
  phaseTable<<<gridFor(static_cast<long long>(ndir) * nparts), 256, 0, s>>>(dirsDev, P, ndir, k, ph.as<double2>());
  farfieldKernel<<<dim3(ndir, q), 256, 0, s>>>(P, ph.as<double2>(), comb.as<double2>(), ntot, ndir,
                                               make_double2(0.0, -k * eta), co, cx);
  TBT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tbt
