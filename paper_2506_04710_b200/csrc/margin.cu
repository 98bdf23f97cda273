// Margin coupling: the B / B^T / C part of the reference
// operator, ToeplitzMatvec::apply = [A xA + B^T xM ; B xA + C xM]
// (proj/src/linsolve.cpp:373-388), for representations with margin parts.
//
//   B1/B2  components 2 and 8 (one part per element row): one-level block
//          Toeplitz over the element rows, block (margin row a, element row
//          b) = G(a - b) of size e_c x (nx*m)           (linsolve.cpp:179-186)
//   B3/B4  components 6 and 4 (one part per element column): for every
//          element row j a one-level block Toeplitz over x, block (margin
//          column a, element (j, b)) = G_j(a - b), e_c x m; the ny rows sum
//          into the same margin segment                   (:187-195, :305-307)
//   B5-B8  corners 3, 9, 1, 7: dense e_c x nA                    (:308-312)
//   C      margin x margin, dense (the reference caches it block-wise as
//          cBlocks, :210-215, :336-349)
//
// As in the reference, the Toeplitz parts go through circulant embeddings of
// length nextPow2(2n-1) (Toe1D, linsolve.cpp:54-134), here bin-major on the
// device: the spectra Ghat[f][i][q] are built once (gather + batched FFT
// pass), every apply transforms x along the element rows / columns once
// (shared by both regions), forms the per-bin products for B and, reading
// the same spectra at the reversed bin, for B^T (the transposed circulant,
// :316-334), and transforms back with the 1/L crop. Corners and C are
// warp-per-row dense products.
//
// Layouts. Internal vectors are [element][rhs][basis] over ne + neM
// elements: the margin unknowns k < nM follow the element part as
// pseudo-elements (element ne + k/m, basis k%m), padded with zeros, so the
// GMRES kernels see one uniform vector. Margin work vectors use the staging
// layout [k][rhs] (k in the reference margin order, array_model.cpp:218-228).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "margin.cuh"

namespace tbt {

namespace {

int gridFor(long long n) { return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 4096))); }

// Circulant sequence of a one-level Toeplitz generator set, bin-major:
// seq[line][s][t] (t = i*q + j over the p x q block, row-major) from raw
// column-major blocks raw[line][idx][j*p + i], idx = shift + (n - 1); shift
// s >= 0 at s < n, negative shift -s' at L - s' (Toe1D::build, :66-81).
__global__ void toeSeq(const double2* __restrict__ raw, double2* __restrict__ seq, int lines, int L, int n, int p,
                       long long q) {
  const long long P = static_cast<long long>(p) * q;
  const long long total = static_cast<long long>(lines) * L * P;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long t = o % P;
    const long long ls = o / P;
    const int s = static_cast<int>(ls % L), line = static_cast<int>(ls / L);
    int shift;
    if (s < n)
      shift = s;
    else if (s > L - n)
      shift = s - L;
    else
      shift = INT_MIN;
    double2 v = make_double2(0.0, 0.0);
    if (shift != INT_MIN) {
      const long long i = t / q, j = t % q;
      const long long blk = static_cast<long long>(line) * (2 * n - 1) + shift + (n - 1);
      v = raw[blk * P + j * p + i];
    }
    seq[o] = v;
  }
}

// out[r][c] = in[c][r] for a rows x cols column-major input (row-major out).
__global__ void transposeCM(const double2* __restrict__ in, double2* __restrict__ out, long long rows,
                            long long cols) {
  const long long total = rows * cols;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = o / cols, c = o % cols;
    out[o] = in[c * rows + r];
  }
}

// xs[k][rhs] = x[((ne + k/m)*K + rhs)*m + k%m]
__global__ void marginGather(const double2* __restrict__ x, double2* __restrict__ xs, long long nM, int ne, int m,
                             int K) {
  const long long total = nM * K;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = o / K;
    const int rhs = static_cast<int>(o % K);
    xs[o] = x[((ne + k / m) * K + rhs) * m + k % m];
  }
}

// y pseudo-elements (zero padding past nM) from ys[k][rhs].
__global__ void marginScatter(const double2* __restrict__ ys, double2* __restrict__ y, long long nM, int ne, int neM,
                              int m, int K) {
  const long long total = static_cast<long long>(neM) * m * K;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    // o enumerates the internal pseudo-element region [e'][rhs][b].
    const int b = static_cast<int>(o % m);
    const long long rest = o / m;
    const int rhs = static_cast<int>(rest % K);
    const long long ep = rest / K;
    const long long k = ep * m + b;
    y[static_cast<long long>(ne) * K * m + o] = k < nM ? ys[k * K + rhs] : make_double2(0.0, 0.0);
  }
}

// B1/B2 per-bin product: hatMs[r][f][i][rhs] = sum_{c,k} G_r[f][i][c*m+k] hatY[f][c][rhs][k].
// One warp per (r, f, i, rhs), lanes over the nx*m sources.
// CTA-wide fixed-order sum (warp butterflies, then warps in order).
__device__ __forceinline__ double2 ctaSum128(double2 v, double2* red) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double2 t = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = cadd(t, red[w]);
  return t;
}

// B1/B2 per-bin product: hatMs[r][f][i][rhs] = sum_{c,k} G_r[f][i][c*m+k] hatY[f][c][rhs][k].
// One CTA per (r, f, i, rhs), threads over the nx*m sources.
__global__ void __launch_bounds__(128) sideProd(const double2* __restrict__ g0, const double2* __restrict__ g1,
                                                int em0, int em1, const double2* __restrict__ hatY,
                                                double2* __restrict__ out0, double2* __restrict__ out1, int Ly,
                                                int nx, int m, int K) {
  __shared__ double2 red[4];
  const int q = nx * m;
  const long long w = blockIdx.x;
  const int rhs = static_cast<int>(w % K);
  const long long rest = w / K;
  const int f = static_cast<int>(rest % Ly);
  int i = static_cast<int>(rest / Ly);
  const int r = i < em0 ? 0 : 1;
  if (r == 1) i -= em0;
  const int em = r == 0 ? em0 : em1;
  const double2* G = (r == 0 ? g0 : g1) + (static_cast<long long>(f) * em + i) * q;
  const double2* X = hatY + static_cast<long long>(f) * nx * K * m;
  double2 acc = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < q; t += blockDim.x) {
    const int c = t / m, k = t - c * m;
    cfma(acc, __ldg(G + t), X[(static_cast<long long>(c) * K + rhs) * m + k]);
  }
  acc = ctaSum128(acc, red);
  if (threadIdx.x == 0) (r == 0 ? out0 : out1)[(static_cast<long long>(f) * em + i) * K + rhs] = acc;
}

// B3/B4 per-bin product: hatMr[r][f][i][rhs] = sum_j sum_k G_r[j][f][i][k] hatX[f][j][rhs][k].
// B3/B4 per-bin product: hatMr[r][f][i][rhs] = sum_j sum_k G_r[j][f][i][k] hatX[f][j][rhs][k].
// One CTA per (r, f, i, rhs), threads over the ny*m sources.
__global__ void __launch_bounds__(128) rowProd(const double2* __restrict__ g0, const double2* __restrict__ g1,
                                               int em0, int em1, const double2* __restrict__ hatX,
                                               double2* __restrict__ out0, double2* __restrict__ out1, int Lx,
                                               int ny, int m, int K) {
  __shared__ double2 red[4];
  const long long w = blockIdx.x;
  const int rhs = static_cast<int>(w % K);
  const long long rest = w / K;
  const int f = static_cast<int>(rest % Lx);
  int i = static_cast<int>(rest / Lx);
  const int r = i < em0 ? 0 : 1;
  if (r == 1) i -= em0;
  const int em = r == 0 ? em0 : em1;
  const double2* G = r == 0 ? g0 : g1;
  double2 acc = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < ny * m; t += blockDim.x) {
    const int j = t / m, k = t - j * m;
    cfma(acc, __ldg(G + ((static_cast<long long>(j) * Lx + f) * em + i) * m + k),
         hatX[((static_cast<long long>(f) * ny + j) * K + rhs) * m + k]);
  }
  acc = ctaSum128(acc, red);
  if (threadIdx.x == 0) (r == 0 ? out0 : out1)[(static_cast<long long>(f) * em + i) * K + rhs] = acc;
}

// B^T over the side regions: hatZy[f][c][rhs][k] = sum_r sum_i G_r[-f][i][c*m+k] hatMs[r][f][i][rhs]
// (Toe1D::applyT's reversed bin, linsolve.cpp:327-329).
__global__ void sideProdT(const double2* __restrict__ g0, const double2* __restrict__ g1, int em0, int em1,
                          const double2* __restrict__ hm0, const double2* __restrict__ hm1,
                          double2* __restrict__ hatZy, int Ly, int nx, int m, int K) {
  const long long q = static_cast<long long>(nx) * m;
  const long long total = static_cast<long long>(Ly) * nx * K * m;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(o % m);
    long long rest = o / m;
    const int rhs = static_cast<int>(rest % K);
    rest /= K;
    const long long c = rest % nx;
    const int f = static_cast<int>(rest / nx);
    const int fr = (Ly - f) % Ly;
    const long long col = c * m + k;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < em0; ++i)
      cfma(acc, g0[(static_cast<long long>(fr) * em0 + i) * q + col], hm0[(static_cast<long long>(f) * em0 + i) * K + rhs]);
    for (int i = 0; i < em1; ++i)
      cfma(acc, g1[(static_cast<long long>(fr) * em1 + i) * q + col], hm1[(static_cast<long long>(f) * em1 + i) * K + rhs]);
    hatZy[o] = acc;
  }
}

// B^T over the row regions: hatZx[f][j][rhs][k] = sum_r sum_i G_r[j][-f][i][k] hatMr[r][f][i][rhs].
__global__ void rowProdT(const double2* __restrict__ g0, const double2* __restrict__ g1, int em0, int em1,
                         const double2* __restrict__ hm0, const double2* __restrict__ hm1, double2* __restrict__ hatZx,
                         int Lx, int ny, int m, int K) {
  const long long total = static_cast<long long>(Lx) * ny * K * m;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(o % m);
    long long rest = o / m;
    const int rhs = static_cast<int>(rest % K);
    rest /= K;
    const long long j = rest % ny;
    const int f = static_cast<int>(rest / ny);
    const int fr = (Lx - f) % Lx;
    double2 acc = make_double2(0.0, 0.0);
    for (int i = 0; i < em0; ++i)
      cfma(acc, g0[((j * Lx + fr) * em0 + i) * m + k], hm0[(static_cast<long long>(f) * em0 + i) * K + rhs]);
    for (int i = 0; i < em1; ++i)
      cfma(acc, g1[((j * Lx + fr) * em1 + i) * m + k], hm1[(static_cast<long long>(f) * em1 + i) * K + rhs]);
    hatZx[o] = acc;
  }
}

struct CornerArgs {
  const double2* bc[4];  // [em][nA] row-major
  int em[4];
  long long start[4];    // margin offsets
};

// B5..B8 (linsolve.cpp:308-312), ys[start_c + i][rhs] = sum_q bc[i][q] xA[q],
// two fixed-order stages: CTA (element block, corner row) partial sums over
// kCornerElems elements, then cornerReduce over the blocks.
constexpr int kCornerElems = 16;

__global__ void __launch_bounds__(256) cornerPart(CornerArgs ca, const double2* __restrict__ x,
                                                  double2* __restrict__ part, int ne, int m, int K, int nblk) {
  __shared__ double2 red[8];
  int i = blockIdx.y, c = 0;
  while (i >= ca.em[c]) i -= ca.em[c++];
  const long long nA = static_cast<long long>(ne) * m;
  const double2* row = ca.bc[c] + static_cast<long long>(i) * nA;
  const int e0 = blockIdx.x * kCornerElems, e1 = min(ne, e0 + kCornerElems);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int rhs = 0; rhs < K; ++rhs) {
    double2 acc = make_double2(0.0, 0.0);
    for (int e = e0 + warp; e < e1; e += 8) {
      const double2* r = row + static_cast<long long>(e) * m;
      const double2* xe = x + (static_cast<long long>(e) * K + rhs) * m;
      for (int k = lane; k < m; k += 32) cfma(acc, r[k], xe[k]);
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
    }
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 t = red[0];
      for (int w = 1; w < 8; ++w) t = cadd(t, red[w]);
      part[(static_cast<long long>(blockIdx.y) * K + rhs) * nblk + blockIdx.x] = t;
    }
    __syncthreads();
  }
}

__global__ void cornerReduce(CornerArgs ca, const double2* __restrict__ part, double2* __restrict__ ys, int K,
                             int nblk) {
  const int rowsTot = ca.em[0] + ca.em[1] + ca.em[2] + ca.em[3];
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= rowsTot * K) return;
  const int rhs = w % K;
  int i = w / K, c = 0;
  const int gRow = i;
  while (i >= ca.em[c]) i -= ca.em[c++];
  const double2* p = part + (static_cast<long long>(gRow) * K + rhs) * nblk;
  double2 acc = make_double2(0.0, 0.0);
  for (int b0 = lane; b0 < nblk; b0 += 256) {  // 8 loads in flight per lane, summed in block order
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = b0 + 32 * q < nblk ? p[b0 + 32 * q] : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = cadd(acc, v[q]);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, off);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, off);
  }
  if (lane == 0) ys[(ca.start[c] + i) * K + rhs] = acc;
}

// ys[k][rhs] += sum_l C[k][l] xs[l][rhs] (applyC, linsolve.cpp:336-349).
// ys[k][rhs] += sum_l C[k][l] xs[l][rhs] (applyC, linsolve.cpp:336-349); CTA per (k, rhs).
__global__ void __launch_bounds__(128) cProd(const double2* __restrict__ C, const double2* __restrict__ xs,
                                             double2* __restrict__ ys, long long nM, int K, int set = 0) {
  __shared__ double2 red[4];
  const long long k = blockIdx.x / K;
  const int rhs = static_cast<int>(blockIdx.x % K);
  const double2* row = C + k * nM;
  double2 acc = make_double2(0.0, 0.0);
  for (long long l = threadIdx.x; l < nM; l += blockDim.x) cfma(acc, __ldg(row + l), xs[l * K + rhs]);
  acc = ctaSum128(acc, red);
  if (threadIdx.x == 0) ys[k * K + rhs] = set ? acc : cadd(ys[k * K + rhs], acc);
}

// yA += zA + zA2 + sum_c bc^T xM_c (B^T's corner part, linsolve.cpp:328-332).
__global__ void addBT(double2* __restrict__ y, const double2* __restrict__ zA, const double2* __restrict__ zA2,
                      CornerArgs ca, const double2* __restrict__ xs, long long nA, int m, int K) {
  const long long total = nA * K;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    // o enumerates the internal element region [e][rhs][b].
    const int b = static_cast<int>(o % m);
    const long long rest = o / m;
    const int rhs = static_cast<int>(rest % K);
    const long long e = rest / K;
    const long long q = e * m + b;
    double2 acc = y[o];
    if (zA) acc = cadd(acc, zA[o]);
    if (zA2) acc = cadd(acc, zA2[o]);
    for (int c = 0; c < 4; ++c)
      for (int i = 0; i < ca.em[c]; ++i)
        cfma(acc, ca.bc[c][static_cast<long long>(i) * nA + q], xs[(ca.start[c] + i) * K + rhs]);
    y[o] = acc;
  }
}


// Dense B (SemiSparse representations, linsolve.cpp:294 / :318).
// ys[k][rhs] += sum_q B[k][q] xA[q][rhs]; CTA per (k, rhs), B row-major,
// xA in the internal layout [e][rhs][b] (q = e*m + b).
__global__ void __launch_bounds__(128) denseBProd(const double2* __restrict__ Bd, const double2* __restrict__ x,
                                                  double2* __restrict__ ys, long long nA, int m, int K) {
  __shared__ double2 red[4];
  const long long k = blockIdx.x / K;
  const int rhs = static_cast<int>(blockIdx.x % K);
  const double2* row = Bd + k * nA;
  double2 acc = make_double2(0.0, 0.0);
  for (long long q = threadIdx.x; q < nA; q += blockDim.x)
    cfma(acc, __ldg(row + q), x[((q / m) * K + rhs) * m + q % m]);
  acc = ctaSum128(acc, red);
  if (threadIdx.x == 0) ys[k * K + rhs] = cadd(ys[k * K + rhs], acc);
}

// yA[q][rhs] += sum_k B[k][q] xs[k][rhs] (B^T xM): thread per (q, rhs), the
// reads of one B row are coalesced across q.
__global__ void denseBTProd(const double2* __restrict__ Bd, const double2* __restrict__ xs, double2* __restrict__ y,
                            long long nA, long long nM, int m, int K) {
  const long long total = nA * K;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = o % nA;
    const int rhs = static_cast<int>(o / nA);
    double2 acc = make_double2(0.0, 0.0);
    for (long long k = 0; k < nM; ++k) cfma(acc, __ldg(Bd + k * nA + q), xs[k * K + rhs]);
    double2& dst = y[((q / m) * K + rhs) * m + q % m];
    dst = cadd(dst, acc);
  }
}

// ---- single-column fused margin products: every generator spectrum and
// corner block is read ONCE per apply and feeds both B (row dots) and B^T
// (column sums at the reversed bin / transposed block). EM bounds the rows
// per region (registers).
constexpr int kFuseThreads = 256;
constexpr int kFuseChunk = 512;  // generator columns per CTA (2 per thread)
constexpr int kCornerQ = 1024;   // corner columns per CTA (256 when that leaves < 4 CTAs per SM)
constexpr int kLoadGroup = 16;   // generator loads issued back to back

__device__ __forceinline__ double2 warpSumM(double2 v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  return v;
}

// Fixed-order CTA reduction of nv per-thread values pv[0..nv) into
// out[v * stride] (thread 0 writes), red: [warps][nv] shared.
template <int NV>
__device__ __forceinline__ void ctaReduceMany(double2 (&pv)[NV], int nv, double2* red, double2* out, long long stride) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (v >= nv) break;
    const double2 t = warpSumM(pv[v]);
    if (lane == 0) red[warp * NV + v] = t;
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nv; v += blockDim.x) {
    double2 t = red[v];
    for (int w = 1; w < nw; ++w) t = cadd(t, red[w * NV + v]);
    out[v * stride] = t;
  }
}

// Prologue of the side/row kernels: the two margin-part spectra at bin hr,
// by direct DFT of the nIn margin unknowns (1-D Toeplitz embedding of
// linsolve.cpp:300-306, zero-padded to L; forward sign as twiddles()):
//   mIn[r*EM + i] = sum_{j<nIn} xs[start_r + j*em_r + i] tw[(hr*j) mod L].
// Dead slots (i >= em_r) get 0. Fixed-order reduction over 8 thread groups.
template <int EM>
__device__ __forceinline__ void marginDft(const double2* __restrict__ xs0, const double2* __restrict__ xs1, int em0,
                                          int em1, int nIn, int hr, int L, const double2* __restrict__ tw,
                                          double2* mIn, double2* scratch /* [8][32] */) {
  static_assert(2 * EM <= 32, "one warp-wide slot per margin row");
  const int v = threadIdx.x & 31, grp = threadIdx.x >> 5, ngrp = blockDim.x >> 5;
  double2 acc = make_double2(0.0, 0.0);
  if (v < 2 * EM) {
    const int r = v / EM, i = v % EM, em = r ? em1 : em0;
    const double2* src = r ? xs1 : xs0;
    if (i < em && src)
      for (int j = grp; j < nIn; j += ngrp)
        cfma(acc, src[static_cast<long long>(j) * em + i], tw[(static_cast<long long>(hr) * j) % L]);
  }
  scratch[grp * 32 + v] = acc;
  __syncthreads();
  if (threadIdx.x < 2 * EM) {
    double2 t = scratch[threadIdx.x];
    for (int g = 1; g < ngrp; ++g) t = cadd(t, scratch[g * 32 + threadIdx.x]);
    mIn[threadIdx.x] = t;
  }
}

// ys[start_r + j*em_r + i] = (1/L) sum_h conj(tw[(h*j) mod L]) sum_ch bpart[(h*2EM + r*EM + i)*nch + ch],
// j < nOut: the chunk reduction and the inverse 1-D transform of the B
// rows in one kernel, CTA per (r, i).
__global__ void __launch_bounds__(256) marginBToYs(const double2* __restrict__ bpart, int EM, int em0, int em1,
                                                  int L, int nch, int nOut, const double2* __restrict__ tw,
                                                  double2* __restrict__ ys0, double2* __restrict__ ys1) {
  extern __shared__ double2 col[];  // [L]
  const int r = blockIdx.x / EM, i = blockIdx.x % EM, em = r ? em1 : em0;
  if (i >= em) return;
  for (int h = threadIdx.x; h < L; h += blockDim.x) {
    const double2* p = bpart + (static_cast<long long>(h) * 2 * EM + r * EM + i) * nch;
    double2 t = make_double2(0.0, 0.0);
    for (int c = 0; c < nch; ++c) t = cadd(t, p[c]);
    col[h] = t;
  }
  __syncthreads();
  const double sc = 1.0 / L;
  double2* out = r ? ys1 : ys0;
  for (int j = threadIdx.x; j < nOut; j += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int h = 0; h < L; ++h) {
      const double2 w = tw[(static_cast<long long>(h) * j) % L];
      cfma(acc, col[h], make_double2(w.x, -w.y));
    }
    out[static_cast<long long>(j) * em + i] = make_double2(acc.x * sc, acc.y * sc);
  }
}

// B1/B2 + their transposes, one column. CTA per (bin h, q-chunk), q = nx*m.
//   bpart[(h*(em0+em1) + r*em0 + i)*nch + ch] = sum_q G_r[h][i][q] xhat_y[h][q]
//   zy[hr][q] = sum_r sum_i G_r[h][i][q] mIn_r[hr][i],  hr = -h mod Ly
template <int EM>
__global__ void __launch_bounds__(kFuseThreads, EM <= 8 ? 2 : 1)
    sideFused(const double2* __restrict__ g0, const double2* __restrict__ g1, int em0, int em1,
              const double2* __restrict__ hatY, const double2* __restrict__ xs0, const double2* __restrict__ xs1,
              int nIn, const double2* __restrict__ tw, double2* __restrict__ zy, double2* __restrict__ bpart, int Ly,
              int q, int nch) {
  __shared__ double2 red[(kFuseThreads / 32) * 32];
  __shared__ double2 mIn[2 * EM];
  __shared__ const double2* rowPtr[2 * EM];
  const int h = blockIdx.x / nch, ch = blockIdx.x % nch;
  const int hr = (Ly - h) % Ly;
  const int qlen = (q + nch - 1) / nch, q0 = ch * qlen, q1 = min(q, q0 + qlen);
  marginDft<EM>(xs0, xs1, em0, em1, nIn, hr, Ly, tw, mIn, red);
  // Rows past em_r read a valid row (hatY) with weight 0 so every load is
  // unconditional and the loads of one t issue back to back.
  if (threadIdx.x < 2 * EM) {
    const int r = threadIdx.x / EM, i = threadIdx.x % EM, em = r ? em1 : em0;
    const double2* g = r ? g1 : g0;
    const bool live = i < em && g != nullptr;
    rowPtr[threadIdx.x] = live ? g + (static_cast<long long>(h) * em + i) * q : hatY + static_cast<long long>(h) * q;
    if (!live) mIn[threadIdx.x] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 pb[2 * EM];
#pragma unroll
  for (int v = 0; v < 2 * EM; ++v) pb[v] = make_double2(0.0, 0.0);
  for (int t = q0 + threadIdx.x; t < q1; t += blockDim.x) {
    const double2 xv = hatY[static_cast<long long>(h) * q + t];
    double2 z = make_double2(0.0, 0.0);
#pragma unroll
    for (int v0 = 0; v0 < 2 * EM; v0 += kLoadGroup) {
      double2 g[kLoadGroup];
#pragma unroll
      for (int v = 0; v < kLoadGroup; ++v) g[v] = __ldg(rowPtr[v0 + v] + t);
#pragma unroll
      for (int v = 0; v < kLoadGroup; ++v) {
        cfma(pb[v0 + v], g[v], xv);
        cfma(z, g[v], mIn[v0 + v]);
      }
    }
    zy[static_cast<long long>(hr) * q + t] = z;
  }
  ctaReduceMany<2 * EM>(pb, 2 * EM, red, bpart + static_cast<long long>(h) * 2 * EM * nch + ch, nch);
}

// B3/B4 + transposes, one column. CTA per (bin h, chunk of t = j*m + k < ny*m).
template <int EM>
__global__ void __launch_bounds__(kFuseThreads, EM <= 8 ? 2 : 1)
    rowFused(const double2* __restrict__ g0, const double2* __restrict__ g1, int em0, int em1,
             const double2* __restrict__ hatX, const double2* __restrict__ xs0, const double2* __restrict__ xs1,
             int nIn, const double2* __restrict__ tw, double2* __restrict__ zx, double2* __restrict__ bpart, int Lx,
             int ny, int m, int nch) {
  __shared__ double2 red[(kFuseThreads / 32) * 32];
  __shared__ double2 mIn[2 * EM];
  __shared__ const double2* rowPtr[2 * EM];  // row base at j = 0; rows step by jStride[r]
  __shared__ long long jStride[2 * EM];
  const int q = ny * m;
  const int h = blockIdx.x / nch, ch = blockIdx.x % nch;
  const int hr = (Lx - h) % Lx;
  const int qlen = (q + nch - 1) / nch, q0 = ch * qlen, q1 = min(q, q0 + qlen);
  marginDft<EM>(xs0, xs1, em0, em1, nIn, hr, Lx, tw, mIn, red);
  if (threadIdx.x < 2 * EM) {  // dead rows: weight 0 on a valid row of hatX
    const int r = threadIdx.x / EM, i = threadIdx.x % EM, em = r ? em1 : em0;
    const double2* g = r ? g1 : g0;
    const bool live = i < em && g != nullptr;
    rowPtr[threadIdx.x] = live ? g + (static_cast<long long>(h) * em + i) * m : hatX + static_cast<long long>(h) * ny * m;
    jStride[threadIdx.x] = live ? static_cast<long long>(Lx) * em * m : m;
    if (!live) mIn[threadIdx.x] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 pb[2 * EM];
#pragma unroll
  for (int v = 0; v < 2 * EM; ++v) pb[v] = make_double2(0.0, 0.0);
  for (int t = q0 + threadIdx.x; t < q1; t += blockDim.x) {
    const int j = t / m, k = t - j * m;
    const double2 xv = hatX[(static_cast<long long>(h) * ny + j) * m + k];
    double2 z = make_double2(0.0, 0.0);
#pragma unroll
    for (int v0 = 0; v0 < 2 * EM; v0 += kLoadGroup) {
      double2 g[kLoadGroup];
#pragma unroll
      for (int v = 0; v < kLoadGroup; ++v) g[v] = __ldg(rowPtr[v0 + v] + j * jStride[v0 + v] + k);
#pragma unroll
      for (int v = 0; v < kLoadGroup; ++v) {
        cfma(pb[v0 + v], g[v], xv);
        cfma(z, g[v], mIn[v0 + v]);
      }
    }
    zx[(static_cast<long long>(hr) * ny + j) * m + k] = z;
  }
  ctaReduceMany<2 * EM>(pb, 2 * EM, red, bpart + static_cast<long long>(h) * 2 * EM * nch + ch, nch);
}

// out_r[h][i] = sum_ch bpart[(h*2EM + r*EM + i)*nch + ch] (fixed order).
__global__ void reduceParts(const double2* __restrict__ bpart, double2* __restrict__ out0, double2* __restrict__ out1,
                            int em0, int em1, int EM, int L, int nch) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < L * 2 * EM; o += gridDim.x * blockDim.x) {
    const int h = o / (2 * EM), v = o % (2 * EM), r = v / EM, i = v % EM;
    if (i >= (r == 0 ? em0 : em1)) continue;
    const double2* p = bpart + static_cast<long long>(o) * nch;
    double2 t = make_double2(0.0, 0.0);
    for (int c = 0; c < nch; ++c) t = cadd(t, p[c]);
    (r == 0 ? out0 : out1)[static_cast<long long>(h) * (r == 0 ? em0 : em1) + i] = t;
  }
}

// Corners, one column: B rows (partials per element block) and the B^T
// corner vector cT[q] = sum_c sum_i bc[i][q] xM_c[i], one read of bc.
// blockIdx.y handles flattened corner rows [16y, 16y + CR) into its own
// cT slice cT + y*nA (summed by marginFinish1).
template <int CR>
__global__ void __launch_bounds__(kFuseThreads, 2) cornerFused(CornerArgs ca, const double2* __restrict__ x,
                                                            const double2* __restrict__ xs,
                                                            double2* __restrict__ part, double2* __restrict__ cT,
                                                            long long nA, int qBlock, int nblk) {
  const int row0 = blockIdx.y * CR;
  cT += blockIdx.y * nA;
  __shared__ double2 red[(kFuseThreads / 32) * CR];
  __shared__ const double2* rowPtr[CR];
  __shared__ double2 mcs[CR];
  const long long q0 = static_cast<long long>(blockIdx.x) * qBlock;
  const long long q1 = min(nA, q0 + qBlock);
  const int rowsTot = ca.em[0] + ca.em[1] + ca.em[2] + ca.em[3];
  const int rows = min(CR, rowsTot - row0);
  if (threadIdx.x < CR) {  // slot u: flattened corner row row0 + u (dead slots re-read the first row, weight 0)
    const int u = threadIdx.x;
    int f = row0 + (u < rows ? u : 0), c = 0;
    while (f >= ca.em[c]) f -= ca.em[c++];
    rowPtr[u] = ca.bc[c] + static_cast<long long>(f) * nA;
    mcs[u] = u < rows ? xs[ca.start[c] + f] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 pb[CR];
#pragma unroll
  for (int u = 0; u < CR; ++u) pb[u] = make_double2(0.0, 0.0);
  for (long long qq = q0 + threadIdx.x; qq < q1; qq += blockDim.x) {
    const double2 xv = x[qq];
    double2 z = make_double2(0.0, 0.0);
#pragma unroll
    for (int u0 = 0; u0 < CR; u0 += 16) {  // all 16 rows' loads in flight at once
      double2 g[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) g[u] = __ldg(rowPtr[u0 + u] + qq);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        cfma(pb[u0 + u], g[u], xv);
        cfma(z, g[u], mcs[u0 + u]);
      }
    }
    cT[qq] = z;
  }
  ctaReduceMany<CR>(pb, rows, red, part + static_cast<long long>(row0) * nblk + blockIdx.x, nblk);
}

// y[q] += zA[q] + zA2[q] + cT[q] (one column).
// One column: yA += zA + zA2 + sum_p cT[p] (B^T parts), and the margin
// pseudo-elements y[nA + k] = ys[k] + ysC[k] (B rows + C xM), zero past nM.
__global__ void marginFinish1(double2* __restrict__ y, const double2* __restrict__ zA,
                              const double2* __restrict__ zA2, const double2* __restrict__ cT, int nT,
                              const double2* __restrict__ ys, const double2* __restrict__ ysC, long long nA,
                              long long nM, long long nPad) {
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < nA + nPad;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (o < nA) {
      double2 acc = y[o];
      if (zA) acc = cadd(acc, zA[o]);
      if (zA2) acc = cadd(acc, zA2[o]);
      for (int p = 0; p < nT; ++p) acc = cadd(acc, cT[p * nA + o]);
      y[o] = acc;
    } else {
      const long long k = o - nA;
      y[o] = k < nM ? cadd(ys[k], ysC[k]) : make_double2(0.0, 0.0);
    }
  }
}

}  // namespace

void marginFree(Ctx& c) {
  delete c.margin;
  c.margin = nullptr;
  c.nM = 0;
  c.neM = 0;
}

void marginSet(Ctx& c, const int* e, const double2* bside, const double2* brow, const double2* bcorner,
               const double2* Cm) {
  TBT_USER_CHECK(e[4] == c.m, "tbt_set_margin: e[4] must equal the element basis size m");
  for (int q = 0; q < 9; ++q) TBT_USER_CHECK(e[q] >= 0, "tbt_set_margin: negative edge count");
  TBT_USER_CHECK(!c.dist, "tbt_set_margin: not supported on a distributed context");
  marginFree(c);
  auto* M = new MarginOp;
  c.margin = M;
  M->stream = c.stream;
  for (int b = 0; b < 2; ++b) {
    TBT_CUDA_CHECK(cudaStreamCreateWithFlags(&M->branch[b], cudaStreamNonBlocking));
    TBT_CUDA_CHECK(cudaEventCreateWithFlags(&M->evJoin[b], cudaEventDisableTiming));
  }
  TBT_CUDA_CHECK(cudaEventCreateWithFlags(&M->evFork, cudaEventDisableTiming));
  const int nx = c.nx, ny = c.ny, m = c.m, K = c.maxNrhs;
  const long long nA = c.n;
  for (int q = 0; q < 9; ++q) M->e[q] = e[q];
  M->nM = static_cast<long long>(ny) * (e[1] + e[7]) + static_cast<long long>(nx) * (e[5] + e[3]) + e[2] + e[8] +
          e[0] + e[6];
  c.nM = M->nM;
  c.neM = static_cast<int>((M->nM + m - 1) / m);
  auto p2 = [](int n) {
    int L = 1;
    while (L < n) L <<= 1;
    return L;
  };
  M->Ly = p2(2 * ny - 1);  // nextPow2(nr + nc - 1), Toe1D::build (linsolve.cpp:70)
  M->Lx = p2(2 * nx - 1);
  M->emSide[0] = e[1];
  M->emSide[1] = e[7];
  M->emRow[0] = e[5];
  M->emRow[1] = e[3];
  const int cc[4] = {3, 9, 1, 7};
  for (int q = 0; q < 4; ++q) M->emCorner[q] = e[cc[q] - 1];
  M->sideStart[0] = 0;
  M->sideStart[1] = static_cast<long long>(ny) * e[1];
  M->rowStart[0] = static_cast<long long>(ny) * (e[1] + e[7]);
  M->rowStart[1] = M->rowStart[0] + static_cast<long long>(nx) * e[5];
  long long cs = M->rowStart[1] + static_cast<long long>(nx) * e[3];
  for (int q = 0; q < 4; ++q) {
    M->cornerStart[q] = cs;
    cs += M->emCorner[q];
  }
  const auto twy = twiddleTable(M->Ly), twx = twiddleTable(M->Lx);
  M->twY = M->alloc(M->Ly);
  M->twX = M->alloc(M->Lx);
  uploadSync(M->twY, twy.data(), twy.size() * sizeof(double2), c.stream);
  uploadSync(M->twX, twx.data(), twx.size() * sizeof(double2), c.stream);
  cudaStream_t s = c.stream;
  // Spectra of B1/B2: seq[s][i][q] then one FFT pass along s.
  const long long qs = static_cast<long long>(nx) * m;
  long long off = 0;
  for (int r = 0; r < 2; ++r) {
    const int em = M->emSide[r];
    const long long P = em * qs, rawCount = (2LL * ny - 1) * P;
    if (em == 0) continue;
    double2* raw = M->alloc(rawCount);
    M->rawSide[r] = raw;
    uploadSync(raw, bside + off, rawCount * sizeof(double2), c.stream);
    double2* seq = M->alloc(static_cast<size_t>(M->Ly) * P);
    toeSeq<<<gridFor(M->Ly * P), 256, 0, s>>>(raw, seq, 1, M->Ly, ny, em, qs);
    M->gSide[r] = M->alloc(static_cast<size_t>(M->Ly) * P);
    FftPass fp;
    fp.in = seq;
    fp.out = M->gSide[r];
    fp.lines = 1;
    fp.in_point_stride = fp.out_point_stride = P;
    fp.n = fp.n_in = fp.n_out = M->Ly;
    fp.batch = static_cast<int>(P);
    fp.tw = M->twY;
    launchFftPass(fp, s);
    off += rawCount;
  }
  // Spectra of B3/B4: per element row j, seq[j][s][i][k].
  off = 0;
  for (int r = 0; r < 2; ++r) {
    const int em = M->emRow[r];
    const long long P = static_cast<long long>(em) * m, rawCount = static_cast<long long>(ny) * (2 * nx - 1) * P;
    if (em == 0) continue;
    double2* raw = M->alloc(rawCount);
    M->rawRow[r] = raw;
    uploadSync(raw, brow + off, rawCount * sizeof(double2), c.stream);
    double2* seq = M->alloc(static_cast<size_t>(ny) * M->Lx * P);
    toeSeq<<<gridFor(static_cast<long long>(ny) * M->Lx * P), 256, 0, s>>>(raw, seq, ny, M->Lx, nx, em, m);
    M->gRow[r] = M->alloc(static_cast<size_t>(ny) * M->Lx * P);
    FftPass fp;
    fp.in = seq;
    fp.out = M->gRow[r];
    fp.lines = ny;
    fp.in_line_stride = fp.out_line_stride = M->Lx * P;
    fp.in_point_stride = fp.out_point_stride = P;
    fp.n = fp.n_in = fp.n_out = M->Lx;
    fp.batch = static_cast<int>(P);
    fp.tw = M->twX;
    launchFftPass(fp, s);
    off += rawCount;
  }
  // Corners (column-major e_c x nA -> row-major) and C.
  off = 0;
  for (int q = 0; q < 4; ++q) {
    const int em = M->emCorner[q];
    if (em == 0) continue;
    double2* raw = M->alloc(static_cast<size_t>(em) * nA);
    uploadSync(raw, bcorner + off, static_cast<size_t>(em) * nA * sizeof(double2), c.stream);
    M->corner[q] = M->alloc(static_cast<size_t>(em) * nA);
    transposeCM<<<gridFor(em * nA), 256, 0, s>>>(raw, M->corner[q], em, nA);
    off += static_cast<long long>(em) * nA;
  }
  if (M->nM > 0) {
    double2* raw = M->alloc(static_cast<size_t>(M->nM) * M->nM);
    uploadSync(raw, Cm, static_cast<size_t>(M->nM) * M->nM * sizeof(double2), c.stream);
    M->C = M->alloc(static_cast<size_t>(M->nM) * M->nM);
    transposeCM<<<gridFor(M->nM * M->nM), 256, 0, s>>>(raw, M->C, M->nM, M->nM);
    M->diag.resize(M->nM);
    for (long long k = 0; k < M->nM; ++k) M->diag[k] = Cm[k * M->nM + k];
  }
  TBT_CUDA_CHECK(cudaGetLastError());
  // Work buffers.
  M->xs = M->alloc(static_cast<size_t>(M->nM) * K);
  M->ys = M->alloc(static_cast<size_t>(M->nM) * K);
  M->hatY = M->alloc(static_cast<size_t>(M->Ly) * nx * K * m);
  M->hatZy = M->alloc(static_cast<size_t>(M->Ly) * nx * K * m);
  M->hatX = M->alloc(static_cast<size_t>(M->Lx) * ny * K * m);
  M->hatZx = M->alloc(static_cast<size_t>(M->Lx) * ny * K * m);
  for (int r = 0; r < 2; ++r) {
    M->hatMs[r] = M->alloc(static_cast<size_t>(M->Ly) * std::max(M->emSide[r], 1) * K);
    M->hatMr[r] = M->alloc(static_cast<size_t>(M->Lx) * std::max(M->emRow[r], 1) * K);
  }
  M->zA = M->alloc(static_cast<size_t>(c.ne) * K * m);
  // Fused single-column path buffers.
  M->chunkS = std::max(1, (nx * m + kFuseChunk - 1) / kFuseChunk);
  M->chunkR = std::max(1, (ny * m + kFuseChunk - 1) / kFuseChunk);
  for (int r = 0; r < 2; ++r) {
    M->hatMsOut[r] = M->alloc(static_cast<size_t>(M->Ly) * std::max(M->emSide[r], 1));
    M->hatMrOut[r] = M->alloc(static_cast<size_t>(M->Lx) * std::max(M->emRow[r], 1));
  }
  M->bpartS = M->alloc(static_cast<size_t>(M->Ly) * 2 * 16 * M->chunkS);  // slots r*EM + i, EM <= 16
  M->bpartR = M->alloc(static_cast<size_t>(M->Lx) * 2 * 16 * M->chunkR);
  M->cornerT = M->alloc(static_cast<size_t>(nA) *
                        std::max(1, (M->emCorner[0] + M->emCorner[1] + M->emCorner[2] + M->emCorner[3] + 15) / 16));
  M->ysC = M->alloc(static_cast<size_t>(M->nM));
  M->cornerPart = M->alloc(static_cast<size_t>(M->emCorner[0] + M->emCorner[1] + M->emCorner[2] + M->emCorner[3]) *
                           std::max<long long>(K * ((c.ne + kCornerElems - 1) / kCornerElems), (nA + 255) / 256));
  M->zA2 = M->alloc(static_cast<size_t>(c.ne) * K * m);
  TBT_CUDA_CHECK(cudaStreamSynchronize(s));
  // The raw uploads and sequences are no longer needed once the spectra exist.
}

// SemiSparse margin coupling: dense B (nM x nA) and C (nM x nM), both
// column-major as the reference stores bFull / cFull (toeplitz.hpp:90-93).
void marginSetDense(Ctx& c, const int* e, const double2* Bm, const double2* Cm) {
  TBT_USER_CHECK(e[4] == c.m, "tbt_set_margin_dense: e[4] must equal the element basis size m");
  for (int q = 0; q < 9; ++q) TBT_USER_CHECK(e[q] >= 0, "tbt_set_margin_dense: negative edge count");
  TBT_USER_CHECK(!c.dist, "tbt_set_margin_dense: not supported on a distributed context");
  marginFree(c);
  auto* M = new MarginOp;
  c.margin = M;
  M->stream = c.stream;
  const int nx = c.nx, ny = c.ny, m = c.m, K = c.maxNrhs;
  const long long nA = c.n;
  for (int q = 0; q < 9; ++q) M->e[q] = e[q];
  M->nM = static_cast<long long>(ny) * (e[1] + e[7]) + static_cast<long long>(nx) * (e[5] + e[3]) + e[2] + e[8] +
          e[0] + e[6];
  c.nM = M->nM;
  c.neM = static_cast<int>((M->nM + m - 1) / m);
  cudaStream_t s = c.stream;
  if (M->nM > 0) {
    double2* raw = M->alloc(static_cast<size_t>(M->nM) * nA);
    uploadSync(raw, Bm, static_cast<size_t>(M->nM) * nA * sizeof(double2), s);
    M->bDense = M->alloc(static_cast<size_t>(M->nM) * nA);
    transposeCM<<<gridFor(M->nM * nA), 256, 0, s>>>(raw, M->bDense, M->nM, nA);
    double2* rawC = M->alloc(static_cast<size_t>(M->nM) * M->nM);
    uploadSync(rawC, Cm, static_cast<size_t>(M->nM) * M->nM * sizeof(double2), s);
    M->C = M->alloc(static_cast<size_t>(M->nM) * M->nM);
    transposeCM<<<gridFor(M->nM * M->nM), 256, 0, s>>>(rawC, M->C, M->nM, M->nM);
    TBT_CUDA_CHECK(cudaGetLastError());
    M->diag.resize(M->nM);
    for (long long k = 0; k < M->nM; ++k) M->diag[k] = Cm[k * M->nM + k];
  }
  M->xs = M->alloc(static_cast<size_t>(M->nM) * K);
  M->ys = M->alloc(static_cast<size_t>(M->nM) * K);
  TBT_CUDA_CHECK(cudaStreamSynchronize(s));
}

void marginDiagonal(const Ctx& c, std::vector<double2>& d) {
  if (!c.margin) return;
  d.insert(d.end(), c.margin->diag.begin(), c.margin->diag.end());
}

namespace {

template <int EM>
void launchSideFused(MarginOp* M, const double2* xs, int nx, int ny, int m, cudaStream_t s) {
  const int q = nx * m;
  sideFused<EM><<<M->Ly * M->chunkS, kFuseThreads, 0, s>>>(
      M->gSide[0], M->gSide[1], M->emSide[0], M->emSide[1], M->hatY, xs + M->sideStart[0], xs + M->sideStart[1], ny,
      M->twY, M->hatZy, M->bpartS, M->Ly, q, M->chunkS);
}
template <int EM>
void launchRowFused(MarginOp* M, const double2* xs, int nx, int ny, int m, cudaStream_t s) {
  rowFused<EM><<<M->Lx * M->chunkR, kFuseThreads, 0, s>>>(
      M->gRow[0], M->gRow[1], M->emRow[0], M->emRow[1], M->hatX, xs + M->rowStart[0], xs + M->rowStart[1], nx,
      M->twX, M->hatZx, M->bpartR, M->Lx, ny, m, M->chunkR);
}

int fuseBound(int a, int b) {
  const int e = std::max(a, b);
  return e <= 8 ? 8 : e <= 16 ? 16 : 0;
}

// One column: B and B^T from a single read of every generator spectrum and
// corner block (hatMs / hatMr hold the transformed margin inputs, the B
// results go to hatMsOut / hatMrOut).
bool marginApplyFused1(Ctx& c, const double2* x, double2* y) {
  MarginOp* M = c.margin;
  const int nx = c.nx, ny = c.ny, m = c.m, ne = c.ne;
  const long long nA = c.n;
  const int emS = fuseBound(M->emSide[0], M->emSide[1]), emR = fuseBound(M->emRow[0], M->emRow[1]);
  const int cornerRows = M->emCorner[0] + M->emCorner[1] + M->emCorner[2] + M->emCorner[3];
  if ((M->anySide() && !emS) || (M->anyRow() && !emR) || !M->hatMsOut[0]) return false;
  // One column: the margin unknowns are contiguous right after the elements.
  const double2* xs = x + nA;
  CornerArgs ca{};
  for (int q = 0; q < 4; ++q) {
    ca.bc[q] = M->corner[q];
    ca.em[q] = M->emCorner[q];
    ca.start[q] = M->cornerStart[q];
  }
  const bool side = M->anySide(), row = M->anyRow();
  // Fork: side products on branch[0], row products on branch[1], C and the
  // corners on the ctx stream; all read x only and write disjoint outputs.
  TBT_CUDA_CHECK(cudaEventRecord(M->evFork, c.stream));
  for (int b = 0; b < 2; ++b) TBT_CUDA_CHECK(cudaStreamWaitEvent(M->branch[b], M->evFork, 0));
  if (side) {
    cudaStream_t s = M->branch[0];
    FftPass fy;
    fy.in = x;
    fy.out = M->hatY;
    fy.lines = 1;
    fy.in_point_stride = fy.out_point_stride = static_cast<long long>(nx) * m;
    fy.n = fy.n_out = M->Ly;
    fy.n_in = ny;
    fy.batch = nx * m;
    fy.tw = M->twY;
    launchFftPass(fy, s);
    if (emS == 8)
      launchSideFused<8>(M, xs, nx, ny, m, s);
    else
      launchSideFused<16>(M, xs, nx, ny, m, s);
    marginBToYs<<<2 * emS, 256, M->Ly * sizeof(double2), s>>>(M->bpartS, emS, M->emSide[0], M->emSide[1], M->Ly,
                                                               M->chunkS, ny, M->twY, M->ys + M->sideStart[0],
                                                               M->ys + M->sideStart[1]);
    FftPass iz;  // B^T side part back to the elements
    iz.in = M->hatZy;
    iz.out = M->zA;
    iz.lines = 1;
    iz.in_point_stride = iz.out_point_stride = static_cast<long long>(nx) * m;
    iz.n = iz.n_in = M->Ly;
    iz.n_out = ny;
    iz.batch = nx * m;
    iz.inverse = 1;
    iz.scale = 1.0 / M->Ly;
    iz.tw = M->twY;
    launchFftPass(iz, s);
  }
  if (row) {
    cudaStream_t s = M->branch[1];
    FftPass fx;
    fx.in = x;
    fx.out = M->hatX;
    fx.lines = ny;
    fx.in_line_stride = static_cast<long long>(nx) * m;
    fx.in_point_stride = m;
    fx.out_line_stride = m;
    fx.out_point_stride = static_cast<long long>(ny) * m;
    fx.n = fx.n_out = M->Lx;
    fx.n_in = nx;
    fx.batch = m;
    fx.tw = M->twX;
    launchFftPass(fx, s);
    if (emR == 8)
      launchRowFused<8>(M, xs, nx, ny, m, s);
    else
      launchRowFused<16>(M, xs, nx, ny, m, s);
    marginBToYs<<<2 * emR, 256, M->Lx * sizeof(double2), s>>>(M->bpartR, emR, M->emRow[0], M->emRow[1], M->Lx,
                                                               M->chunkR, nx, M->twX, M->ys + M->rowStart[0],
                                                               M->ys + M->rowStart[1]);
    FftPass iz;
    iz.in = M->hatZx;
    iz.out = M->zA2;
    iz.lines = ny;
    iz.in_line_stride = m;
    iz.in_point_stride = static_cast<long long>(ny) * m;
    iz.out_line_stride = static_cast<long long>(nx) * m;
    iz.out_point_stride = m;
    iz.n = iz.n_in = M->Lx;
    iz.n_out = nx;
    iz.batch = m;
    iz.inverse = 1;
    iz.scale = 1.0 / M->Lx;
    iz.tw = M->twX;
    launchFftPass(iz, s);
  }
  cudaStream_t s = c.stream;
  cProd<<<static_cast<unsigned>(M->nM), 128, 0, s>>>(M->C, xs, M->ysC, M->nM, 1, 1);
  const int passes = (cornerRows + 15) / 16;
  if (cornerRows > 0) {
    const int qBlock = (nA + kCornerQ - 1) / kCornerQ >= 4LL * smCount(c.device) ? kCornerQ : 256;
    const int nblk = static_cast<int>((nA + qBlock - 1) / qBlock);
    // 16 rows per pass (blockIdx.y) keeps the kernel at 2 CTAs/SM.
    cornerFused<16><<<dim3(nblk, passes), kFuseThreads, 0, s>>>(ca, x, xs, M->cornerPart, M->cornerT, nA, qBlock,
                                                                nblk);
    cornerReduce<<<(cornerRows * 32 + 255) / 256, 256, 0, s>>>(ca, M->cornerPart, M->ys, 1, nblk);
  }
  for (int b = 0; b < 2; ++b) {  // join
    TBT_CUDA_CHECK(cudaEventRecord(M->evJoin[b], M->branch[b]));
    TBT_CUDA_CHECK(cudaStreamWaitEvent(c.stream, M->evJoin[b], 0));
  }
  const long long nPad = static_cast<long long>(c.neM) * m;
  marginFinish1<<<gridFor(nA + nPad), 256, 0, s>>>(y, side ? M->zA : nullptr, row ? M->zA2 : nullptr, M->cornerT,
                                                   cornerRows > 0 ? passes : 0, M->ys, M->ysC, nA, M->nM, nPad);
  TBT_CUDA_CHECK(cudaGetLastError());
  return true;
}

}  // namespace

void marginApply(Ctx& c, const double2* x, double2* y, int K) {
  MarginOp* M = c.margin;
  if (!M || M->nM == 0) return;
  static const bool noFuse = getenv("TBT_MARGIN_UNFUSED") != nullptr;
  cudaStream_t s = c.stream;
  const int nx = c.nx, ny = c.ny, m = c.m, ne = c.ne;
  const long long nA = c.n, B = static_cast<long long>(K) * m;
  if (M->bDense) {
    // SemiSparse: yM = B xA + C xM, yA += B^T xM (linsolve.cpp:294,318,338).
    marginGather<<<gridFor(M->nM * K), 256, 0, s>>>(x, M->xs, M->nM, ne, m, K);
    cProd<<<static_cast<unsigned>(M->nM * K), 128, 0, s>>>(M->C, M->xs, M->ys, M->nM, K, 1);
    denseBProd<<<static_cast<unsigned>(M->nM * K), 128, 0, s>>>(M->bDense, x, M->ys, nA, m, K);
    denseBTProd<<<gridFor(nA * K), 256, 0, s>>>(M->bDense, M->xs, y, nA, M->nM, m, K);
    marginScatter<<<gridFor(static_cast<long long>(c.neM) * K * m), 256, 0, s>>>(M->ys, y, M->nM, ne, c.neM, m, K);
    TBT_CUDA_CHECK(cudaGetLastError());
    return;
  }
  if (K == 1 && !noFuse && marginApplyFused1(c, x, y)) return;
  marginGather<<<gridFor(M->nM * K), 256, 0, s>>>(x, M->xs, M->nM, ne, m, K);
  CornerArgs ca{};
  for (int q = 0; q < 4; ++q) {
    ca.bc[q] = M->corner[q];
    ca.em[q] = M->emCorner[q];
    ca.start[q] = M->cornerStart[q];
  }
  const bool side = M->anySide(), row = M->anyRow();
  if (side) {
    // x along the element rows (level 1): hatY[f][c][rhs][k].
    FftPass fy;
    fy.in = x;
    fy.out = M->hatY;
    fy.lines = 1;
    fy.in_point_stride = fy.out_point_stride = nx * B;
    fy.n = fy.n_out = M->Ly;
    fy.n_in = ny;
    fy.batch = static_cast<int>(nx * B);
    fy.tw = M->twY;
    launchFftPass(fy, s);
    // Margin side segments along their ny parts.
    for (int r = 0; r < 2; ++r) {
      if (M->emSide[r] == 0) continue;
      FftPass fm;
      fm.in = M->xs + M->sideStart[r] * K;
      fm.out = M->hatMs[r];
      fm.lines = 1;
      fm.in_point_stride = fm.out_point_stride = static_cast<long long>(M->emSide[r]) * K;
      fm.n = fm.n_out = M->Ly;
      fm.n_in = ny;
      fm.batch = M->emSide[r] * K;
      fm.tw = M->twY;
      launchFftPass(fm, s);
    }
  }
  if (row) {
    // x along the element columns (level 0) per row: hatX[f][j][rhs][k].
    FftPass fx;
    fx.in = x;
    fx.out = M->hatX;
    fx.lines = ny;
    fx.in_line_stride = nx * B;
    fx.in_point_stride = B;
    fx.out_line_stride = B;
    fx.out_point_stride = ny * B;
    fx.n = fx.n_out = M->Lx;
    fx.n_in = nx;
    fx.batch = static_cast<int>(B);
    fx.tw = M->twX;
    launchFftPass(fx, s);
    for (int r = 0; r < 2; ++r) {
      if (M->emRow[r] == 0) continue;
      FftPass fm;
      fm.in = M->xs + M->rowStart[r] * K;
      fm.out = M->hatMr[r];
      fm.lines = 1;
      fm.in_point_stride = fm.out_point_stride = static_cast<long long>(M->emRow[r]) * K;
      fm.n = fm.n_out = M->Lx;
      fm.n_in = nx;
      fm.batch = M->emRow[r] * K;
      fm.tw = M->twX;
      launchFftPass(fm, s);
    }
  }
  // B^T parts first (they read hatMs / hatMr before the B products reuse them).
  if (side) {
    sideProdT<<<gridFor(static_cast<long long>(M->Ly) * nx * B), 256, 0, s>>>(
        M->gSide[0], M->gSide[1], M->emSide[0], M->emSide[1], M->hatMs[0], M->hatMs[1], M->hatZy, M->Ly, nx, m, K);
    FftPass iz;
    iz.in = M->hatZy;
    iz.out = M->zA;
    iz.lines = 1;
    iz.in_point_stride = iz.out_point_stride = nx * B;
    iz.n = iz.n_in = M->Ly;
    iz.n_out = ny;
    iz.batch = static_cast<int>(nx * B);
    iz.inverse = 1;
    iz.scale = 1.0 / M->Ly;
    iz.tw = M->twY;
    launchFftPass(iz, s);
  }
  if (row) {
    rowProdT<<<gridFor(static_cast<long long>(M->Lx) * ny * B), 256, 0, s>>>(
        M->gRow[0], M->gRow[1], M->emRow[0], M->emRow[1], M->hatMr[0], M->hatMr[1], M->hatZx, M->Lx, ny, m, K);
    FftPass iz;
    iz.in = M->hatZx;
    iz.out = M->zA2;
    iz.lines = ny;
    iz.in_line_stride = B;
    iz.in_point_stride = ny * B;
    iz.out_line_stride = nx * B;
    iz.out_point_stride = B;
    iz.n = iz.n_in = M->Lx;
    iz.n_out = nx;
    iz.batch = static_cast<int>(B);
    iz.inverse = 1;
    iz.scale = 1.0 / M->Lx;
    iz.tw = M->twX;
    launchFftPass(iz, s);
  }
  addBT<<<gridFor(nA * K), 256, 0, s>>>(y, side ? M->zA : nullptr, row ? M->zA2 : nullptr, ca, M->xs, nA, m, K);
  // B xA into the margin staging vector.
  if (side) {
    sideProd<<<static_cast<unsigned>(static_cast<long long>(M->emSide[0] + M->emSide[1]) * M->Ly * K), 128, 0, s>>>(
        M->gSide[0], M->gSide[1], M->emSide[0], M->emSide[1], M->hatY, M->hatMs[0], M->hatMs[1], M->Ly, nx, m, K);
    for (int r = 0; r < 2; ++r) {
      if (M->emSide[r] == 0) continue;
      FftPass im;
      im.in = M->hatMs[r];
      im.out = M->ys + M->sideStart[r] * K;
      im.lines = 1;
      im.in_point_stride = im.out_point_stride = static_cast<long long>(M->emSide[r]) * K;
      im.n = im.n_in = M->Ly;
      im.n_out = ny;
      im.batch = M->emSide[r] * K;
      im.inverse = 1;
      im.scale = 1.0 / M->Ly;
      im.tw = M->twY;
      launchFftPass(im, s);
    }
  }
  if (row) {
    rowProd<<<static_cast<unsigned>(static_cast<long long>(M->emRow[0] + M->emRow[1]) * M->Lx * K), 128, 0, s>>>(
        M->gRow[0], M->gRow[1], M->emRow[0], M->emRow[1], M->hatX, M->hatMr[0], M->hatMr[1], M->Lx, ny, m, K);
    for (int r = 0; r < 2; ++r) {
      if (M->emRow[r] == 0) continue;
      FftPass im;
      im.in = M->hatMr[r];
      im.out = M->ys + M->rowStart[r] * K;
      im.lines = 1;
      im.in_point_stride = im.out_point_stride = static_cast<long long>(M->emRow[r]) * K;
      im.n = im.n_in = M->Lx;
      im.n_out = nx;
      im.batch = M->emRow[r] * K;
      im.inverse = 1;
      im.scale = 1.0 / M->Lx;
      im.tw = M->twX;
      launchFftPass(im, s);
    }
  }
  const int cornerRows = ca.em[0] + ca.em[1] + ca.em[2] + ca.em[3];
  if (cornerRows > 0) {
    const int nblk = (ne + kCornerElems - 1) / kCornerElems;
    cornerPart<<<dim3(nblk, cornerRows), 256, 0, s>>>(ca, x, M->cornerPart, ne, m, K, nblk);
    cornerReduce<<<(cornerRows * K * 32 + 255) / 256, 256, 0, s>>>(ca, M->cornerPart, M->ys, K, nblk);
  }
  cProd<<<static_cast<unsigned>(M->nM * K), 128, 0, s>>>(M->C, M->xs, M->ys, M->nM, K);
  marginScatter<<<gridFor(static_cast<long long>(c.neM) * m * K), 256, 0, s>>>(M->ys, y, M->nM, ne, c.neM, m, K);
  TBT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tbt
