// The operator application: K2 (forward 2-D transform, two batched line
// passes) -> K3 (bin-pair product) -> K4 (inverse 2-D transform, crop,
// 1/L) -> spatial terms. Replaces ToeplitzMatvec::applyA / apply
// (proj/src/linsolve.cpp:260-290,373-388).
//
// Zero-padding is pruned: the forward x-pass reads only the nx non-zero
// points of the ny non-zero rows; the forward y-pass reads ny of L1 points;
// the inverse y-pass keeps ny rows and the inverse x-pass keeps nx points
// (the crop of linsolve.cpp:284-287).
#include <algorithm>

#include "tbt_internal.cuh"

namespace tbt {
namespace {

// Column-major n x nrhs  <->  internal [e][rhs][a].
__global__ void layoutKernel(const double2* __restrict__ in, double2* __restrict__ out, long long n, int m,
                             int nrhs, int toInternal) {
  const long long total = n * nrhs;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    // q indexes the internal layout.
    const long long a = q % m;
    const long long rest = q / m;
    const long long rhs = rest % nrhs, e = rest / nrhs;
    const long long ext = rhs * n + e * m + a;
    if (toInternal)
      out[q] = in[ext];
    else
      out[ext] = in[q];
  }
}

}  // namespace

void launchLayout(const double2* in, double2* out, long long n, int nrhs, bool toInternal, cudaStream_t s,
                  int m) {
  const long long total = n * nrhs;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
  layoutKernel<<<blocks, 256, 0, s>>>(in, out, n, m, nrhs, toInternal ? 1 : 0);
  TBT_CUDA_CHECK(cudaGetLastError());
}

void applyInternal(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr) {
  const long long B = static_cast<long long>(nrhs) * c.m;
  cudaStream_t s = c.stream;

  FftPass fa;  // forward, level 0 (x): one line per element row r < ny
  fa.in = x;
  fa.out = c.dT;
  fa.lines = c.ny;
  fa.in_line_stride = static_cast<long long>(c.nx) * B;
  fa.in_point_stride = B;
  fa.out_line_stride = static_cast<long long>(c.L0) * B;
  fa.out_point_stride = B;
  fa.n = c.L0;
  fa.n_in = c.nx;
  fa.n_out = c.L0;
  fa.batch = static_cast<int>(B);
  fa.tw = c.dTw0;
  launchFftPass(fa, s);

  FftPass fb;  // forward, level 1 (y): one line per column s0
  fb.in = c.dT;
  fb.out = c.dXhat;
  fb.lines = c.L0;
  fb.in_line_stride = B;
  fb.in_point_stride = static_cast<long long>(c.L0) * B;
  fb.out_line_stride = B;
  fb.out_point_stride = static_cast<long long>(c.L0) * B;
  fb.n = c.L1;
  fb.n_in = c.ny;
  fb.n_out = c.L1;
  fb.batch = static_cast<int>(B);
  fb.tw = c.dTw1;
  launchFftPass(fb, s);

  if (c.timeBinprod) {
    if (c.tCount == static_cast<int>(c.tEvA.size())) {
      cudaEvent_t a, b;
      TBT_CUDA_CHECK(cudaEventCreate(&a));
      TBT_CUDA_CHECK(cudaEventCreate(&b));
      c.tEvA.push_back(a);
      c.tEvB.push_back(b);
    }
    TBT_CUDA_CHECK(cudaEventRecord(c.tEvA[c.tCount], s));
    launchBinProduct(c, nrhs);
    TBT_CUDA_CHECK(cudaEventRecord(c.tEvB[c.tCount], s));
    ++c.tCount;
  } else {
    launchBinProduct(c, nrhs);
  }

  FftPass ib;  // inverse, level 1: keep the ny element rows
  ib.in = c.dYhat;
  ib.out = c.dT;
  ib.lines = c.L0;
  ib.in_line_stride = B;
  ib.in_point_stride = static_cast<long long>(c.L0) * B;
  ib.out_line_stride = B;
  ib.out_point_stride = static_cast<long long>(c.L0) * B;
  ib.n = c.L1;
  ib.n_in = c.L1;
  ib.n_out = c.ny;
  ib.batch = static_cast<int>(B);
  ib.inverse = 1;
  ib.tw = c.dTw1;
  launchFftPass(ib, s);

  FftPass ia;  // inverse, level 0: keep the nx element columns, scale 1/L
  ia.in = c.dT;
  ia.out = y;
  ia.lines = c.ny;
  ia.in_line_stride = static_cast<long long>(c.L0) * B;
  ia.in_point_stride = B;
  ia.out_line_stride = static_cast<long long>(c.nx) * B;
  ia.out_point_stride = B;
  ia.n = c.L0;
  ia.n_in = c.L0;
  ia.n_out = c.nx;
  ia.batch = static_cast<int>(B);
  ia.inverse = 1;
  ia.scale = 1.0 / static_cast<double>(c.L);
  ia.tw = c.dTw0;
  launchFftPass(ia, s);

  launchAntisym(c, x, y, nrhs);
  if (withCorr) launchCorrection(c, x, y, nrhs);
}

}  // namespace tbt
