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
__global__ void layoutKernel(const double2* __restrict__ in, double2* __restrict__ out, long long nUser,
                             long long nInt, int m, int nrhs, int toInternal) {
  const long long total = nInt * nrhs;
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    // q indexes the internal layout [e][rhs][a]; rows past nUser are the
    // zero padding of the margin pseudo-elements.
    const long long a = q % m;
    const long long rest = q / m;
    const long long rhs = rest % nrhs, e = rest / nrhs;
    const long long row = e * m + a;
    if (row >= nUser) {
      if (toInternal) out[q] = make_double2(0.0, 0.0);
      continue;
    }
    const long long ext = rhs * nUser + row;
    if (toInternal)
      out[q] = in[ext];
    else
      out[ext] = in[q];
  }
}

}  // namespace

void launchLayoutU(const double2* in, double2* out, long long nUser, long long nInt, int nrhs, bool toInternal,
                   cudaStream_t s, int m) {
  const long long total = nInt * nrhs;
  const int blocks = static_cast<int>(std::min<long long>((total + 255) / 256, 148LL * 16));
  layoutKernel<<<blocks, 256, 0, s>>>(in, out, nUser, nInt, m, nrhs, toInternal ? 1 : 0);
  TBT_CUDA_CHECK(cudaGetLastError());
}

void launchLayout(const double2* in, double2* out, long long n, int nrhs, bool toInternal, cudaStream_t s,
                  int m) {
  launchLayoutU(in, out, n, n, nrhs, toInternal, s, m);
}

namespace {

void binProductTimed(Ctx& c, int nrhs) {
  cudaStream_t s = c.stream;
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
    launchBinProductAnti(c, nrhs);
    TBT_CUDA_CHECK(cudaEventRecord(c.tEvB[c.tCount], s));
    ++c.tCount;
  } else {
    launchBinProduct(c, nrhs);
    launchBinProductAnti(c, nrhs);
  }
}

// K2 -> K3 -> K4 with the cluster-fused transforms; the correction's rank-r
// projections run in a parallel branch (side stream) joined before K4.
bool applyFused(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr) {
  const int B = nrhs * c.m;
  int CL = 1, BC = 16;
  fft2dPlan(c.L0, c.L1, c.nx, c.ny, B, smCount(c.device), &CL, &BC);
  const bool corr = withCorr && c.haveCorr && c.nTerms > 0;
  const bool proj = corr;
  if (proj) {
    TBT_CUDA_CHECK(cudaEventRecord(c.evFork, c.stream));
    TBT_CUDA_CHECK(cudaStreamWaitEvent(c.side, c.evFork, 0));
    launchCorrVector(c, x, c.dYcorr, nrhs, c.side);
    TBT_CUDA_CHECK(cudaEventRecord(c.evJoin, c.side));
  }
  Fft2dArgs f;
  f.in = x;
  f.out = c.dXhat;
  f.nx = c.nx;
  f.ny = c.ny;
  f.L0 = c.L0;
  f.L1 = c.L1;
  f.B = B;
  f.tw0 = c.dTw0;
  f.tw1 = c.dTw1;
  if (!launchFft2d(f, CL, BC, false, c.stream)) {
    if (proj) TBT_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.evJoin, 0));
    return false;
  }
  binProductTimed(c, nrhs);
  if (proj) TBT_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.evJoin, 0));
  Fft2dArgs iv = f;
  iv.in = c.dYhat;
  iv.out = y;
  iv.scale = 1.0 / static_cast<double>(c.L);
  if (corr) {
    iv.corr = 1;
    iv.tPtr = c.dElemPtr;
    iv.ycorr = c.dYcorr;
  }
  if (!launchFft2d(iv, CL, BC, true, c.stream)) throw Error{TBT_CUDA_ERROR, "inverse 2-D transform launch"};
  TBT_CUDA_CHECK(cudaGetLastError());
  launchAntisym(c, x, y, nrhs);
  return true;
}

}  // namespace

namespace {

bool regPassesServe(const Ctx& c, int nrhs) {
  return static_cast<long long>(nrhs) * c.m >= 1024 && c.L0 <= 64 && c.L1 <= 64 && !c.forceFused2d;
}

// The four 1-D passes around K3 (user = x / y in the caller's column-major
// layout, register passes only).
void applyPasses(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr, bool regPasses, bool user) {
  const long long B = static_cast<long long>(nrhs) * c.m;
  cudaStream_t s = c.stream;
  // The correction's term vectors depend on x only: a parallel branch joined
  // before the last pass, which adds them in its store epilogue.
  const bool corrBranch = regPasses && withCorr && c.haveCorr && c.nTerms > 0;
  if (corrBranch) {
    TBT_CUDA_CHECK(cudaEventRecord(c.evFork, s));
    TBT_CUDA_CHECK(cudaStreamWaitEvent(c.side, c.evFork, 0));
    launchCorrVector(c, x, c.dYcorr, nrhs, c.side, user ? c.n : 0);
    TBT_CUDA_CHECK(cudaEventRecord(c.evJoin, c.side));
  }
  auto pass = [&](const FftPass& p) {
    if (!(regPasses && launchFftPassReg(p, s))) {
      if (p.inUser || p.outUser) throw Error{TBT_CUDA_ERROR, "user-layout transform pass without the register kernel"};
      launchFftPass(p, s);
    }
  };
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
  if (user) {
    fa.inUser = 1;
    fa.userNx = c.nx;
    fa.userM = c.m;
    fa.userN = c.n;
  }
  pass(fa);

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
  pass(fb);

  binProductTimed(c, nrhs);

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
  pass(ib);

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
  if (corrBranch) {
    TBT_CUDA_CHECK(cudaStreamWaitEvent(s, c.evJoin, 0));
    ia.tPtr = c.dElemPtr;
    ia.ycorr = c.dYcorr;
    ia.corrNx = c.nx;
  }
  if (user) {
    ia.outUser = 1;
    ia.userNx = c.nx;
    ia.userM = c.m;
    ia.userN = c.n;
  }
  pass(ia);

  if (!user) {
    launchAntisym(c, x, y, nrhs);
    if (withCorr && !corrBranch) launchCorrection(c, x, y, nrhs);
  }
}


}  // namespace

void applyInternal(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr) {
  if (c.dist) {
    applyDist(c, x, y, nrhs, withCorr);
    return;
  }
  if (nrhs == 1 && clusterSmallSupported(c, 1)) {  // tiny operators: one cluster, one launch
    launchClusterApply(c, x, y, withCorr);
    return;
  }
  if (nrhs == 1 && c.persistent && !c.timeBinprod && launchPersistentApply(c, x, y, withCorr)) return;
  // Wide batches (many right-hand sides) with short lines: register line
  // passes (one thread per line and batch entry, fft.cu) beat the cluster
  // 2-D kernels (C3: see DESIGN.md section 4.2); TBT_FFT=fused keeps those.
  const bool regPasses = regPassesServe(c, nrhs);
  if (!regPasses && c.fused2d && !c.forceMultiPass && applyFused(c, x, y, nrhs, withCorr)) return;
  applyPasses(c, x, y, nrhs, withCorr, regPasses, false);
}

bool applyUserLayout(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr) {
  if (nrhs < 2 || c.dist || c.margin || c.hasAntisym || !regPassesServe(c, nrhs)) return false;
  applyPasses(c, x, y, nrhs, withCorr, true, true);
  return true;
}

}  // namespace tbt

namespace tbt {

void applyOperator(Ctx& c, const double2* x, double2* y, int nrhs, bool withCorr) {
  applyInternal(c, x, y, nrhs, withCorr);
  if (withCorr && c.margin) marginApply(c, x, y, nrhs);
}

}  // namespace tbt
