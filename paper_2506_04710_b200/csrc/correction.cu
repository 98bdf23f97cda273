// Non-Toeplitz terms of the operator, applied in the spatial domain after
// the inverse transform:
//  * the synthetic nine-component edge/corner correction (BASELINE.json;
//    include/tbt_gen.h), the stand-in for ToeplitzMatvec::apply's margin
//    coupling (proj/src/linsolve.cpp:384-386): per term
//        y_t += diag(d) x_s + U (V^T x_s)      (P)
//        y_t += diag(d) x_s + V (U^T x_s)      (P^T)
//    as a rank-r projection pass plus a per-target accumulation pass;
//  * the antisymmetric part K of Z(0,0) (see spectra.cu): y_e += K x_e.
// Internal vector layout is [element][rhs][basis].
#include <algorithm>

#include "tbt_internal.cuh"

namespace tbt {
namespace {

// One warp per (term, rhs): proj[t][rhs][q] = sum_a W[s][q][a] x[src][rhs][a].
__global__ void corrProject(const int* __restrict__ termInfo, int nTerms, const double2* __restrict__ U,
                            const double2* __restrict__ V, const double2* __restrict__ x, double2* __restrict__ proj,
                            int m, int rank, int nrhs) {
  const int warpsPerBlock = blockDim.x / 32;
  const long long wid = static_cast<long long>(blockIdx.x) * warpsPerBlock + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (wid >= static_cast<long long>(nTerms) * nrhs) return;
  const int t = static_cast<int>(wid / nrhs), rhs = static_cast<int>(wid % nrhs);
  const int src = termInfo[4 * t + 1], slot = termInfo[4 * t + 2], trans = termInfo[4 * t + 3];
  const double2* W = (trans ? U : V) + static_cast<long long>(slot) * rank * m;
  const double2* xs = x + (static_cast<long long>(src) * nrhs + rhs) * m;
  for (int q = 0; q < rank; ++q) {
    double2 s = make_double2(0.0, 0.0);
    for (int a = lane; a < m; a += 32) cfma(s, W[static_cast<long long>(q) * m + a], xs[a]);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
    }
    if (lane == 0) proj[(static_cast<long long>(t) * nrhs + rhs) * rank + q] = s;
  }
}

// One CTA per (target, rhs), threads over the basis index.
__global__ void corrApply(const int* __restrict__ termInfo, const int* __restrict__ targetList,
                          const int* __restrict__ targetPtr, const double2* __restrict__ D,
                          const double2* __restrict__ U, const double2* __restrict__ V,
                          const double2* __restrict__ x, const double2* __restrict__ proj, double2* __restrict__ y,
                          int m, int rank, int nrhs) {
  const int ti = blockIdx.x, rhs = blockIdx.y;
  const int e = targetList[ti];
  const int t0 = targetPtr[ti], t1 = targetPtr[ti + 1];
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int t = t0; t < t1; ++t) {
      const int src = termInfo[4 * t + 1], slot = termInfo[4 * t + 2], trans = termInfo[4 * t + 3];
      cfma(acc, D[static_cast<long long>(slot) * m + a], x[(static_cast<long long>(src) * nrhs + rhs) * m + a]);
      const double2* W2 = (trans ? V : U) + static_cast<long long>(slot) * rank * m;
      const double2* pr = proj + (static_cast<long long>(t) * nrhs + rhs) * rank;
      for (int q = 0; q < rank; ++q) cfma(acc, W2[static_cast<long long>(q) * m + a], pr[q]);
    }
    double2* out = y + (static_cast<long long>(e) * nrhs + rhs) * m + a;
    *out = cadd(*out, acc);
  }
}

// One CTA per (target element, rhs): the rank-r projections of all the
// target's terms (one warp per term) into shared memory, then
// ycorr[e][rhs][a] = sum_t diag(d_t) x_src + W2_t proj_t. Depends on x only,
// so it runs in a parallel branch beside the transforms and the bin product.
__global__ void __launch_bounds__(256) corrFused(const int* __restrict__ termInfo, const int* __restrict__ targetList,
                                                 const int* __restrict__ targetPtr, const double2* __restrict__ D,
                                                 const double2* __restrict__ U, const double2* __restrict__ V,
                                                 const double2* __restrict__ x, double2* __restrict__ ycorr, int m,
                                                 int rank, int nrhs, long long xE, long long xR) {
  extern __shared__ double2 sproj[];  // [terms of this target][rank]
  const int ti = blockIdx.x, rhs = blockIdx.y;
  const int e = targetList[ti];
  const int t0 = targetPtr[ti], t1 = targetPtr[ti + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = t0 + warp; t < t1; t += blockDim.x / 32) {
    const int src = termInfo[4 * t + 1], slot = termInfo[4 * t + 2], trans = termInfo[4 * t + 3];
    const double2* W = (trans ? U : V) + static_cast<long long>(slot) * rank * m;
    const double2* xs = x + src * xE + rhs * xR;
    for (int q = 0; q < rank; ++q) {
      double2 s = make_double2(0.0, 0.0);
      for (int a = lane; a < m; a += 32) cfma(s, __ldg(W + static_cast<long long>(q) * m + a), __ldg(xs + a));
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, off);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, off);
      }
      if (lane == 0) sproj[(t - t0) * rank + q] = s;
    }
  }
  __syncthreads();
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int t = t0; t < t1; ++t) {
      const int src = termInfo[4 * t + 1], slot = termInfo[4 * t + 2], trans = termInfo[4 * t + 3];
      cfma(acc, __ldg(D + static_cast<long long>(slot) * m + a), __ldg(x + src * xE + rhs * xR + a));
      const double2* W2 = (trans ? V : U) + static_cast<long long>(slot) * rank * m + a;
      for (int q = 0; q < rank; ++q) cfma(acc, __ldg(W2 + static_cast<long long>(q) * m), sproj[(t - t0) * rank + q]);
    }
    ycorr[(static_cast<long long>(e) * nrhs + rhs) * m + a] = acc;
  }
}

// Many right-hand sides: one CTA per (target, chunk of 32 columns). Each
// term's d, U, V (rank RANK, m = 32*KPL) are staged once in shared memory and
// reused by all 32 columns of the chunk (instead of once per column); every
// warp owns 4 columns whose sums stay in registers across the term list.
template <int KPL, int RANK>
__global__ void __launch_bounds__(256) corrMulti(const int* __restrict__ termInfo, const int* __restrict__ targetList,
                                                 const int* __restrict__ targetPtr, const double2* __restrict__ D,
                                                 const double2* __restrict__ U, const double2* __restrict__ V,
                                                 const double2* __restrict__ x, double2* __restrict__ ycorr,
                                                 int nrhs, long long xE, long long xR) {
  constexpr int M = 32 * KPL;
  constexpr int RPW = 4;  // columns per warp
  constexpr int RC = 8 * RPW;
  __shared__ double2 sW[RANK][M], sW2[RANK][M], sD[M];
  const int ti = blockIdx.x;
  const int r0 = blockIdx.y * RC;
  const int e = targetList[ti];
  const int t0 = targetPtr[ti], t1 = targetPtr[ti + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 acc[RPW][KPL];
#pragma unroll
  for (int j = 0; j < RPW; ++j)
#pragma unroll
    for (int k = 0; k < KPL; ++k) acc[j][k] = make_double2(0.0, 0.0);
  for (int t = t0; t < t1; ++t) {
    const int src = termInfo[4 * t + 1], slot = termInfo[4 * t + 2], trans = termInfo[4 * t + 3];
    const double2* W = (trans ? U : V) + static_cast<long long>(slot) * RANK * M;
    const double2* W2 = (trans ? V : U) + static_cast<long long>(slot) * RANK * M;
    __syncthreads();
    for (int q = threadIdx.x; q < RANK * M; q += blockDim.x) {
      (&sW[0][0])[q] = __ldg(W + q);
      (&sW2[0][0])[q] = __ldg(W2 + q);
    }
    for (int q = threadIdx.x; q < M; q += blockDim.x) sD[q] = __ldg(D + static_cast<long long>(slot) * M + q);
    __syncthreads();
    // All RPW columns advance together through the rank loop: one shared
    // memory read of U/V row q serves RPW columns, and the RPW butterfly
    // reductions interleave.
    double2 xv[RPW][KPL];
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int r = r0 + warp * RPW + j;
      const double2* xs = x + src * xE + static_cast<long long>(r) * xR;
#pragma unroll
      for (int k = 0; k < KPL; ++k) xv[j][k] = r < nrhs ? __ldg(xs + lane + 32 * k) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const double2 d = sD[lane + 32 * k];
#pragma unroll
      for (int j = 0; j < RPW; ++j) cfma(acc[j][k], d, xv[j][k]);
    }
#pragma unroll 1
    for (int q = 0; q < RANK; ++q) {
      double2 p[RPW];
#pragma unroll
      for (int j = 0; j < RPW; ++j) p[j] = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < KPL; ++k) {
        const double2 w = sW[q][lane + 32 * k];
#pragma unroll
        for (int j = 0; j < RPW; ++j) cfma(p[j], w, xv[j][k]);
      }
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
        for (int j = 0; j < RPW; ++j) {
          p[j].x += __shfl_xor_sync(0xffffffffu, p[j].x, off);
          p[j].y += __shfl_xor_sync(0xffffffffu, p[j].y, off);
        }
#pragma unroll
      for (int k = 0; k < KPL; ++k) {
        const double2 w2 = sW2[q][lane + 32 * k];
#pragma unroll
        for (int j = 0; j < RPW; ++j) cfma(acc[j][k], w2, p[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RPW; ++j) {
    const int r = r0 + warp * RPW + j;
    if (r >= nrhs) break;
#pragma unroll
    for (int k = 0; k < KPL; ++k) ycorr[(static_cast<long long>(e) * nrhs + r) * M + lane + 32 * k] = acc[j][k];
  }
}

// y[e][rhs][a] += sum_b K[a][b] x[e][rhs][b].
__global__ void antisymApply(const double2* __restrict__ K, const double2* __restrict__ x, double2* __restrict__ y,
                             int m, int nrhs) {
  extern __shared__ double2 sx[];
  const long long base = (static_cast<long long>(blockIdx.x) * nrhs + blockIdx.y) * m;
  for (int b = threadIdx.x; b < m; b += blockDim.x) sx[b] = x[base + b];
  __syncthreads();
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int b = 0; b < m; ++b) cfma(s, K[static_cast<long long>(a) * m + b], sx[b]);
    y[base + a] = cadd(y[base + a], s);
  }
}

}  // namespace

void launchCorrVectorOn(Ctx& c, const CorrTables& t, const double2* x, double2* ycorr, int nrhs, cudaStream_t s,
                        long long xUserN) {
  if (t.nTargets == 0) return;
  // x's element / column strides: internal [e][rhs][a], or the user's
  // column-major n x nrhs (xUserN = n > 0).
  const long long xE = xUserN > 0 ? c.m : static_cast<long long>(nrhs) * c.m;
  const long long xR = xUserN > 0 ? xUserN : c.m;
  if (nrhs >= 8 && (c.rank == 4 || c.rank == 8) && (c.m == 64 || c.m == 128)) {
    dim3 grid(t.nTargets, (nrhs + 31) / 32);
    auto k = c.m == 64 ? (c.rank == 4 ? corrMulti<2, 4> : corrMulti<2, 8>)
                       : (c.rank == 4 ? corrMulti<4, 4> : corrMulti<4, 8>);
    k<<<grid, 256, 0, s>>>(t.termInfo, t.targetList, t.targetPtr, c.dCorrD, c.dCorrU, c.dCorrV, x, ycorr, nrhs, xE, xR);
    TBT_CUDA_CHECK(cudaGetLastError());
    return;
  }
  dim3 grid(t.nTargets, nrhs);
  const size_t smem = static_cast<size_t>(t.maxTerms) * std::max(c.rank, 1) * sizeof(double2);
  corrFused<<<grid, 256, smem, s>>>(t.termInfo, t.targetList, t.targetPtr, c.dCorrD, c.dCorrU, c.dCorrV, x, ycorr,
                                    c.m, c.rank, nrhs, xE, xR);
  TBT_CUDA_CHECK(cudaGetLastError());
}

void launchCorrVector(Ctx& c, const double2* x, double2* ycorr, int nrhs, cudaStream_t s, long long xUserN) {
  if (!c.haveCorr || c.nTerms == 0) return;
  launchCorrVectorOn(c, CorrTables{c.dTermInfo, c.dTargetList, c.dTargetPtr, c.nTargets, c.maxTermsPerTarget}, x,
                     ycorr, nrhs, s, xUserN);
}

void launchCorrection(Ctx& c, const double2* x, double2* y, int nrhs) {
  if (!c.haveCorr || c.nTerms == 0) return;
  if (c.rank > 0) {
    const long long warps = static_cast<long long>(c.nTerms) * nrhs;
    const int blocks = static_cast<int>((warps + 7) / 8);
    corrProject<<<blocks, 256, 0, c.stream>>>(c.dTermInfo, c.nTerms, c.dCorrU, c.dCorrV, x, c.dProj, c.m, c.rank,
                                              nrhs);
    TBT_CUDA_CHECK(cudaGetLastError());
  }
  dim3 grid(c.nTargets, nrhs);
  corrApply<<<grid, 64, 0, c.stream>>>(c.dTermInfo, c.dTargetList, c.dTargetPtr, c.dCorrD, c.dCorrU, c.dCorrV, x,
                                       c.dProj, y, c.m, c.rank, nrhs);
  TBT_CUDA_CHECK(cudaGetLastError());
}

void launchAntisym(Ctx& c, const double2* x, double2* y, int nrhs, int nElems) {
  if (!c.hasAntisym) return;
  if (nElems < 0) nElems = c.ne;
  if (nElems == 0) return;
  dim3 grid(nElems, nrhs);
  antisymApply<<<grid, 64, c.m * sizeof(double2), c.stream>>>(c.dAntisym, x, y, c.m, nrhs);
  TBT_CUDA_CHECK(cudaGetLastError());
}

}  // namespace tbt
