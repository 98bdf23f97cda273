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
#include <atomic>
#include <cstdlib>
#include <string>

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

// Many right-hand sides: one CTA per (target, chunk of 8*RPW columns). Each
// term's d, U, V (rank RANK, m = 32*KPL) are staged once in shared memory and
// reused by all columns of the chunk (instead of once per column); every
// warp owns RPW columns whose sums stay in registers across the term list.
// The term list is a latency chain (stage, barrier, x loads, rank loop with
// warp reductions): the next term's d, U, V arrive through a second cp.async
// stage and its x values are loaded before the current term's arithmetic,
// and RPW = 2 keeps two CTAs (16 warps) on an SM. With RPW = 4, one stage and
// one CTA per SM the kernel took 136 us at C3 and, although on a side stream,
// cost 108 us of the 663 us apply.
__device__ __forceinline__ void corrCpAsync16(void* dst, const void* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}

template <int KPL, int RANK, int RPW>
__global__ void __launch_bounds__(256, RPW <= 2 ? 2 : 1)
corrMulti(const int* __restrict__ termInfo, const int* __restrict__ targetList, const int* __restrict__ targetPtr,
          const int* __restrict__ order, const double2* __restrict__ D, const double2* __restrict__ U, const double2* __restrict__ V,
          const double2* __restrict__ x, double2* __restrict__ ycorr, int nrhs, long long xE, long long xR) {
  constexpr int M = 32 * KPL;
  constexpr int RC = 8 * RPW;
  constexpr int STG = (2 * RANK + 1) * M;  // W, W2, d
  extern __shared__ __align__(16) double2 csm[];  // [2][STG]
  const int ti = order ? order[blockIdx.y] : blockIdx.y;  // grid (column chunks, targets): a target's chunks adjacent
  const int r0 = blockIdx.x * RC;
  const int e = targetList[ti];
  const int t0 = targetPtr[ti], t1 = targetPtr[ti + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 acc[RPW][KPL];
#pragma unroll
  for (int j = 0; j < RPW; ++j)
#pragma unroll
    for (int k = 0; k < KPL; ++k) acc[j][k] = make_double2(0.0, 0.0);

  auto stage = [&](int t, int st) {
    const int slot = termInfo[4 * t + 2], trans = termInfo[4 * t + 3];
    const double2* W = (trans ? U : V) + static_cast<long long>(slot) * RANK * M;
    const double2* W2 = (trans ? V : U) + static_cast<long long>(slot) * RANK * M;
    double2* sW = csm + st * STG;
    for (int q = threadIdx.x; q < RANK * M; q += 256) {
      corrCpAsync16(sW + q, W + q);
      corrCpAsync16(sW + RANK * M + q, W2 + q);
    }
    for (int q = threadIdx.x; q < M; q += 256) corrCpAsync16(sW + 2 * RANK * M + q, D + static_cast<long long>(slot) * M + q);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto loadX = [&](int t, double2 (&xv)[RPW][KPL]) {
    const int src = termInfo[4 * t + 1];
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int r = r0 + warp * RPW + j;
      const double2* xs = x + src * xE + static_cast<long long>(r) * xR;
#pragma unroll
      for (int k = 0; k < KPL; ++k) xv[j][k] = r < nrhs ? __ldg(xs + lane + 32 * k) : make_double2(0.0, 0.0);
    }
  };

  double2 xv[RPW][KPL], xn[RPW][KPL];
  if (t0 < t1) {
    stage(t0, 0);
    loadX(t0, xv);
  }
  for (int t = t0; t < t1; ++t) {
    const int st = (t - t0) & 1;
    if (t + 1 < t1) {
      stage(t + 1, st ^ 1);  // read last in iteration t - 1, which ended with a barrier
      loadX(t + 1, xn);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double2* sW = csm + st * STG;
    const double2* sW2 = sW + RANK * M;
    const double2* sD = sW2 + RANK * M;
    // All RPW columns advance together through the rank loop: one shared
    // memory read of U/V row q serves RPW columns.
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const double2 d = sD[lane + 32 * k];
#pragma unroll
      for (int j = 0; j < RPW; ++j) cfma(acc[j][k], d, xv[j][k]);
    }
    // Rank rows in groups of four: the four projections of a column are
    // reduced together (lanes trade two values at offset 16, one at offset
    // 8, then a 3-level butterfly on the single remaining value; the totals
    // come back by indexed shuffles): 10 shuffles and 6 additions per value
    // pair and group instead of 20 and 20 with one butterfly per row.
#pragma unroll 1
    for (int q0 = 0; q0 < RANK; q0 += 4) {
      double2 p[4][RPW];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int j = 0; j < RPW; ++j) p[i][j] = make_double2(0.0, 0.0);
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
          const double2 w = sW[(q0 + i) * M + lane + 32 * k];
#pragma unroll
          for (int j = 0; j < RPW; ++j) cfma(p[i][j], w, xv[j][k]);
        }
      }
      const bool b4 = lane & 16, b3 = lane & 8;
#pragma unroll
      for (int j = 0; j < RPW; ++j) {
        const double2 s0 = b4 ? p[0][j] : p[2][j], s1 = b4 ? p[1][j] : p[3][j];
        double2 r0 = b4 ? p[2][j] : p[0][j], r1 = b4 ? p[3][j] : p[1][j];
        r0.x += __shfl_xor_sync(0xffffffffu, s0.x, 16);
        r0.y += __shfl_xor_sync(0xffffffffu, s0.y, 16);
        r1.x += __shfl_xor_sync(0xffffffffu, s1.x, 16);
        r1.y += __shfl_xor_sync(0xffffffffu, s1.y, 16);
        const double2 s = b3 ? r0 : r1;
        double2 v = b3 ? r1 : r0;
        v.x += __shfl_xor_sync(0xffffffffu, s.x, 8);
        v.y += __shfl_xor_sync(0xffffffffu, s.y, 8);
#pragma unroll
        for (int off = 4; off >= 1; off >>= 1) {
          v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
          v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
        }
        // lane l now holds the total of row q0 + (l >> 3)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          p[i][j].x = __shfl_sync(0xffffffffu, v.x, 8 * i);
          p[i][j].y = __shfl_sync(0xffffffffu, v.y, 8 * i);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
          const double2 w2 = sW2[(q0 + i) * M + lane + 32 * k];
#pragma unroll
          for (int j = 0; j < RPW; ++j) cfma(acc[j][k], w2, p[i][j]);
        }
    }
    __syncthreads();  // stage st is refilled in the next iteration
    if (t + 1 < t1) {
#pragma unroll
      for (int j = 0; j < RPW; ++j)
#pragma unroll
        for (int k = 0; k < KPL; ++k) xv[j][k] = xn[j][k];
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

template <int KPL, int RANK, int RPW>
void launchCorrMulti(Ctx& c, const CorrTables& t, const double2* x, double2* ycorr, int nrhs, cudaStream_t s,
                     long long xE, long long xR) {
  constexpr size_t SMEM = 2 * (2 * RANK + 1) * 32 * KPL * sizeof(double2);
  static std::atomic<unsigned long long> attr{0};
  oncePerDevice(attr, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(corrMulti<KPL, RANK, RPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(SMEM)));
  });
  dim3 grid((nrhs + 8 * RPW - 1) / (8 * RPW), t.nTargets);
  corrMulti<KPL, RANK, RPW><<<grid, 256, SMEM, s>>>(t.termInfo, t.targetList, t.targetPtr, t.order, c.dCorrD,
                                                    c.dCorrU, c.dCorrV, x, ycorr, nrhs, xE, xR);
}

// Rank-8 terms on the FP64 tensor path (the default; TBT_CORR=vec selects
// corrMulti): a warp owns 8
// columns; per term P(8 x 8 cols) = W(8 x m) X(m x 8 cols) and
// Y(m x 8 cols) += W2^T(m x 8) P as mma.sync.m8n8k4.f64 tiles (4M complex
// form: four real DMMAs per complex tile), X fragments straight from global
// memory (each value is used once per warp), P turned from the accumulator
// layout into the B-operand layout through 1 KB of warp-private shared
// memory; the diagonal term stays on DFMA. No cross-lane reductions.
__device__ __forceinline__ void corrDmmaOp(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int KPL>
__global__ void __launch_bounds__(128, 2)
corrDmma(const int* __restrict__ termInfo, const int* __restrict__ targetList, const int* __restrict__ targetPtr,
         const int* __restrict__ order, const double2* __restrict__ D, const double2* __restrict__ U, const double2* __restrict__ V,
         const double2* __restrict__ x, double2* __restrict__ ycorr, int nrhs, long long xE, long long xR) {
  constexpr int M = 32 * KPL, RANK = 8, MBLK = M / 8;
  constexpr int LDW = M + 4, LDW2 = M + 2;  // row pitches: conflict-free A fragments of W (rows = q) and W2 (k = q)
  constexpr int STG = RANK * LDW + RANK * LDW2 + M;
  constexpr int NBAT = M / 16;  // batches of 4 k steps = 16 basis rows = 2 m-blocks
  extern __shared__ __align__(16) double2 csm[];  // [2][STG], then per warp: P [64], X batch [16][8]
  const int ti = order ? order[blockIdx.y] : blockIdx.y;
  const int e = targetList[ti];
  const int t0 = targetPtr[ti], t1 = targetPtr[ti + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  double2* sP = csm + 2 * STG + warp * 192;
  double2* sX = sP + 64;
  const int c0 = blockIdx.x * 32 + warp * 8;
  const bool active = c0 < nrhs;
  const int cb = c0 + gid;  // the column of this lane's B fragments
  const bool cbok = cb < nrhs;
  const long long xcol = static_cast<long long>(cbok ? cb : 0) * xR + tig;
  double yr[MBLK][2], yi[MBLK][2];
#pragma unroll
  for (int mb = 0; mb < MBLK; ++mb) yr[mb][0] = yr[mb][1] = yi[mb][0] = yi[mb][1] = 0.0;

  auto stage = [&](int t, int st) {
    const int slot = termInfo[4 * t + 2], trans = termInfo[4 * t + 3];
    const double2* W = (trans ? U : V) + static_cast<long long>(slot) * RANK * M;
    const double2* W2 = (trans ? V : U) + static_cast<long long>(slot) * RANK * M;
    double2* sW = csm + st * STG;
    double2* sW2 = sW + RANK * LDW;
    for (int q = threadIdx.x; q < RANK * M; q += 128) {
      const int r = q / M, a = q % M;
      corrCpAsync16(sW + r * LDW + a, W + q);
      corrCpAsync16(sW2 + r * LDW2 + a, W2 + q);
    }
    for (int q = threadIdx.x; q < M; q += 128) corrCpAsync16(sW2 + RANK * LDW2 + q, D + static_cast<long long>(slot) * M + q);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // X fragments of one batch: rows 16 bt + 4 u + tig of column cb.
  auto loadX = [&](const double2* xs, int bt, double2 (&xq)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) xq[u] = cbok ? __ldg(xs + bt * 16 + u * 4) : make_double2(0.0, 0.0);
  };

  double2 xq[2][4];
  if (t0 < t1) {
    stage(t0, 0);
    if (active) loadX(x + termInfo[4 * t0 + 1] * xE + xcol, 0, xq[0]);
  }
  for (int t = t0; t < t1; ++t) {
    const int st = (t - t0) & 1;
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // term t's stage has landed everywhere; everyone is done with term t - 1's
    if (t + 1 < t1) stage(t + 1, st ^ 1);
    if (!active) continue;
    const double2* sW = csm + st * STG;
    const double2* sW2 = sW + RANK * LDW;
    const double2* sD = sW2 + RANK * LDW2;
    const double2* xs = x + termInfo[4 * t + 1] * xE + xcol;
    double pr[2] = {0.0, 0.0}, pi[2] = {0.0, 0.0};
#pragma unroll
    for (int bt = 0; bt < NBAT; ++bt) {
      if (bt + 1 < NBAT) loadX(xs, bt + 1, xq[(bt + 1) & 1]);
      double2(&xb)[4] = xq[bt & 1];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 w = sW[gid * LDW + bt * 16 + u * 4 + tig];
        corrDmmaOp(pr, w.x, xb[u].x);
        corrDmmaOp(pr, -w.y, xb[u].y);
        corrDmmaOp(pi, w.x, xb[u].y);
        corrDmmaOp(pi, w.y, xb[u].x);
      }
      // Diagonal term: the batch's X values go from the B layout (row 4u +
      // tig, column gid) to the accumulator layout (row gid of m-block 2 bt +
      // mbl, columns 2 tig + {0,1}) through warp-private shared memory
      // (column index XOR row: conflict-free reads, 2-way writes).
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = u * 4 + tig;
        sX[r * 8 + (gid ^ (r & 7))] = xb[u];
      }
      __syncwarp();
#pragma unroll
      for (int mbl = 0; mbl < 2; ++mbl) {
        const int mb = 2 * bt + mbl;
        const double2 d = sD[mb * 8 + gid];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 xv = sX[(mbl * 8 + gid) * 8 + ((2 * tig + h) ^ gid)];
          yr[mb][h] = fma(d.x, xv.x, fma(-d.y, xv.y, yr[mb][h]));
          yi[mb][h] = fma(d.x, xv.y, fma(d.y, xv.x, yi[mb][h]));
        }
      }
      __syncwarp();
    }
    // accumulator layout (row q = gid, columns 2 tig + {0,1}) -> B layout (k = q = tig (+4), column gid)
    sP[gid * 8 + 2 * tig] = make_double2(pr[0], pi[0]);
    sP[gid * 8 + 2 * tig + 1] = make_double2(pr[1], pi[1]);
    __syncwarp();
    const double2 pb0 = sP[tig * 8 + gid], pb1 = sP[(4 + tig) * 8 + gid];
    __syncwarp();
    // the next term's first X batch arrives under this term's second product
    if (t + 1 < t1) loadX(x + termInfo[4 * (t + 1) + 1] * xE + xcol, 0, xq[0]);
#pragma unroll
    for (int mb = 0; mb < MBLK; ++mb) {
      const double2 w0 = sW2[tig * LDW2 + mb * 8 + gid], w1 = sW2[(4 + tig) * LDW2 + mb * 8 + gid];
      corrDmmaOp(yr[mb], w0.x, pb0.x);
      corrDmmaOp(yr[mb], -w0.y, pb0.y);
      corrDmmaOp(yi[mb], w0.x, pb0.y);
      corrDmmaOp(yi[mb], w0.y, pb0.x);
      corrDmmaOp(yr[mb], w1.x, pb1.x);
      corrDmmaOp(yr[mb], -w1.y, pb1.y);
      corrDmmaOp(yi[mb], w1.x, pb1.y);
      corrDmmaOp(yi[mb], w1.y, pb1.x);
    }
  }
  if (!active) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = c0 + 2 * tig + h;
    if (c >= nrhs) continue;
#pragma unroll
    for (int mb = 0; mb < MBLK; ++mb)
      ycorr[(static_cast<long long>(e) * nrhs + c) * M + mb * 8 + gid] = make_double2(yr[mb][h], yi[mb][h]);
  }
}

template <int KPL>
void launchCorrDmma(Ctx& c, const CorrTables& t, const double2* x, double2* ycorr, int nrhs, cudaStream_t s,
                    long long xE, long long xR) {
  constexpr int M = 32 * KPL;
  constexpr size_t SMEM = (2 * (8 * (M + 4) + 8 * (M + 2) + M) + 4 * 192) * sizeof(double2);
  static std::atomic<unsigned long long> attr{0};
  oncePerDevice(attr, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(corrDmma<KPL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(SMEM)));
  });
  dim3 grid((nrhs + 31) / 32, t.nTargets);
  corrDmma<KPL><<<grid, 128, SMEM, s>>>(t.termInfo, t.targetList, t.targetPtr, t.order, c.dCorrD, c.dCorrU, c.dCorrV, x,
                                        ycorr, nrhs, xE, xR);
}

bool corrUseDmma() {
  static const bool on = [] {
    const char* e = getenv("TBT_CORR");
    return !(e && std::string(e) == "vec");  // TBT_CORR=vec: the DFMA / shuffle kernel (corrMulti) for rank 8 too
  }();
  return on;
}

// Columns per warp of corrMulti (TBT_CORR_RPW = 1 | 2 | 4; default 2).
int corrRpw() {
  static const int v = [] {
    const char* e = getenv("TBT_CORR_RPW");
    const int r = e ? atoi(e) : 2;
    return r == 1 || r == 4 ? r : 2;
  }();
  return v;
}

template <int KPL, int RANK>
void launchCorrMultiRpw(Ctx& c, const CorrTables& t, const double2* x, double2* ycorr, int nrhs, cudaStream_t s,
                        long long xE, long long xR) {
  switch (corrRpw()) {
    case 1: launchCorrMulti<KPL, RANK, 1>(c, t, x, ycorr, nrhs, s, xE, xR); break;
    case 4: launchCorrMulti<KPL, RANK, 4>(c, t, x, ycorr, nrhs, s, xE, xR); break;
    default: launchCorrMulti<KPL, RANK, 2>(c, t, x, ycorr, nrhs, s, xE, xR);
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
    if (c.rank == 8 && corrUseDmma())
      c.m == 64 ? launchCorrDmma<2>(c, t, x, ycorr, nrhs, s, xE, xR) : launchCorrDmma<4>(c, t, x, ycorr, nrhs, s, xE, xR);
    else if (c.m == 64)
      c.rank == 4 ? launchCorrMultiRpw<2, 4>(c, t, x, ycorr, nrhs, s, xE, xR)
                  : launchCorrMultiRpw<2, 8>(c, t, x, ycorr, nrhs, s, xE, xR);
    else
      c.rank == 4 ? launchCorrMultiRpw<4, 4>(c, t, x, ycorr, nrhs, s, xE, xR)
                  : launchCorrMultiRpw<4, 8>(c, t, x, ycorr, nrhs, s, xE, xR);
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
  launchCorrVectorOn(c, CorrTables{c.dTermInfo, c.dTargetList, c.dTargetPtr, c.nTargets, c.maxTermsPerTarget,
                                   c.dTargetList + c.nTargets},
                     x,
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
