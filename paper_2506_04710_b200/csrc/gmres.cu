// Kernel group K5: restarted GMRES on the device, columns in lockstep.
//
// Restates gmres (proj/src/linsolve.cpp:425-515) per column: x0 = 0, true
// relative residual at every restart, left Jacobi, modified Gram-Schmidt
// with the conjugated inner product, complex Givens rotations, inner exit
// at |g_{j+1}|/beta < 0.1 tol, lucky breakdown, back substitution; maxIter
// counts inner iterations. All Krylov data stays in HBM/L2; the host only
// enqueues and polls a few bytes of per-column state.
//
// The Arnoldi step is ONE cooperative kernel per iteration: the fused MGS
// sweep "w -= h_i v_i; partial <v_{i+1}, w>" needs one grid barrier per
// projection (j+2 barriers per step). Cross-CTA reductions read the per-CTA
// partials in a fixed order (every warp reduces them itself, butterfly), so
// every CTA derives bitwise-identical h values and runs are reproducible.
// For one column with at most FAST_K slots per thread, w and the basis
// vectors being projected out live in registers (gmresArnoldi1).
// The Givens sweep and the back substitution run on staged shared-memory /
// register copies of H, cs, sn, g (one memory round trip, not one per entry).
#include <algorithm>
#include <mutex>
#include <cmath>

#include <cstdio>
#include <cstring>

#include "gmres_dev.cuh"

namespace tbt {

namespace {

using namespace gmresdev;

// Last column of a lagged restart cycle (matvec_persistent.cu LAGGED): its
// w' norm from the G per-CTA partials of the last node, and its Givens step.
__global__ void gmresLaggedFinish(GmresArgs A, int j, int G) {
  __shared__ double2 sh[3 * RMAX + 4];
  const volatile GmresState* st = A.st;
  if (!st->cycleActive || st->stopInner) return;  // a node already ended the cycle
  const double hn = sqrt(warpTotalN(partSlotN(A, 0, 0, G), G).x);
  givensWarp(A, 0, j, hn, sh);
}

__global__ void __launch_bounds__(kThreads) gmresInit(GmresArgs A) {
  __shared__ double2 scratch[kWarps];
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int col = 0; col < A.ncols; ++col) {
    double2 acc = make_double2(0.0, 0.0);
    for (long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; s < slots; s += stride) {
      const double2 v = A.b[slotIndex(s, col, A.ncols, A.m)];
      acc.x += v.x * v.x + v.y * v.y;
    }
    blockPartial(acc, scratch, partSlot(A, 0, col));
    __syncthreads();
  }
  gridBarrier(A.bar);
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    for (int col = 0; col < A.ncols; ++col) {
      const double2 tot = warpTotal(partSlot(A, 0, col));
      if (threadIdx.x == 0) {
        GmresState& st = A.st[col];
        st.bnorm = sqrt(tot.x);
        st.beta = 0.0;
        st.beta0 = 0.0;
        st.residual = 0.0;
        st.iterations = 0;
        st.ncount = 0;
        st.stopInner = 1;
        st.cycleActive = 0;
        st.histLen = 0;
        st.done = st.bnorm == 0.0 ? 1 : 0;
        st.converged = st.done;
      }
    }
  }
}

// r = b - A x, residual test, z = M r, beta, v0 = z / beta (linsolve.cpp:446-461).
constexpr int kCyU = 4;  // element-wise passes: slots in flight per thread

__global__ void __launch_bounds__(kThreads) gmresCycleStart(GmresArgs A) {
  __shared__ double2 scratch[kWarps];
  extern __shared__ int sFlag[];  // [ncols]: 1 = this cycle runs
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long s0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  for (int col = 0; col < A.ncols; ++col) {
    const bool run = !A.st[col].done;
    if (threadIdx.x == 0) sFlag[col] = run ? 1 : 0;
    double2 acc = make_double2(0.0, 0.0);
    if (run)
      for (long long sb = s0; sb < slots; sb += kCyU * stride) {  // kCyU slots in flight per thread
        double2 bv[kCyU], av[kCyU];
#pragma unroll
        for (int u = 0; u < kCyU; ++u) {
          const long long s = sb + u * stride;
          const long long q = slotIndex(s < slots ? s : sb, col, A.ncols, A.m);
          bv[u] = A.b[q];
          av[u] = A.ax[q];
        }
#pragma unroll
        for (int u = 0; u < kCyU; ++u) {
          const long long s = sb + u * stride;
          if (s >= slots) continue;
          const double2 r = csub(bv[u], av[u]);
          A.w[slotIndex(s, col, A.ncols, A.m)] = r;
          acc.x += r.x * r.x + r.y * r.y;
        }
      }
    blockPartial(acc, scratch, partSlot(A, 0, col));
    __syncthreads();
  }
  gridBarrier(A.bar);
  for (int col = 0; col < A.ncols; ++col) {
    if (!sFlag[col]) continue;
    const double2 tot = warpTotal(partSlot(A, 0, col));
    const double res = sqrt(tot.x) / A.st[col].bnorm;
    int decision = 0;  // 0 run, 1 converged, 2 out of iterations
    if (res < A.tol)
      decision = 1;
    else if (A.st[col].iterations >= A.maxIter)
      decision = 2;
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      GmresState& st = A.st[col];
      st.residual = res;
      pushHist(A, col, decision == 2 ? 2.0 : 0.0, res);
      if (decision != 0) {
        st.done = 1;
        st.converged = decision == 1 ? 1 : 0;
        st.cycleActive = 0;
        st.stopInner = 1;
      }
    }
    if (threadIdx.x == 0) sFlag[col] = decision == 0 ? 1 : 0;
    __syncthreads();
    double2 acc = make_double2(0.0, 0.0);
    if (sFlag[col])
      for (long long sb = s0; sb < slots; sb += kCyU * stride) {
        double2 wv[kCyU], dv[kCyU];
#pragma unroll
        for (int u = 0; u < kCyU; ++u) {
          const long long s = sb + u * stride;
          const long long sc = s < slots ? s : sb;
          wv[u] = A.w[slotIndex(sc, col, A.ncols, A.m)];
          dv[u] = A.dinv ? A.dinv[sc] : make_double2(1.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < kCyU; ++u) {
          const long long s = sb + u * stride;
          if (s >= slots) continue;
          const double2 z = A.dinv ? cmul(wv[u], dv[u]) : wv[u];
          A.V[slotIndex(s, col, A.ncols, A.m)] = z;
          acc.x += z.x * z.x + z.y * z.y;
        }
      }
    blockPartial(acc, scratch, partSlot(A, 1, col));
    __syncthreads();
  }
  gridBarrier(A.bar);
  for (int col = 0; col < A.ncols; ++col) {
    if (!sFlag[col]) continue;
    const double beta = sqrt(warpTotal(partSlot(A, 1, col)).x);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      GmresState& st = A.st[col];
      if (beta == 0.0) {
        st.done = 1;
        st.converged = 1;
        st.cycleActive = 0;
        st.stopInner = 1;
      } else {
        st.beta = beta;
        if (st.beta0 == 0.0) st.beta0 = beta;
        st.ncount = 0;
        st.stopInner = 0;
        st.cycleActive = 1;
        double2* g = A.g + static_cast<long long>(col) * (A.restart + 1);
        for (int k = 0; k <= A.restart; ++k) g[k] = make_double2(0.0, 0.0);
        g[0] = make_double2(beta, 0.0);
      }
    }
    if (beta != 0.0)
      for (long long sb = s0; sb < slots; sb += kCyU * stride) {
        double2 zv[kCyU];
#pragma unroll
        for (int u = 0; u < kCyU; ++u) {
          const long long s = sb + u * stride;
          zv[u] = A.V[slotIndex(s < slots ? s : sb, col, A.ncols, A.m)];
        }
#pragma unroll
        for (int u = 0; u < kCyU; ++u) {
          const long long s = sb + u * stride;
          if (s < slots) A.V[slotIndex(s, col, A.ncols, A.m)] = make_double2(zv[u].x / beta, zv[u].y / beta);
        }
      }
  }
}

// One Arnoldi step j, single column, w and the basis vector being projected
// out held in registers (FAST_K slots per thread, grid-strided).
__global__ void __launch_bounds__(kThreads) gmresArnoldi1(GmresArgs A) {
  __shared__ double2 scratch[kWarps];
  __shared__ double2 hcol[RMAX + 2];
  __shared__ double2 sh[3 * RMAX + 4];
  const int run = A.st[0].cycleActive && !A.st[0].stopInner;
  if (!run) return;  // uniform over the grid
  const int j = A.j;
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long s0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  double2 w[FAST_K], vc[FAST_K], vn[FAST_K];
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < FAST_K; ++k) {
    const long long s = s0 + k * stride;
    w[k] = vc[k] = vn[k] = make_double2(0.0, 0.0);
    if (s < slots) {
      double2 wv = A.w[s];
      if (A.dinv) wv = cmul(wv, A.dinv[s]);
      w[k] = wv;
      vc[k] = A.V[s];
      cfma_conj(acc, vc[k], wv);
    }
  }
  blockPartial(acc, scratch, partSlot(A, 0, 0));
  gridBarrier(A.bar);
  for (int i = 0; i <= j; ++i) {
    if (i < j) {
      const double2* vnext = A.V + static_cast<long long>(i + 1) * slots;
#pragma unroll
      for (int k = 0; k < FAST_K; ++k) {
        const long long s = s0 + k * stride;
        vn[k] = s < slots ? vnext[s] : make_double2(0.0, 0.0);
      }
    }
    const double2 h = warpTotal(partSlot(A, i, 0));
    if (blockIdx.x == 0 && threadIdx.x == 0) hcol[i] = h;
    acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < FAST_K; ++k) {
      w[k] = csub(w[k], cmul(h, vc[k]));
      if (i < j)
        cfma_conj(acc, vn[k], w[k]);
      else
        acc.x += w[k].x * w[k].x + w[k].y * w[k].y;
      vc[k] = vn[k];
    }
    blockPartial(acc, scratch, partSlot(A, i + 1, 0));
    gridBarrier(A.bar);
  }
  const double hn = sqrt(warpTotal(partSlot(A, j + 1, 0)).x);
  if (hn > 0.0) {
    double2* vout = A.V + static_cast<long long>(j + 1) * slots;
#pragma unroll
    for (int k = 0; k < FAST_K; ++k) {
      const long long s = s0 + k * stride;
      if (s < slots) vout[s] = make_double2(w[k].x / hn, w[k].y / hn);
    }
  }
  if (blockIdx.x == 0) givensStep(A, 0, j, hn, hcol, sh);
}

// One Arnoldi step j, single column, low-synchronisation MGS (gmres_dev.cuh).
__global__ void __launch_bounds__(kThreads) gmresArnoldiLS(GmresArgs A, double2* S, double2* dots,
                                                           double2* dotPart) {
  extern __shared__ double2 shw[];
  __shared__ double2 scratch[kWarps];
  __shared__ double2 hcol[RMAX + 2];
  __shared__ double2 sh[3 * RMAX + 4];
  arnoldiLS(A, A.j, S, dots, dotPart, shw, scratch, hcol, sh, A.bar);
}

// One Arnoldi step j, single column, low-synchronisation MGS, for vectors
// whose per-CTA row chunk does not fit shared memory (C4: 3.5 k rows, C5:
// 21 k rows per SM): the same recurrence as arnoldiLS (h = (I + L)^{-1} c,
// c = V^H M w, S_j = V^H v_j; two passes over the basis, two grid barriers)
// with the chunk streamed in sub-chunks of kBigSub rows:
//   pass 1  per sub-chunk: M w and v_j staged in shared memory; every warp
//           owns a contiguous slice of the sub-chunk and sweeps ALL basis
//           vectors over it, four at a time (8 rows per lane per vector:
//           32 loads in flight per lane), so all warps stream at any j;
//           per-(warp, vector) partials accumulate in shared memory in
//           sub-chunk order and are summed over the warps in warp order
//   -- barrier --  every CTA reduces every dot, forward substitution
//   pass 2  w' = M w - V h written to v_{j+1} unnormalised, ||w'||^2
//           (4 rows per thread, 8 vectors unrolled: 32 loads in flight),
//           row blocks in reverse order so the first ones hit what pass 1
//           left in L2 (C5: 4.20 -> 4.18 ms per iteration)
//   -- barrier --  v_{j+1} /= ||w'|| (the chunk rereads its own rows, L2),
//                  Givens (CTA 0)
// All sums are fixed-order: bitwise reproducible. Measured alternatives
// (C4, same box): a bulk-copy ring for pass 1 (tiles w, v_j, v_k through
// shared memory, warp-owned row slices) 0.533 vs 0.520 ms per iteration;
// (vector, segment) work items with register accumulators 0.545.
constexpr int kBigSub = 2048;
constexpr int kBigRowsPerLane = kBigSub / (kWarps * 32);  // 8
constexpr int kBigVec = 4;                                 // basis vectors per sweep step

size_t lsBigSmem(int restart) {  // dynamic: ws, vj sub-chunks + packed L + per-warp partials
  return sizeof(double2) * (2 * kBigSub + static_cast<size_t>(restart) * (restart + 1) / 2 +
                            2 * static_cast<size_t>(kWarps) * (restart + 1));
}

__global__ void __launch_bounds__(kThreads, 1) gmresArnoldiLSBig(GmresArgs A, double2* S, double2* dotPart) {
  extern __shared__ double2 dyn[];
  const int lds = A.restart + 1;
  double2* ws = dyn;                                          // [kBigSub]
  double2* vj = dyn + kBigSub;                                // [kBigSub]
  double2* sL = vj + kBigSub;                                 // packed rows of L: row i at i*(i-1)/2
  double2* wpart = sL + static_cast<long long>(A.restart) * (A.restart + 1) / 2;  // [2][kWarps][lds]
  __shared__ double2 cv[RMAX + 1];
  __shared__ double2 scratch[kWarps];
  __shared__ double2 hcol[RMAX + 2];
  __shared__ double2 sh[3 * RMAX + 4];
  const int run = A.st[0].cycleActive && !A.st[0].stopInner;
  if (!run) return;  // uniform over the grid
  const int j = A.j;
  const long long n = static_cast<long long>(A.ne) * A.m;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk;
  const long long cnt = r0 >= n ? 0 : (n - r0 < chunk ? n - r0 : chunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int nw = kWarps;
  const double2* Vj = A.V + static_cast<long long>(j) * n + r0;
  const double2* w = A.w + r0;
  const double2* dinv = A.dinv ? A.dinv + r0 : nullptr;
  for (int t = threadIdx.x; t < 2 * nw * lds; t += blockDim.x) wpart[t] = make_double2(0.0, 0.0);
  // ---- pass 1
  for (long long s0 = 0; s0 < cnt; s0 += kBigSub) {
    const int sc = static_cast<int>(cnt - s0 < kBigSub ? cnt - s0 : kBigSub);
    __syncthreads();  // previous sub-chunk's readers are done
    {  // stage M w and v_j: all of a thread's loads issued before its stores
      constexpr int PT = kBigSub / kThreads;
      double2 lw[PT], ld[PT], lv[PT];
#pragma unroll
      for (int u = 0; u < PT; ++u) {
        const int r = threadIdx.x + u * kThreads;
        const bool ok = r < sc;
        lw[u] = ok ? w[s0 + r] : make_double2(0.0, 0.0);
        ld[u] = ok && dinv ? dinv[s0 + r] : make_double2(1.0, 0.0);
        lv[u] = ok ? Vj[s0 + r] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < PT; ++u) {
        const int r = threadIdx.x + u * kThreads;
        ws[r] = dinv ? cmul(lw[u], ld[u]) : lw[u];
        vj[r] = lv[u];
      }
    }
    __syncthreads();
    const int rw = warp * 32 * kBigRowsPerLane;  // this warp's slice of the sub-chunk
    for (int k0 = 0; k0 <= j; k0 += kBigVec) {
      double2 c[kBigVec], q[kBigVec];
      double2 v[kBigVec][kBigRowsPerLane];
#pragma unroll
      for (int t = 0; t < kBigVec; ++t) {
        c[t] = q[t] = make_double2(0.0, 0.0);
        const int k = k0 + t <= j ? k0 + t : j;
        const double2* Vk = A.V + static_cast<long long>(k) * n + r0 + s0 + rw;
#pragma unroll
        for (int u = 0; u < kBigRowsPerLane; ++u) {
          const int rr = rw + lane + 32 * u;
          v[t][u] = (rr < sc && k0 + t <= j) ? Vk[lane + 32 * u] : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < kBigRowsPerLane; ++u) {
        const int rr = rw + lane + 32 * u;
        const double2 wv = rr < sc ? ws[rr] : make_double2(0.0, 0.0);
        const double2 vv = rr < sc ? vj[rr] : make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < kBigVec; ++t) {
          cfma_conj(c[t], v[t][u], wv);
          cfma_conj(q[t], vv, v[t][u]);
        }
      }
#pragma unroll
      for (int t = 0; t < kBigVec; ++t) {
        const double2 ct = warpSum(c[t]), qt = warpSum(q[t]);
        if (lane == 0 && k0 + t <= j) {  // the warp owns its slots: sub-chunks in order
          double2& pc = wpart[static_cast<long long>(warp) * lds + k0 + t];
          double2& pq = wpart[static_cast<long long>(nw + warp) * lds + k0 + t];
          pc = cadd(pc, ct);
          pq = cadd(pq, qt);
        }
      }
    }
  }
  __syncthreads();
  for (int k = threadIdx.x; k <= j; k += blockDim.x) {
    double2 tc = wpart[k], tq = wpart[static_cast<long long>(nw) * lds + k];
    for (int w2 = 1; w2 < nw; ++w2) {
      tc = cadd(tc, wpart[static_cast<long long>(w2) * lds + k]);
      tq = cadd(tq, wpart[static_cast<long long>(nw + w2) * lds + k]);
    }
    dotPart[static_cast<long long>(k) * gridDim.x + blockIdx.x] = tc;
    if (k < j) dotPart[static_cast<long long>(lds + k) * gridDim.x + blockIdx.x] = tq;
  }
  gridBarrier(A.bar);
  // ---- grid totals, reduced by every CTA in the same fixed order
  double2* sLrow = sL;
  {
    const int ndots = 2 * j + 1;
    const int grp = lane >> 4, gl = lane & 15;
    const int G = static_cast<int>(gridDim.x);
    for (int d0 = warp * 2; d0 < ndots; d0 += nw * 2) {
      const int d = d0 + grp;
      double2 t = make_double2(0.0, 0.0);
      if (d < ndots) {
        const double2* pp = dotPart + static_cast<long long>(d <= j ? d : lds + (d - j - 1)) * G;
        double2 v[10];
        for (int k0 = gl; k0 < G; k0 += 160) {
#pragma unroll
          for (int q = 0; q < 10; ++q) {
            const int k = k0 + 16 * q;
            v[q] = k < G ? __ldcg(pp + k) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int q = 0; q < 10; ++q) t = cadd(t, v[q]);
        }
      }
#pragma unroll
      for (int off = 8; off >= 1; off >>= 1) {
        t.x += __shfl_xor_sync(0xffffffffu, t.x, off);
        t.y += __shfl_xor_sync(0xffffffffu, t.y, off);
      }
      if (gl == 0 && d < ndots) {
        if (d <= j) {
          cv[d] = t;
        } else {
          sLrow[j * (j - 1) / 2 + (d - j - 1)] = t;
          if (blockIdx.x == 0) S[static_cast<long long>(j) * lds + (d - j - 1)] = t;
        }
      }
    }
  }
  for (int i = 1 + warp; i < j; i += nw)
    for (int k = lane; k < i; k += 32) sLrow[i * (i - 1) / 2 + k] = __ldcg(S + static_cast<long long>(i) * lds + k);
  __syncthreads();
  if (warp == 0) {
    if (A.restart < 64)
      forwardSubstWarp<2>(cv, sLrow, j, lane);
    else
      forwardSubstWarp<(RMAX + 31) / 32 + 1>(cv, sLrow, j, lane);
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i <= j; i += blockDim.x) hcol[i] = cv[i];
  // ---- pass 2: w' = M w - V h -> v_{j+1} (unnormalised), ||w'||^2; four
  // rows per thread, the update order over k unchanged per row.
  double2* vout = A.V + static_cast<long long>(j + 1) * n + r0;
  double2 acc = make_double2(0.0, 0.0);
  const int bd = static_cast<int>(blockDim.x);
  constexpr int RT = 4;
  const long long nblk = (cnt + RT * bd - 1) / (RT * bd);
  for (long long bi = nblk - 1; bi >= 0; --bi) {  // reverse: pass 1's last rows are still in L2
    const long long ra = bi * RT * bd + threadIdx.x;
    double2 wr[RT];
    long long rs[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const long long r = ra + t * bd;
      rs[t] = r < cnt ? r : ra;
      wr[t] = w[rs[t]];
      if (dinv) wr[t] = cmul(wr[t], dinv[rs[t]]);
    }
    int k = 0;
    for (; k + 8 <= j + 1; k += 8) {
      double2 vv[8][RT];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int t = 0; t < RT; ++t) vv[u][t] = A.V[static_cast<long long>(k + u) * n + r0 + rs[t]];
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int t = 0; t < RT; ++t) wr[t] = csub(wr[t], cmul(cv[k + u], vv[u][t]));
    }
    for (; k <= j; ++k)
#pragma unroll
      for (int t = 0; t < RT; ++t) wr[t] = csub(wr[t], cmul(cv[k], A.V[static_cast<long long>(k) * n + r0 + rs[t]]));
#pragma unroll
    for (int t = 0; t < RT; ++t)
      if (ra + t * bd < cnt) {
        vout[ra + t * bd] = wr[t];
        acc.x += wr[t].x * wr[t].x + wr[t].y * wr[t].y;
      }
  }
  blockPartial(acc, scratch, partSlot(A, 0, 0));
  if (blockIdx.x == 0) givensStage(A, 0, j, hcol, sh);  // made visible by the barrier
  gridBarrier(A.bar);
  const double hn = sqrt(warpTotal(partSlot(A, 0, 0)).x);
  if (hn > 0.0) {
    constexpr int PT = 8;  // loads in flight per thread
    for (long long rb = threadIdx.x; rb < cnt; rb += PT * static_cast<long long>(blockDim.x)) {
      double2 v[PT];
#pragma unroll
      for (int u = 0; u < PT; ++u) {
        const long long r = rb + u * static_cast<long long>(blockDim.x);
        v[u] = r < cnt ? __ldcg(vout + r) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < PT; ++u) {
        const long long r = rb + u * static_cast<long long>(blockDim.x);
        if (r < cnt) vout[r] = make_double2(v[u].x / hn, v[u].y / hn);
      }
    }
  }
  if (blockIdx.x == 0) givensFinish(A, 0, j, hn, sh);
}

// One Arnoldi step j for many columns: one CTA per column runs the
// reference's MGS sweep (linsolve.cpp:465-468) with CTA-level reductions
// only, so columns proceed independently without grid barriers; w lives in
// global memory (L2), each projection is one fused sweep
// "w -= h_i v_i; partial <v_{i+1}, w>".
__global__ void __launch_bounds__(kThreads) gmresArnoldiCols(GmresArgs A) {
  __shared__ double2 scratch[kWarps];
  __shared__ double2 hcol[RMAX + 2];
  __shared__ double2 sh[3 * RMAX + 4];
  __shared__ double2 bcast;
  const int col = blockIdx.x;
  if (col >= A.ncols) return;
  const GmresState st = A.st[col];
  if (!(st.cycleActive && !st.stopInner)) return;
  const int j = A.j;
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long nall = slots * A.ncols;
  // Column col's entries: element e's m values at (e*ncols + col)*m. Each
  // thread walks a fixed basis index over a strided set of elements (no
  // index division in the sweeps).
  const int m = A.m;
  const int tpe = static_cast<int>(blockDim.x) >= m ? static_cast<int>(blockDim.x) / m : 1;  // threads per element slot
  const int a = static_cast<int>(threadIdx.x) % m;
  const int e0 = static_cast<int>(threadIdx.x) / m;
  const bool activeT = static_cast<int>(threadIdx.x) < tpe * m;
  const long long qStep = static_cast<long long>(tpe) * A.ncols * m;
  const long long q0 = (static_cast<long long>(e0) * A.ncols + col) * m + a;
  const long long sStep = static_cast<long long>(tpe) * m;
  const long long s0 = static_cast<long long>(e0) * m + a;
  const int nIter = activeT ? (A.ne - e0 + tpe - 1) / tpe : 0;
  auto total = [&](double2 v) {  // CTA sum, broadcast to every thread
    v = warpSum(v);
    if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double2 t = scratch[0];
      for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) t = cadd(t, scratch[k]);
      bcast = t;
    }
    __syncthreads();
    const double2 r = bcast;
    __syncthreads();
    return r;
  };
  constexpr int U = 4;
  double2 acc = make_double2(0.0, 0.0);
  for (int it = 0; it < nIter; ++it) {
    const long long qq = q0 + it * qStep;
    double2 wv = A.w[qq];
    if (A.dinv) wv = cmul(wv, A.dinv[s0 + it * sStep]);
    A.w[qq] = wv;
    cfma_conj(acc, A.V[qq], wv);
  }
  double2 h = total(acc);
  for (int i = 0; i <= j; ++i) {
    if (threadIdx.x == 0) hcol[i] = h;
    const double2* vi = A.V + static_cast<long long>(i) * nall;
    const double2* vn = A.V + static_cast<long long>(i + 1) * nall;
    acc = make_double2(0.0, 0.0);
    int it = 0;
    for (; it + U <= nIter; it += U) {
      double2 wv[U], v0[U], v1[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long qq = q0 + (it + u) * qStep;
        wv[u] = A.w[qq];
        v0[u] = vi[qq];
        v1[u] = i < j ? vn[qq] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        wv[u] = csub(wv[u], cmul(h, v0[u]));
        A.w[q0 + (it + u) * qStep] = wv[u];
        if (i < j)
          cfma_conj(acc, v1[u], wv[u]);
        else
          acc.x += wv[u].x * wv[u].x + wv[u].y * wv[u].y;
      }
    }
    for (; it < nIter; ++it) {
      const long long qq = q0 + it * qStep;
      const double2 wv = csub(A.w[qq], cmul(h, vi[qq]));
      A.w[qq] = wv;
      if (i < j)
        cfma_conj(acc, vn[qq], wv);
      else
        acc.x += wv.x * wv.x + wv.y * wv.y;
    }
    h = total(acc);
  }
  const double hn = sqrt(h.x);
  if (hn > 0.0) {
    double2* vout = A.V + static_cast<long long>(j + 1) * nall;
    for (int it = 0; it < nIter; ++it) {
      const long long qq = q0 + it * qStep;
      const double2 wv = A.w[qq];
      vout[qq] = make_double2(wv.x / hn, wv.y / hn);
    }
  }
  givensStep(A, col, j, hn, hcol, sh);
}

// ---------------------------------------------------------------------------
// Column-blocked GMRES kernels: many columns (C3) and the multi-GPU solve.
// Grids are (element blocks) x (columns), one warp per element with the m
// basis values lane-strided in registers (KPL = ceil(m/32) <= 8). Every
// reduction is two-stage and fixed-order: per-CTA partials
// part[col][slot][blk], then colReduce sums them per (slot, col) into
// tot[slot][col] -- the contiguous array a multi-GPU solve all-reduces
// (ncclAllReduce, the only collective of the solve) before the consumers
// read it. Low-synchronisation MGS (the arnoldiLS recurrence,
// gmres_dev.cuh) batched over the columns:
//   lsColsDots    c_k = <v_k, M w> (slot k), S_jk = <v_j, v_k> (slot j+1+k)
//   lsColsSolve   CTA per column: h = (I + L)^{-1} c (forward substitution)
//   lsColsUpdate  w' = M w - V h, ||w'||^2 partials
//   lsColsFinish  v_{j+1} = w' / ||w'||, Givens (first CTA of each column)
// Two passes over the basis per step; the per-projection sweep reads it j+1
// times and rewrites w each time.
struct ColsLS {
  double2* part;  // [ncols][2*(restart+1)][nblk]
  double2* tot;   // [2*(restart+1)][ncols]
  double2* S;     // [ncols][restart+1][restart+1], S(i,k) = <v_i, v_k>, k < i
  double2* h;     // [ncols][restart+1]
  int* run;       // [ncols] column runs this step / cycle
  int nblk;
};
constexpr int kColsElems = kWarps;  // elements per CTA, one per warp

__device__ __forceinline__ long long colsPart(const GmresArgs& A, const ColsLS& L, int col, int slot) {
  return (static_cast<long long>(col) * 2 * (A.restart + 1) + slot) * L.nblk + blockIdx.x;
}

// CTA sum of a per-warp value in fixed order, written as partial `slot`.
__device__ __forceinline__ void colsBlockPartial(const GmresArgs& A, const ColsLS& L, int col, int slot, double2 v,
                                                 double2* scratch) {
  v = warpSum(v);
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = scratch[0];
    for (int q = 1; q < kWarps; ++q) t = cadd(t, scratch[q]);
    L.part[colsPart(A, L, col, slot)] = t;
  }
}

// tot[slot][col] = sum_blk part[col][slot][blk], slots [0, nslots): one warp
// per (slot, col), lanes over the blocks, fixed-order butterfly.
__global__ void colReduce(GmresArgs A, ColsLS L, int nslots) {
  const int col = blockIdx.y;
  const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (slot >= nslots) return;
  const int lane = threadIdx.x & 31;
  const double2* p = L.part + (static_cast<long long>(col) * 2 * (A.restart + 1) + slot) * L.nblk;
  double2 t = make_double2(0.0, 0.0);
  for (int b0 = lane; b0 < L.nblk; b0 += 256) {  // 8 loads in flight per lane, summed in block order
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = b0 + 32 * q < L.nblk ? p[b0 + 32 * q] : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 8; ++q) t = cadd(t, v[q]);
  }
  t = warpSum(t);
  if (lane == 0) L.tot[static_cast<long long>(slot) * A.ncols + col] = t;
}

// Element-wise passes of init / cycle start, partial |.|^2 in slot 0:
//   0  |b|^2                         (gmresInit)
//   1  w = r = b - A x, |r|^2         (columns not done)
//   2  v_0 = z = M r, |z|^2           (columns with run = 1)
//   3  v_0 /= beta                    (run = 1, beta = sqrt(tot[0][col]) > 0)
template <int KPL>
__global__ void __launch_bounds__(kThreads) colsVecPass(GmresArgs A, ColsLS L, int mode) {
  __shared__ double2 scratch[kWarps];
  const int col = blockIdx.y;
  if (mode == 1 && A.st[col].done) return;
  if ((mode == 2 || mode == 3) && !L.run[col]) return;
  double beta = 1.0;
  if (mode == 3) {
    beta = sqrt(L.tot[col].x);
    if (beta == 0.0) return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, m = A.m;
  const int e = blockIdx.x * kColsElems + warp;
  const long long base = (static_cast<long long>(e) * A.ncols + col) * m;
  double2 acc = make_double2(0.0, 0.0);
  if (e < A.ne) {
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int a = lane + 32 * k;
      if (a >= m) continue;
      const long long q = base + a;
      double2 v;
      if (mode == 0) {
        v = A.b[q];
      } else if (mode == 1) {
        v = csub(A.b[q], A.ax[q]);
        A.w[q] = v;
      } else if (mode == 2) {
        v = A.w[q];
        if (A.dinv) v = cmul(v, A.dinv[static_cast<long long>(e) * m + a]);
        A.V[q] = v;
      } else {
        const double2 z = A.V[q];
        A.V[q] = make_double2(z.x / beta, z.y / beta);
        continue;
      }
      acc.x += v.x * v.x + v.y * v.y;
    }
  }
  if (mode != 3) colsBlockPartial(A, L, col, 0, acc, scratch);
}

// Per-column state transitions (one thread per column) on the totals:
//   0  after |b|^2: gmresInit's state
//   1  after |r|^2: restart residual test (linsolve.cpp:446-452), run flag
//   2  after |z|^2: beta, g (linsolve.cpp:453-461); run = beta > 0
__global__ void colsState(GmresArgs A, ColsLS L, int phase) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= A.ncols) return;
  GmresState& st = A.st[col];
  const double t = L.tot[col].x;
  if (phase == 0) {
    st.bnorm = sqrt(t);
    st.beta = st.beta0 = st.residual = 0.0;
    st.iterations = st.ncount = st.histLen = 0;
    st.stopInner = 1;
    st.cycleActive = 0;
    st.done = st.bnorm == 0.0 ? 1 : 0;
    st.converged = st.done;
    return;
  }
  if (phase == 1) {
    if (st.done) {
      L.run[col] = 0;
      return;
    }
    const double res = sqrt(t) / st.bnorm;
    int decision = 0;
    if (res < A.tol)
      decision = 1;
    else if (st.iterations >= A.maxIter)
      decision = 2;
    st.residual = res;
    pushHist(A, col, decision == 2 ? 2.0 : 0.0, res);
    if (decision != 0) {
      st.done = 1;
      st.converged = decision == 1 ? 1 : 0;
      st.cycleActive = 0;
      st.stopInner = 1;
    }
    L.run[col] = decision == 0 ? 1 : 0;
    return;
  }
  if (!L.run[col]) return;
  const double beta = sqrt(t);
  if (beta == 0.0) {
    st.done = 1;
    st.converged = 1;
    st.cycleActive = 0;
    st.stopInner = 1;
    L.run[col] = 0;
    return;
  }
  st.beta = beta;
  if (st.beta0 == 0.0) st.beta0 = beta;
  st.ncount = 0;
  st.stopInner = 0;
  st.cycleActive = 1;
  double2* g = A.g + static_cast<long long>(col) * (A.restart + 1);
  for (int k = 0; k <= A.restart; ++k) g[k] = make_double2(0.0, 0.0);
  g[0] = make_double2(beta, 0.0);
}

// Snapshot of "column runs this Arnoldi step" (the Givens step of
// lsColsFinish may stop a column while other CTAs of it still work).
__global__ void colsRunFlags(GmresArgs A, ColsLS L) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= A.ncols) return;
  const GmresState st = A.st[col];
  L.run[col] = st.cycleActive && !st.stopInner;
}

template <int KPL>
__global__ void __launch_bounds__(kThreads) lsColsDots(GmresArgs A, ColsLS L) {
  __shared__ double2 red[kWarps][2 * (RMAX + 1)];
  const int col = blockIdx.y;
  if (!L.run[col]) return;
  const int j = A.j, m = A.m;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * kColsElems + warp;
  const bool ev = e < A.ne;
  const long long nall = static_cast<long long>(A.ne) * m * A.ncols;
  const long long base = (static_cast<long long>(e) * A.ncols + col) * m;
  double2 w[KPL], vj[KPL];
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int a = lane + 32 * k;
    w[k] = vj[k] = make_double2(0.0, 0.0);
    if (ev && a < m) {
      double2 wv = A.w[base + a];
      if (A.dinv) wv = cmul(wv, A.dinv[static_cast<long long>(e) * m + a]);
      w[k] = wv;
      vj[k] = A.V[static_cast<long long>(j) * nall + base + a];
    }
  }
  for (int kk = 0; kk <= j; kk += 2) {
    const bool two = kk + 1 <= j;
    double2 v0[KPL], v1[KPL];
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int a = lane + 32 * k;
      const bool ok = ev && a < m;
      v0[k] = ok ? A.V[static_cast<long long>(kk) * nall + base + a] : make_double2(0.0, 0.0);
      v1[k] = ok && two ? A.V[static_cast<long long>(kk + 1) * nall + base + a] : make_double2(0.0, 0.0);
    }
    double2 c0 = make_double2(0.0, 0.0), c1 = c0, s0 = c0, s1 = c0;
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      cfma_conj(c0, v0[k], w[k]);
      cfma_conj(c1, v1[k], w[k]);
      cfma_conj(s0, vj[k], v0[k]);
      cfma_conj(s1, vj[k], v1[k]);
    }
    c0 = warpSum(c0);
    c1 = warpSum(c1);
    s0 = warpSum(s0);
    s1 = warpSum(s1);
    if (lane == 0) {
      red[warp][kk] = c0;
      if (kk < j) red[warp][j + 1 + kk] = s0;
      if (two) {
        red[warp][kk + 1] = c1;
        if (kk + 1 < j) red[warp][j + 2 + kk] = s1;
      }
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 2 * j + 1; d += blockDim.x) {
    double2 t = red[0][d];
    for (int q = 1; q < kWarps; ++q) t = cadd(t, red[q][d]);
    L.part[colsPart(A, L, col, d)] = t;
  }
}

// Dynamic shared memory: cv[RMAX+1] + packed strictly-lower rows of L.
__global__ void __launch_bounds__(kThreads) lsColsSolve(GmresArgs A, ColsLS L) {
  extern __shared__ double2 shs[];
  const int col = blockIdx.x;
  if (!L.run[col]) return;
  const int j = A.j, lds = A.restart + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* cv = shs;
  double2* sL = shs + RMAX + 1;  // row i (1..j) at i*(i-1)/2
  double2* S = L.S + static_cast<long long>(col) * lds * lds;
  for (int d = threadIdx.x; d < 2 * j + 1; d += blockDim.x) {
    const double2 t = L.tot[static_cast<long long>(d) * A.ncols + col];
    if (d <= j) {
      cv[d] = t;
    } else {
      const int k = d - j - 1;
      S[static_cast<long long>(j) * lds + k] = t;
      sL[j * (j - 1) / 2 + k] = t;
    }
  }
  for (int i = 1 + warp; i < j; i += kWarps)
    for (int k = lane; k < i; k += 32) sL[i * (i - 1) / 2 + k] = S[static_cast<long long>(i) * lds + k];
  __syncthreads();
  if (warp == 0) {
    constexpr int RPL = (RMAX + 31) / 32 + 1;
    double2 hv[RPL];
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int i = lane + 32 * t;
      hv[t] = i <= j ? cv[i] : make_double2(0.0, 0.0);
    }
    for (int k = 0; k < j; ++k) {
      double2 hk = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < RPL; ++t)
        if (t == (k >> 5)) hk = hv[t];
      hk = shfl2(hk, k & 31);
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        if (i > k && i <= j) hv[t] = csub(hv[t], cmul(sL[i * (i - 1) / 2 + k], hk));
      }
    }
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int i = lane + 32 * t;
      if (i <= j) L.h[static_cast<long long>(col) * lds + i] = hv[t];
    }
  }
}

template <int KPL>
__global__ void __launch_bounds__(kThreads) lsColsUpdate(GmresArgs A, ColsLS L) {
  __shared__ double2 hs[RMAX + 1];
  __shared__ double2 scratch[kWarps];
  const int col = blockIdx.y;
  if (!L.run[col]) return;
  const int j = A.j, m = A.m, lds = A.restart + 1;
  for (int i = threadIdx.x; i <= j; i += blockDim.x) hs[i] = L.h[static_cast<long long>(col) * lds + i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int e = blockIdx.x * kColsElems + warp;
  const bool ev = e < A.ne;
  const long long nall = static_cast<long long>(A.ne) * m * A.ncols;
  const long long base = (static_cast<long long>(e) * A.ncols + col) * m;
  double2 w[KPL];
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int a = lane + 32 * k;
    w[k] = make_double2(0.0, 0.0);
    if (ev && a < m) {
      double2 wv = A.w[base + a];
      if (A.dinv) wv = cmul(wv, A.dinv[static_cast<long long>(e) * m + a]);
      w[k] = wv;
    }
  }
  int kk = 0;
  for (; kk + 2 <= j + 1; kk += 2) {
    double2 v0[KPL], v1[KPL];
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int a = lane + 32 * k;
      const bool ok = ev && a < m;
      v0[k] = ok ? A.V[static_cast<long long>(kk) * nall + base + a] : make_double2(0.0, 0.0);
      v1[k] = ok ? A.V[static_cast<long long>(kk + 1) * nall + base + a] : make_double2(0.0, 0.0);
    }
    const double2 h0 = hs[kk], h1 = hs[kk + 1];
#pragma unroll
    for (int k = 0; k < KPL; ++k) w[k] = csub(csub(w[k], cmul(h0, v0[k])), cmul(h1, v1[k]));
  }
  if (kk <= j) {
    const double2 h0 = hs[kk];
#pragma unroll
    for (int k = 0; k < KPL; ++k) {
      const int a = lane + 32 * k;
      if (ev && a < m) w[k] = csub(w[k], cmul(h0, A.V[static_cast<long long>(kk) * nall + base + a]));
    }
  }
  double2 acc = make_double2(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < KPL; ++k) {
    const int a = lane + 32 * k;
    if (ev && a < m) {
      A.w[base + a] = w[k];
      acc.x += w[k].x * w[k].x + w[k].y * w[k].y;
    }
  }
  colsBlockPartial(A, L, col, 0, acc, scratch);
}

__global__ void __launch_bounds__(kThreads) lsColsFinish(GmresArgs A, ColsLS L) {
  __shared__ double2 hcol[RMAX + 2];
  __shared__ double2 sh[3 * RMAX + 4];
  const int col = blockIdx.y;
  if (!L.run[col]) return;
  const int j = A.j, m = A.m, lds = A.restart + 1;
  const double hn = sqrt(L.tot[col].x);
  if (hn > 0.0) {
    const long long nall = static_cast<long long>(A.ne) * m * A.ncols;
    const int e0 = blockIdx.x * kColsElems;
    const int e1 = min(A.ne, e0 + kColsElems);
    for (int q = threadIdx.x; q < (e1 - e0) * m; q += blockDim.x) {
      const int e = e0 + q / m, a = q % m;
      const long long idx = (static_cast<long long>(e) * A.ncols + col) * m + a;
      const double2 wv = A.w[idx];
      A.V[static_cast<long long>(j + 1) * nall + idx] = make_double2(wv.x / hn, wv.y / hn);
    }
  }
  if (blockIdx.x == 0) {
    for (int i = threadIdx.x; i <= j; i += blockDim.x) hcol[i] = L.h[static_cast<long long>(col) * lds + i];
    givensStep(A, col, j, hn, hcol, sh);
  }
}

size_t lsColsSolveSmem(int restart) {
  return sizeof(double2) * (RMAX + 1 + static_cast<size_t>(restart) * (restart + 1) / 2);
}

// Host side of the column-blocked solve: `reduce(nslots)` = colReduce, then
// (multi-GPU) the all-reduce of tot[0 .. nslots*ncols).
struct ColsRunner {
  GmresArgs* A;
  ColsLS L;
  int kpl;
  size_t solveSmem;
  Ctx* c;
  cudaStream_t s;

  void reduce(int nslots) {
    colReduce<<<dim3((nslots + 7) / 8, A->ncols), 256, 0, s>>>(*A, L, nslots);
    TBT_CUDA_CHECK(cudaGetLastError());
    if (c->dist) c->comm->allReduceSum(reinterpret_cast<double*>(L.tot), static_cast<size_t>(nslots) * A->ncols * 2, s);
  }
  template <int K>
  void vecPass(int mode) {
    colsVecPass<K><<<dim3(L.nblk, A->ncols), kThreads, 0, s>>>(*A, L, mode);
  }
  void vec(int mode) {
    switch (kpl) {
      case 1: vecPass<1>(mode); break;
      case 2: vecPass<2>(mode); break;
      case 4: vecPass<4>(mode); break;
      default: vecPass<8>(mode); break;
    }
    TBT_CUDA_CHECK(cudaGetLastError());
  }
  void state(int phase) {
    colsState<<<(A->ncols + 127) / 128, 128, 0, s>>>(*A, L, phase);
    TBT_CUDA_CHECK(cudaGetLastError());
  }
  void init() {
    vec(0);
    reduce(1);
    state(0);
  }
  void cycleStart() {
    vec(1);
    reduce(1);
    state(1);
    vec(2);
    reduce(1);
    state(2);
    vec(3);
  }
  template <int K>
  void arnoldiK() {
    const dim3 grid(L.nblk, A->ncols);
    colsRunFlags<<<(A->ncols + 127) / 128, 128, 0, s>>>(*A, L);
    lsColsDots<K><<<grid, kThreads, 0, s>>>(*A, L);
    reduce(2 * A->j + 1);
    lsColsSolve<<<A->ncols, kThreads, solveSmem, s>>>(*A, L);
    lsColsUpdate<K><<<grid, kThreads, 0, s>>>(*A, L);
    reduce(1);
    lsColsFinish<<<grid, kThreads, 0, s>>>(*A, L);
    TBT_CUDA_CHECK(cudaGetLastError());
  }
  void arnoldi() {
    switch (kpl) {
      case 1: arnoldiK<1>(); break;
      case 2: arnoldiK<2>(); break;
      case 4: arnoldiK<4>(); break;
      default: arnoldiK<8>(); break;
    }
  }
};

// One Arnoldi step j for every running column (any column count / size).
__global__ void __launch_bounds__(kThreads) gmresArnoldi(GmresArgs A) {
  __shared__ double2 scratch[kWarps];
  __shared__ double2 sh[3 * RMAX + 4];
  extern __shared__ int sFlag[];
  const int j = A.j;
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long nall = slots * A.ncols;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long s0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int ldh = A.restart + 1;
  for (int col = 0; col < A.ncols; ++col) {
    const bool run = A.st[col].cycleActive && !A.st[col].stopInner;
    if (threadIdx.x == 0) sFlag[col] = run ? 1 : 0;
    double2 acc = make_double2(0.0, 0.0);
    if (run)
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        double2 wv = A.w[q];
        if (A.dinv) wv = cmul(wv, A.dinv[s]);
        A.w[q] = wv;
        cfma_conj(acc, A.V[q], wv);
      }
    blockPartial(acc, scratch, partSlot(A, 0, col));
    __syncthreads();
  }
  gridBarrier(A.bar);
  for (int i = 0; i <= j; ++i) {
    for (int col = 0; col < A.ncols; ++col) {
      if (!sFlag[col]) continue;
      const double2 h = warpTotal(partSlot(A, i, col));
      if (blockIdx.x == 0 && threadIdx.x == 0) A.H[static_cast<long long>(col) * ldh * A.restart + i + j * ldh] = h;
      const double2* vi = A.V + static_cast<long long>(i) * nall;
      const double2* vn = A.V + static_cast<long long>(i + 1) * nall;
      double2 acc = make_double2(0.0, 0.0);
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        const double2 wv = csub(A.w[q], cmul(h, vi[q]));
        A.w[q] = wv;
        if (i < j)
          cfma_conj(acc, vn[q], wv);
        else
          acc.x += wv.x * wv.x + wv.y * wv.y;
      }
      blockPartial(acc, scratch, partSlot(A, i + 1, col));
      __syncthreads();
    }
    gridBarrier(A.bar);
  }
  for (int col = 0; col < A.ncols; ++col) {
    if (!sFlag[col]) continue;
    const double hn = sqrt(warpTotal(partSlot(A, j + 1, col)).x);
    if (hn > 0.0) {
      double2* vout = A.V + static_cast<long long>(j + 1) * nall;
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        const double2 wv = A.w[q];
        vout[q] = make_double2(wv.x / hn, wv.y / hn);
      }
    }
    // Columns are spread over CTAs for the (sequential) Givens sweep; H(.,j)
    // was written by CTA 0 before the last barrier.
    if (col % static_cast<int>(gridDim.x) == static_cast<int>(blockIdx.x)) givensStep(A, col, j, hn, nullptr, sh);
  }
}

// Back substitution and x += sum_i y_i v_i (linsolve.cpp:503-510). One CTA
// per column stages the triangle of H in shared memory; warp 0 then solves
// with its rows in registers.
__global__ void __launch_bounds__(kThreads) gmresUpdate(GmresArgs A) {
  extern __shared__ double2 shH[];  // [(restart+1)*restart]
  const int ldh = A.restart + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int RPL = RMAX / 32;  // rows per lane
  for (int col = blockIdx.x; col < A.ncols; col += gridDim.x) {
    const GmresState st = A.st[col];
    if (!st.cycleActive) continue;
    const double2* H = A.H + static_cast<long long>(col) * ldh * A.restart;
    const double2* g = A.g + static_cast<long long>(col) * (A.restart + 1);
    double2* y = A.ycoef + static_cast<long long>(col) * A.restart;
    const int nc = st.ncount;
    __syncthreads();
    for (int q = threadIdx.x; q < ldh * nc; q += blockDim.x) shH[q] = H[q];
    __syncthreads();
    if (warp == 0) {
      double2 s[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int i = lane + 32 * t;
        s[t] = i < nc ? g[i] : make_double2(0.0, 0.0);
      }
      for (int i0 = nc - 1; i0 >= 0; --i0) {
        const int owner = i0 & 31, tt = i0 >> 5;
        double2 mine = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < RPL; ++t)
          if (t == tt) mine = s[t];
        double2 yi = cdiv(mine, shH[i0 + i0 * ldh]);
        yi = shfl2(yi, owner);
        if (lane == owner) y[i0] = yi;
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int i = lane + 32 * t;
          if (i < i0) s[t] = csub(s[t], cmul(shH[i + i0 * ldh], yi));
        }
      }
    }
  }
  gridBarrier(A.bar);
  // x += V y over all (slot, column) entries at once (internal layout
  // [e][col][a]); y and the column state come through L1.
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long nall = slots * A.ncols;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  if (A.ncols == 1) {
    // One column: y in shared memory, four slots per thread with eight basis
    // loads each in flight (per slot the order over i is unchanged).
    if (!A.st[0].cycleActive) return;
    const int nc = A.st[0].ncount;
    __syncthreads();
    for (int i = threadIdx.x; i < nc; i += blockDim.x) shH[i] = __ldcg(A.ycoef + i);
    __syncthreads();
    constexpr int QT = 4;  // slots per thread per trip: 32 basis loads in flight
    for (long long qa = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; qa < nall;
         qa += QT * stride) {
      long long qs[QT];
      double2 xv[QT];
#pragma unroll
      for (int t = 0; t < QT; ++t) {
        const long long q = qa + t * stride;
        qs[t] = q < nall ? q : qa;
        xv[t] = A.x[qs[t]];
      }
      int i = 0;
      for (; i + 8 <= nc; i += 8) {
        double2 v[8][QT];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int t = 0; t < QT; ++t) v[u][t] = A.V[static_cast<long long>(i + u) * nall + qs[t]];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int t = 0; t < QT; ++t) xv[t] = cadd(xv[t], cmul(shH[i + u], v[u][t]));
      }
      for (; i < nc; ++i)
#pragma unroll
        for (int t = 0; t < QT; ++t) xv[t] = cadd(xv[t], cmul(shH[i], A.V[static_cast<long long>(i) * nall + qs[t]]));
#pragma unroll
      for (int t = 0; t < QT; ++t)
        if (qa + t * stride < nall) A.x[qa + t * stride] = xv[t];
    }
    return;
  }
  for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < nall; q += stride) {
    const int col = static_cast<int>((q / A.m) % A.ncols);
    if (!A.st[col].cycleActive) continue;
    const int nc = A.st[col].ncount;
    const double2* sy = A.ycoef + static_cast<long long>(col) * A.restart;
    double2 xv = A.x[q];
    int i = 0;
    for (; i + 8 <= nc; i += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = A.V[static_cast<long long>(i + u) * nall + q];
#pragma unroll
      for (int u = 0; u < 8; ++u) xv = cadd(xv, cmul(__ldcg(sy + i + u), v[u]));
    }
    for (; i < nc; ++i) xv = cadd(xv, cmul(__ldcg(sy + i), A.V[static_cast<long long>(i) * nall + q]));
    A.x[q] = xv;
  }
}

void coopLaunch(const void* fn, int grid, size_t smem, GmresArgs& args, cudaStream_t s) {
  // Same (maximal) shared-memory carveout as the persistent apply kernel, so
  // alternating launches do not reconfigure L1/shared memory on every SM.
  // Per (kernel, device), under a lock: contexts on other threads / GPUs.
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> configured;
  {
    int dev = 0;
    TBT_CUDA_CHECK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(fn, dev);
    if (std::find(configured.begin(), configured.end(), key) == configured.end()) {
      TBT_CUDA_CHECK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          cudaSharedmemCarveoutMaxShared));
      configured.push_back(key);
    }
  }
  void* params[] = {&args};
  TBT_CUDA_CHECK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), params, smem, s));
}

}  // namespace

// Host driver (iterativeSolve, linsolve.cpp:551-593, columns in lockstep).
void gmresSolve(Ctx& c, const double2* b, double2* x, int ncols, const tbt_gmres_opts& o, bool useAOnly,
                std::vector<GmresState>& out, std::vector<double>& hist, int& matvecs) {
  const int R = o.restart;
  TBT_USER_CHECK(R <= RMAX, "tbt_gmres: restart above " + std::to_string(RMAX));
  struct SolveScope {  // applies of this solve alternate their pair order (matvec_persistent.cu)
    Ctx& c;
    explicit SolveScope(Ctx& cc) : c(cc) { c.inSolve = true; }
    ~SolveScope() { c.inSolve = false; }
  } scope(c);
  // Multi-GPU: this rank's element-row slab (dist.cu); every reduction of
  // the solve is all-reduced, so all ranks take identical decisions.
  // Margin parts (full operator): the neM pseudo-elements join the vector.
  const bool withMargin = c.margin && !useAOnly;
  const int neLoc = c.dist ? c.myRows * c.nx : c.ne + (withMargin ? c.neM : 0);
  const long long nloc = static_cast<long long>(neLoc) * c.m;
  const long long nall = nloc * ncols;
  cudaStream_t s = c.stream;
  const int sms = smCount(c.device);
  // One CTA per SM: always co-resident, as the grid barrier requires
  // (cudaLaunchCooperativeKernel rejects a grid that is not).
  const int grid = sms;
  // Column-blocked kernels + all-reduces for the multi-GPU solve (always
  // low-synchronisation MGS there) and for many columns.
  // One column: the LS step fused into the persistent apply for small
  // vectors (C2: per-CTA row chunk in shared memory, no extra launches);
  // from C4 up the column-blocked kernels are faster (measured: C4 0.553 vs
  // 0.573 ms per iteration, C5 4.6 vs 5.2).
  const long long lsChunk = (nloc + grid - 1) / grid;
  // One column, large vectors (row chunk beyond shared memory, C4 / C5):
  // the streamed low-sync step, two launches per iteration (apply + LS).
  const bool bigLS = !c.dist && !withMargin && o.orthog == 1 && ncols == 1 && lsChunk > 2048 && !c.forceCols;
  const bool colsLS = !bigLS && (c.dist || withMargin ||
                                 (o.orthog == 1 && c.m <= 256 && (ncols > 1 || lsChunk > 2048 || c.forceCols)));
  TBT_USER_CHECK(!withMargin || c.m <= 256, "tbt_gmres: margin solves support m <= 256");
  TBT_USER_CHECK(!c.dist || c.m <= 256, "tbt_gmres: distributed solve supports m <= 256");
  const bool fast = !colsLS && ncols == 1 && nloc <= static_cast<long long>(grid) * kThreads * FAST_K;
  const bool lowSync = !colsLS && !bigLS && o.orthog == 1 && ncols == 1 && lsChunk <= 2048;
  const int colsKpl = c.m <= 32 ? 1 : c.m <= 64 ? 2 : c.m <= 128 ? 4 : 8;
  const size_t colsSolveSmem = lsColsSolveSmem(R);
  const size_t lsSmem = static_cast<size_t>(arnoldiLSSmem(lsChunk, R)) * sizeof(double2);

  GmresArgs A{};
  A.ncols = ncols;
  A.restart = R;
  A.maxIter = o.max_iter;
  A.histCap = std::max(0, o.hist_cap);
  A.precondition = o.precondition;
  A.tol = o.tol;
  A.ne = neLoc;
  A.m = c.m;
  // Device workspace, cached in the context across solves of the same shape
  // (allocation and graph instantiation are per-solve costs otherwise).
  GmresWs& W = *gmresWorkspace(c);
  const long long key[6] = {ncols, R, nall, std::max(1, A.histCap), grid, colsLS ? 1 : 0};
  if (std::memcmp(key, W.key, sizeof(key)) != 0) {
    W.release();
    auto dalloc = [&](size_t bytes) {
      void* p = nullptr;
      TBT_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
      W.allocs.push_back(p);
      return p;
    };
    W.st = static_cast<GmresState*>(dalloc(sizeof(GmresState) * ncols));
    W.H = static_cast<double2*>(dalloc(sizeof(double2) * ncols * (R + 1) * R));
    W.g = static_cast<double2*>(dalloc(sizeof(double2) * ncols * (R + 1)));
    W.cs = static_cast<double2*>(dalloc(sizeof(double2) * ncols * R));
    W.sn = static_cast<double2*>(dalloc(sizeof(double2) * ncols * R));
    W.ycoef = static_cast<double2*>(dalloc(sizeof(double2) * ncols * R));
    W.hist = static_cast<double*>(dalloc(sizeof(double) * 2 * ncols * std::max(1, A.histCap)));
    W.partial = static_cast<double2*>(dalloc(sizeof(double2) * 2 * ncols * grid));
    W.bar = static_cast<unsigned long long*>(dalloc(sizeof(unsigned long long)));
    W.ax = static_cast<double2*>(dalloc(sizeof(double2) * nall));
    W.w = static_cast<double2*>(dalloc(sizeof(double2) * nall));
    W.V = static_cast<double2*>(dalloc(sizeof(double2) * nall * (R + 1)));
    W.lsS = static_cast<double2*>(dalloc(sizeof(double2) * (R + 1) * (R + 1)));
    W.lsDots = static_cast<double2*>(dalloc(sizeof(double2) * 2 * (R + 1)));
    W.lsPart = static_cast<double2*>(dalloc(sizeof(double2) * 2 * (R + 1) * grid));
    if (colsLS) {
      const long long nblk = (neLoc + kColsElems - 1) / kColsElems;
      W.clPart = static_cast<double2*>(dalloc(sizeof(double2) * ncols * 2 * (R + 1) * nblk));
      W.clTot = static_cast<double2*>(dalloc(sizeof(double2) * ncols * 2 * (R + 1)));
      W.clS = static_cast<double2*>(dalloc(sizeof(double2) * ncols * (R + 1) * (R + 1)));
      W.clH = static_cast<double2*>(dalloc(sizeof(double2) * ncols * (R + 1)));
      W.clRun = static_cast<int*>(dalloc(sizeof(int) * ncols));
    }
    TBT_CUDA_CHECK(cudaMemsetAsync(W.bar, 0, sizeof(unsigned long long), s));
    std::memcpy(W.key, key, sizeof(key));
  }
  A.st = W.st;
  A.H = W.H;
  A.g = W.g;
  A.cs = W.cs;
  A.sn = W.sn;
  A.ycoef = W.ycoef;
  A.hist = W.hist;
  A.partial = W.partial;
  A.bar = W.bar;
  A.ax = W.ax;
  A.w = W.w;
  A.V = W.V;
  A.b = b;
  A.x = x;
  double2* lsS = W.lsS;
  double2* lsDots = W.lsDots;
  double2* lsPart = W.lsPart;
  ColsRunner cols{&A, ColsLS{W.clPart, W.clTot, W.clS, W.clH, W.clRun, (neLoc + kColsElems - 1) / kColsElems},
                  colsKpl, colsSolveSmem, &c, s};
  try {
    if (colsLS && colsSolveSmem > 48 * 1024)
      TBT_CUDA_CHECK(cudaFuncSetAttribute(lsColsSolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(colsSolveSmem)));
    if (bigLS)
      TBT_CUDA_CHECK(cudaFuncSetAttribute(gmresArnoldiLSBig, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(lsBigSmem(R))));
    if (lowSync) {
      TBT_CUDA_CHECK(cudaFuncSetAttribute(gmresArnoldiLS, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(lsSmem)));
      TBT_CUDA_CHECK(cudaFuncSetAttribute(gmresArnoldiLS, cudaFuncAttributePreferredSharedMemoryCarveout,
                                          cudaSharedmemCarveoutMaxShared));
    }
    TBT_CUDA_CHECK(cudaMemsetAsync(A.V, 0, sizeof(double2) * nall * (R + 1), s));
    TBT_CUDA_CHECK(cudaMemsetAsync(A.H, 0, sizeof(double2) * ncols * (R + 1) * R, s));
    TBT_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double2) * nall, s));
    A.dinv = o.precondition ? (useAOnly ? c.dDiagInvA : c.dDiagInv) : nullptr;
    static const bool lsProf = getenv("TBT_LSPROF") != nullptr;  // debug: LS section timing (CTA 0)
    A.prof = lsProf ? c.dPhaseNs + 24 : nullptr;
    if (lsProf) memsetSync(c.dPhaseNs + 24, 0, 5 * sizeof(unsigned long long), s);
    if (A.dinv && c.dist) A.dinv += static_cast<long long>(c.myRow0) * c.nx * c.m;
    const size_t smem = sizeof(int) * ncols;

    matvecs = 0;
    if (ncols == 1 && !withMargin && clusterSmallSupported(c, R)) {
      // Tiny operator: the whole solve in one cluster launch (cluster_small.cu).
      launchClusterGmres(c, A, !useAOnly);
      std::vector<GmresState> st(1);
      TBT_CUDA_CHECK(cudaMemcpyAsync(st.data(), A.st, sizeof(GmresState), cudaMemcpyDeviceToHost, s));
      hist.assign(static_cast<size_t>(2) * std::max(1, A.histCap), 0.0);
      if (A.histCap > 0)
        TBT_CUDA_CHECK(cudaMemcpyAsync(hist.data(), A.hist, sizeof(double) * 2 * A.histCap, cudaMemcpyDeviceToHost, s));
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));
      // matvecs: one per true-residual check (each restart and the final
      // one, counted by the kernel) + one per inner iteration.
      matvecs = st[0].checks + st[0].iterations;
      out = st;
      return;
    }
    if (colsLS)
      cols.init();
    else
      coopLaunch(reinterpret_cast<const void*>(gmresInit), grid, smem, A, s);
    std::vector<GmresState> st(ncols);
    auto pull = [&]() {
      TBT_CUDA_CHECK(cudaMemcpyAsync(st.data(), A.st, sizeof(GmresState) * ncols, cudaMemcpyDeviceToHost, s));
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));
    };
    auto arnoldi = [&](int j) {
      A.j = j;
      if (bigLS) {
        void* params[] = {&A, &lsS, &lsPart};
        TBT_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(gmresArnoldiLSBig), dim3(grid),
                                                   dim3(kThreads), params, lsBigSmem(R), s));
      } else if (lowSync) {
        void* params[] = {&A, &lsS, &lsDots, &lsPart};
        TBT_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(gmresArnoldiLS), dim3(grid),
                                                   dim3(kThreads), params, lsSmem, s));
      } else if (fast) {
        coopLaunch(reinterpret_cast<const void*>(gmresArnoldi1), grid, 0, A, s);
      } else if (colsLS) {
        cols.arnoldi();
      } else if (ncols > 1 && c.m <= kThreads) {
        gmresArnoldiCols<<<ncols, kThreads, 0, s>>>(A);
        TBT_CUDA_CHECK(cudaGetLastError());
      } else {
        coopLaunch(reinterpret_cast<const void*>(gmresArnoldi), grid, smem, A, s);
      }
    };
    // One inner iteration: the apply and the Arnoldi step, fused into the
    // persistent apply kernel when possible (one cooperative launch).
    const bool fuse = lowSync && !c.timeBinprod && !c.dist && !c.forceUnfused;
    // Single column: the whole inner loop of a cycle is one CUDA graph
    // (restart x [apply, Arnoldi]); every node turns into a no-op once the
    // column's inner loop stopped (device flag), so the host synchronises
    // once per restart cycle.
    const bool useGraph = ncols == 1 && !c.timeBinprod && !c.dist && !withMargin;
    // Fused nodes with lagged normalisation (matvec_persistent.cu LAGGED):
    // node j finishes column j-1 (norm, Givens step, stop decision) under
    // its own phase A1 and the nodes are serialised programmatically (PDL),
    // so a node's CTAs are placed as the previous node's exit; a last node
    // finishes column restart-1. TBT_GMRES=nolag keeps the unlagged nodes.
    static const bool noLagEnv = getenv("TBT_GMRES") && std::string(getenv("TBT_GMRES")) == "nolag";
    const bool lagged = useGraph && fuse && !noLagEnv && persistentLaggedFits(c, A);
    auto iteration = [&](int j) {
      A.j = j;
      if (fuse && launchPersistentApply(c, A.V + static_cast<long long>(j) * nall, A.w, !useAOnly, &A, lsS, lsDots,
                                        lsPart, lagged))
        return;
      applyOperator(c, A.V + static_cast<long long>(j) * nall, A.w, ncols, !useAOnly);
      arnoldi(j);
    };
    GmresArgs keyA = A;  // what the captured nodes bake in (b, x unused by them)
    keyA.b = nullptr;
    keyA.x = nullptr;
    keyA.j = 0;
    const int flags = (fuse ? 1 : 0) | (lowSync ? 2 : 0) | (fast ? 4 : 0) | (useAOnly ? 8 : 0) | (bigLS ? 16 : 0) |
                      (lagged ? 32 : 0) | (plainLaunchOk(c) ? 64 : 0);  // plain vs cooperative nodes
    if (useGraph && (!W.inner || std::memcmp(&keyA, &W.graphKey, sizeof(GmresArgs)) != 0 || W.graphFlags != flags)) {
      if (W.inner) cudaGraphExecDestroy(W.inner);
      W.inner = nullptr;
      c.skipFlag = &A.st[0].stopInner;
      // Plain (programmatically serialised) nodes need this context's
      // co-residency check: one cooperative apply of scratch first.
      if (lagged && !c.coopChecked) launchPersistentApply(c, A.V, A.w, false);
      cudaGraph_t gph;
      TBT_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        for (int j = 0; j < R; ++j) iteration(j);
        if (lagged) {
          gmresLaggedFinish<<<1, 32, 0, s>>>(A, R - 1, smCount(c.device));
          TBT_CUDA_CHECK(cudaGetLastError());
        }
      } catch (...) {
        cudaStreamEndCapture(s, &gph);
        c.skipFlag = nullptr;
        throw;
      }
      TBT_CUDA_CHECK(cudaStreamEndCapture(s, &gph));
      c.skipFlag = nullptr;
      const cudaError_t e = cudaGraphInstantiate(&W.inner, gph, 0);
      cudaGraphDestroy(gph);
      TBT_CUDA_CHECK(e);
      W.graphKey = keyA;
      W.graphFlags = flags;
    }
    cudaGraphExec_t inner = useGraph ? W.inner : nullptr;
    try {
      pull();
      bool open = !st[0].done;
      for (size_t k = 1; k < st.size(); ++k) open |= !st[k].done;
      while (open) {
        applyOperator(c, x, W.ax, ncols, !useAOnly);
        ++matvecs;
        if (colsLS)
          cols.cycleStart();
        else
          coopLaunch(reinterpret_cast<const void*>(gmresCycleStart), grid, smem, A, s);
        if (useGraph) {
          // The cycle start may have ended the solve (budget or tolerance
          // reached): then the 'restart' no-op nodes are not worth a launch.
          pull();
          if (st[0].cycleActive && !st[0].stopInner) TBT_CUDA_CHECK(cudaGraphLaunch(inner, s));
        } else {
          pull();
          bool anyRun = false;
          for (auto& v : st) anyRun |= (v.cycleActive && !v.stopInner);
          for (int j = 0; anyRun && j < R; ++j) {
            iteration(j);
            if ((j + 1) % 8 == 0 && j + 1 < R) {
              pull();
              bool more = false;
              for (auto& v : st) more |= (v.cycleActive && !v.stopInner);
              if (!more) break;
            }
          }
        }
        coopLaunch(reinterpret_cast<const void*>(gmresUpdate), grid, sizeof(double2) * (R + 1) * R, A, s);
        pull();
        open = false;
        for (auto& v : st) open |= !v.done;
      }
    } catch (...) {
      throw;
    }
    // Matvecs issued: one per cycle start plus one per inner iteration.
    {
      int it = 0;
      for (auto& v : st) it = std::max(it, v.iterations);
      matvecs += it;
    }
    out = st;
    if (lsProf) {
      unsigned long long ns[5];
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));
      TBT_CUDA_CHECK(cudaMemcpy(ns, c.dPhaseNs + 24, sizeof(ns), cudaMemcpyDeviceToHost));
      const double it = ns[4] > 0 ? static_cast<double>(ns[4]) : 1.0;
      fprintf(stderr, "LS step per iteration (us): dots %.2f reduce %.2f subst+update %.2f normalize+givens %.2f (%llu)\n",
              1e-3 * ns[0] / it, 1e-3 * ns[1] / it, 1e-3 * ns[2] / it, 1e-3 * ns[3] / it, ns[4]);
    }
    hist.assign(static_cast<size_t>(2) * ncols * std::max(1, A.histCap), 0.0);
    if (A.histCap > 0)
      TBT_CUDA_CHECK(cudaMemcpy(hist.data(), A.hist, sizeof(double) * 2 * ncols * A.histCap, cudaMemcpyDeviceToHost));
  } catch (...) {
    cudaStreamSynchronize(s);
    W.release();  // state unknown after a failure: rebuild next time
    throw;
  }
  cudaStreamSynchronize(s);
}

void freeGmresWorkspace(Ctx& c) {
  if (c.gmresWs) {
    c.gmresWs->release();
    if (c.gmresWs->bufB) cudaFree(c.gmresWs->bufB);
    if (c.gmresWs->bufX) cudaFree(c.gmresWs->bufX);
    delete c.gmresWs;
    c.gmresWs = nullptr;
  }
}

GmresWs* gmresWorkspace(Ctx& c) {
  if (!c.gmresWs) c.gmresWs = new GmresWs;
  return c.gmresWs;
}

void GmresWs::release() {
  if (inner) cudaGraphExecDestroy(inner);
  inner = nullptr;
  for (void* p : allocs) cudaFree(p);
  allocs.clear();
  std::memset(key, 0, sizeof(key));
}

}  // namespace tbt
