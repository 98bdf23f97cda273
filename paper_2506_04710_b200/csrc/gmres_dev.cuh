// Device-side GMRES pieces shared by gmres.cu and the fused apply+Arnoldi
// step of matvec_persistent.cu (see gmres.cu for the algorithm notes).
#pragma once

#include <cmath>
#include <vector>

#include "grid_sync.cuh"
#include "tbt_internal.cuh"

namespace tbt {

struct GmresArgs {
  int ncols, restart, maxIter, histCap, precondition;
  double tol;
  int ne, m;
  GmresState* st;
  double2* H;       // [ncols][(restart+1)*restart], H(i,j) at i + j*(restart+1)
  double2* g;       // [ncols][restart+1]
  double2* cs;      // [ncols][restart]
  double2* sn;      // [ncols][restart]
  double2* ycoef;   // [ncols][restart]
  double* hist;     // [ncols][histCap][2]
  double2* partial; // [2][ncols][grid]
  unsigned long long* bar;  // monotonic grid-barrier counter
  const double2* b;
  double2* x;
  const double2* ax;
  double2* w;
  double2* V;       // [restart+1][ne*ncols*m]
  const double2* dinv;  // [ne*m] or null
  int j;            // Arnoldi column of this launch
  unsigned long long* prof;  // optional (TBT_LSPROF): accumulated ns per LS section, CTA 0
};

// Device workspace of gmresSolve, cached in the context (gmres.cu).
struct GmresWs {
  long long key[6] = {0, 0, 0, 0, 0, 0};  // ncols, restart, n*ncols, hist cap, grid, column-blocked
  std::vector<void*> allocs;
  GmresState* st = nullptr;
  double2 *H = nullptr, *g = nullptr, *cs = nullptr, *sn = nullptr, *ycoef = nullptr;
  double* hist = nullptr;
  double2* partial = nullptr;
  unsigned long long* bar = nullptr;
  double2 *ax = nullptr, *w = nullptr, *V = nullptr;
  double2 *lsS = nullptr, *lsDots = nullptr, *lsPart = nullptr;
  double2 *clPart = nullptr, *clTot = nullptr, *clS = nullptr, *clH = nullptr;  // column-blocked solve
  int* clRun = nullptr;
  double2 *bufB = nullptr, *bufX = nullptr;  // tbt_gmres staging
  long long bufLen = 0;
  cudaGraphExec_t inner = nullptr;  // captured inner loop of a restart cycle
  GmresArgs graphKey{};
  int graphFlags = 0;
  void release();
};
GmresWs* gmresWorkspace(Ctx& c);
void launchClusterGmres(Ctx& c, const GmresArgs& A, bool withCorr);  // cluster_small.cu

namespace gmresdev {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int FAST_K = 8;  // slots per thread in the register-resident Arnoldi
constexpr int RMAX = 128;  // largest restart the staged Givens / solve support

__device__ __forceinline__ void gridBarrier(unsigned long long* bar) { gridBarrierMono(bar); }

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  v.x = __shfl_sync(0xffffffffu, v.x, src);
  v.y = __shfl_sync(0xffffffffu, v.y, src);
  return v;
}

// Butterfly sum: every lane ends with the same bits.
__device__ __forceinline__ double2 warpSum(double2 v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  return v;
}

// Per-CTA partial of v written to part[blockIdx.x] (thread 0).
__device__ __forceinline__ void blockPartial(double2 v, double2* scratch, double2* part) {
  v = warpSum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 s = scratch[0];
    for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) s = cadd(s, scratch[k]);
    part[blockIdx.x] = s;
  }
}

// Grid total of the partials, computed by each warp independently in a
// fixed order (bitwise identical in every warp and CTA).
__device__ __forceinline__ double2 warpTotalN(const double2* part, int G) {
  const int lane = threadIdx.x & 31;
  double2 s = make_double2(0.0, 0.0);
  for (int k0 = lane; k0 < G; k0 += 256) {  // up to 8 loads in flight per lane, summed in k order
    double2 v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) v[q] = k0 + 32 * q < G ? __ldcg(part + k0 + 32 * q) : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 8; ++q) s = cadd(s, v[q]);
  }
  return warpSum(s);
}
__device__ __forceinline__ double2 warpTotal(const double2* part) {
  return warpTotalN(part, static_cast<int>(gridDim.x));
}

// Partials of a launch with G CTAs (gridDim.x by default).
__device__ __forceinline__ double2* partSlotN(const GmresArgs& A, int phase, int col, int G) {
  return A.partial + (static_cast<long long>(phase & 1) * A.ncols + col) * G;
}
__device__ __forceinline__ double2* partSlot(const GmresArgs& A, int phase, int col) {
  return partSlotN(A, phase, col, static_cast<int>(gridDim.x));
}

__device__ __forceinline__ long long slotIndex(long long s, int col, int ncols, int m) {
  const long long e = s / m, a = s % m;
  return (e * ncols + col) * m + a;
}

__device__ inline void pushHist(const GmresArgs& A, int col, double kind, double v) {
  GmresState& st = A.st[col];
  if (st.histLen < A.histCap) {
    A.hist[(static_cast<long long>(col) * A.histCap + st.histLen) * 2] = kind;
    A.hist[(static_cast<long long>(col) * A.histCap + st.histLen) * 2 + 1] = v;
  }
  st.histLen++;
}

__device__ __forceinline__ double cabs2(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// Smith's complex division a / b.
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

// Givens sweep for Arnoldi column j of one GMRES column (linsolve.cpp:472-501),
// executed by one CTA: H(0..j, j), cs, sn staged in shared memory by all
// threads, the sequential rotations by thread 0, results written back.
// hcolIn (optional) already holds H(0..j, j) in shared memory.
// Split in two so callers can stage the inputs (givensStage, independent
// of hn) before a grid barrier and finish after it.
__device__ inline void givensStage(const GmresArgs& A, int col, int j, const double2* hcolIn, double2* sh) {
  const int ldh = A.restart + 1;
  const double2* H = A.H + static_cast<long long>(col) * ldh * A.restart;
  const double2* cs = A.cs + static_cast<long long>(col) * A.restart;
  const double2* sn = A.sn + static_cast<long long>(col) * A.restart;
  double2* hc = sh;               // [j+2]
  double2* scs = sh + RMAX + 2;   // [j]
  double2* ssn = scs + RMAX;      // [j]
  for (int t = threadIdx.x; t <= j; t += blockDim.x) hc[t] = hcolIn ? hcolIn[t] : H[t + j * ldh];
  for (int t = threadIdx.x; t < j; t += blockDim.x) {
    scs[t] = cs[t];
    ssn[t] = sn[t];
  }
}

// The sequential part of the Givens step (one thread): rotations 0..j-1 on
// the staged column, the new rotation, g, the state and the stop decision.
__device__ inline void givensCore(const GmresArgs& A, int col, int j, double hn, double2* sh) {
  double2* cs = A.cs + static_cast<long long>(col) * A.restart;
  double2* sn = A.sn + static_cast<long long>(col) * A.restart;
  double2* g = A.g + static_cast<long long>(col) * (A.restart + 1);
  double2* hc = sh;
  double2* scs = sh + RMAX + 2;
  double2* ssn = scs + RMAX;
  {
    GmresState& st = A.st[col];
    // Global state the tail needs, loaded before the sequential sweep so
    // the loads overlap it.
    const double beta = st.beta, beta0 = st.beta0;
    const int iters = st.iterations;
    const double2 gj = g[j];
    hc[j + 1] = make_double2(hn, 0.0);
    // Rotations 0..j-1 with the running entry carried in registers.
    double2 carry = hc[0];
    for (int i = 0; i < j; ++i) {
      const double2 a0 = carry, a1 = hc[i + 1];
      hc[i] = cadd(cmul(scs[i], a0), cmul(ssn[i], a1));
      carry = cadd(cmul(make_double2(-ssn[i].x, ssn[i].y), a0), cmul(cconj(scs[i]), a1));
    }
    hc[j] = carry;
    const double2 hjj = hc[j], hj1 = hc[j + 1];
    const double den = sqrt((hjj.x * hjj.x + hjj.y * hjj.y) + (hj1.x * hj1.x + hj1.y * hj1.y));
    double2 c, s;
    if (den == 0.0) {
      c = make_double2(1.0, 0.0);
      s = make_double2(0.0, 0.0);
    } else {
      c = make_double2(hjj.x / den, -hjj.y / den);
      s = make_double2(hj1.x / den, -hj1.y / den);
    }
    cs[j] = c;
    sn[j] = s;
    hc[j] = cadd(cmul(c, hjj), cmul(s, hj1));
    hc[j + 1] = make_double2(0.0, 0.0);
    g[j] = cmul(c, gj);
    const double2 gj1 = cmul(make_double2(-s.x, s.y), gj);
    g[j + 1] = gj1;
    st.iterations = iters + 1;
    st.ncount = j + 1;
    const double rel = cabs2(gj1) / beta;
    pushHist(A, col, 1.0, cabs2(gj1) / beta0);
    if (rel < 0.1 * A.tol || !(hn > 0.0) || j + 1 >= A.restart || iters + 1 >= A.maxIter) st.stopInner = 1;
  }
}

// Needs givensStage's shared-memory staging visible (a __syncthreads after it).
__device__ inline void givensFinish(const GmresArgs& A, int col, int j, double hn, double2* sh) {
  const int ldh = A.restart + 1;
  double2* H = A.H + static_cast<long long>(col) * ldh * A.restart;
  if (threadIdx.x == 0) givensCore(A, col, j, hn, sh);
  __syncthreads();
  for (int t = threadIdx.x; t <= j + 1; t += blockDim.x) H[t + j * ldh] = sh[t];
  __syncthreads();
}

// The whole Givens step of column j on ONE warp (the restart-cycle kernel's
// auxiliary warp), the unrotated column read from H (written by the LS step
// of column j), sh: 3*RMAX+4 entries of this warp's shared memory.
__device__ inline void givensWarp(const GmresArgs& A, int col, int j, double hn, double2* sh) {
  const int lane = threadIdx.x & 31;
  const int ldh = A.restart + 1;
  double2* H = A.H + static_cast<long long>(col) * ldh * A.restart;
  const double2* cs = A.cs + static_cast<long long>(col) * A.restart;
  const double2* sn = A.sn + static_cast<long long>(col) * A.restart;
  double2* scs = sh + RMAX + 2;
  double2* ssn = scs + RMAX;
  for (int t = lane; t <= j; t += 32) sh[t] = __ldcg(H + t + j * ldh);
  for (int t = lane; t < j; t += 32) {
    scs[t] = __ldcg(cs + t);
    ssn[t] = __ldcg(sn + t);
  }
  __syncwarp();
  if (lane == 0) givensCore(A, col, j, hn, sh);
  __syncwarp();
  for (int t = lane; t <= j + 1; t += 32) H[t + j * ldh] = sh[t];
  __syncwarp();
}

__device__ inline void givensStep(const GmresArgs& A, int col, int j, double hn, const double2* hcolIn,
                                  double2* sh /* >= 3*RMAX+4 */) {
  __syncthreads();
  givensStage(A, col, j, hcolIn, sh);
  __syncthreads();
  givensFinish(A, col, j, hn, sh);
}

// cv[0..j] <- (I + L)^{-1} cv on one warp, L packed by rows (row i at
// i(i-1)/2); RPL rows per lane (RPL * 32 > j).
template <int RPL>
__device__ __forceinline__ void forwardSubstWarp(double2* cv, const double2* sL, int j, int lane) {
  double2 hv[RPL];
  int rowBase[RPL];
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    const int i = lane + 32 * t;
    hv[t] = i <= j ? cv[i] : make_double2(0.0, 0.0);
    rowBase[t] = i * (i - 1) / 2;
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
      if (i > k && i <= j) hv[t] = csub(hv[t], cmul(sL[rowBase[t] + k], hk));
    }
  }
  __syncwarp();
#pragma unroll
  for (int t = 0; t < RPL; ++t) {
    const int i = lane + 32 * t;
    if (i <= j) cv[i] = hv[t];
  }
}

// One Arnoldi step j, single column, low-synchronisation MGS (device
// function: the gmresArnoldiLS kernel and the fused apply+Arnoldi of
// matvec_persistent.cu run it): the MGS
// coefficients h_i = <v_i, (I - v_{i-1}v_{i-1}^H)...(I - v_0 v_0^H) w> are
// obtained as h = (I + L)^{-1} c with c = V^H w and L the strictly lower
// part of the basis Gram matrix V^H V (identical to the MGS sweep in exact
// arithmetic; L accumulates one row per iteration). Two grid barriers per
// step instead of j + 2:
//   pass 1  per-CTA partials of c_k = <v_k, w> and S_jk = <v_j, v_k>
//           (a warp per two k, the CTA's row chunk of w and v_j in smem)
//   -- barrier --  every CTA reduces every dot (fixed order, same bits),
//                  forward substitution for h (warp 0)
//   pass 2  w' = w - V h, ||w'||^2
//   -- barrier --  v_{j+1} = w' / ||w'||, Givens (CTA 0)
// (`dots` is unused since the totals stay in shared memory.)
// shw: dynamic shared memory of arnoldiLSSmem(chunk) double2; scratch:
// blockDim/32 entries; hcol: RMAX+2; sh: 3*RMAX+4.
//
// Lagged normalisation (lagged = true, the restart-cycle kernel): v_j arrives
// unnormalised (w' of the previous step) with its norm hnPrev known since the
// step's first grid barrier; the staging divides it by hnPrev and writes the
// normalised rows back, pass 2 stores w' unnormalised straight into v_{j+1}
// and publishes the CTA's ||w'||^2 partial; the w' norm, v_{j+1}'s
// normalisation and the Givens step of column j move into the next step (no
// third grid barrier, no normalisation pass). The unrotated column h is left
// in H(:, j) for that Givens step.
__device__ inline void arnoldiLS(const GmresArgs& A, int j, double2* S, double2* dots, double2* dotPart, double2* shw,
                          double2* scratch, double2* hcol, double2* sh, unsigned long long* bar,
                          bool lagged = false, double hnPrev = 1.0, unsigned long long* traceDots = nullptr) {
  // Written by CTA 0 before a grid barrier (or before this launch): read
  // through L1 (the persistent restart-cycle loop re-reads it per column).
  const volatile GmresState* stv = A.st;
  const int run = stv->cycleActive && !stv->stopInner;
  if (!run) return;  // uniform over the grid
  unsigned long long pt[5] = {0, 0, 0, 0, 0};
  auto mark = [&](int k) {
    if (A.prof && blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt[k]));
  };
  mark(0);
  const int lds = A.restart + 1;
  const long long n = static_cast<long long>(A.ne) * A.m;
  const long long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long long r0 = blockIdx.x * chunk;
  const int cnt = static_cast<int>(r0 >= n ? 0 : (n - r0 < chunk ? n - r0 : chunk));
  double2* ws = shw;
  double2* vj = shw + chunk;
  double2* cv = vj + chunk;  // [j+1] totals of c, later h
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2* Vj = A.V + static_cast<long long>(j) * n;
  const bool rescale = lagged && hnPrev != 1.0;
  for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
    double2 wv = A.w[r0 + r];
    if (A.dinv) wv = cmul(wv, A.dinv[r0 + r]);
    ws[r] = wv;
    double2 vv = __ldcg(Vj + r0 + r);
    if (rescale) {
      vv = make_double2(vv.x / hnPrev, vv.y / hnPrev);
      A.V[static_cast<long long>(j) * n + r0 + r] = vv;
    }
    vj[r] = vv;
  }
  __syncthreads();
  // Pass 1: warp w owns dots k = w, w + nw, ...; it takes them two at a
  // time with 16 rows per lane per vector in flight (32 loads: one trip for
  // row chunks up to 512, i.e. C2), c_k in slot k, S_jk in slot lds + k.
  {
    constexpr int U1 = 16;
    const int nw = static_cast<int>(blockDim.x >> 5);
    for (int k0 = warp; k0 <= j; k0 += 2 * nw) {
      const int k1 = k0 + nw;
      const bool two = k1 <= j;
      const double2* V0 = A.V + static_cast<long long>(k0) * n + r0;
      const double2* V1 = A.V + static_cast<long long>(two ? k1 : k0) * n + r0;
      // Lagged: v_j's rows were just rewritten (normalised) by this CTA: read them from vj.
      const bool sm0 = lagged && k0 == j, sm1 = lagged && two && k1 == j;
      double2 c0 = make_double2(0.0, 0.0), c1 = c0, s0 = c0, s1 = c0;
      for (int r = lane; r < cnt; r += 32 * U1) {
        double2 v0[U1], v1[U1];
#pragma unroll
        for (int u = 0; u < U1; ++u) {
          const int rr = r + 32 * u;
          v0[u] = rr < cnt ? (sm0 ? vj[rr] : __ldcg(V0 + rr)) : make_double2(0.0, 0.0);
          v1[u] = rr < cnt && two ? (sm1 ? vj[rr] : __ldcg(V1 + rr)) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < U1; ++u) {
          const int rr = r + 32 * u;
          if (rr < cnt) {
            const double2 wv = ws[rr], vv = vj[rr];
            cfma_conj(c0, v0[u], wv);
            cfma_conj(s0, vv, v0[u]);
            cfma_conj(c1, v1[u], wv);
            cfma_conj(s1, vv, v1[u]);
          }
        }
      }
      const double2 t0 = warpSum(c0), u0 = warpSum(s0);
      const double2 t1 = warpSum(c1), u1 = warpSum(s1);
      if (lane == 0) {
        dotPart[static_cast<long long>(k0) * gridDim.x + blockIdx.x] = t0;
        if (k0 < j) dotPart[static_cast<long long>(lds + k0) * gridDim.x + blockIdx.x] = u0;
        if (two) {
          dotPart[static_cast<long long>(k1) * gridDim.x + blockIdx.x] = t1;
          if (k1 < j) dotPart[static_cast<long long>(lds + k1) * gridDim.x + blockIdx.x] = u1;
        }
      }
    }
  }
  gridBarrier(bar);
  mark(1);
  if (traceDots && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    traceDots[blockIdx.x] = t;
  }
  // Grid totals, reduced by EVERY CTA itself (no second grid barrier):
  // 16 lanes per dot slot, 2 slots per warp; lane q of a group sums the
  // partials q, q+16, ... in order, then a 4-step butterfly — the same bits
  // in every CTA. Slots: c_0..c_j, then S_j0..S_j,j-1 (CTA 0 also records
  // row j of S for the later iterations).
  double2* sL = cv + RMAX + 1;  // lower triangle of L, packed rows: row i at i*(i-1)/2
  {
    const int ndots = 2 * j + 1;
    const int grp = lane >> 4, gl = lane & 15;
    const int nw = static_cast<int>(blockDim.x >> 5);
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
          sL[j * (j - 1) / 2 + (d - j - 1)] = t;
          if (blockIdx.x == 0) S[static_cast<long long>(j) * lds + (d - j - 1)] = t;
        }
      }
    }
  }
  mark(2);
  // Rows 1..j-1 of L from the earlier iterations.
  for (int i = 1 + warp; i < j; i += static_cast<int>(blockDim.x >> 5))  // row i: warp, lanes over k < i
    for (int k = lane; k < i; k += 32) sL[i * (i - 1) / 2 + k] = __ldcg(S + static_cast<long long>(i) * lds + k);
  __syncthreads();
  // h = (I + L)^{-1} c, column-oriented on warp 0 (rows in registers; the
  // register count follows the restart length).
  if (warp == 0) {
    if (A.restart < 64)
      forwardSubstWarp<2>(cv, sL, j, lane);
    else
      forwardSubstWarp<(RMAX + 31) / 32 + 1>(cv, sL, j, lane);
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i <= j; i += blockDim.x) {
      hcol[i] = cv[i];
      if (lagged) A.H[i + static_cast<long long>(j) * (A.restart + 1)] = cv[i];
    }
  // Pass 2: w' = w - V h and ||w'||^2. Two rows per thread at a time
  // (16 loads in flight); per row the update order over k is unchanged.
  double2 acc = make_double2(0.0, 0.0);
  const int bd = static_cast<int>(blockDim.x);
  for (int ra = threadIdx.x; ra < cnt; ra += 2 * bd) {
    const int rb = ra + bd;
    const bool hb = rb < cnt;
    const int rbs = hb ? rb : ra;
    double2 wa = ws[ra], wb = ws[rbs];
    const double2* Va = A.V + r0 + ra;
    const double2* Vb = A.V + r0 + rbs;
    int k = 0;
    const int kEnd = lagged ? j : j + 1;  // lagged: the k = j term from vj below (same order)
    for (; k + 8 <= kEnd; k += 8) {
      double2 va[8], vb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        va[u] = __ldcg(Va + static_cast<long long>(k + u) * n);
        vb[u] = __ldcg(Vb + static_cast<long long>(k + u) * n);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        wa = csub(wa, cmul(cv[k + u], va[u]));
        wb = csub(wb, cmul(cv[k + u], vb[u]));
      }
    }
    for (; k < kEnd; ++k) {
      const double2 va = __ldcg(Va + static_cast<long long>(k) * n), vb = __ldcg(Vb + static_cast<long long>(k) * n);
      wa = csub(wa, cmul(cv[k], va));
      wb = csub(wb, cmul(cv[k], vb));
    }
    if (lagged) {
      wa = csub(wa, cmul(cv[j], vj[ra]));
      wb = csub(wb, cmul(cv[j], vj[rbs]));
    }
    ws[ra] = wa;
    acc.x += wa.x * wa.x + wa.y * wa.y;
    if (lagged) A.V[static_cast<long long>(j + 1) * n + r0 + ra] = wa;
    if (hb) {
      ws[rb] = wb;
      acc.x += wb.x * wb.x + wb.y * wb.y;
      if (lagged) A.V[static_cast<long long>(j + 1) * n + r0 + rb] = wb;
    }
  }
  blockPartial(acc, scratch, partSlot(A, 0, 0));
  if (lagged) {
    if (A.prof && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t3;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
      A.prof[0] += pt[1] - pt[0];
      A.prof[1] += pt[2] - pt[1];
      A.prof[2] += t3 - pt[2];
      A.prof[4] += 1;
    }
    return;
  }
  if (blockIdx.x == 0) givensStage(A, 0, j, hcol, sh);  // made visible by the barrier
  gridBarrier(bar);
  mark(3);
  const double hn = sqrt(warpTotal(partSlot(A, 0, 0)).x);
  if (hn > 0.0) {
    double2* vout = A.V + static_cast<long long>(j + 1) * n + r0;
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) vout[r] = make_double2(ws[r].x / hn, ws[r].y / hn);
  }
  if (blockIdx.x == 0) givensFinish(A, 0, j, hn, sh);
  if (A.prof && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t4;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t4));
    A.prof[0] += pt[1] - pt[0];
    A.prof[1] += pt[2] - pt[1];
    A.prof[2] += pt[3] - pt[2];
    A.prof[3] += t4 - pt[3];
    A.prof[4] += 1;
  }
}

// Dynamic shared memory (double2 count) the LS step needs for a row chunk.
__host__ __device__ inline long long arnoldiLSSmem(long long chunk, int restart) {
  return 2 * chunk + RMAX + 1 + static_cast<long long>(restart) * (restart + 1) / 2;
}

}  // namespace gmresdev
}  // namespace tbt
