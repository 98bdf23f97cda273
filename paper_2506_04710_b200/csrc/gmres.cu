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
#include <cmath>

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
};

namespace {

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
    for (int k = 1; k < kWarps; ++k) s = cadd(s, scratch[k]);
    part[blockIdx.x] = s;
  }
}

// Grid total of the partials, computed by each warp independently in a
// fixed order (bitwise identical in every warp and CTA).
__device__ __forceinline__ double2 warpTotal(const double2* part) {
  const int lane = threadIdx.x & 31;
  double2 s = make_double2(0.0, 0.0);
  for (int k = lane; k < static_cast<int>(gridDim.x); k += 32) s = cadd(s, __ldcg(part + k));
  return warpSum(s);
}

__device__ __forceinline__ double2* partSlot(const GmresArgs& A, int phase, int col) {
  return A.partial + (static_cast<long long>(phase & 1) * A.ncols + col) * gridDim.x;
}

__device__ __forceinline__ long long slotIndex(long long s, int col, int ncols, int m) {
  const long long e = s / m, a = s % m;
  return (e * ncols + col) * m + a;
}

__device__ void pushHist(const GmresArgs& A, int col, double kind, double v) {
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
__device__ void givensStep(const GmresArgs& A, int col, int j, double hn, const double2* hcolIn,
                           double2* sh /* >= 3*RMAX+4 */) {
  const int ldh = A.restart + 1;
  double2* H = A.H + static_cast<long long>(col) * ldh * A.restart;
  double2* cs = A.cs + static_cast<long long>(col) * A.restart;
  double2* sn = A.sn + static_cast<long long>(col) * A.restart;
  double2* g = A.g + static_cast<long long>(col) * (A.restart + 1);
  double2* hc = sh;               // [j+2]
  double2* scs = sh + RMAX + 2;   // [j]
  double2* ssn = scs + RMAX;      // [j]
  __syncthreads();
  for (int t = threadIdx.x; t <= j; t += blockDim.x) hc[t] = hcolIn ? hcolIn[t] : H[t + j * ldh];
  for (int t = threadIdx.x; t < j; t += blockDim.x) {
    scs[t] = cs[t];
    ssn[t] = sn[t];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    GmresState& st = A.st[col];
    hc[j + 1] = make_double2(hn, 0.0);
    for (int i = 0; i < j; ++i) {
      const double2 a0 = hc[i], a1 = hc[i + 1];
      hc[i] = cadd(cmul(scs[i], a0), cmul(ssn[i], a1));
      hc[i + 1] = cadd(cmul(make_double2(-ssn[i].x, ssn[i].y), a0), cmul(cconj(scs[i]), a1));
    }
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
    const double2 gj = g[j];
    g[j] = cmul(c, gj);
    const double2 gj1 = cmul(make_double2(-s.x, s.y), gj);
    g[j + 1] = gj1;
    st.iterations += 1;
    st.ncount = j + 1;
    const double rel = cabs2(gj1) / st.beta;
    pushHist(A, col, 1.0, cabs2(gj1) / st.beta0);
    if (rel < 0.1 * A.tol || !(hn > 0.0) || st.ncount >= A.restart || st.iterations >= A.maxIter) st.stopInner = 1;
  }
  __syncthreads();
  for (int t = threadIdx.x; t <= j + 1; t += blockDim.x) H[t + j * ldh] = hc[t];
  __syncthreads();
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
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        const double2 r = csub(A.b[q], A.ax[q]);
        A.w[q] = r;
        acc.x += r.x * r.x + r.y * r.y;
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
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        double2 z = A.w[q];
        if (A.dinv) z = cmul(z, A.dinv[s]);
        A.V[q] = z;
        acc.x += z.x * z.x + z.y * z.y;
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
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        const double2 z = A.V[q];
        A.V[q] = make_double2(z.x / beta, z.y / beta);
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

// One Arnoldi step j, single column, low-synchronisation MGS: the MGS
// coefficients h_i = <v_i, (I - v_{i-1}v_{i-1}^H)...(I - v_0 v_0^H) w> are
// obtained as h = (I + L)^{-1} c with c = V^H w and L the strictly lower
// part of the basis Gram matrix V^H V (identical to the MGS sweep in exact
// arithmetic; L accumulates one row per iteration). Three grid barriers per
// step instead of j + 2:
//   pass 1  per-CTA partials of c_k = <v_k, w> and S_jk = <v_j, v_k>
//           (one warp per k, the CTA's row chunk of w and v_j in smem)
//   -- barrier --  CTA k reduces dot k over the grid
//   -- barrier --  every CTA: forward substitution for h (warp 0)
//   pass 2  w' = w - V h, ||w'||^2
//   -- barrier --  v_{j+1} = w' / ||w'||, Givens (CTA 0)
__global__ void __launch_bounds__(kThreads) gmresArnoldiLS(GmresArgs A, double2* S, double2* dots,
                                                           double2* dotPart) {
  extern __shared__ double2 shw[];  // [chunk] w, [chunk] v_j, [RMAX+1] c/h, [(RMAX+1)] S row staging
  __shared__ double2 scratch[kWarps];
  __shared__ double2 hcol[RMAX + 2];
  __shared__ double2 sh[3 * RMAX + 4];
  const int run = A.st[0].cycleActive && !A.st[0].stopInner;
  if (!run) return;  // uniform over the grid
  const int j = A.j;
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
  for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
    double2 wv = A.w[r0 + r];
    if (A.dinv) wv = cmul(wv, A.dinv[r0 + r]);
    ws[r] = wv;
    vj[r] = Vj[r0 + r];
  }
  __syncthreads();
  // Pass 1: dot k by warp k % 8; c_k in slot k, S_jk in slot lds + k.
  for (int k = warp; k <= j; k += kWarps) {
    const double2* Vk = A.V + static_cast<long long>(k) * n + r0;
    double2 c0 = make_double2(0.0, 0.0), c1 = c0, s0 = c0, s1 = c0;
    int r = lane;
    for (; r + 96 < cnt; r += 128) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = Vk[r + 32 * u];
      cfma_conj(c0, v[0], ws[r]);
      cfma_conj(c1, v[1], ws[r + 32]);
      cfma_conj(c0, v[2], ws[r + 64]);
      cfma_conj(c1, v[3], ws[r + 96]);
      if (k < j) {
        cfma_conj(s0, vj[r], v[0]);
        cfma_conj(s1, vj[r + 32], v[1]);
        cfma_conj(s0, vj[r + 64], v[2]);
        cfma_conj(s1, vj[r + 96], v[3]);
      }
    }
    for (; r < cnt; r += 32) {
      const double2 v = Vk[r];
      cfma_conj(c0, v, ws[r]);
      if (k < j) cfma_conj(s0, vj[r], v);
    }
    const double2 c = warpSum(cadd(c0, c1));
    const double2 sjk = warpSum(cadd(s0, s1));
    if (lane == 0) {
      dotPart[static_cast<long long>(k) * gridDim.x + blockIdx.x] = c;
      if (k < j) dotPart[static_cast<long long>(lds + k) * gridDim.x + blockIdx.x] = sjk;
    }
  }
  gridBarrier(A.bar);
  // Grid totals: CTA d reduces dot d (c_0..c_j, then S_j0..S_j,j-1).
  const int ndots = 2 * j + 1;
  for (int d = blockIdx.x; d < ndots; d += gridDim.x) {
    const int slot = d <= j ? d : lds + (d - j - 1);
    if (warp == 0) {
      const double2 t = warpTotal(dotPart + static_cast<long long>(slot) * gridDim.x);
      if (lane == 0) {
        dots[slot] = t;
        if (d > j) S[static_cast<long long>(j) * lds + (d - j - 1)] = t;
      }
    }
  }
  gridBarrier(A.bar);
  // Stage the lower triangle rows 1..j of L (shared memory after cv).
  double2* sL = cv + RMAX + 1;  // packed rows: row i at i*(i-1)/2
  for (int q = threadIdx.x; q < j * (j + 1) / 2; q += blockDim.x) {
    // q -> (i, k) with i >= 1, k < i
    int i = static_cast<int>((1.0 + sqrt(1.0 + 8.0 * q)) * 0.5);
    while (i * (i - 1) / 2 > q) --i;
    while ((i + 1) * i / 2 <= q) ++i;
    const int k = q - i * (i - 1) / 2;
    sL[q] = __ldcg(S + static_cast<long long>(i) * lds + k);
  }
  for (int i = threadIdx.x; i <= j; i += blockDim.x) cv[i] = __ldcg(dots + i);
  __syncthreads();
  // h = (I + L)^{-1} c, column-oriented on warp 0 (rows in registers).
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
    __syncwarp();
#pragma unroll
    for (int t = 0; t < RPL; ++t) {
      const int i = lane + 32 * t;
      if (i <= j) cv[i] = hv[t];
    }
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i <= j; i += blockDim.x) hcol[i] = cv[i];
  // Pass 2: w' = w - V h and ||w'||^2.
  double2 acc = make_double2(0.0, 0.0);
  for (int r = threadIdx.x; r < cnt; r += blockDim.x) {
    double2 wv = ws[r];
    int k = 0;
    for (; k + 8 <= j + 1; k += 8) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = A.V[static_cast<long long>(k + u) * n + r0 + r];
#pragma unroll
      for (int u = 0; u < 8; ++u) wv = csub(wv, cmul(cv[k + u], v[u]));
    }
    for (; k <= j; ++k) wv = csub(wv, cmul(cv[k], A.V[static_cast<long long>(k) * n + r0 + r]));
    ws[r] = wv;
    acc.x += wv.x * wv.x + wv.y * wv.y;
  }
  blockPartial(acc, scratch, partSlot(A, 0, 0));
  gridBarrier(A.bar);
  const double hn = sqrt(warpTotal(partSlot(A, 0, 0)).x);
  if (hn > 0.0) {
    double2* vout = A.V + static_cast<long long>(j + 1) * n + r0;
    for (int r = threadIdx.x; r < cnt; r += blockDim.x) vout[r] = make_double2(ws[r].x / hn, ws[r].y / hn);
  }
  if (blockIdx.x == 0) givensStep(A, 0, j, hn, hcol, sh);
}

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
  extern __shared__ double2 shH[];  // [(restart+1)*restart] + [restart] y
  __shared__ int sFlagU[1];
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
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long nall = slots * A.ncols;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  double2* sy = shH;  // reuse: y of the current column
  for (int col = 0; col < A.ncols; ++col) {
    __syncthreads();
    if (threadIdx.x == 0) sFlagU[0] = A.st[col].cycleActive;
    const int nc = A.st[col].ncount;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) sy[i] = __ldcg(A.ycoef + static_cast<long long>(col) * A.restart + i);
    __syncthreads();
    if (!sFlagU[0]) continue;
    for (long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; s < slots; s += stride) {
      const long long q = slotIndex(s, col, A.ncols, A.m);
      double2 xv = A.x[q];
      int i = 0;
      for (; i + 8 <= nc; i += 8) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = A.V[static_cast<long long>(i + u) * nall + q];
#pragma unroll
        for (int u = 0; u < 8; ++u) xv = cadd(xv, cmul(sy[i + u], v[u]));
      }
      for (; i < nc; ++i) xv = cadd(xv, cmul(sy[i], A.V[static_cast<long long>(i) * nall + q]));
      A.x[q] = xv;
    }
  }
}

void coopLaunch(const void* fn, int grid, size_t smem, GmresArgs& args, cudaStream_t s) {
  void* params[] = {&args};
  TBT_CUDA_CHECK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), params, smem, s));
}

}  // namespace

// Host driver (iterativeSolve, linsolve.cpp:551-593, columns in lockstep).
void gmresSolve(Ctx& c, const double2* b, double2* x, int ncols, const tbt_gmres_opts& o, bool useAOnly,
                std::vector<GmresState>& out, std::vector<double>& hist, int& matvecs) {
  const int R = o.restart;
  TBT_USER_CHECK(R <= RMAX, "tbt_gmres: restart above " + std::to_string(RMAX));
  const long long nall = c.n * ncols;
  cudaStream_t s = c.stream;
  const int sms = smCount(c.device);
  // One CTA per SM: always co-resident, as the grid barrier requires
  // (cudaLaunchCooperativeKernel rejects a grid that is not).
  const int grid = sms;
  const bool fast = ncols == 1 && c.n <= static_cast<long long>(grid) * kThreads * FAST_K;
  const long long lsChunk = (c.n + grid - 1) / grid;
  const bool lowSync = o.orthog == 1 && ncols == 1 && lsChunk <= 4096;
  const size_t lsSmem = (2 * lsChunk + RMAX + 1 + static_cast<size_t>(R) * (R + 1) / 2) * sizeof(double2);

  GmresArgs A{};
  A.ncols = ncols;
  A.restart = R;
  A.maxIter = o.max_iter;
  A.histCap = std::max(0, o.hist_cap);
  A.precondition = o.precondition;
  A.tol = o.tol;
  A.ne = c.ne;
  A.m = c.m;
  // Device allocations for this solve.
  std::vector<void*> allocs;
  auto dalloc = [&](size_t bytes) {
    void* p = nullptr;
    TBT_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    allocs.push_back(p);
    return p;
  };
  try {
    A.st = static_cast<GmresState*>(dalloc(sizeof(GmresState) * ncols));
    A.H = static_cast<double2*>(dalloc(sizeof(double2) * ncols * (R + 1) * R));
    A.g = static_cast<double2*>(dalloc(sizeof(double2) * ncols * (R + 1)));
    A.cs = static_cast<double2*>(dalloc(sizeof(double2) * ncols * R));
    A.sn = static_cast<double2*>(dalloc(sizeof(double2) * ncols * R));
    A.ycoef = static_cast<double2*>(dalloc(sizeof(double2) * ncols * R));
    A.hist = static_cast<double*>(dalloc(sizeof(double) * 2 * ncols * std::max(1, A.histCap)));
    A.partial = static_cast<double2*>(dalloc(sizeof(double2) * 2 * ncols * grid));
    A.bar = static_cast<unsigned long long*>(dalloc(sizeof(unsigned long long)));
    A.b = b;
    A.x = x;
    double2* ax = static_cast<double2*>(dalloc(sizeof(double2) * nall));
    A.ax = ax;
    A.w = static_cast<double2*>(dalloc(sizeof(double2) * nall));
    A.V = static_cast<double2*>(dalloc(sizeof(double2) * nall * (R + 1)));
    double2* lsS = static_cast<double2*>(dalloc(sizeof(double2) * (R + 1) * (R + 1)));
    double2* lsDots = static_cast<double2*>(dalloc(sizeof(double2) * 2 * (R + 1)));
    double2* lsPart = static_cast<double2*>(dalloc(sizeof(double2) * 2 * (R + 1) * grid));
    if (lowSync)
      TBT_CUDA_CHECK(cudaFuncSetAttribute(gmresArnoldiLS, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(lsSmem)));
    TBT_CUDA_CHECK(cudaMemsetAsync(A.bar, 0, sizeof(unsigned long long), s));
    TBT_CUDA_CHECK(cudaMemsetAsync(A.V, 0, sizeof(double2) * nall * (R + 1), s));
    TBT_CUDA_CHECK(cudaMemsetAsync(A.H, 0, sizeof(double2) * ncols * (R + 1) * R, s));
    TBT_CUDA_CHECK(cudaMemsetAsync(x, 0, sizeof(double2) * nall, s));
    A.dinv = o.precondition ? (useAOnly ? c.dDiagInvA : c.dDiagInv) : nullptr;
    const size_t smem = sizeof(int) * ncols;

    matvecs = 0;
    coopLaunch(reinterpret_cast<const void*>(gmresInit), grid, smem, A, s);
    std::vector<GmresState> st(ncols);
    auto pull = [&]() {
      TBT_CUDA_CHECK(cudaMemcpyAsync(st.data(), A.st, sizeof(GmresState) * ncols, cudaMemcpyDeviceToHost, s));
      TBT_CUDA_CHECK(cudaStreamSynchronize(s));
    };
    auto arnoldi = [&](int j) {
      A.j = j;
      if (lowSync) {
        void* params[] = {&A, &lsS, &lsDots, &lsPart};
        TBT_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(gmresArnoldiLS), dim3(grid),
                                                   dim3(kThreads), params, lsSmem, s));
      } else if (fast) {
        coopLaunch(reinterpret_cast<const void*>(gmresArnoldi1), grid, 0, A, s);
      } else {
        coopLaunch(reinterpret_cast<const void*>(gmresArnoldi), grid, smem, A, s);
      }
    };
    // Single column: the whole inner loop of a cycle is one CUDA graph
    // (restart x [apply, Arnoldi]); every node turns into a no-op once the
    // column's inner loop stopped (device flag), so the host synchronises
    // once per restart cycle.
    cudaGraphExec_t inner = nullptr;
    const bool useGraph = ncols == 1 && !c.timeBinprod;
    if (useGraph) {
      c.skipFlag = &A.st[0].stopInner;
      cudaGraph_t gph;
      TBT_CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        for (int j = 0; j < R; ++j) {
          applyInternal(c, A.V + static_cast<long long>(j) * nall, A.w, ncols, !useAOnly);
          arnoldi(j);
        }
      } catch (...) {
        cudaStreamEndCapture(s, &gph);
        c.skipFlag = nullptr;
        throw;
      }
      TBT_CUDA_CHECK(cudaStreamEndCapture(s, &gph));
      c.skipFlag = nullptr;
      const cudaError_t e = cudaGraphInstantiate(&inner, gph, 0);
      cudaGraphDestroy(gph);
      TBT_CUDA_CHECK(e);
    }
    try {
      pull();
      bool open = !st[0].done;
      for (size_t k = 1; k < st.size(); ++k) open |= !st[k].done;
      while (open) {
        applyInternal(c, x, ax, ncols, !useAOnly);
        ++matvecs;
        coopLaunch(reinterpret_cast<const void*>(gmresCycleStart), grid, smem, A, s);
        if (useGraph) {
          TBT_CUDA_CHECK(cudaGraphLaunch(inner, s));
        } else {
          pull();
          bool anyRun = false;
          for (auto& v : st) anyRun |= (v.cycleActive && !v.stopInner);
          for (int j = 0; anyRun && j < R; ++j) {
            applyInternal(c, A.V + static_cast<long long>(j) * nall, A.w, ncols, !useAOnly);
            arnoldi(j);
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
      if (inner) cudaGraphExecDestroy(inner);
      throw;
    }
    if (inner) cudaGraphExecDestroy(inner);
    // Matvecs issued: one per cycle start plus one per inner iteration.
    {
      int it = 0;
      for (auto& v : st) it = std::max(it, v.iterations);
      matvecs += it;
    }
    out = st;
    hist.assign(static_cast<size_t>(2) * ncols * std::max(1, A.histCap), 0.0);
    if (A.histCap > 0)
      TBT_CUDA_CHECK(cudaMemcpy(hist.data(), A.hist, sizeof(double) * 2 * ncols * A.histCap, cudaMemcpyDeviceToHost));
  } catch (...) {
    cudaStreamSynchronize(s);
    for (void* p : allocs) cudaFree(p);
    throw;
  }
  cudaStreamSynchronize(s);
  for (void* p : allocs) cudaFree(p);
}

}  // namespace tbt
