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
// projection (j+2 barriers per step) instead of 2(j+1) kernel launches.
// Cross-CTA reductions read the per-CTA partials in a fixed order, so every
// CTA derives bitwise-identical h values and runs are reproducible.
#include <algorithm>
#include <cmath>

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
  double2* partial; // [ncols][grid]
  unsigned* bar;    // [2] barrier counter / generation
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

__device__ __forceinline__ void gridBarrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vgen = bar + 1;
    const unsigned gen = *vgen;
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*vgen == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double2 warpSum(double2 v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, off);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, off);
  }
  return v;
}

// Block sum; the result is valid in thread 0.
__device__ double2 blockSum(double2 v, double2* scratch) {
  v = warpSum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  if (threadIdx.x == 0)
    for (int k = 0; k < kThreads / 32; ++k) s = cadd(s, scratch[k]);
  return s;
}

// Sum of the grid's partials for one column, identical in every CTA.
__device__ double2 gridTotal(const double2* part, double2* scratch) {
  __syncthreads();
  if (threadIdx.x < 32) {
    double2 s = make_double2(0.0, 0.0);
    for (int k = threadIdx.x; k < static_cast<int>(gridDim.x); k += 32) s = cadd(s, __ldcg(part + k));
    s = warpSum(s);
    if (threadIdx.x == 0) scratch[0] = s;
  }
  __syncthreads();
  const double2 r = scratch[0];
  __syncthreads();
  return r;
}

// Per-CTA partials are double-buffered by barrier parity: a CTA may write
// the next phase's partial while slower CTAs still sum the previous one.
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

// Smith's complex division a / b.
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

__global__ void __launch_bounds__(kThreads) gmresInit(GmresArgs A) {
  __shared__ double2 scratch[kThreads / 32];
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int col = 0; col < A.ncols; ++col) {
    double2 acc = make_double2(0.0, 0.0);
    for (long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; s < slots; s += stride) {
      const double2 v = A.b[slotIndex(s, col, A.ncols, A.m)];
      acc.x += v.x * v.x + v.y * v.y;
    }
    const double2 t = blockSum(acc, scratch);
    if (threadIdx.x == 0) partSlot(A, 0, col)[blockIdx.x] = t;
  }
  gridBarrier(A.bar);
  for (int col = 0; col < A.ncols; ++col) {
    const double2 tot = gridTotal(partSlot(A, 0, col), scratch);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
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

// r = b - A x, residual test, z = M r, beta, v0 = z / beta (linsolve.cpp:446-461).
__global__ void __launch_bounds__(kThreads) gmresCycleStart(GmresArgs A) {
  __shared__ double2 scratch[kThreads / 32];
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
    const double2 t = blockSum(acc, scratch);
    if (threadIdx.x == 0) partSlot(A, 0, col)[blockIdx.x] = t;
  }
  gridBarrier(A.bar);
  const long long nall = slots * A.ncols;
  for (int col = 0; col < A.ncols; ++col) {
    if (!sFlag[col]) continue;
    const double2 tot = gridTotal(partSlot(A, 0, col), scratch);
    const double bnorm = A.st[col].bnorm;
    const double res = sqrt(tot.x) / bnorm;
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
    const double2 t = blockSum(acc, scratch);
    if (threadIdx.x == 0) partSlot(A, 1, col)[blockIdx.x] = t;
  }
  gridBarrier(A.bar);
  for (int col = 0; col < A.ncols; ++col) {
    if (!sFlag[col]) continue;
    const double2 tot = gridTotal(partSlot(A, 1, col), scratch);
    const double beta = sqrt(tot.x);
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
  (void)nall;
}

// One Arnoldi step j for every running column (linsolve.cpp:463-502).
__global__ void __launch_bounds__(kThreads) gmresArnoldi(GmresArgs A) {
  __shared__ double2 scratch[kThreads / 32];
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
    const double2 t = blockSum(acc, scratch);
    if (threadIdx.x == 0) partSlot(A, 0, col)[blockIdx.x] = t;
  }
  gridBarrier(A.bar);
  for (int i = 0; i <= j; ++i) {
    for (int col = 0; col < A.ncols; ++col) {
      if (!sFlag[col]) continue;
      const double2 h = gridTotal(partSlot(A, i, col), scratch);
      if (blockIdx.x == 0 && threadIdx.x == 0) A.H[static_cast<long long>(col) * ldh * A.restart + i + j * ldh] = h;
      const double2* vi = A.V + static_cast<long long>(i) * nall;
      const double2* vn = A.V + static_cast<long long>(i + 1) * nall;
      double2 acc = make_double2(0.0, 0.0);
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        const double2 hv = cmul(h, vi[q]);
        const double2 wv = csub(A.w[q], hv);
        A.w[q] = wv;
        if (i < j)
          cfma_conj(acc, vn[q], wv);
        else
          acc.x += wv.x * wv.x + wv.y * wv.y;
      }
      const double2 t = blockSum(acc, scratch);
      if (threadIdx.x == 0) partSlot(A, i + 1, col)[blockIdx.x] = t;
    }
    gridBarrier(A.bar);
  }
  for (int col = 0; col < A.ncols; ++col) {
    if (!sFlag[col]) continue;
    const double2 tot = gridTotal(partSlot(A, j + 1, col), scratch);
    const double hn = sqrt(tot.x);
    if (hn > 0.0) {
      double2* vn = A.V + static_cast<long long>(j + 1) * nall;
      for (long long s = s0; s < slots; s += stride) {
        const long long q = slotIndex(s, col, A.ncols, A.m);
        const double2 wv = A.w[q];
        vn[q] = make_double2(wv.x / hn, wv.y / hn);
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) A.H[static_cast<long long>(col) * ldh * A.restart + (j + 1) + j * ldh] = make_double2(hn, 0.0);
  }
  if (blockIdx.x != 0) return;
  __syncthreads();
  // Givens rotations and exit tests, one thread per column.
  for (int col = threadIdx.x; col < A.ncols; col += blockDim.x) {
    if (!sFlag[col]) continue;
    GmresState& st = A.st[col];
    double2* H = A.H + static_cast<long long>(col) * ldh * A.restart;
    double2* cs = A.cs + static_cast<long long>(col) * A.restart;
    double2* sn = A.sn + static_cast<long long>(col) * A.restart;
    double2* g = A.g + static_cast<long long>(col) * (A.restart + 1);
    auto h = [&](int r, int c) -> double2& { return H[r + c * ldh]; };
    const double hn = h(j + 1, j).x;
    for (int i = 0; i < j; ++i) {
      const double2 t = cadd(cmul(cs[i], h(i, j)), cmul(sn[i], h(i + 1, j)));
      const double2 lo = cadd(cmul(make_double2(-sn[i].x, sn[i].y), h(i, j)), cmul(cconj(cs[i]), h(i + 1, j)));
      h(i + 1, j) = lo;
      h(i, j) = t;
    }
    const double2 hjj = h(j, j), hj1 = h(j + 1, j);
    const double den = sqrt((hjj.x * hjj.x + hjj.y * hjj.y) + (hj1.x * hj1.x + hj1.y * hj1.y));
    if (den == 0.0) {
      cs[j] = make_double2(1.0, 0.0);
      sn[j] = make_double2(0.0, 0.0);
    } else {
      cs[j] = make_double2(hjj.x / den, -hjj.y / den);
      sn[j] = make_double2(hj1.x / den, -hj1.y / den);
    }
    h(j, j) = cadd(cmul(cs[j], hjj), cmul(sn[j], hj1));
    h(j + 1, j) = make_double2(0.0, 0.0);
    const double2 gj = g[j];
    g[j] = cmul(cs[j], gj);
    g[j + 1] = cmul(make_double2(-sn[j].x, sn[j].y), gj);
    st.iterations += 1;
    st.ncount = j + 1;
    const double rel = cabs2(g[j + 1]) / st.beta;
    pushHist(A, col, 1.0, cabs2(g[j + 1]) / st.beta0);
    if (rel < 0.1 * A.tol || !(hn > 0.0) || st.ncount >= A.restart || st.iterations >= A.maxIter) st.stopInner = 1;
  }
}

// Back substitution and x += sum_i y_i v_i (linsolve.cpp:503-510).
__global__ void __launch_bounds__(kThreads) gmresUpdate(GmresArgs A) {
  extern __shared__ int sFlag[];
  const int ldh = A.restart + 1;
  if (blockIdx.x == 0) {
    for (int col = threadIdx.x; col < A.ncols; col += blockDim.x) {
      const GmresState& st = A.st[col];
      if (!st.cycleActive) continue;
      const double2* H = A.H + static_cast<long long>(col) * ldh * A.restart;
      const double2* g = A.g + static_cast<long long>(col) * (A.restart + 1);
      double2* y = A.ycoef + static_cast<long long>(col) * A.restart;
      const int nc = st.ncount;
      for (int i = nc - 1; i >= 0; --i) {
        double2 s = g[i];
        for (int k = i + 1; k < nc; ++k) s = csub(s, cmul(H[i + k * ldh], y[k]));
        y[i] = cdiv(s, H[i + i * ldh]);
      }
    }
  }
  for (int col = 0; col < A.ncols; ++col)
    if (threadIdx.x == 0) sFlag[col] = A.st[col].cycleActive;
  gridBarrier(A.bar);
  const long long slots = static_cast<long long>(A.ne) * A.m;
  const long long nall = slots * A.ncols;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int col = 0; col < A.ncols; ++col) {
    if (!sFlag[col]) continue;
    const int nc = A.st[col].ncount;
    const double2* y = A.ycoef + static_cast<long long>(col) * A.restart;
    for (long long s = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; s < slots; s += stride) {
      const long long q = slotIndex(s, col, A.ncols, A.m);
      double2 xv = A.x[q];
      for (int i = 0; i < nc; ++i) xv = cadd(xv, cmul(__ldcg(y + i), A.V[static_cast<long long>(i) * nall + q]));
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
struct GmresWork {
  long long cap = 0;
};

void gmresSolve(Ctx& c, const double2* b, double2* x, int ncols, const tbt_gmres_opts& o, bool useAOnly,
                std::vector<GmresState>& out, std::vector<double>& hist, int& matvecs) {
  const int R = o.restart;
  const long long nall = c.n * ncols;
  cudaStream_t s = c.stream;
  const int sms = smCount(c.device);
  // One CTA per SM: always co-resident, as the grid barrier requires
  // (cudaLaunchCooperativeKernel rejects a grid that is not).
  const int grid = sms;

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
    A.bar = static_cast<unsigned*>(dalloc(sizeof(unsigned) * 2));
    A.b = b;
    A.x = x;
    double2* ax = static_cast<double2*>(dalloc(sizeof(double2) * nall));
    A.ax = ax;
    A.w = static_cast<double2*>(dalloc(sizeof(double2) * nall));
    A.V = static_cast<double2*>(dalloc(sizeof(double2) * nall * (R + 1)));
    TBT_CUDA_CHECK(cudaMemsetAsync(A.bar, 0, sizeof(unsigned) * 2, s));
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
    for (;;) {
      pull();
      bool anyOpen = false;
      for (auto& v : st) anyOpen |= !v.done;
      if (!anyOpen) break;
      applyInternal(c, x, ax, ncols, !useAOnly);
      ++matvecs;
      coopLaunch(reinterpret_cast<const void*>(gmresCycleStart), grid, smem, A, s);
      pull();
      bool anyRun = false;
      for (auto& v : st) anyRun |= (v.cycleActive && !v.stopInner);
      if (!anyRun) continue;
      for (int j = 0; j < R; ++j) {
        applyInternal(c, A.V + static_cast<long long>(j) * nall, A.w, ncols, !useAOnly);
        ++matvecs;
        A.j = j;
        coopLaunch(reinterpret_cast<const void*>(gmresArnoldi), grid, smem, A, s);
        if ((j + 1) % 8 == 0 && j + 1 < R) {
          pull();
          bool more = false;
          for (auto& v : st) more |= (v.cycleActive && !v.stopInner);
          if (!more) break;
        }
      }
      coopLaunch(reinterpret_cast<const void*>(gmresUpdate), grid, smem, A, s);
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
