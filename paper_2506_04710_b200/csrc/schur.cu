// Schur-complement driver: schurSolve, the reference's
// default solver (proj/src/linsolve.cpp:595-682, config.hpp:42), on the
// device. For Z = [A  B^T; B  C] and excitations that vanish on the margin
// rows:
//   A [U F] = [V1  B^T]     p + nM A-only GMRES columns (gmres.cu, batches
//                           of max_nrhs columns in lockstep; Jacobi of A)
//   S = C - B F             TN complex GEMM over nA (zgemmTN)
//   S = P L U               right-looking LU with partial pivoting, the
//                           pivot-ratio check of checkLu (:517-528)
//   I2 = -S^{-1} (B U),  I1 = U - F I2
// then the relative residual of every column under the same operator.
// B^T is materialised densely from the uploaded margin generators (buildBT);
// everything stays in HBM, the host only sequences launches and reads the
// few bytes of pivots / norms it reports.
#include <algorithm>
#include <cmath>
#include <limits>

#include "dense.cuh"
#include "margin.cuh"

namespace tbt {
namespace {

int gridFor(long long n) { return static_cast<int>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 8192))); }

struct BTArgs {
  int nx, ny, m;
  long long nA, nM;
  int emSide[2], emRow[2], emCorner[4];
  long long sideStart[2], rowStart[2], cornerStart[4];
  const double2* rawSide[2];
  const double2* rawRow[2];
  const double2* corner[4];
  const double2* dense;  // SemiSparse: B row-major [nM][nA] (margin.cuh bDense)
};

// bt[q + k*nA] = (B^T)_{q,k} = B_{k,q}: the margin unknown k's coupling to
// element unknown q (regions as in margin.cu; raw layouts of tbt_gen.h).
__global__ void buildBT(BTArgs a, double2* __restrict__ bt) {
  const long long total = a.nA * a.nM;
  const long long rowLen = static_cast<long long>(a.nx) * a.m;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = o % a.nA, k = o / a.nA;
    if (a.dense) {  // bt[k*nA + q] = B[k][q]: the same index as the row-major B
      bt[o] = a.dense[o];
      continue;
    }
    double2 v = make_double2(0.0, 0.0);
    bool done = false;
    for (int r = 0; r < 2 && !done; ++r) {
      const int em = a.emSide[r];
      const long long kk = k - a.sideStart[r];
      if (em > 0 && kk >= 0 && kk < static_cast<long long>(a.ny) * em) {
        const int rowM = static_cast<int>(kk / em), i = static_cast<int>(kk % em);
        const int b = static_cast<int>(q / rowLen);
        const long long qq = q % rowLen;
        const int s = rowM - b;
        v = a.rawSide[r][(static_cast<long long>(s + a.ny - 1) * rowLen + qq) * em + i];
        done = true;
      }
    }
    for (int r = 0; r < 2 && !done; ++r) {
      const int em = a.emRow[r];
      const long long kk = k - a.rowStart[r];
      if (em > 0 && kk >= 0 && kk < static_cast<long long>(a.nx) * em) {
        const int colM = static_cast<int>(kk / em), i = static_cast<int>(kk % em);
        const long long e = q / a.m;
        const int j = static_cast<int>(e / a.nx), cEl = static_cast<int>(e % a.nx), b = static_cast<int>(q % a.m);
        const int s = colM - cEl;
        const long long blk = static_cast<long long>(j) * (2 * a.nx - 1) + s + a.nx - 1;
        v = a.rawRow[r][(blk * a.m + b) * em + i];
        done = true;
      }
    }
    for (int c = 0; c < 4 && !done; ++c) {
      const long long kk = k - a.cornerStart[c];
      if (a.emCorner[c] > 0 && kk >= 0 && kk < a.emCorner[c]) {
        v = a.corner[c][kk * a.nA + q];
        done = true;
      }
    }
    bt[o] = v;
  }
}

// out(k, l) = base(k, l) + sgn * sum_q A[q + k*lda] B[q + l*ldb]   (column-major out)
// base = Crm[k*ldc + l] (row-major C) or 0. 32 x 32 output tile per CTA,
// 16 x 16 threads with 2 x 2 outputs each, K staged through shared memory.
constexpr int TT = 32, TK = 16;
__global__ void __launch_bounds__(256) zgemmTN(const double2* __restrict__ A, long long lda,
                                               const double2* __restrict__ B, long long ldb, double2* __restrict__ out,
                                               long long ldo, int M, int N, long long K, const double2* __restrict__ Crm,
                                               long long ldc, double sgn) {
  __shared__ double2 As[TK][TT + 1], Bs[TK][TT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int k0 = blockIdx.y * TT, l0 = blockIdx.x * TT;
  double2 acc[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j] = make_double2(0.0, 0.0);
  for (long long q0 = 0; q0 < K; q0 += TK) {
    for (int t = threadIdx.x; t < TK * TT; t += 256) {
      const int qq = t % TK, cc = t / TK;
      const long long q = q0 + qq;
      As[qq][cc] = (q < K && k0 + cc < M) ? A[q + static_cast<long long>(k0 + cc) * lda] : make_double2(0.0, 0.0);
      Bs[qq][cc] = (q < K && l0 + cc < N) ? B[q + static_cast<long long>(l0 + cc) * ldb] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int qq = 0; qq < TK; ++qq) {
      const double2 a0 = As[qq][ty], a1 = As[qq][ty + 16];
      const double2 b0 = Bs[qq][tx], b1 = Bs[qq][tx + 16];
      cfma(acc[0][0], a0, b0);
      cfma(acc[0][1], a0, b1);
      cfma(acc[1][0], a1, b0);
      cfma(acc[1][1], a1, b1);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int k = k0 + ty + 16 * i, l = l0 + tx + 16 * j;
      if (k < M && l < N) {
        double2 v = make_double2(sgn * acc[i][j].x, sgn * acc[i][j].y);
        if (Crm) v = cadd(v, Crm[static_cast<long long>(k) * ldc + l]);
        out[k + static_cast<long long>(l) * ldo] = v;
      }
    }
}

// X(:, c) = [U(:, c) + F Y(:, c); -Y(:, c)]  with Y = S^{-1} B U  (I2 = -Y).
__global__ void combineX(const double2* __restrict__ UF, const double2* __restrict__ Y, double2* __restrict__ X,
                         long long nA, long long nM, int p) {
  const long long ntot = nA + nM;
  const long long total = ntot * p;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = o % ntot;
    const int c = static_cast<int>(o / ntot);
    const double2* y = Y + static_cast<long long>(c) * nM;
    if (q < nA) {
      double2 acc = UF[q + static_cast<long long>(c) * nA];
      const double2* F = UF + static_cast<long long>(p) * nA + q;
      for (long long k = 0; k < nM; ++k) cfma(acc, F[k * nA], y[k]);
      X[o] = acc;
    } else {
      const double2 v = y[q - nA];
      X[o] = make_double2(-v.x, -v.y);
    }
  }
}

// dst (nA x nc, column-major) = columns [c0, c0+nc) of [V1 | B^T].
__global__ void gatherRhs(const double2* __restrict__ b, long long ldb, const double2* __restrict__ bt,
                          double2* __restrict__ dst, long long nA, int p, int c0, int nc) {
  const long long total = nA * nc;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = o % nA;
    const int c = c0 + static_cast<int>(o / nA);
    dst[o] = c < p ? b[q + static_cast<long long>(c) * ldb] : bt[q + static_cast<long long>(c - p) * nA];
  }
}

__global__ void marginRowsNonzero(const double2* __restrict__ b, long long ntot, long long nA, int p, int* flag) {
  const long long nM = ntot - nA;
  const long long total = nM * p;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double2 v = b[nA + o % nM + (o / nM) * ntot];
    if (v.x != 0.0 || v.y != 0.0) atomicOr(flag, 1);
  }
}

// Per column: |y - b|^2 and |b|^2 (fixed-order per CTA, CTA per column).
__global__ void residualNorms(const double2* __restrict__ y, const double2* __restrict__ b, long long n,
                              double* __restrict__ out) {
  __shared__ double s1[256], s2[256];
  const int c = blockIdx.x;
  double a = 0.0, bb = 0.0;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 yv = y[i + c * n], bv = b[i + c * n];
    const double dx = yv.x - bv.x, dy = yv.y - bv.y;
    a += dx * dx + dy * dy;
    bb += bv.x * bv.x + bv.y * bv.y;
  }
  s1[threadIdx.x] = a;
  s2[threadIdx.x] = bb;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      s1[threadIdx.x] += s1[threadIdx.x + off];
      s2[threadIdx.x] += s2[threadIdx.x + off];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * c] = s1[0];
    out[2 * c + 1] = s2[0];
  }
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { TBT_CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

}  // namespace

// b, x: device, (nA + nM) x p column-major. Fills iterations / residual.
void schurSolve(Ctx& c, const double2* b, double2* x, int p, const tbt_gmres_opts& o, std::vector<int>& iterations,
                std::vector<double>& residual) {
  cudaStream_t s = c.stream;
  const MarginOp* M = c.margin;
  const long long nA = c.n, nM = M ? M->nM : 0, ntot = nA + nM;
  {
    DevBuf flag(sizeof(int));
    memsetSync(flag.p, 0, sizeof(int), s);
    if (nM > 0) marginRowsNonzero<<<gridFor(nM * p), 256, 0, s>>>(b, ntot, nA, p, flag.as<int>());
    int h = 0;
    TBT_CUDA_CHECK(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    TBT_CUDA_CHECK(cudaStreamSynchronize(s));
    TBT_USER_CHECK(h == 0, "schurSolve: excitation must vanish on margin rows");
  }
  const long long cols = p + nM;
  DevBuf bt(static_cast<size_t>(nA) * std::max<long long>(nM, 1) * sizeof(double2));
  if (nM > 0) {
    BTArgs a{};
    a.nx = c.nx;
    a.ny = c.ny;
    a.m = c.m;
    a.nA = nA;
    a.nM = nM;
    a.dense = M->bDense;
    for (int r = 0; r < 2; ++r) {
      a.emSide[r] = M->emSide[r];
      a.emRow[r] = M->emRow[r];
      a.sideStart[r] = M->sideStart[r];
      a.rowStart[r] = M->rowStart[r];
      a.rawSide[r] = M->rawSide[r];
      a.rawRow[r] = M->rawRow[r];
    }
    for (int q = 0; q < 4; ++q) {
      a.emCorner[q] = M->emCorner[q];
      a.cornerStart[q] = M->cornerStart[q];
      a.corner[q] = M->corner[q];
    }
    buildBT<<<gridFor(nA * nM), 256, 0, s>>>(a, bt.as<double2>());
    TBT_CUDA_CHECK(cudaGetLastError());
  }
  // A [U F] = [V1 B^T]: batches of max_nrhs columns through the A-only GMRES.
  DevBuf uf(static_cast<size_t>(nA) * cols * sizeof(double2));
  const int K = c.maxNrhs;
  DevBuf chunk(static_cast<size_t>(nA) * K * sizeof(double2));
  DevBuf ib(static_cast<size_t>(nA) * K * sizeof(double2)), ix(static_cast<size_t>(nA) * K * sizeof(double2));
  tbt_gmres_opts oi = o;
  oi.hist_cap = 0;
  oi.use_a_only = 1;
  iterations.assign(p, 0);
  std::string failure;
  for (long long c0 = 0; c0 < cols; c0 += K) {
    const int nc = static_cast<int>(std::min<long long>(K, cols - c0));
    gatherRhs<<<gridFor(nA * nc), 256, 0, s>>>(b, ntot, bt.as<double2>(), chunk.as<double2>(), nA, p,
                                               static_cast<int>(c0), nc);
    launchLayoutU(chunk.as<double2>(), ib.as<double2>(), nA, nA, nc, true, s, c.m);
    std::vector<GmresState> st;
    std::vector<double> hist;
    int mv = 0;
    gmresSolve(c, ib.as<double2>(), ix.as<double2>(), nc, oi, true, st, hist, mv);
    launchLayoutU(ix.as<double2>(), uf.as<double2>() + c0 * nA, nA, nA, nc, false, s, c.m);
    for (int k = 0; k < nc; ++k) {
      const long long col = c0 + k;
      if (col < p) iterations[col] = st[k].iterations;
      if (!st[k].converged && failure.empty())
        failure = "schur inner solve did not converge (column " + std::to_string(col) + ", best residual " +
                  std::to_string(st[k].residual) + ")";
    }
  }
  if (!failure.empty()) throw Error{TBT_NUMERIC_ERROR, failure};
  DevBuf y(static_cast<size_t>(std::max<long long>(nM, 1)) * p * sizeof(double2));
  if (nM > 0) {
    // S = C - B F (= C - (B^T)^T F, plain transpose as linsolve.cpp:669).
    DevBuf S(static_cast<size_t>(nM) * nM * sizeof(double2));
    const dim3 g1((nM + TT - 1) / TT, (nM + TT - 1) / TT);
    zgemmTN<<<g1, 256, 0, s>>>(bt.as<double2>(), nA, uf.as<double2>() + static_cast<long long>(p) * nA, nA,
                               S.as<double2>(), nM, static_cast<int>(nM), static_cast<int>(nM), nA, M->C, nM, -1.0);
    DevBuf perm(static_cast<size_t>(nM) * sizeof(int));
    {
      std::vector<int> id(nM);
      for (long long i = 0; i < nM; ++i) id[i] = static_cast<int>(i);
      uploadSync(perm.p, id.data(), nM * sizeof(int), s);
    }
    if (nM <= 512) {  // one CTA, barriers between steps
      dense::luFactorSmall<<<1, 1024, 0, s>>>(S.as<double2>(), static_cast<int>(nM), perm.as<int>());
    } else {
      for (int k = 0; k < nM; ++k) {
        dense::luPivot<<<1, 256, 0, s>>>(S.as<double2>(), static_cast<int>(nM), k, perm.as<int>());
        if (k + 1 < nM) {
          const long long rest = (nM - k - 1) * (nM - k - 1);
          dense::luUpdate<<<gridFor(rest), 256, 0, s>>>(S.as<double2>(), static_cast<int>(nM), k);
        }
      }
    }
    TBT_CUDA_CHECK(cudaGetLastError());
    // checkLu (linsolve.cpp:517-528): pivot ratio of U's diagonal.
    std::vector<double2> diag(nM);
    TBT_CUDA_CHECK(cudaMemcpy2DAsync(diag.data(), sizeof(double2), S.p, (nM + 1) * sizeof(double2), sizeof(double2),
                                     nM, cudaMemcpyDeviceToHost, s));
    TBT_CUDA_CHECK(cudaStreamSynchronize(s));
    double maxAbs = 0.0, minAbs = std::numeric_limits<double>::infinity();
    for (const double2& d : diag) {
      const double a = std::hypot(d.x, d.y);
      maxAbs = std::max(maxAbs, a);
      minAbs = std::min(minAbs, a);
    }
    if (!(minAbs > 1e-14 * maxAbs))
      throw Error{TBT_NUMERIC_ERROR, "singular matrix in schur complement (pivot ratio " +
                                         std::to_string(minAbs / (maxAbs > 0 ? maxAbs : 1.0)) + ")"};
    // Y = S^{-1} (B U); I2 = -Y.
    const dim3 g2((p + TT - 1) / TT, (nM + TT - 1) / TT);
    zgemmTN<<<g2, 256, 0, s>>>(bt.as<double2>(), nA, uf.as<double2>(), nA, y.as<double2>(), nM, static_cast<int>(nM),
                               p, nA, nullptr, 0, 1.0);
    DevBuf scratch(static_cast<size_t>(nM) * p * sizeof(double2));
    dense::luSolveCols<<<p, 256, 0, s>>>(S.as<double2>(), perm.as<int>(), static_cast<int>(nM), y.as<double2>(),
                                  scratch.as<double2>());
    TBT_CUDA_CHECK(cudaGetLastError());
  }
  // X = [U - F I2; I2] = [U + F Y; -Y].
  combineX<<<gridFor(ntot * p), 256, 0, s>>>(uf.as<double2>(), y.as<double2>(), x, nA, nM, p);
  TBT_CUDA_CHECK(cudaGetLastError());
  // Residual of every column under the Schur system [A B^T; B C].
  residual.assign(p, 0.0);
  const long long nInt = static_cast<long long>(c.ne + c.neM) * c.m;
  DevBuf xi(static_cast<size_t>(nInt) * K * sizeof(double2)), yi(static_cast<size_t>(nInt) * K * sizeof(double2));
  DevBuf yu(static_cast<size_t>(ntot) * K * sizeof(double2));
  DevBuf norms(static_cast<size_t>(2) * K * sizeof(double));
  for (int c0 = 0; c0 < p; c0 += K) {
    const int nc = std::min(K, p - c0);
    launchLayoutU(x + static_cast<long long>(c0) * ntot, xi.as<double2>(), ntot, nInt, nc, true, s, c.m);
    applyInternal(c, xi.as<double2>(), yi.as<double2>(), nc, false);
    if (c.margin) marginApply(c, xi.as<double2>(), yi.as<double2>(), nc);
    launchLayoutU(yi.as<double2>(), yu.as<double2>(), ntot, nInt, nc, false, s, c.m);
    residualNorms<<<nc, 256, 0, s>>>(yu.as<double2>(), b + static_cast<long long>(c0) * ntot, ntot,
                                     norms.as<double>());
    std::vector<double> h(2 * nc);
    TBT_CUDA_CHECK(cudaMemcpyAsync(h.data(), norms.p, 2 * nc * sizeof(double), cudaMemcpyDeviceToHost, s));
    TBT_CUDA_CHECK(cudaStreamSynchronize(s));
    for (int k = 0; k < nc; ++k) residual[c0 + k] = std::sqrt(h[2 * k]) / (h[2 * k + 1] > 0 ? std::sqrt(h[2 * k + 1]) : 1.0);
  }
}

}  // namespace tbt
