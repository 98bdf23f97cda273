// Small dense complex kernels shared by the Schur driver (schur.cu) and
// the port network (postproc.cu): right-looking LU with partial pivoting,
// column-wise substitution.
#pragma once

#include "tbt_internal.cuh"

namespace tbt {
namespace dense {
namespace {  // per translation unit (kernels in a header)

// LU step k (one CTA): pivot = first row of maximal |S(i,k)|, i >= k; swap
// rows k and pivot over all columns; scale the column below the diagonal.
__global__ void luPivot(double2* __restrict__ S, int n, int k, int* __restrict__ perm) {
  __shared__ double bestV[256];
  __shared__ int bestI[256];
  double bv = -1.0;
  int bi = n;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double2 v = S[i + static_cast<long long>(k) * n];
    const double a = hypot(v.x, v.y);
    if (a > bv) {
      bv = a;
      bi = i;
    }
  }
  bestV[threadIdx.x] = bv;
  bestI[threadIdx.x] = bi;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off) {
      const double ov = bestV[threadIdx.x + off];
      const int oi = bestI[threadIdx.x + off];
      if (ov > bestV[threadIdx.x] || (ov == bestV[threadIdx.x] && oi < bestI[threadIdx.x])) {
        bestV[threadIdx.x] = ov;
        bestI[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const int p = bestI[0];
  if (p != k && p < n) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const long long a = k + static_cast<long long>(j) * n, b = p + static_cast<long long>(j) * n;
      const double2 t = S[a];
      S[a] = S[b];
      S[b] = t;
    }
    if (threadIdx.x == 0) {
      const int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
  }
  __syncthreads();
  const double2 piv = S[k + static_cast<long long>(k) * n];
  if (piv.x == 0.0 && piv.y == 0.0) return;
  const double d = piv.x * piv.x + piv.y * piv.y;
  const double2 inv = make_double2(piv.x / d, -piv.y / d);
  for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
    const long long a = i + static_cast<long long>(k) * n;
    S[a] = cmul(S[a], inv);
  }
}

// Trailing update S(i,j) -= L(i,k) U(k,j), i, j > k.
__global__ void luUpdate(double2* __restrict__ S, int n, int k) {
  const int m = n - k - 1;
  const long long total = static_cast<long long>(m) * m;
  for (long long o = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = k + 1 + static_cast<int>(o % m), j = k + 1 + static_cast<int>(o / m);
    const double2 l = S[i + static_cast<long long>(k) * n], u = S[k + static_cast<long long>(j) * n];
    double2& s = S[i + static_cast<long long>(j) * n];
    s = csub(s, cmul(l, u));
  }
}

// In place: R <- U^{-1} L^{-1} P R, one CTA per column (column-oriented
// substitution, one barrier per step). y is n x p scratch.
__global__ void luSolveCols(const double2* __restrict__ LU, const int* __restrict__ perm, int n,
                            double2* __restrict__ R, double2* __restrict__ y) {
  const int c = blockIdx.x;
  double2* r = R + static_cast<long long>(c) * n;
  double2* t = y + static_cast<long long>(c) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t[i] = r[perm[i]];
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double2 tk = t[k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x)
      t[i] = csub(t[i], cmul(LU[i + static_cast<long long>(k) * n], tk));
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {
    if (threadIdx.x == 0) {
      const double2 d = LU[k + static_cast<long long>(k) * n];
      const double dd = d.x * d.x + d.y * d.y;
      t[k] = cmul(t[k], make_double2(d.x / dd, -d.y / dd));
    }
    __syncthreads();
    const double2 tk = t[k];
    for (int i = threadIdx.x; i < k; i += blockDim.x) t[i] = csub(t[i], cmul(LU[i + static_cast<long long>(k) * n], tk));
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) r[i] = t[i];
}


// The whole factorisation in one CTA (small n): the same pivot rule and
// update order as luPivot / luUpdate, barriers instead of launches.
__global__ void __launch_bounds__(1024) luFactorSmall(double2* __restrict__ S, int n, int* __restrict__ perm) {
  __shared__ double bestV[32];
  __shared__ int bestI[33];
  for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    double bv = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      const double2 v = S[i + static_cast<long long>(k) * n];
      const double a = hypot(v.x, v.y);
      if (a > bv) {
        bv = a;
        bi = i;
      }
    }
    // Largest |v|, ties to the lowest row: warp shuffles, then warp 0 over
    // the per-warp winners.
    for (int off = 16; off > 0; off >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      bestV[threadIdx.x >> 5] = bv;
      bestI[threadIdx.x >> 5] = bi;
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int nw = static_cast<int>(blockDim.x >> 5);
      bv = threadIdx.x < nw ? bestV[threadIdx.x] : -1.0;
      bi = threadIdx.x < nw ? bestI[threadIdx.x] : n;
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      if (threadIdx.x == 0) bestI[32] = bi;
    }
    __syncthreads();
    const int p = bestI[32];
    if (p != k && p < n) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const long long a = k + static_cast<long long>(j) * n, b = p + static_cast<long long>(j) * n;
        const double2 t = S[a];
        S[a] = S[b];
        S[b] = t;
      }
      if (threadIdx.x == 0) {
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    const double2 piv = S[k + static_cast<long long>(k) * n];
    if (!(piv.x == 0.0 && piv.y == 0.0)) {
      const double d = piv.x * piv.x + piv.y * piv.y;
      const double2 inv = make_double2(piv.x / d, -piv.y / d);
      for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) {
        const long long a = i + static_cast<long long>(k) * n;
        S[a] = cmul(S[a], inv);
      }
    }
    __syncthreads();
    const int m = n - k - 1;
    for (int o = threadIdx.x; o < m * m; o += blockDim.x) {
      const int i = k + 1 + o % m, j = k + 1 + o / m;
      const double2 l = S[i + static_cast<long long>(k) * n], u = S[k + static_cast<long long>(j) * n];
      double2& sv = S[i + static_cast<long long>(j) * n];
      sv = csub(sv, cmul(l, u));
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace dense
}  // namespace tbt
