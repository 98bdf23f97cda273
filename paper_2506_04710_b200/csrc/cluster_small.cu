// Latency-bound sizes (C1: 4 x 4 elements, m = 24, 64 bins): the operator
// application and the WHOLE restarted GMRES in one kernel launch on one
// 8-CTA thread-block cluster.
//
// At C1 the multi-kernel apply is a chain of launch latencies (~18 us for a
// ~2 MFLOP operator) and a GMRES iteration a dozen of them. Here:
//  * each CTA keeps its share of the half spectrum (pairs p = rank mod 8) in
//    shared memory for the whole solve, and owns a contiguous slice of the
//    elements (its slice of every Krylov vector lives in its shared memory);
//  * an apply all-gathers the input slices through distributed shared
//    memory, evaluates x^ for its own bins directly (2-D DFT over the
//    nx*ny elements with exact twiddles), multiplies by its blocks (A or
//    A^T), cluster-barrier, gathers every bin's y^ through DSMEM and
//    evaluates the inverse DFT + 1/L + K + edge/corner terms for its
//    elements only;
//  * GMRES (gmres.cu semantics: x0 = 0, true residual per restart, Jacobi,
//    low-synchronisation MGS h = (I+L)^-1 V^H w, Givens, inner exit at
//    |g_{j+1}|/beta < 0.1 tol, back substitution) reduces dot products as
//    per-CTA partials summed by every CTA in the same order after a cluster
//    barrier (bitwise-identical scalars everywhere); the scalar recurrences
//    run redundantly per CTA, CTA 0 publishes state and history.
// Same definitions as linsolve.cpp:260-290 (applyA), :373-388 (+ the BASELINE
// correction), :425-515 (gmres).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "gmres_dev.cuh"

namespace cg = cooperative_groups;

namespace tbt {
namespace {

constexpr int CL = 8;          // CTAs in the cluster
constexpr int CT = 256;        // threads per CTA
constexpr int CW = CT / 32;

struct CsArgs {
  int nx, ny, m, L0, L1, L, ne, n;
  double scale;
  const double2* S;      // half spectrum [pair][a][b]
  const int* pairF;
  const int* pairG;
  int npairs, kp;        // pairs, max pairs per CTA
  const int4* binMap;    // [L]: {owner CTA, slot, trans, 0}
  const double2* tw0;
  const double2* tw1;
  int corr;
  const int* tInfo;
  const int* elemPtr;
  const double2* D;
  const double2* U;
  const double2* V;
  int rank;
  const double2* K;      // antisymmetric part of Z(0,0) (row-major) or null
  int elemPerCta, nloc;  // element slice per CTA, nloc = elemPerCta * m
  // shared-memory carve (double2 offsets)
  int oSpec, oX, oXh, oYh, oYall, oV, oW, oXs, oB, oDinv, oS, oH, oG, oCs, oSn, oPart, oTot, oY;
  int oTw0, oTw1, oScr;  // twiddles, per-warp scratch (corrections / inverse partials)
  int oBin;              // bin map copy (int4 per bin, 16 bytes like a double2)
  unsigned long long* prof;  // optional: accumulated ns per section (CTA 0)
  int smemD2;
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct CsCtx {
  const CsArgs& a;
  double2* sm;
  cg::cluster_group cl;
  int rank;
  int epoch = 0;  // which half of the double-buffered partials the next reduction uses
  __device__ double2* at(int off) const { return sm + off; }
  __device__ double2* part() const { return sm + a.oPart + (epoch & 1) * 2 * (gmresdev::RMAX + 1); }
};

// Fixed-order cluster all-reduce of cnt partials (part()[0..cnt) in every
// CTA) into tot[0..cnt) in every CTA. The partials are double-buffered by
// epoch, so one cluster barrier per reduction suffices: a CTA can only
// overwrite this half again after the NEXT reduction's barrier, which every
// CTA reaches after finishing its reads here.
__device__ void clusterSum(CsCtx& c, int cnt) {
  double2* part = c.part();
  double2* tot = c.at(c.a.oTot);
  c.cl.sync();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    double2 v[CL];  // all remote loads in flight, then the fixed-order sum
#pragma unroll
    for (int r = 0; r < CL; ++r) v[r] = c.cl.map_shared_rank(part, r)[i];
    double2 t = v[0];
#pragma unroll
    for (int r = 1; r < CL; ++r) t = cadd(t, v[r]);
    tot[i] = t;
  }
  __syncthreads();
  ++c.epoch;
}

// CTA-level partial sum of v into part[slot] (fixed order).
__device__ void ctaPartial(CsCtx& c, double2 v, int slot, double2* red) {
  v = gmresdev::warpSum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = red[0];
    for (int w = 1; w < CW; ++w) t = cadd(t, red[w]);
    c.part()[slot] = t;
  }
}

// y (slice, smem at oY) = Z v, v given as this CTA's slice at vloc (smem).
__device__ void clusterApply(CsCtx& c, const double2* vloc, bool withCorr) {
  const CsArgs& a = c.a;
  const int m = a.m, nx = a.nx, ny = a.ny, L0 = a.L0, L1 = a.L1;
  double2* X = c.at(a.oX);
  double2* xh = c.at(a.oXh);
  double2* yh = c.at(a.oYh);
  double2* yall = c.at(a.oYall);
  double2* out = c.at(a.oY);
  const double2* tw0 = c.at(a.oTw0);
  const double2* tw1 = c.at(a.oTw1);
  // 1. All-gather the input slices (each CTA published vloc before).
  c.cl.sync();
  for (int i0 = threadIdx.x; i0 < a.n; i0 += 4 * blockDim.x) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      const int r = i / a.nloc;
      v[u] = i < a.n ? c.cl.map_shared_rank(const_cast<double2*>(vloc), r)[i - r * a.nloc] : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * blockDim.x < a.n) X[i0 + u * blockDim.x] = v[u];
  }
  __syncthreads();
  // 2. x^ for the own bins: slot s -> pair rank + CL*(s/2), bin f or g.
  const int nslot = 2 * a.kp;
  for (int t = threadIdx.x; t < nslot * m; t += blockDim.x) {
    const int s = t / m, b = t % m;
    const int p = c.rank + CL * (s >> 1);
    if (p >= a.npairs) continue;
    const int f = (s & 1) ? a.pairG[p] : a.pairF[p];
    const int s1 = f / L0, s0 = f % L0;
    double2 acc = make_double2(0.0, 0.0);
    for (int r = 0; r < ny; ++r) {
      const double2 w1 = tw1[(s1 * r) % L1];
      double2 row = make_double2(0.0, 0.0);
      for (int cc = 0; cc < nx; ++cc) cfma(row, X[(r * nx + cc) * m + b], tw0[(s0 * cc) % L0]);
      cfma(acc, row, w1);
    }
    xh[t] = acc;
  }
  __syncthreads();
  // 3. y^ = A x^ (representative bin) or A^T x^ (partner), blocks in smem.
  const double2* spec = c.at(a.oSpec);
  for (int t = threadIdx.x; t < nslot * m; t += blockDim.x) {
    const int s = t / m, i = t % m;
    const int p = c.rank + CL * (s >> 1);
    if (p >= a.npairs) continue;
    if ((s & 1) && a.pairG[p] == a.pairF[p]) continue;
    const double2* A = spec + static_cast<size_t>(s >> 1) * m * m;
    const double2* xv = xh + s * m;
    double2 acc = make_double2(0.0, 0.0);
    if (s & 1)
      for (int j = 0; j < m; ++j) cfma(acc, A[j * m + i], xv[j]);
    else
      for (int j = 0; j < m; ++j) cfma(acc, A[i * m + j], xv[j]);
    yh[t] = acc;
  }
  // 4. Every CTA gathers all bins' y^ (DSMEM).
  c.cl.sync();
  for (int t0 = threadIdx.x; t0 < a.L * m; t0 += 4 * blockDim.x) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int t = t0 + u * blockDim.x;
      v[u] = make_double2(0.0, 0.0);
      if (t < a.L * m) {
        const int4 bm = reinterpret_cast<const int4*>(c.at(a.oBin))[t / m];
        v[u] = c.cl.map_shared_rank(yh, bm.x)[bm.y * m + t % m];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (t0 + u * blockDim.x < a.L * m) yall[t0 + u * blockDim.x] = v[u];
  }
  __syncthreads();
  // 5. Inverse DFT for the own elements: partial rows per (output, s1) in
  //    scratch, then the s1 sum in order, 1/L, + K x_e.
  const int e0 = min(c.rank * a.elemPerCta, a.ne);
  const int ecount = max(0, min(a.elemPerCta, a.ne - e0));  // trailing CTAs may own no element
  double2* scr = c.at(a.oScr);
  for (int t = threadIdx.x; t < a.nloc * L1; t += blockDim.x) {
    const int s1 = t / a.nloc, q = t % a.nloc;
    const int el = q / m, i = q % m;
    double2 row = make_double2(0.0, 0.0);
    if (el < ecount) {
      const int e = e0 + el, r = e / nx, cc = e % nx;
      for (int s0 = 0; s0 < L0; ++s0) {
        double2 w0 = tw0[(s0 * cc) % L0];
        w0.y = -w0.y;
        cfma(row, yall[(s1 * L0 + s0) * m + i], w0);
      }
      double2 w1 = tw1[(s1 * r) % L1];
      w1.y = -w1.y;
      row = cmul(row, w1);
    }
    scr[t] = row;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < a.nloc; t += blockDim.x) {
    const int el = t / m, i = t % m;
    double2 acc = make_double2(0.0, 0.0);
    if (el < ecount) {
      for (int s1 = 0; s1 < L1; ++s1) acc = cadd(acc, scr[s1 * a.nloc + t]);
      acc = make_double2(acc.x * a.scale, acc.y * a.scale);
      if (a.K) {
        const int e = e0 + el;
        for (int j = 0; j < m; ++j) cfma(acc, a.K[i * m + j], X[e * m + j]);
      }
    }
    out[t] = acc;
  }
  __syncthreads();
  // 6. Edge/corner terms of the own elements: the terms of the slice are
  //    spread over the warps (each warp adds its terms' vectors into its own
  //    scratch row), then summed over warps in order.
  if (withCorr && a.corr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double2* wsum = scr + static_cast<size_t>(warp) * a.nloc;
    for (int t = lane; t < a.nloc; t += 32) wsum[t] = make_double2(0.0, 0.0);
    const int t0 = a.elemPtr[e0], t1 = a.elemPtr[e0 + ecount];
    for (int tt = t0 + warp; tt < t1; tt += CW) {
      const int tgt = a.tInfo[4 * tt], src = a.tInfo[4 * tt + 1], slot = a.tInfo[4 * tt + 2];
      const int trans = a.tInfo[4 * tt + 3];
      const double2* W = (trans ? a.U : a.V) + static_cast<long long>(slot) * a.rank * m;
      const double2* W2 = (trans ? a.V : a.U) + static_cast<long long>(slot) * a.rank * m;
      const double2* xs = X + src * m;
      double2* o = wsum + (tgt - e0) * m;
      // All of the term's U / V / d values a lane needs are loaded up front
      // (one latency instead of one per projection); m <= 64, rank <= 8.
      constexpr int QM = 8;
      double2 wv[QM][2], w2v[QM][2], dv[2], xv[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = lane + 32 * h;
        const bool ok = i < m;
        dv[h] = ok ? __ldg(a.D + slot * m + i) : make_double2(0.0, 0.0);
        xv[h] = ok ? xs[i] : make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < QM; ++q) {
          const bool oq = ok && q < a.rank;
          wv[q][h] = oq ? __ldg(W + q * m + i) : make_double2(0.0, 0.0);
          w2v[q][h] = oq ? __ldg(W2 + q * m + i) : make_double2(0.0, 0.0);
        }
      }
      double2 acc[2] = {cmul(dv[0], xv[0]), cmul(dv[1], xv[1])};
#pragma unroll
      for (int q = 0; q < QM; ++q) {
        if (q >= a.rank) break;
        double2 pr = make_double2(0.0, 0.0);
        cfma(pr, wv[q][0], xv[0]);
        cfma(pr, wv[q][1], xv[1]);
        pr = gmresdev::warpSum(pr);
        cfma(acc[0], w2v[q][0], pr);
        cfma(acc[1], w2v[q][1], pr);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (lane + 32 * h < m) o[lane + 32 * h] = cadd(o[lane + 32 * h], acc[h]);
    }
    __syncthreads();
    for (int t = threadIdx.x; t < a.nloc; t += blockDim.x) {
      double2 acc = out[t];
      for (int w2 = 0; w2 < CW; ++w2) acc = cadd(acc, scr[static_cast<size_t>(w2) * a.nloc + t]);
      out[t] = acc;
    }
    __syncthreads();
  }
}

__device__ void loadSpectrum(CsCtx& c) {
  const CsArgs& a = c.a;
  for (int t = threadIdx.x; t < a.L; t += blockDim.x) reinterpret_cast<int4*>(c.at(a.oBin))[t] = a.binMap[t];
  for (int t = threadIdx.x; t < a.L0; t += blockDim.x) c.at(a.oTw0)[t] = a.tw0[t];
  for (int t = threadIdx.x; t < a.L1; t += blockDim.x) c.at(a.oTw1)[t] = a.tw1[t];
  double2* spec = c.at(a.oSpec);
  const int mm = a.m * a.m;
  // Batches of 8 independent loads per thread (one latency per batch).
  const int total = a.kp * mm;
  for (int t0 = threadIdx.x; t0 < total; t0 += 8 * blockDim.x) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * blockDim.x;
      const int p = c.rank + CL * (t / mm);
      v[u] = (t < total && p < a.npairs) ? __ldg(a.S + static_cast<long long>(p) * mm + t % mm) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int t = t0 + u * blockDim.x;
      if (t < total) spec[t] = v[u];
    }
  }
  __syncthreads();
}

__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(CT) clusterApplyKernel(CsArgs a, const double2* x,
                                                                                     double2* y, int withCorr) {
  extern __shared__ double2 smc[];
  CsCtx c{a, smc, cg::this_cluster(), static_cast<int>(cg::this_cluster().block_rank())};
  loadSpectrum(c);
  double2* xs = c.at(a.oXs);
  for (int t = threadIdx.x; t < a.nloc; t += blockDim.x) {
    const int q = c.rank * a.nloc + t;
    xs[t] = q < a.n ? x[q] : make_double2(0.0, 0.0);
  }
  clusterApply(c, xs, withCorr != 0);
  const double2* out = c.at(a.oY);
  for (int t = threadIdx.x; t < a.nloc; t += blockDim.x) {
    const int q = c.rank * a.nloc + t;
    if (q < a.n) y[q] = out[t];
  }
  c.cl.sync();  // no CTA exits while others may still read its shared memory
}

// The complete solve. A: the usual GmresArgs (b, x, st, hist in global).
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(CT) clusterGmresKernel(CsArgs a, GmresArgs A,
                                                                                     int withCorr) {
  extern __shared__ double2 smc[];
  __shared__ double2 red[CW];
  __shared__ double2 hcol[gmresdev::RMAX + 2];
  __shared__ int sStop;
  CsCtx c{a, smc, cg::this_cluster(), static_cast<int>(cg::this_cluster().block_rank())};
  loadSpectrum(c);
  const int nloc = a.nloc, R = A.restart, lds = R + 1;
  const int base = c.rank * nloc;
  double2* Vl = c.at(a.oV);   // [R+1][nloc]
  double2* w = c.at(a.oW);
  double2* xl = c.at(a.oXs);  // solution slice
  double2* bl = c.at(a.oB);
  double2* dl = c.at(a.oDinv);
  double2* Sm = c.at(a.oS);   // [R+1][R+1] Gram rows
  double2* H = c.at(a.oH);    // [(R+1)*R]
  double2* g = c.at(a.oG);
  double2* cs = c.at(a.oCs);
  double2* sn = c.at(a.oSn);
  double2* tot = c.at(a.oTot);
  const double2* y = c.at(a.oY);
  const bool lead = c.rank == 0 && threadIdx.x == 0;
  for (int t = threadIdx.x; t < nloc; t += blockDim.x) {
    const int q = base + t;
    bl[t] = q < a.n ? A.b[q] : make_double2(0.0, 0.0);
    dl[t] = (q < a.n && A.dinv) ? A.dinv[q] : make_double2(1.0, 0.0);
    xl[t] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  auto norm2 = [&](const double2* v) {
    double2 s = make_double2(0.0, 0.0);
    for (int t = threadIdx.x; t < nloc; t += blockDim.x) s.x += v[t].x * v[t].x + v[t].y * v[t].y;
    ctaPartial(c, s, 0, red);
    clusterSum(c, 1);
    return tot[0].x;
  };
  auto push = [&](double kind, double v, int& histLen) {
    if (lead && histLen < A.histCap) {
      A.hist[2 * histLen] = kind;
      A.hist[2 * histLen + 1] = v;
    }
    ++histLen;
  };
  const double bnorm = sqrt(norm2(bl));
  int iterations = 0, histLen = 0, converged = bnorm == 0.0 ? 1 : 0, done = converged, checks = 0;
  double residual = 0.0, beta0 = 0.0, beta = 0.0;
  while (!done) {
    // r = b - A x, residual (linsolve.cpp:446-452).
    clusterApply(c, xl, withCorr != 0);
    ++checks;
    for (int t = threadIdx.x; t < nloc; t += blockDim.x) w[t] = csub(bl[t], y[t]);
    __syncthreads();
    const double res = sqrt(norm2(w)) / bnorm;
    residual = res;
    int decision = 0;
    if (res < A.tol)
      decision = 1;
    else if (iterations >= A.maxIter)
      decision = 2;
    push(decision == 2 ? 2.0 : 0.0, res, histLen);
    if (decision != 0) {
      converged = decision == 1;
      break;
    }
    for (int t = threadIdx.x; t < nloc; t += blockDim.x) Vl[t] = cmul(w[t], dl[t]);
    __syncthreads();
    beta = sqrt(norm2(Vl));
    if (beta == 0.0) {
      converged = 1;
      break;
    }
    if (beta0 == 0.0) beta0 = beta;
    for (int k = threadIdx.x; k <= R; k += blockDim.x) g[k] = make_double2(0.0, 0.0);
    for (int t = threadIdx.x; t < nloc; t += blockDim.x) Vl[t] = make_double2(Vl[t].x / beta, Vl[t].y / beta);
    __syncthreads();
    if (threadIdx.x == 0) {
      g[0] = make_double2(beta, 0.0);
      sStop = 0;
    }
    __syncthreads();
    int ncount = 0;
    for (int j = 0; j < R && !sStop; ++j) {
      const double2* vj = Vl + static_cast<size_t>(j) * nloc;
      unsigned long long tp0 = gtime();
      clusterApply(c, vj, withCorr != 0);
      unsigned long long tp1 = gtime();
      for (int t = threadIdx.x; t < nloc; t += blockDim.x) w[t] = cmul(y[t], dl[t]);
      __syncthreads();
      // Low-sync MGS: c_k = <v_k, w> (slot k), S_jk = <v_j, v_k> (slot j+1+k).
      {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int d = warp; d < 2 * j + 1; d += CW) {  // one warp per dot, fixed lane order
          const int k = d <= j ? d : d - j - 1;
          const double2* vk = Vl + static_cast<size_t>(k) * nloc;
          double2 acc = make_double2(0.0, 0.0);
          if (d <= j)
            for (int t = lane; t < nloc; t += 32) cfma_conj(acc, vk[t], w[t]);
          else
            for (int t = lane; t < nloc; t += 32) cfma_conj(acc, vj[t], vk[t]);
          acc = gmresdev::warpSum(acc);
          if (lane == 0) c.part()[d] = acc;
        }
      }
      clusterSum(c, 2 * j + 1);
      unsigned long long tp2 = gtime();
      for (int k = threadIdx.x; k < j; k += blockDim.x) Sm[j * lds + k] = tot[j + 1 + k];
      __syncthreads();
      if (threadIdx.x < 32) {  // h = (I + L)^-1 c: column-oriented forward substitution on warp 0
        constexpr int RPL = (gmresdev::RMAX + 31) / 32 + 1;
        const int lane = threadIdx.x;
        double2 hv[RPL];
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int i = lane + 32 * t;
          hv[t] = i <= j ? tot[i] : make_double2(0.0, 0.0);
        }
        for (int k = 0; k < j; ++k) {
          double2 hk = make_double2(0.0, 0.0);
#pragma unroll
          for (int t = 0; t < RPL; ++t)
            if (t == (k >> 5)) hk = hv[t];
          hk = gmresdev::shfl2(hk, k & 31);
#pragma unroll
          for (int t = 0; t < RPL; ++t) {
            const int i = lane + 32 * t;
            if (i > k && i <= j) hv[t] = csub(hv[t], cmul(Sm[i * lds + k], hk));
          }
        }
#pragma unroll
        for (int t = 0; t < RPL; ++t) {
          const int i = lane + 32 * t;
          if (i <= j) hcol[i] = hv[t];
        }
      }
      __syncthreads();
      double2 nacc = make_double2(0.0, 0.0);
      for (int t = threadIdx.x; t < nloc; t += blockDim.x) {
        double2 wv = w[t];
        for (int k = 0; k <= j; ++k) wv = csub(wv, cmul(hcol[k], Vl[static_cast<size_t>(k) * nloc + t]));
        w[t] = wv;
        nacc.x += wv.x * wv.x + wv.y * wv.y;
      }
      unsigned long long tp3 = gtime();
      ctaPartial(c, nacc, 0, red);
      clusterSum(c, 1);
      const double hn = sqrt(tot[0].x);
      if (hn > 0.0)
        for (int t = threadIdx.x; t < nloc; t += blockDim.x)
          Vl[static_cast<size_t>(j + 1) * nloc + t] = make_double2(w[t].x / hn, w[t].y / hn);
      // Givens (linsolve.cpp:472-501), redundantly in every CTA.
      if (threadIdx.x == 0) {
        double2* hc = H + static_cast<size_t>(j) * lds;
        for (int i = 0; i <= j; ++i) hc[i] = hcol[i];
        hc[j + 1] = make_double2(hn, 0.0);
        for (int i = 0; i < j; ++i) {
          const double2 a0 = hc[i], a1 = hc[i + 1];
          hc[i] = cadd(cmul(cs[i], a0), cmul(sn[i], a1));
          hc[i + 1] = cadd(cmul(make_double2(-sn[i].x, sn[i].y), a0), cmul(gmresdev::cconj(cs[i]), a1));
        }
        const double2 hjj = hc[j], hj1 = hc[j + 1];
        const double den = sqrt((hjj.x * hjj.x + hjj.y * hjj.y) + (hj1.x * hj1.x + hj1.y * hj1.y));
        double2 cc, ss;
        if (den == 0.0) {
          cc = make_double2(1.0, 0.0);
          ss = make_double2(0.0, 0.0);
        } else {
          cc = make_double2(hjj.x / den, -hjj.y / den);
          ss = make_double2(hj1.x / den, -hj1.y / den);
        }
        cs[j] = cc;
        sn[j] = ss;
        hc[j] = cadd(cmul(cc, hjj), cmul(ss, hj1));
        hc[j + 1] = make_double2(0.0, 0.0);
        const double2 gj = g[j];
        g[j] = cmul(cc, gj);
        const double2 gj1 = cmul(make_double2(-ss.x, ss.y), gj);
        g[j + 1] = gj1;
        const double rel = gmresdev::cabs2(gj1) / beta;
        if (c.rank == 0 && histLen < A.histCap) {
          A.hist[2 * histLen] = 1.0;
          A.hist[2 * histLen + 1] = gmresdev::cabs2(gj1) / beta0;
        }
        sStop = (rel < 0.1 * A.tol || !(hn > 0.0) || j + 1 >= R || iterations + 1 >= A.maxIter) ? 1 : 0;
      }
      ++histLen;
      ++iterations;
      ncount = j + 1;
      if (a.prof && lead) {
        const unsigned long long tp4 = gtime();
        a.prof[0] += tp1 - tp0;
        a.prof[1] += tp2 - tp1;
        a.prof[2] += tp3 - tp2;
        a.prof[3] += tp4 - tp3;
        a.prof[4] += 1;
      }
      __syncthreads();
    }
    // Back substitution and x += V y (:504-510); y coefficients in hcol.
    if (threadIdx.x == 0) {
      for (int i0 = ncount - 1; i0 >= 0; --i0) {
        double2 s = g[i0];
        for (int k = i0 + 1; k < ncount; ++k) s = csub(s, cmul(H[static_cast<size_t>(k) * lds + i0], hcol[k]));
        hcol[i0] = gmresdev::cdiv(s, H[static_cast<size_t>(i0) * lds + i0]);
      }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nloc; t += blockDim.x) {
      double2 xv = xl[t];
      for (int i = 0; i < ncount; ++i) xv = cadd(xv, cmul(hcol[i], Vl[static_cast<size_t>(i) * nloc + t]));
      xl[t] = xv;
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nloc; t += blockDim.x) {
    const int q = base + t;
    if (q < a.n) A.x[q] = xl[t];
  }
  if (lead) {
    GmresState& st = A.st[0];
    st.bnorm = bnorm;
    st.beta = beta;
    st.beta0 = beta0;
    st.residual = residual;
    st.iterations = iterations;
    st.ncount = 0;
    st.stopInner = 1;
    st.done = 1;
    st.converged = converged;
    st.cycleActive = 0;
    st.histLen = histLen;
    st.checks = checks;
  }
  c.cl.sync();
}

}  // namespace

struct ClusterSmall {
  CsArgs a{};
  int4* dBinMap = nullptr;
  size_t smem = 0;
  bool ok = false;
};

namespace {

bool buildArgs(Ctx& c, CsArgs& a, size_t& smemBytes) {
  a.nx = c.nx;
  a.ny = c.ny;
  a.m = c.m;
  a.L0 = c.L0;
  a.L1 = c.L1;
  a.L = static_cast<int>(c.L);
  a.ne = c.ne;
  a.n = static_cast<int>(c.n);
  a.scale = 1.0 / static_cast<double>(c.L);
  a.S = c.dSpectra;
  a.pairF = c.dPairF;
  a.pairG = c.dPairG;
  a.npairs = static_cast<int>(c.npairs);
  a.kp = (a.npairs + CL - 1) / CL;
  a.tw0 = c.dTw0;
  a.tw1 = c.dTw1;
  a.corr = (c.haveCorr && c.nTerms > 0) ? 1 : 0;
  a.tInfo = c.dTermInfo;
  a.elemPtr = c.dElemPtr;
  a.D = c.dCorrD;
  a.U = c.dCorrU;
  a.V = c.dCorrV;
  a.rank = c.rank;
  a.K = c.hasAntisym ? c.dAntisym : nullptr;
  a.elemPerCta = (c.ne + CL - 1) / CL;
  a.nloc = a.elemPerCta * c.m;
  const int R = gmresdev::RMAX;  // carve for the largest restart
  const int m = c.m;
  int off = 0;
  auto take = [&](long long cnt) {
    const int o = off;
    off += static_cast<int>(cnt);
    return o;
  };
  a.oSpec = take(static_cast<long long>(a.kp) * m * m);
  a.oX = take(a.n);
  a.oXh = take(2LL * a.kp * m);
  a.oYh = take(2LL * a.kp * m);
  a.oYall = take(static_cast<long long>(a.L) * m);
  a.oY = take(a.nloc);
  a.oXs = take(a.nloc);
  a.oW = take(a.nloc);
  a.oB = take(a.nloc);
  a.oDinv = take(a.nloc);
  a.oPart = take(4 * (R + 1));  // two halves
  a.oTot = take(2 * (R + 1));
  a.oG = take(R + 1);
  a.oCs = take(R);
  a.oSn = take(R);
  a.oBin = take(c.L);
  a.oTw0 = take(c.L0);
  a.oTw1 = take(c.L1);
  a.oScr = take(std::max<long long>(static_cast<long long>(CW) * 2 * a.nloc, static_cast<long long>(c.L1) * a.nloc));
  a.oV = take(0);  // sized per solve (restart): V, S, H follow
  a.smemD2 = off;
  smemBytes = static_cast<size_t>(off) * sizeof(double2);
  return true;
}

}  // namespace

// Whether the one-cluster path serves this context (tiny operators only).
bool clusterSmallSupported(const Ctx& c, int restart) {
  if (c.dist || c.margin || c.forceMultiPass || c.timeBinprod || c.fullMode) return false;
  if (c.L > 256 || c.m > 64 || c.ne > 256 || c.npairs < 1 || c.rank > 8) return false;
  CsArgs a{};
  size_t base = 0;
  buildArgs(const_cast<Ctx&>(c), a, base);
  const int R = std::max(1, restart);
  const size_t extra = sizeof(double2) * (static_cast<size_t>(R + 1) * a.nloc + static_cast<size_t>(R + 1) * (R + 1) +
                                          static_cast<size_t>(R + 1) * R);
  return base + extra <= 200 * 1024;
}

namespace {
int4* binMapFor(Ctx& c) {
  static thread_local std::vector<int4> host;
  host.assign(static_cast<size_t>(c.L), make_int4(0, 0, 0, 0));
  for (long long p = 0; p < c.npairs; ++p) {
    const int owner = static_cast<int>(p % CL), lp = static_cast<int>(p / CL);
    host[c.pairF[p]] = make_int4(owner, 2 * lp, 0, 0);
    if (c.pairG[p] != c.pairF[p]) host[c.pairG[p]] = make_int4(owner, 2 * lp + 1, 1, 0);
  }
  int4* d = nullptr;
  TBT_CUDA_CHECK(cudaMalloc(&d, host.size() * sizeof(int4)));
  uploadSync(d, host.data(), host.size() * sizeof(int4), c.stream);
  return d;
}
}  // namespace

void clusterSmallFree(Ctx& c) {
  if (c.clusterSmall) {
    if (c.clusterSmall->dBinMap) cudaFree(c.clusterSmall->dBinMap);
    delete c.clusterSmall;
    c.clusterSmall = nullptr;
  }
}

static ClusterSmall& prepared(Ctx& c) {
  if (!c.clusterSmall) {
    c.clusterSmall = new ClusterSmall;
    c.clusterSmall->dBinMap = binMapFor(c);
  }
  return *c.clusterSmall;
}

void launchClusterApply(Ctx& c, const double2* x, double2* y, bool withCorr) {
  ClusterSmall& cs = prepared(c);
  CsArgs a{};
  size_t smem = 0;
  buildArgs(c, a, smem);
  a.binMap = cs.dBinMap;
  static std::atomic<unsigned long long> attr{0};
  oncePerDevice(attr, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(clusterApplyKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  clusterApplyKernel<<<CL, CT, smem, c.stream>>>(a, x, y, withCorr ? 1 : 0);
  TBT_CUDA_CHECK(cudaGetLastError());
}

void launchClusterGmres(Ctx& c, const GmresArgs& A, bool withCorr) {
  ClusterSmall& cs = prepared(c);
  CsArgs a{};
  size_t smem = 0;
  buildArgs(c, a, smem);
  static const bool prof = getenv("TBT_CLPROF") != nullptr;  // debug: per-section ns in dPhaseNs[24..28]
  a.prof = prof ? c.dPhaseNs + 24 : nullptr;
  if (prof) memsetSync(c.dPhaseNs + 24, 0, 5 * sizeof(unsigned long long), c.stream);
  a.binMap = cs.dBinMap;
  const int R = A.restart;
  a.oS = a.oV + (R + 1) * a.nloc;
  a.oH = a.oS + (R + 1) * (R + 1);
  smem += sizeof(double2) * (static_cast<size_t>(R + 1) * a.nloc + static_cast<size_t>(R + 1) * (R + 1) +
                             static_cast<size_t>(R + 1) * R);
  static std::atomic<unsigned long long> attr{0};
  oncePerDevice(attr, [] {
    TBT_CUDA_CHECK(cudaFuncSetAttribute(clusterGmresKernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  clusterGmresKernel<<<CL, CT, smem, c.stream>>>(a, A, withCorr ? 1 : 0);
  TBT_CUDA_CHECK(cudaGetLastError());
  if (prof) {
    unsigned long long ns[5];
    TBT_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    TBT_CUDA_CHECK(cudaMemcpy(ns, c.dPhaseNs + 24, sizeof(ns), cudaMemcpyDeviceToHost));
    const double it = ns[4] > 0 ? static_cast<double>(ns[4]) : 1.0;
    fprintf(stderr, "cluster gmres per iteration (us): apply %.2f dots %.2f subst+update %.2f norm+givens %.2f (%llu its)\n",
            1e-3 * ns[0] / it, 1e-3 * ns[1] / it, 1e-3 * ns[2] / it, 1e-3 * ns[3] / it, ns[4]);
  }
}

}  // namespace tbt
